// fit.cu — gradient-boosted regression trees, exact greedy squared error (host code).
//
// Reference: knobtuner/cost_model.py fit (:367-398), _grow (:328-364), _best_split
// (:292-325), Tree.predict (:83-97).  SURVEY §8(f) row 1: the surrogate is refit every
// tuning round (driver.py:142-148) and is the dominant host cost of a tune; this is a
// native restatement in numpy's exact operation order so the model is byte-identical:
//
//   * canonical row order = np.lexsort((targets, f_{n-1}, ..., f_0)): stable, feature 0
//     primary;
//   * means / SSEs use numpy's pairwise summation (np.add.reduce on contiguous
//     float64: 8 accumulators, 128-element blocks, split n/2 - (n/2 % 8));
//   * split search uses sequential cumsums over the node's per-feature stable order,
//     numpy's elementwise expression order, first maximum (smallest threshold), and
//     a strictly greater gain to switch features (lowest feature wins ties);
//   * children keep canonical / per-feature order (stable partition), preorder node ids.
//
// Host-only (no device work): the training set is at most the tuning budget (~10^3-10^4
// rows), far below where a GPU launch pays; kept native so a round's refit costs
// milliseconds instead of the reference's Python recursion.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>

#include "common.cuh"

namespace kt {
namespace {

// numpy pairwise_sum (numpy/_core/src/umath/loops_utils.h.src), unit stride.
double pw_sum(const double* a, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; ++i) res += a[i];
        return res;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pw_sum(a, n2) + pw_sum(a + n2, n - n2);
}

struct Grower {
    const double* X;  // canonical order, row-major [m][n]
    int64_t m;
    int n;
    int max_depth;
    double shrink;
    std::vector<double> resid;
    // output (one tree)
    std::vector<int32_t> feature, left, right;
    std::vector<double> threshold, value;
    std::vector<double> buf, xs, rs, csum, csq;
    std::vector<uint8_t> in_left;

    int add() {
        feature.push_back(-1);
        threshold.push_back(0.0);
        left.push_back(-1);
        right.push_back(-1);
        value.push_back(0.0);
        return int(feature.size()) - 1;
    }

    double x(int64_t row, int j) const { return X[size_t(row) * n + j]; }

    // _best_split (cost_model.py:292-325); returns false when no feature has a boundary
    bool best_split(const std::vector<std::vector<int64_t>>& orders, int& bf, double& bt) {
        const int64_t mm = int64_t(orders[0].size());
        bool have = false;
        double best_gain = 0.0;
        xs.resize(mm);
        rs.resize(mm);
        csum.resize(mm);
        csq.resize(mm);
        for (int j = 0; j < n; ++j) {
            const auto& ord = orders[j];
            for (int64_t k = 0; k < mm; ++k) {
                xs[k] = x(ord[k], j);
                rs[k] = resid[ord[k]];
            }
            bool any = false;
            for (int64_t k = 0; k + 1 < mm && !any; ++k) any = xs[k] != xs[k + 1];
            if (!any) continue;
            double c = 0.0, q = 0.0;
            for (int64_t k = 0; k < mm; ++k) {
                c = k ? c + rs[k] : rs[k];
                q = k ? q + rs[k] * rs[k] : rs[k] * rs[k];
                csum[k] = c;
                csq[k] = q;
            }
            const double total = csum[mm - 1], total_sq = csq[mm - 1];
            const double parent_sse = total_sq - total * total / double(mm);
            double g_best = 0.0;
            int64_t b_best = -1;
            for (int64_t b = 0; b + 1 < mm; ++b) {
                if (!(xs[b] != xs[b + 1])) continue;
                const double ln = double(b + 1), rn = double(mm - (b + 1));
                const double ls = csum[b], lq = csq[b];
                const double sse_left = lq - ls * ls / ln;
                const double d = total - ls;
                const double sse_right = (total_sq - lq) - d * d / rn;
                const double gain = parent_sse - sse_left - sse_right;
                // np.argmax: first maximum; a NaN is the maximum (first NaN wins)
                if (b_best < 0) {
                    g_best = gain;
                    b_best = b;
                } else if (!std::isnan(g_best) && (std::isnan(gain) || gain > g_best)) {
                    g_best = gain;
                    b_best = b;
                }
            }
            const double thr = (xs[b_best] + xs[b_best + 1]) / 2.0;
            if (!have || g_best > best_gain) {
                have = true;
                best_gain = g_best;
                bf = j;
                bt = thr;
            }
        }
        return have;
    }

    // _grow (cost_model.py:328-364)
    int grow(const std::vector<int64_t>& rows, const std::vector<std::vector<int64_t>>& orders, int depth) {
        const int node = add();
        const int64_t cnt = int64_t(rows.size());
        buf.resize(cnt);
        for (int64_t i = 0; i < cnt; ++i) buf[i] = resid[rows[i]];
        const double mean = pw_sum(buf.data(), cnt) / double(cnt);
        for (int64_t i = 0; i < cnt; ++i) {
            const double d = buf[i] - mean;
            buf[i] = d * d;
        }
        const double sse = pw_sum(buf.data(), cnt);
        int j = -1;
        double t = 0.0;
        const bool split = depth < max_depth && sse > 0.0 && best_split(orders, j, t);
        if (!split) {
            value[node] = shrink * mean;
            return node;
        }
        std::vector<int64_t> lrows, rrows;
        in_left.assign(size_t(m), 0);
        for (int64_t r : rows) {
            if (x(r, j) <= t) {
                lrows.push_back(r);
                in_left[r] = 1;
            } else {
                rrows.push_back(r);
            }
        }
        std::vector<std::vector<int64_t>> lo(n), ro(n);
        for (int f = 0; f < n; ++f) {
            lo[f].reserve(lrows.size());
            ro[f].reserve(rrows.size());
            for (int64_t r : orders[f]) (in_left[r] ? lo[f] : ro[f]).push_back(r);
        }
        feature[node] = j;
        threshold[node] = t;
        const int l = grow(lrows, lo, depth + 1);
        left[node] = l;
        const int rr = grow(rrows, ro, depth + 1);
        right[node] = rr;
        return node;
    }
};

}  // namespace
}  // namespace kt

extern "C" int kt_fit_trees(const double* features, const double* targets, int64_t m, int n, int rounds, int depth,
                            double learning_rate, int32_t* feature_out, double* threshold_out, int32_t* left_out,
                            int32_t* right_out, double* value_out, int64_t node_capacity, int32_t* tree_offsets_out,
                            double* base_out) {
    KT_API_BEGIN
    using namespace kt;
    if (m < 1) fail(KT_ERR_VALUE, "training set is empty");
    if (n < 1) fail(KT_ERR_VALUE, "training set needs at least one feature");
    if (rounds < 1) fail(KT_ERR_VALUE, "rounds must be >= 1, got " + std::to_string(rounds));
    if (depth < 1) fail(KT_ERR_VALUE, "depth must be >= 1, got " + std::to_string(depth));
    if (!(learning_rate > 0.0 && learning_rate <= 1.0)) fail(KT_ERR_VALUE, "learning_rate must be in (0, 1]");
    // canonical order: np.lexsort(np.vstack([targets, features.T[::-1]])) — feature 0 primary
    std::vector<int64_t> order(static_cast<size_t>(m));
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
        for (int j = 0; j < n; ++j) {
            const double xa = features[size_t(a) * n + j], xb = features[size_t(b) * n + j];
            if (xa < xb) return true;
            if (xb < xa) return false;
        }
        return targets[a] < targets[b];
    });
    std::vector<double> X(static_cast<size_t>(m) * n), y(static_cast<size_t>(m));
    for (int64_t i = 0; i < m; ++i) {
        std::memcpy(&X[size_t(i) * n], features + size_t(order[i]) * n, sizeof(double) * n);
        y[i] = targets[order[i]];
    }
    const double base = pw_sum(y.data(), m) / double(m);
    std::vector<double> pred(static_cast<size_t>(m), base);
    std::vector<int64_t> all_rows(static_cast<size_t>(m));
    std::iota(all_rows.begin(), all_rows.end(), 0);
    std::vector<std::vector<int64_t>> root(n, all_rows);
    for (int j = 0; j < n; ++j)
        std::stable_sort(root[j].begin(), root[j].end(),
                         [&](int64_t a, int64_t b) { return X[size_t(a) * n + j] < X[size_t(b) * n + j]; });
    Grower g;
    g.X = X.data();
    g.m = m;
    g.n = n;
    g.max_depth = depth;
    g.shrink = learning_rate;
    g.resid.resize(size_t(m));
    int64_t used = 0;
    for (int r = 0; r < rounds; ++r) {
        for (int64_t i = 0; i < m; ++i) g.resid[i] = y[i] - pred[i];
        g.feature.clear(), g.left.clear(), g.right.clear(), g.threshold.clear(), g.value.clear();
        g.grow(all_rows, root, 0);
        const int64_t nodes = int64_t(g.feature.size());
        if (used + nodes > node_capacity) fail(KT_ERR_VALUE, "node capacity exceeded");
        tree_offsets_out[r] = int32_t(used);
        for (int64_t k = 0; k < nodes; ++k) {
            feature_out[used + k] = g.feature[k];
            threshold_out[used + k] = g.threshold[k];
            left_out[used + k] = g.left[k];
            right_out[used + k] = g.right[k];
            value_out[used + k] = g.value[k];
        }
        used += nodes;
        // pred += tree.predict(X)
        for (int64_t i = 0; i < m; ++i) {
            int node = 0;
            while (g.feature[node] >= 0)
                node = X[size_t(i) * n + g.feature[node]] <= g.threshold[node] ? g.left[node] : g.right[node];
            pred[i] += g.value[node];
        }
    }
    tree_offsets_out[rounds] = int32_t(used);
    *base_out = base;
    KT_API_END
}
