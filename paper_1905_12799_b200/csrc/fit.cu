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
    double* pred = nullptr;  // running prediction, canonical row order
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

    // Row-id storage without per-node allocation: the rows and the n per-feature orders of
    // every node at depth d live in the node's segment [off, off + cnt) of level d's arrays
    // (children partition their parent's segment: left part first, stable).
    std::vector<std::vector<int64_t>> lvl_rows;   // [depth + 1][m]
    std::vector<std::vector<int64_t>> lvl_ord;    // [depth + 1][n * m]

    void setup_levels(const std::vector<std::vector<int64_t>>& root_orders) {
        lvl_rows.assign(size_t(max_depth) + 1, std::vector<int64_t>(size_t(m)));
        lvl_ord.assign(size_t(max_depth) + 1, std::vector<int64_t>(size_t(n) * size_t(m)));
        for (int64_t i = 0; i < m; ++i) lvl_rows[0][i] = i;
        for (int f = 0; f < n; ++f) std::copy(root_orders[f].begin(), root_orders[f].end(), lvl_ord[0].begin() + size_t(f) * m);
        in_left.assign(size_t(m), 0);
    }

    // _best_split (cost_model.py:292-325) over feature orders ord[f * m + off .. + cnt)
    bool best_split(const int64_t* ord, int64_t off, int64_t mm, int& bf, double& bt) {
        bool have = false;
        double best_gain = 0.0;
        xs.resize(mm);
        rs.resize(mm);
        csum.resize(mm);
        csq.resize(mm);
        for (int j = 0; j < n; ++j) {
            const int64_t* o = ord + size_t(j) * m + off;
            // one pass: gather, sequential cumsums (np.cumsum order), boundary detection
            double c = 0.0, q = 0.0;
            bool any = false;
            for (int64_t k = 0; k < mm; ++k) {
                const int64_t row = o[k];
                const double xv = x(row, j), rv = resid[row];
                xs[k] = xv;
                any |= k > 0 && xv != xs[k - 1];
                c = k ? c + rv : rv;
                q = k ? q + rv * rv : rv * rv;
                csum[k] = c;
                csq[k] = q;
            }
            if (!any) continue;
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

    // _grow (cost_model.py:328-364) for the node owning segment [off, off + cnt) of level `depth`
    int grow(int64_t off, int64_t cnt, int depth) {
        const int node = add();
        const int64_t* rows = lvl_rows[depth].data() + off;
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
        const bool split = depth < max_depth && sse > 0.0 && best_split(lvl_ord[depth].data(), off, cnt, j, t);
        if (!split) {
            const double v = shrink * mean;
            value[node] = v;
            // pred += tree.predict(X): the rows this leaf owns are exactly the training rows
            // Tree.predict routes here (same x[f] <= t rule), so no tree walk is needed
            for (int64_t i = 0; i < cnt; ++i) pred[rows[i]] += v;
            return node;
        }
        // stable partition of the rows and of every feature order into level depth + 1
        int64_t* nrows = lvl_rows[depth + 1].data() + off;
        int64_t nl = 0;
        for (int64_t i = 0; i < cnt; ++i) {
            const int64_t r = rows[i];
            const bool lft = x(r, j) <= t;
            in_left[r] = lft;
            nl += lft;
        }
        int64_t li = 0, ri = nl;
        for (int64_t i = 0; i < cnt; ++i) {
            const int64_t r = rows[i];
            nrows[in_left[r] ? li++ : ri++] = r;
        }
        for (int f = 0; f < n && depth + 1 < max_depth; ++f) {  // children at max depth are leaves: no orders
            const int64_t* o = lvl_ord[depth].data() + size_t(f) * m + off;
            int64_t* no = lvl_ord[depth + 1].data() + size_t(f) * m + off;
            int64_t a2 = 0, b2 = nl;
            for (int64_t i = 0; i < cnt; ++i) {
                const int64_t r = o[i];
                no[in_left[r] ? a2++ : b2++] = r;
            }
        }
        feature[node] = j;
        threshold[node] = t;
        const int l = grow(off, nl, depth + 1);
        left[node] = l;
        const int rr = grow(off + nl, cnt - nl, depth + 1);
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
    g.setup_levels(root);
    g.pred = pred.data();
    int64_t used = 0;
    for (int r = 0; r < rounds; ++r) {
        for (int64_t i = 0; i < m; ++i) g.resid[i] = y[i] - pred[i];
        g.feature.clear(), g.left.clear(), g.right.clear(), g.threshold.clear(), g.value.clear();
        g.grow(0, m, 0);
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
        used += nodes;  // pred was updated at the leaves during growth
    }
    tree_offsets_out[rounds] = int32_t(used);
    *base_out = base;
    KT_API_END
}
