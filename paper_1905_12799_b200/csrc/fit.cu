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
// Two engines, same bytes: kt_fit_trees_device runs the whole boosting loop (every round,
// every level) in one single-CTA kernel on the GPU — one warp per node of a level, one lane
// per feature for the split scans, warp-stable partitions — with the float64 operations in
// the reference's order and rounding (explicit _rn intrinsics, no FMA contraction);
// kt_fit_trees is the same algorithm on the host for CPU-only callers.  The host does the
// O(m log m) canonical sorts (np.lexsort / stable argsort order) for both.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <vector>

#include "common.cuh"
#include "pwsum_warp.cuh"

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
    std::vector<double> buf, xs, csum, csq, gbuf;
    std::vector<int64_t> bnd;
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

    // _best_split (cost_model.py:292-325) over feature orders ord[f * m + off .. + cnt).
    // Features are scanned G at a time in one pass over the rows, so the G per-feature
    // sequential cumsum chains (np.cumsum order) run side by side; the pass also records the
    // boundaries (value changes), so the gain evaluation visits only those.
    template <int G>
    void scan_group(const int64_t* ord, int64_t off, int64_t mm, int j0, bool& have, double& best_gain, int& bf,
                    double& bt) {
        const int64_t* o[G];
        double c[G], q[G], prev[G];
        int64_t nb[G];
        double* xsj[G];
        double* csj[G];
        double* cqj[G];
        int64_t* bj[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            o[g] = ord + size_t(j0 + g) * m + off;
            c[g] = q[g] = prev[g] = 0.0;
            nb[g] = 0;
            xsj[g] = xs.data() + size_t(g) * mm;
            csj[g] = csum.data() + size_t(g) * mm;
            cqj[g] = csq.data() + size_t(g) * mm;
            bj[g] = bnd.data() + size_t(g) * mm;
        }
        for (int64_t k = 0; k < mm; ++k) {
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const int64_t row = o[g][k];
                const double xv = x(row, j0 + g), rv = resid[row];
                c[g] = k ? c[g] + rv : rv;
                q[g] = k ? q[g] + rv * rv : rv * rv;
                csj[g][k] = c[g];
                cqj[g][k] = q[g];
                xsj[g][k] = xv;
                bj[g][nb[g]] = k - 1;  // boundary between k - 1 and k
                nb[g] += k > 0 && xv != prev[g];
                prev[g] = xv;
            }
        }
        for (int g = 0; g < G; ++g) {
            if (!nb[g]) continue;  // constant feature: no split
            const double* cs = csj[g];
            const double* cq = cqj[g];
            const double total = cs[mm - 1], total_sq = cq[mm - 1];
            const double parent_sse = total_sq - total * total / double(mm);
            // gains at every boundary first (independent divisions pipeline), then np.argmax
            const int64_t nbg = nb[g];
            double* gains = gbuf.data();
            for (int64_t i = 0; i < nbg; ++i) {
                const int64_t b = bj[g][i];
                const double ln = double(b + 1), rn = double(mm - (b + 1));
                const double ls = cs[b], lq = cq[b];
                const double sse_left = lq - ls * ls / ln;
                const double d = total - ls;
                const double sse_right = (total_sq - lq) - d * d / rn;
                gains[i] = parent_sse - sse_left - sse_right;
            }
            // np.argmax: first maximum; a NaN is the maximum (first NaN wins)
            double g_best = gains[0];
            int64_t i_best = 0;
            for (int64_t i = 1; i < nbg && !std::isnan(g_best); ++i) {
                const double gain = gains[i];
                if (std::isnan(gain) || gain > g_best) {
                    g_best = gain;
                    i_best = i;
                }
            }
            const int64_t b_best = bj[g][i_best];
            const double thr = (xsj[g][b_best] + xsj[g][b_best + 1]) / 2.0;
            if (!have || g_best > best_gain) {
                have = true;
                best_gain = g_best;
                bf = j0 + g;
                bt = thr;
            }
        }
    }

    bool best_split(const int64_t* ord, int64_t off, int64_t mm, int& bf, double& bt) {
        constexpr int kG = 4;
        bool have = false;
        double best_gain = 0.0;
        const size_t need = size_t(kG) * size_t(mm);
        if (xs.size() < need) {
            xs.resize(need);
            csum.resize(need);
            csq.resize(need);
            bnd.resize(need);
        }
        if (gbuf.size() < size_t(mm)) gbuf.resize(size_t(mm));
        int j = 0;
        for (; j + kG <= n; j += kG) scan_group<kG>(ord, off, mm, j, have, best_gain, bf, bt);
        switch (n - j) {
            case 1: scan_group<1>(ord, off, mm, j, have, best_gain, bf, bt); break;
            case 2: scan_group<2>(ord, off, mm, j, have, best_gain, bf, bt); break;
            case 3: scan_group<3>(ord, off, mm, j, have, best_gain, bf, bt); break;
            default: break;
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
        // branch-free (the side of a row is data-dependent: branches mispredict half the time)
        auto partition = [&](const int64_t* src, int64_t* dst) {
            int64_t a2 = 0, b2 = nl;
            for (int64_t i = 0; i < cnt; ++i) {
                const int64_t r = src[i];
                const int64_t lft = in_left[r];
                dst[b2 + (a2 - b2) * lft] = r;
                a2 += lft;
                b2 += 1 - lft;
            }
        };
        partition(rows, nrows);
        for (int f = 0; f < n && depth + 1 < max_depth; ++f)  // children at max depth are leaves: no orders
            partition(lvl_ord[depth].data() + size_t(f) * m + off, lvl_ord[depth + 1].data() + size_t(f) * m + off);
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

// ============================================================ device engine
// One CTA of kFitThreads; level lists in shared memory; rows / orders / scratch in global.
constexpr int kFitThreads = 512;
constexpr int kFitWarps = kFitThreads / 32;
constexpr int kFitMaxDepth = 7;  // static shared memory bound; deeper trees use kt_fit_trees
constexpr int kFitMaxNodes = (1 << (kFitMaxDepth + 1)) - 1;
constexpr int kFitMaxLevel = 1 << kFitMaxDepth;  // nodes of the deepest level

struct FitDevArgs {
    const double* X;     // canonical order [m][n]
    const double* y;     // canonical order
    const int32_t* root_ord;  // [n][m] stable argsort per feature
    int64_t m;
    int n, rounds, depth;
    double lr, base;
    int32_t* lvl_rows;   // [depth + 1][m]
    int32_t* lvl_ord;    // [depth + 1][n][m]
    double* resid;       // [m]
    double* pred;        // [m]
    double* buf;         // [m] per-node segments
    uint8_t* in_left;    // [m]
    const uint16_t* codes;  // [n][m] rank of each row's value among the feature's distinct values (or null)
    double* xs;          // [n][m] the node's feature values in its per-feature order (segment-local)
    double* rs;          // [n][m] residuals in the same order
    double* csum;        // [n][m] np.cumsum(rs) of the segment
    double* csq;         // [n][m] np.cumsum(rs * rs)
    // outputs (preorder per tree, concatenated)
    int32_t* feature;
    double* threshold;
    int32_t* left;
    int32_t* right;
    double* value;
    int32_t* tree_offsets;  // [rounds + 1]
};

// numpy pairwise_sum, unit stride (same as pw_sum above), device side.  Iterative post-order
// walk of the same split tree (device recursion would need an unbounded stack).
__device__ double pw_leaf_dev(const double* a, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
        return res;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
}
__device__ double pw_sum_dev(const double* a, int64_t n) {
    if (n <= 128) return pw_leaf_dev(a, n);
    constexpr int kMaxFrames = 32;  // halving from n < 2^31 to <= 128 rows
    int32_t off[kMaxFrames], len[kMaxFrames];
    double lsum[kMaxFrames];
    bool right[kMaxFrames];  // the frame's left half is done, its right half is on top
    int sp = 0;
    off[0] = 0, len[0] = int32_t(n), right[0] = false;
    for (;;) {
        // descend to the leftmost leaf of the frame on top
        while (len[sp] > 128) {
            int32_t n2 = len[sp] / 2;
            n2 -= n2 % 8;
            off[sp + 1] = off[sp];
            len[sp + 1] = n2;
            right[sp + 1] = false;
            ++sp;
        }
        double v = pw_leaf_dev(a + off[sp], len[sp]);
        // climb: a finished left half starts its sibling, a finished right half folds up
        for (;;) {
            if (sp == 0) return v;
            const int p = sp - 1;
            int32_t n2 = len[p] / 2;
            n2 -= n2 % 8;
            if (!right[sp]) {
                lsum[p] = v;
                off[sp] = off[p] + n2;
                len[sp] = len[p] - n2;
                right[sp] = true;
                break;
            }
            v = __dadd_rn(lsum[p], v);
            --sp;
        }
    }
}


struct FitNode {  // BFS record of one tree
    int off, cnt;
    int feature;      // -1 leaf
    double thr, value;
    int lchild, rchild;  // BFS ids
};

// np.argmax order over (gain, boundary index): first maximum, a NaN is the maximum (first NaN wins)
__device__ __forceinline__ bool argmax_better(double g, int64_t i, double gb, int64_t ib) {
    if (ib < 0) return i >= 0;
    if (i < 0) return false;
    const bool nan_g = isnan(g), nan_b = isnan(gb);
    if (nan_g || nan_b) return nan_g && (!nan_b || i < ib);
    return g > gb || (g == gb && i < ib);
}

__global__ void __launch_bounds__(kFitThreads, 1) fit_kernel(FitDevArgs a) {
    __shared__ FitNode nodes[kFitMaxNodes];
    __shared__ int level_begin[kFitMaxDepth + 2];
    __shared__ int n_nodes;
    __shared__ double feat_gain[kFitMaxLevel][kMaxKnobs];
    __shared__ double feat_thr[kFitMaxLevel][kMaxKnobs];
    __shared__ uint8_t feat_have[kFitMaxLevel][kMaxKnobs];
    __shared__ int node_split[kFitMaxLevel];
    __shared__ uint8_t node_try[kFitMaxLevel];
    __shared__ int preorder[kFitMaxNodes];
    __shared__ int used;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t m = a.m;
    const int n = a.n;
    for (int64_t i = tid; i < m; i += blockDim.x) {
        a.pred[i] = a.base;
        a.lvl_rows[i] = int32_t(i);
    }
    for (int64_t i = tid; i < int64_t(n) * m; i += blockDim.x) a.lvl_ord[i] = a.root_ord[i];
    if (tid == 0) used = 0;
    __syncthreads();
    for (int round = 0; round < a.rounds; ++round) {
        for (int64_t i = tid; i < m; i += blockDim.x) a.resid[i] = __dsub_rn(a.y[i], a.pred[i]);
        if (tid == 0) {
            nodes[0].off = 0;
            nodes[0].cnt = int(m);
            n_nodes = 1;
            level_begin[0] = 0;
            level_begin[1] = 1;
        }
        __syncthreads();
        for (int d = 0; d <= a.depth; ++d) {
            const int lb = level_begin[d], le = level_begin[d + 1];
            const int32_t* rows_d = a.lvl_rows + int64_t(d) * m;
            const int32_t* ord_d = a.lvl_ord + int64_t(d) * n * m;
            // ---- node statistics (mean, SSE in numpy's pairwise order) and split search
            for (int q = lb + warp; q < le; q += kFitWarps) {
                const int off = nodes[q].off, cnt = nodes[q].cnt, li = q - lb;
                const int32_t* rows = rows_d + off;
                const double* resid = a.resid;
                const double mean =
                    __ddiv_rn(pw_sum_warp([&](int i) { return resid[rows[i]]; }, cnt), double(cnt));
                const double sse = pw_sum_warp(
                    [&](int i) {
                        const double dd = __dsub_rn(resid[rows[i]], mean);
                        return __dmul_rn(dd, dd);
                    },
                    cnt);
                const bool try_split = d < a.depth && sse > 0.0;
                if (lane == 0) {
                    node_try[li] = try_split;
                    nodes[q].value = __dmul_rn(a.lr, mean);  // used if the node ends up a leaf
                    nodes[q].lchild = nodes[q].rchild = -1;
                }
            }
            __syncthreads();
            // ---- split search (_best_split, cost_model.py:292-325), in three block-wide phases:
            // gather each candidate's per-feature (x, resid) sequences contiguously (parallel) ...
            for (int q = lb; q < le; ++q) {
                const int li = q - lb;
                if (!node_try[li]) continue;
                const int off = nodes[q].off, cnt = nodes[q].cnt;
                for (int idx = tid; idx < n * cnt; idx += blockDim.x) {
                    const int f = idx / cnt, k = idx - f * cnt;
                    const int row = ord_d[int64_t(f) * m + off + k];
                    a.xs[int64_t(f) * m + off + k] = a.X[int64_t(row) * n + f];
                    a.rs[int64_t(f) * m + off + k] = a.resid[row];
                }
            }
            __syncthreads();
            // ... sequential cumsums (np.cumsum order), one warp per (candidate, feature): lanes
            // load 32 elements at a time (coalesced, next chunk prefetched), every lane runs the
            // same sequential chain over shuffled values and keeps the prefix at its position
            for (int pair = warp; pair < (le - lb) * n; pair += kFitWarps) {
                const int li = pair / n, f = pair - li * n, q = lb + li;
                if (!node_try[li]) {
                    if (lane == 0) feat_have[li][f] = 0;
                    continue;
                }
                const int off = nodes[q].off, cnt = nodes[q].cnt;
                const double* __restrict__ xs = a.xs + int64_t(f) * m + off;
                const double* __restrict__ rs = a.rs + int64_t(f) * m + off;
                double* __restrict__ cs = a.csum + int64_t(f) * m + off;
                double* __restrict__ cq = a.csq + int64_t(f) * m + off;
                double c = 0.0, qq = 0.0, xlast = 0.0;
                bool any = false;
                double rv = lane < cnt ? rs[lane] : 0.0, xv = lane < cnt ? xs[lane] : 0.0;
                for (int k0 = 0; k0 < cnt; k0 += 32) {
                    const int k = k0 + lane, kn = k + 32;
                    const double rv_n = kn < cnt ? rs[kn] : 0.0, xv_n = kn < cnt ? xs[kn] : 0.0;  // prefetch
                    const double xprev = __shfl_up_sync(0xffffffffu, xv, 1);
                    any |= __any_sync(0xffffffffu, k < cnt && k > 0 && xv != (lane ? xprev : xlast));
                    const double r2 = __dmul_rn(rv, rv);
                    double myc = 0.0, myq = 0.0;
                    const int lim = min(32, cnt - k0);
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        if (i >= lim) break;
                        const double r = __shfl_sync(0xffffffffu, rv, i), rr = __shfl_sync(0xffffffffu, r2, i);
                        if (k0 + i == 0) {  // np.cumsum's first element is the value itself (-0.0 kept)
                            c = r;
                            qq = rr;
                        } else {
                            c = __dadd_rn(c, r);
                            qq = __dadd_rn(qq, rr);
                        }
                        if (lane == i) {
                            myc = c;
                            myq = qq;
                        }
                    }
                    if (k < cnt) {
                        cs[k] = myc;
                        cq[k] = myq;
                    }
                    xlast = __shfl_sync(0xffffffffu, xv, 31);
                    rv = rv_n;
                    xv = xv_n;
                }
                if (lane == 0) feat_have[li][f] = any;
            }
            __syncthreads();
            // ... and the gains at every boundary + first-maximum argmax, one warp per pair
            for (int pair = warp; pair < (le - lb) * n; pair += kFitWarps) {
                const int li = pair / n, f = pair - li * n, q = lb + li;
                if (!node_try[li] || !feat_have[li][f]) continue;
                const int off = nodes[q].off, cnt = nodes[q].cnt;
                const double* xs = a.xs + int64_t(f) * m + off;
                const double* cs = a.csum + int64_t(f) * m + off;
                const double* cq = a.csq + int64_t(f) * m + off;
                const double total = cs[cnt - 1], total_sq = cq[cnt - 1];
                const double parent_sse = __dsub_rn(total_sq, __ddiv_rn(__dmul_rn(total, total), double(cnt)));
                double gb = 0.0;
                int64_t ib = -1;
                for (int b = lane; b + 1 < cnt; b += 32) {
                    if (!(xs[b] != xs[b + 1])) continue;
                    const double ln = double(b + 1), rn = double(cnt - (b + 1));
                    const double ls = cs[b], lq = cq[b];
                    const double sse_left = __dsub_rn(lq, __ddiv_rn(__dmul_rn(ls, ls), ln));
                    const double dd = __dsub_rn(total, ls);
                    const double sse_right = __dsub_rn(__dsub_rn(total_sq, lq), __ddiv_rn(__dmul_rn(dd, dd), rn));
                    const double gain = __dsub_rn(__dsub_rn(parent_sse, sse_left), sse_right);
                    if (argmax_better(gain, b, gb, ib)) {
                        gb = gain;
                        ib = b;
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const double g2 = __shfl_xor_sync(0xffffffffu, gb, o);
                    const int64_t i2 = __shfl_xor_sync(0xffffffffu, ib, o);
                    if (argmax_better(g2, i2, gb, ib)) {
                        gb = g2;
                        ib = i2;
                    }
                }
                if (lane == 0) {
                    feat_gain[li][f] = gb;
                    feat_thr[li][f] = __ddiv_rn(__dadd_rn(xs[ib], xs[ib + 1]), 2.0);
                }
            }
            __syncthreads();
            // ---- per node: lowest feature unless a later one is strictly better; leaves update pred
            for (int q = lb + warp; q < le; q += kFitWarps) {
                const int li = q - lb, off = nodes[q].off, cnt = nodes[q].cnt;
                const int32_t* rows = rows_d + off;
                if (lane == 0) {
                    int bf = -1;
                    double bg = 0.0, bt = 0.0;
                    if (node_try[li])
                        for (int j = 0; j < n; ++j)
                            if (feat_have[li][j] && (bf < 0 || feat_gain[li][j] > bg)) {
                                bf = j;
                                bg = feat_gain[li][j];
                                bt = feat_thr[li][j];
                            }
                    node_split[li] = bf;
                    nodes[q].feature = bf;
                    nodes[q].thr = bf >= 0 ? bt : 0.0;
                    if (bf >= 0) nodes[q].value = 0.0;
                }
                __syncwarp();
                if (node_split[li] < 0) {  // leaf: pred += its value for the rows it owns
                    const double v = nodes[q].value;
                    for (int i = lane; i < cnt; i += 32) {
                        const int r = rows[i];
                        a.pred[r] = __dadd_rn(a.pred[r], v);
                    }
                }
            }
            __syncthreads();
            if (d == a.depth) break;
            // ---- children (BFS ids in parent order, left first) and stable partitions
            if (tid == 0) {
                int nn = n_nodes;
                for (int q = lb; q < le; ++q)
                    if (nodes[q].feature >= 0) {
                        nodes[q].lchild = nn++;
                        nodes[q].rchild = nn++;
                    }
                level_begin[d + 2] = nn;
                n_nodes = nn;
            }
            __syncthreads();
            int32_t* rows_n = a.lvl_rows + int64_t(d + 1) * m;
            int32_t* ord_n = a.lvl_ord + int64_t(d + 1) * n * m;
            for (int q = lb + warp; q < le; q += kFitWarps) {
                const int j = nodes[q].feature;
                if (j < 0) continue;
                const int off = nodes[q].off, cnt = nodes[q].cnt;
                const double t = nodes[q].thr;
                // left flags + stable compaction of the rows (left part first)
                int nl = 0;
                for (int i0 = 0; i0 < cnt; i0 += 32) {
                    const int i = i0 + lane;
                    bool lft = false;
                    if (i < cnt) {
                        const int r = rows_d[off + i];
                        lft = a.X[int64_t(r) * n + j] <= t;
                        a.in_left[r] = lft;
                    }
                    nl += __popc(__ballot_sync(0xffffffffu, lft));
                }
                __syncwarp();
                const int nordered = d + 1 < a.depth ? n : 0;  // children at max depth are leaves
                for (int f = -1; f < nordered; ++f) {
                    const int32_t* src = f < 0 ? rows_d + off : ord_d + int64_t(f) * m + off;
                    int32_t* dst = f < 0 ? rows_n + off : ord_n + int64_t(f) * m + off;
                    int li2 = 0, ri2 = nl;
                    for (int i0 = 0; i0 < cnt; i0 += 32) {
                        const int i = i0 + lane;
                        const int r = i < cnt ? src[i] : 0;
                        const bool lft = i < cnt && a.in_left[r];
                        const unsigned bl = __ballot_sync(0xffffffffu, lft);
                        const unsigned br = __ballot_sync(0xffffffffu, i < cnt && !lft);
                        const unsigned below = (1u << lane) - 1u;
                        if (i < cnt) dst[lft ? li2 + __popc(bl & below) : ri2 + __popc(br & below)] = r;
                        li2 += __popc(bl);
                        ri2 += __popc(br);
                    }
                }
                __syncwarp();
                if (lane == 0) {
                    FitNode& L = nodes[nodes[q].lchild];
                    FitNode& R = nodes[nodes[q].rchild];
                    L.off = off, L.cnt = nl;
                    R.off = off + nl, R.cnt = cnt - nl;
                }
            }
            __syncthreads();
        }
        // ---- preorder numbering (the reference's recursive _Builder order) and output
        if (tid == 0) {
            int stack[kFitMaxDepth + 2];
            int sp = 0, next = 0;
            stack[sp++] = 0;
            while (sp) {
                const int q = stack[--sp];
                preorder[q] = next++;
                if (nodes[q].feature >= 0) {
                    stack[sp++] = nodes[q].rchild;
                    stack[sp++] = nodes[q].lchild;
                }
            }
            a.tree_offsets[round] = used;
        }
        __syncthreads();
        const int nn = n_nodes;
        for (int q = tid; q < nn; q += blockDim.x) {
            const int o = used + preorder[q];
            const bool split = nodes[q].feature >= 0;
            a.feature[o] = nodes[q].feature;
            a.threshold[o] = nodes[q].thr;
            a.left[o] = split ? preorder[nodes[q].lchild] : -1;  // tree-local node ids
            a.right[o] = split ? preorder[nodes[q].rchild] : -1;
            a.value[o] = nodes[q].value;
        }
        __syncthreads();
        if (tid == 0) used += nn;
        __syncthreads();
    }
    if (tid == 0) a.tree_offsets[a.rounds] = used;
}

// Shared-memory engine (the tuning loop's sizes: m <= ~1300 rows): the training matrix
// (feature-major), residuals, predictions and two levels of row / per-feature orders (uint16)
// live in shared memory for the whole boosting loop, so every phase is on-chip.  The split
// scan of a (node, feature) is one warp: pass 1 runs the cumsum chain for the totals, pass 2
// runs it again with every lane keeping the prefix at its own position and evaluating the gain
// there (boundaries in parallel), then a first-maximum argmax across the warp.
__host__ __device__ inline size_t fit_smem_bytes(int64_t m, int n) {
    return size_t(2) * n * m * 8 + size_t(m) * 8 * 2 + size_t(2) * m * 2 + size_t(2) * n * m * 2 + size_t(n) * m * 2 +
           size_t(m) + 64;
}

__global__ void __launch_bounds__(kFitThreads, 1) fit_smem_kernel(FitDevArgs a) {
    extern __shared__ __align__(16) unsigned char fs_dyn[];
    __shared__ FitNode nodes[kFitMaxNodes];
    __shared__ int level_begin[kFitMaxDepth + 2];
    __shared__ int n_nodes;
    __shared__ double feat_gain[kFitMaxLevel][kMaxKnobs];
    __shared__ double feat_thr[kFitMaxLevel][kMaxKnobs];
    __shared__ uint8_t feat_have[kFitMaxLevel][kMaxKnobs];
    __shared__ uint8_t node_try[kFitMaxLevel];
    __shared__ int preorder[kFitMaxNodes];
    __shared__ int used;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int m = int(a.m), n = a.n;
    double* csum = reinterpret_cast<double*>(fs_dyn);     // [n][m] np.cumsum(rs) per (node, feature) segment
    double* csq = csum + size_t(n) * m;                    // [n][m] np.cumsum(rs * rs)
    double* resid = csq + size_t(n) * m;                   // [m]
    double* pred = resid + m;                              // [m]
    uint16_t* rows2 = reinterpret_cast<uint16_t*>(pred + m);  // [2][m]
    uint16_t* ord2 = rows2 + 2 * m;                        // [2][n][m]
    uint16_t* codes = ord2 + size_t(2) * n * m;            // [n][m] value ranks: boundary tests on chip
    uint8_t* in_left = reinterpret_cast<uint8_t*>(codes + size_t(n) * m);
    const double* Xg = a.xs;  // feature-major copy in global memory (L2-resident), [n][m]
    for (int i = tid; i < n * m; i += blockDim.x) {
        const int f = i / m, r = i - f * m;
        a.xs[i] = a.X[int64_t(r) * n + f];
    }
    for (int i = tid; i < m; i += blockDim.x) pred[i] = a.base;
    for (int i = tid; i < n * m; i += blockDim.x) codes[i] = a.codes[i];
    if (tid == 0) used = 0;
    __syncthreads();
    for (int round = 0; round < a.rounds; ++round) {
        for (int i = tid; i < m; i += blockDim.x) {
            resid[i] = __dsub_rn(a.y[i], pred[i]);
            rows2[i] = uint16_t(i);
        }
        for (int i = tid; i < n * m; i += blockDim.x) ord2[i] = uint16_t(a.root_ord[i]);
        if (tid == 0) {
            nodes[0].off = 0;
            nodes[0].cnt = m;
            n_nodes = 1;
            level_begin[0] = 0;
            level_begin[1] = 1;
        }
        __syncthreads();
        for (int d = 0; d <= a.depth; ++d) {
            const int lb = level_begin[d], le = level_begin[d + 1];
            const uint16_t* rows_d = rows2 + (d & 1) * m;
            const uint16_t* ord_d = ord2 + size_t(d & 1) * n * m;
            // ---- node statistics: mean, SSE (numpy pairwise order), split candidacy
            for (int q = lb + warp; q < le; q += kFitWarps) {
                const int off = nodes[q].off, cnt = nodes[q].cnt, li = q - lb;
                const uint16_t* rows = rows_d + off;
                const double mean = __ddiv_rn(pw_sum_warp([&](int i) { return resid[rows[i]]; }, cnt), double(cnt));
                const double sse = pw_sum_warp(
                    [&](int i) {
                        const double dd = __dsub_rn(resid[rows[i]], mean);
                        return __dmul_rn(dd, dd);
                    },
                    cnt);
                if (lane == 0) {
                    node_try[li] = d < a.depth && sse > 0.0;
                    nodes[q].value = __dmul_rn(a.lr, mean);
                    nodes[q].feature = -1;
                    nodes[q].thr = 0.0;
                    nodes[q].lchild = nodes[q].rchild = -1;
                }
            }
            __syncthreads();
            // ---- split scans (_best_split): the cumsum chains, one thread per (candidate node,
            // feature), prefixes kept in shared memory ...
            for (int pair = tid; pair < (le - lb) * n; pair += blockDim.x) {
                const int li = pair / n, f = pair - li * n, q = lb + li;
                if (!node_try[li]) continue;
                const int off = nodes[q].off, cnt = nodes[q].cnt;
                const uint16_t* __restrict__ o = ord_d + size_t(f) * m + off;
                double* __restrict__ cs = csum + size_t(f) * m + off;
                double* __restrict__ cq = csq + size_t(f) * m + off;
                const double* __restrict__ rsd = resid;
                double c = rsd[o[0]];
                double qq = __dmul_rn(c, c);
                cs[0] = c;
                cq[0] = qq;
                // the residuals of 8 positions are gathered before their 8 chain steps, so the
                // two dependent shared-memory loads per element overlap the float64 add chain
                int kk = 1;
                for (; kk + 8 <= cnt; kk += 8) {
                    double rv[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) rv[u] = rsd[o[kk + u]];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        c = __dadd_rn(c, rv[u]);
                        qq = __dadd_rn(qq, __dmul_rn(rv[u], rv[u]));
                        cs[kk + u] = c;
                        cq[kk + u] = qq;
                    }
                }
                for (; kk < cnt; ++kk) {
                    const double rv = rsd[o[kk]];
                    c = __dadd_rn(c, rv);
                    qq = __dadd_rn(qq, __dmul_rn(rv, rv));
                    cs[kk] = c;
                    cq[kk] = qq;
                }
            }
            __syncthreads();
            // ... then the gains at every boundary in parallel + first-maximum argmax, a warp per pair
            for (int pair = warp; pair < (le - lb) * n; pair += kFitWarps) {
                const int li = pair / n, f = pair - li * n, q = lb + li;
                if (!node_try[li]) {
                    if (lane == 0) feat_have[li][f] = 0;
                    continue;
                }
                const int off = nodes[q].off, cnt = nodes[q].cnt;
                const uint16_t* o = ord_d + size_t(f) * m + off;
                const double* cs = csum + size_t(f) * m + off;
                const double* cq = csq + size_t(f) * m + off;
                const double* xf = Xg + size_t(f) * m;
                const uint16_t* cf = codes + size_t(f) * m;
                const double total = cs[cnt - 1], total_sq = cq[cnt - 1];
                const double parent_sse = __dsub_rn(total_sq, __ddiv_rn(__dmul_rn(total, total), double(cnt)));
                double gb = 0.0, tb = 0.0;
                int64_t ib = -1;
                bool any = false;
                for (int kk = lane; kk + 1 < cnt; kk += 32) {
                    if (cf[o[kk]] == cf[o[kk + 1]]) continue;  // equal values (distinct values have distinct ranks)
                    any = true;
                    const double ln = double(kk + 1), rn = double(cnt - (kk + 1));
                    const double ls = cs[kk], lq = cq[kk];
                    const double sse_left = __dsub_rn(lq, __ddiv_rn(__dmul_rn(ls, ls), ln));
                    const double dd = __dsub_rn(total, ls);
                    const double sse_right = __dsub_rn(__dsub_rn(total_sq, lq), __ddiv_rn(__dmul_rn(dd, dd), rn));
                    const double gain = __dsub_rn(__dsub_rn(parent_sse, sse_left), sse_right);
                    if (argmax_better(gain, kk, gb, ib)) {
                        gb = gain;
                        ib = kk;
                    }
                }
                any = __any_sync(0xffffffffu, any);
#pragma unroll
                for (int s2 = 16; s2 > 0; s2 >>= 1) {
                    const double g2 = __shfl_xor_sync(0xffffffffu, gb, s2);
                    const int64_t i2 = __shfl_xor_sync(0xffffffffu, ib, s2);
                    if (argmax_better(g2, i2, gb, ib)) {
                        gb = g2;
                        ib = i2;
                    }
                }
                if (lane == 0) {
                    feat_have[li][f] = any;
                    feat_gain[li][f] = gb;
                    // the winning boundary's midpoint (float64 values from the global copy)
                    if (any) tb = __ddiv_rn(__dadd_rn(xf[o[ib]], xf[o[ib + 1]]), 2.0);
                    feat_thr[li][f] = tb;
                }
            }
            __syncthreads();
            // ---- per node: lowest feature unless a later one is strictly better; leaves update pred
            for (int q = lb + warp; q < le; q += kFitWarps) {
                const int li = q - lb, off = nodes[q].off, cnt = nodes[q].cnt;
                int bf = -1;
                double bg = 0.0, bt = 0.0;
                if (node_try[li])
                    for (int j = 0; j < n; ++j)
                        if (feat_have[li][j] && (bf < 0 || feat_gain[li][j] > bg)) {
                            bf = j;
                            bg = feat_gain[li][j];
                            bt = feat_thr[li][j];
                        }
                __syncwarp();
                if (lane == 0 && bf >= 0) {
                    nodes[q].feature = bf;
                    nodes[q].thr = bt;
                    nodes[q].value = 0.0;
                }
                if (bf < 0) {
                    const double v = nodes[q].value;
                    for (int i = lane; i < cnt; i += 32) {
                        const int r = rows_d[off + i];
                        pred[r] = __dadd_rn(pred[r], v);
                    }
                }
            }
            __syncthreads();
            if (d == a.depth) break;
            if (tid == 0) {
                int nn = n_nodes;
                for (int q = lb; q < le; ++q)
                    if (nodes[q].feature >= 0) {
                        nodes[q].lchild = nn++;
                        nodes[q].rchild = nn++;
                    }
                level_begin[d + 2] = nn;
                n_nodes = nn;
            }
            __syncthreads();
            // ---- stable partitions into the other level buffers (left part first): the left
            // flags and counts per split node (a warp per node), then every (node, array) pair —
            // the rows and each feature's order — partitioned by its own warp
            uint16_t* rows_n = rows2 + ((d + 1) & 1) * m;
            uint16_t* ord_n = ord2 + size_t((d + 1) & 1) * n * m;
            for (int q = lb + warp; q < le; q += kFitWarps) {
                const int j = nodes[q].feature;
                if (j < 0) continue;
                const int off = nodes[q].off, cnt = nodes[q].cnt;
                const double t = nodes[q].thr;
                const double* xj = Xg + size_t(j) * m;
                int nl = 0;
                for (int i0 = 0; i0 < cnt; i0 += 32) {
                    const int i = i0 + lane;
                    bool lft = false;
                    if (i < cnt) {
                        const int r = rows_d[off + i];
                        lft = xj[r] <= t;
                        in_left[r] = lft;
                    }
                    nl += __popc(__ballot_sync(0xffffffffu, lft));
                }
                if (lane == 0) {
                    FitNode& L = nodes[nodes[q].lchild];
                    FitNode& R = nodes[nodes[q].rchild];
                    L.off = off, L.cnt = nl;
                    R.off = off + nl, R.cnt = cnt - nl;
                }
            }
            __syncthreads();
            const int narr = 1 + (d + 1 < a.depth ? n : 0);  // children at max depth are leaves: no orders
            for (int pair = warp; pair < (le - lb) * narr; pair += kFitWarps) {
                const int q = lb + pair / narr, f = pair % narr - 1;
                if (nodes[q].feature < 0) continue;
                const int off = nodes[q].off, cnt = nodes[q].cnt, nl = nodes[nodes[q].lchild].cnt;
                const uint16_t* src = f < 0 ? rows_d + off : ord_d + size_t(f) * m + off;
                uint16_t* dst = f < 0 ? rows_n + off : ord_n + size_t(f) * m + off;
                int li2 = 0, ri2 = nl;
                for (int i0 = 0; i0 < cnt; i0 += 32) {
                    const int i = i0 + lane;
                    const int r = i < cnt ? src[i] : 0;
                    const bool lft = i < cnt && in_left[r];
                    const unsigned bl = __ballot_sync(0xffffffffu, lft);
                    const unsigned br = __ballot_sync(0xffffffffu, i < cnt && !lft);
                    const unsigned below = (1u << lane) - 1u;
                    if (i < cnt) dst[lft ? li2 + __popc(bl & below) : ri2 + __popc(br & below)] = uint16_t(r);
                    li2 += __popc(bl);
                    ri2 += __popc(br);
                }
            }
            __syncthreads();
        }
        if (tid == 0) {
            int stack[kFitMaxDepth + 2];
            int sp = 0, next = 0;
            stack[sp++] = 0;
            while (sp) {
                const int q = stack[--sp];
                preorder[q] = next++;
                if (nodes[q].feature >= 0) {
                    stack[sp++] = nodes[q].rchild;
                    stack[sp++] = nodes[q].lchild;
                }
            }
            a.tree_offsets[round] = used;
        }
        __syncthreads();
        const int nn = n_nodes;
        for (int q = tid; q < nn; q += blockDim.x) {
            const int o = used + preorder[q];
            const bool split = nodes[q].feature >= 0;
            a.feature[o] = nodes[q].feature;
            a.threshold[o] = nodes[q].thr;
            a.left[o] = split ? preorder[nodes[q].lchild] : -1;
            a.right[o] = split ? preorder[nodes[q].rchild] : -1;
            a.value[o] = nodes[q].value;
        }
        __syncthreads();
        if (tid == 0) used += nn;
        __syncthreads();
    }
    if (tid == 0) a.tree_offsets[a.rounds] = used;
}

}  // namespace kt

namespace kt {
namespace {
// Validation + canonical order (np.lexsort((targets, f_{n-1}, ..., f_0))) + per-feature stable
// argsorts, shared by the host and device engines.
struct Canonical {
    std::vector<double> X, y;
    std::vector<std::vector<int64_t>> root;
    double base = 0.0;
};
Canonical canonical(const double* features, const double* targets, int64_t m, int n, int rounds, int depth,
                    double learning_rate) {
    if (m < 1) fail(KT_ERR_VALUE, "training set is empty");
    if (n < 1) fail(KT_ERR_VALUE, "training set needs at least one feature");
    if (rounds < 1) fail(KT_ERR_VALUE, "rounds must be >= 1, got " + std::to_string(rounds));
    if (depth < 1) fail(KT_ERR_VALUE, "depth must be >= 1, got " + std::to_string(depth));
    if (!(learning_rate > 0.0 && learning_rate <= 1.0)) fail(KT_ERR_VALUE, "learning_rate must be in (0, 1]");
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
    Canonical c;
    c.X.resize(static_cast<size_t>(m) * n);
    c.y.resize(static_cast<size_t>(m));
    for (int64_t i = 0; i < m; ++i) {
        std::memcpy(&c.X[size_t(i) * n], features + size_t(order[i]) * n, sizeof(double) * n);
        c.y[i] = targets[order[i]];
    }
    c.base = pw_sum(c.y.data(), m) / double(m);
    std::vector<int64_t> all_rows(static_cast<size_t>(m));
    std::iota(all_rows.begin(), all_rows.end(), 0);
    c.root.assign(n, all_rows);
    for (int j = 0; j < n; ++j)
        std::stable_sort(c.root[j].begin(), c.root[j].end(),
                         [&](int64_t a, int64_t b) { return c.X[size_t(a) * n + j] < c.X[size_t(b) * n + j]; });
    return c;
}
}  // namespace
}  // namespace kt

extern "C" int kt_fit_trees(const double* features, const double* targets, int64_t m, int n, int rounds, int depth,
                            double learning_rate, int32_t* feature_out, double* threshold_out, int32_t* left_out,
                            int32_t* right_out, double* value_out, int64_t node_capacity, int32_t* tree_offsets_out,
                            double* base_out) {
    KT_API_BEGIN
    using namespace kt;
    Canonical c = canonical(features, targets, m, n, rounds, depth, learning_rate);
    std::vector<double>& X = c.X;
    std::vector<double>& y = c.y;
    const double base = c.base;
    std::vector<double> pred(static_cast<size_t>(m), base);
    std::vector<std::vector<int64_t>>& root = c.root;
    (void)y;
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
        for (int64_t i = 0; i < m; ++i) g.resid[i] = c.y[i] - pred[i];
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

extern "C" int kt_fit_trees_device(kt_engine* e, const double* features, const double* targets, int64_t m, int n,
                                   int rounds, int depth, double learning_rate, int32_t* feature_out,
                                   double* threshold_out, int32_t* left_out, int32_t* right_out, double* value_out,
                                   int64_t node_capacity, int32_t* tree_offsets_out, double* base_out) {
    KT_API_BEGIN
    using namespace kt;
    Canonical c = canonical(features, targets, m, n, rounds, depth, learning_rate);
    if (depth > kFitMaxDepth) fail(KT_ERR_UNSUPPORTED, "device fit supports depth <= 7 (use kt_fit_trees)");
    if (n > kMaxKnobs) fail(KT_ERR_UNSUPPORTED, "device fit supports at most 8 features");
    if (m >= (int64_t(1) << 31)) fail(KT_ERR_UNSUPPORTED, "training set too large");
    const int64_t per_tree = (int64_t(1) << (depth + 1)) - 1;
    if (node_capacity < int64_t(rounds) * per_tree) fail(KT_ERR_VALUE, "node capacity below rounds * (2^(depth+1) - 1)");
    // one upload: X, y, root orders (int32); outputs come back in one copy
    const size_t xb = size_t(m) * n * 8, yb = size_t(m) * 8, ob = size_t(n) * m * 4;
    const size_t cap = size_t(rounds) * size_t(per_tree);
    const size_t outb = cap * (4 + 8 + 4 + 4 + 8) + size_t(rounds + 1) * 4 + 6 * 16;
    auto* h = static_cast<unsigned char*>(e->staging("fit.host", xb + yb + ob + size_t(n) * m * 2 + outb + 64));
    std::memcpy(h, c.X.data(), xb);
    std::memcpy(h + xb, c.y.data(), yb);
    auto* ho = reinterpret_cast<int32_t*>(h + xb + yb);
    for (int j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) ho[size_t(j) * m + i] = int32_t(c.root[j][i]);
    // value ranks per feature (walk each stable argsort; NaN-free inputs only — NaN compares unequal
    // to itself, which ranks cannot express, so such inputs take the global kernel)
    bool finite = m < 65536;
    for (size_t i = 0; i < c.X.size() && finite; ++i) finite = !std::isnan(c.X[i]);
    auto* hcodes = reinterpret_cast<uint16_t*>(ho + size_t(n) * m);
    if (finite)
        for (int j = 0; j < n; ++j) {
            int code = 0;
            for (int64_t i = 0; i < m; ++i) {
                const int64_t r = c.root[j][i];
                if (i && c.X[size_t(r) * n + j] != c.X[size_t(c.root[j][i - 1]) * n + j]) ++code;
                hcodes[size_t(j) * m + r] = uint16_t(code);
            }
        }
    const size_t cb = size_t(n) * m * 2;
    auto* d = static_cast<unsigned char*>(e->scratch("fit.in", xb + yb + ob + cb + 64));
    KT_CUDA(cudaMemcpyAsync(d, h, xb + yb + ob + cb, cudaMemcpyHostToDevice, e->stream));
    FitDevArgs a{};
    a.X = reinterpret_cast<const double*>(d);
    a.y = reinterpret_cast<const double*>(d + xb);
    a.root_ord = reinterpret_cast<const int32_t*>(d + xb + yb);
    a.codes = finite ? reinterpret_cast<const uint16_t*>(d + xb + yb + ob) : nullptr;
    a.m = m, a.n = n, a.rounds = rounds, a.depth = depth, a.lr = learning_rate, a.base = c.base;
    const size_t wb = size_t(depth + 1) * m * 4 + size_t(depth + 1) * n * m * 4 + size_t(m) * (8 * 3 + 1) +
                      size_t(4) * n * m * 8 + 10 * 16;
    auto* w = static_cast<unsigned char*>(e->scratch("fit.work", wb));
    size_t o = 0;
    auto take = [&](size_t bytes) { unsigned char* p = w + o; o += (bytes + 15) & ~size_t(15); return p; };
    a.lvl_rows = reinterpret_cast<int32_t*>(take(size_t(depth + 1) * m * 4));
    a.lvl_ord = reinterpret_cast<int32_t*>(take(size_t(depth + 1) * n * m * 4));
    a.resid = reinterpret_cast<double*>(take(size_t(m) * 8));
    a.pred = reinterpret_cast<double*>(take(size_t(m) * 8));
    a.buf = reinterpret_cast<double*>(take(size_t(m) * 8));
    a.in_left = take(size_t(m));
    a.xs = reinterpret_cast<double*>(take(size_t(n) * m * 8));
    a.rs = reinterpret_cast<double*>(take(size_t(n) * m * 8));
    a.csum = reinterpret_cast<double*>(take(size_t(n) * m * 8));
    a.csq = reinterpret_cast<double*>(take(size_t(n) * m * 8));
    auto* dout = static_cast<unsigned char*>(e->scratch("fit.out", outb + 64));
    size_t oo = 0;
    auto takeo = [&](size_t bytes) { unsigned char* p = dout + oo; oo += (bytes + 15) & ~size_t(15); return p; };
    a.feature = reinterpret_cast<int32_t*>(takeo(cap * 4));
    a.left = reinterpret_cast<int32_t*>(takeo(cap * 4));
    a.right = reinterpret_cast<int32_t*>(takeo(cap * 4));
    a.tree_offsets = reinterpret_cast<int32_t*>(takeo(size_t(rounds + 1) * 4));
    a.threshold = reinterpret_cast<double*>(takeo(cap * 8));
    a.value = reinterpret_cast<double*>(takeo(cap * 8));
    KT_CUDA(cudaMemsetAsync(dout, 0, oo, e->stream));  // read back whole: trees use <= the capacity
    const size_t smem = fit_smem_bytes(m, n);
    int optin = 0;
    KT_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, e->device));
    cudaFuncAttributes fa{};
    KT_CUDA(cudaFuncGetAttributes(&fa, (const void*)fit_smem_kernel));
    const bool on_chip = finite && smem + fa.sharedSizeBytes <= size_t(optin) && !std::getenv("KT_FIT_GLOBAL");
    e->pre_launch("fit_trees");
    if (on_chip) {
        allow_dynamic_smem((const void*)fit_smem_kernel);
        fit_smem_kernel<<<1, kFitThreads, smem, e->stream>>>(a);
    } else {
        fit_kernel<<<1, kFitThreads, 0, e->stream>>>(a);
    }
    e->check_launch("fit_trees");
    unsigned char* hout = h + xb + yb + ob + cb;
    KT_CUDA(cudaMemcpyAsync(hout, dout, oo, cudaMemcpyDeviceToHost, e->stream));
    e->sync();
    const int32_t* offs = reinterpret_cast<const int32_t*>(hout + (reinterpret_cast<unsigned char*>(a.tree_offsets) - dout));
    const int64_t used = offs[rounds];
    auto at = [&](const void* dp) { return hout + (static_cast<const unsigned char*>(dp) - dout); };
    std::memcpy(feature_out, at(a.feature), size_t(used) * 4);
    std::memcpy(left_out, at(a.left), size_t(used) * 4);
    std::memcpy(right_out, at(a.right), size_t(used) * 4);
    std::memcpy(threshold_out, at(a.threshold), size_t(used) * 8);
    std::memcpy(value_out, at(a.value), size_t(used) * 8);
    std::memcpy(tree_offsets_out, offs, size_t(rounds + 1) * 4);
    *base_out = c.base;
    KT_API_END
}
