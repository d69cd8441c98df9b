// pairwise.cu — see pairwise.cuh.
#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "pairwise.cuh"

namespace kt {

struct Builder {
    PairwiseTree& t;
    struct Tmp {
        int32_t l, r, h;
    };
    std::vector<Tmp> tmp;
    // returns encoded id: leaf -> (id), internal -> -(tmp index) - 1
    int64_t build(int64_t s, int64_t n, int* height) {
        if (n <= 128) {
            t.leaf_start.push_back(s);
            t.leaf_len.push_back(int32_t(n));
            *height = 0;
            return int64_t(t.leaf_start.size()) - 1;
        }
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        int hl, hr;
        int64_t a = build(s, n2, &hl);
        int64_t b = build(s + n2, n - n2, &hr);
        *height = 1 + std::max(hl, hr);
        tmp.push_back({int32_t(a), int32_t(b), *height});
        return -int64_t(tmp.size());
    }
};

std::shared_ptr<PairwiseTree> make_tree(int64_t m) {
    auto t = std::make_shared<PairwiseTree>();
    t->m = m;
    Builder b{*t, {}};
    int h;
    int64_t root = b.build(0, m, &h);
    const int L = int(t->leaf_start.size());
    // final ids: leaves 0..L-1; internal nodes L.. ordered by height
    const int I = int(b.tmp.size());
    std::vector<int> order(I);
    for (int i = 0; i < I; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return b.tmp[x].h < b.tmp[y].h; });
    std::vector<int> final_id(I);
    for (int i = 0; i < I; ++i) final_id[order[i]] = L + i;
    auto enc = [&](int64_t v) -> int32_t { return v >= 0 ? int32_t(v) : final_id[-v - 1]; };
    t->node_left.resize(I);
    t->node_right.resize(I);
    int cur_h = -1;
    for (int i = 0; i < I; ++i) {
        const auto& nd = b.tmp[order[i]];
        t->node_left[i] = enc(nd.l);
        t->node_right[i] = enc(nd.r);
        if (nd.h != cur_h) {
            t->level_start.push_back(i);
            cur_h = nd.h;
        }
    }
    t->level_start.push_back(I);
    t->n_levels = int(t->level_start.size()) - 1;
    t->root = enc(root);
    // one device allocation and one copy for the five arrays (a new length costs one cudaMalloc
    // and one synchronous copy instead of five each: the tuning loop's lengths change every round)
    const size_t o_len = size_t(std::max(1, L)) * 8, o_left = o_len + size_t(std::max(1, L)) * 4;
    const size_t o_right = o_left + size_t(std::max(1, I)) * 4, o_level = o_right + size_t(std::max(1, I)) * 4;
    const size_t total = o_level + t->level_start.size() * 4;
    std::vector<unsigned char> hb(total, 0);
    std::memcpy(hb.data(), t->leaf_start.data(), size_t(L) * 8);
    std::memcpy(hb.data() + o_len, t->leaf_len.data(), size_t(L) * 4);
    if (I) {
        std::memcpy(hb.data() + o_left, t->node_left.data(), size_t(I) * 4);
        std::memcpy(hb.data() + o_right, t->node_right.data(), size_t(I) * 4);
    }
    std::memcpy(hb.data() + o_level, t->level_start.data(), t->level_start.size() * 4);
    KT_CUDA(cudaMalloc(&t->d_block, total));
    KT_CUDA(cudaMemcpy(t->d_block, hb.data(), total, cudaMemcpyHostToDevice));
    auto* base = static_cast<unsigned char*>(t->d_block);
    t->d_leaf_start = reinterpret_cast<int64_t*>(base);
    t->d_leaf_len = reinterpret_cast<int32_t*>(base + o_len);
    t->d_left = reinterpret_cast<int32_t*>(base + o_left);
    t->d_right = reinterpret_cast<int32_t*>(base + o_right);
    t->d_level = reinterpret_cast<int32_t*>(base + o_level);
    return t;
}

// Shared by every engine of the process (shard threads run concurrently): the cache is
// locked, and callers hold a reference so an eviction never frees a tree in use.
static std::mutex g_trees_mu;
static std::map<std::pair<int, int64_t>, std::shared_ptr<PairwiseTree>> g_trees;

std::shared_ptr<const PairwiseTree> pairwise_tree(int device, int64_t m) {
    auto key = std::make_pair(device, m);
    std::lock_guard<std::mutex> lock(g_trees_mu);
    auto it = g_trees.find(key);
    if (it != g_trees.end()) return it->second;
    if (g_trees.size() > 64) g_trees.clear();
    auto t = make_tree(m);
    g_trees[key] = t;
    return t;
}

// ---------------------------------------------------------------- kernels
// One warp per leaf (<= 128 values): lanes evaluate the values into shared
// memory, lanes 0..7 run numpy's 8 strided accumulators in order, lane 0
// folds them as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) and adds the tail.
constexpr int kLeafWarps = 4;

template <class Value>
__device__ __forceinline__ void warp_leaf(int l, const int64_t* leaf_start, const int32_t* leaf_len, double* vals,
                                          double* buf, Value value) {
    const int lane = threadIdx.x & 31;
    const int64_t s = leaf_start[l];
    const int len = leaf_len[l];
    double v[4];  // a leaf holds <= 128 values: all four per lane in flight at once
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int i = lane + 32 * q;
        v[q] = i < len ? value(s + i) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
        if (lane + 32 * q < len) buf[lane + 32 * q] = v[q];
    __syncwarp();
    double r = 0.0;
    const int body = len - (len % 8);
    if (len >= 8 && lane < 8) {
        r = buf[lane];
        for (int i = 8 + lane; i < body; i += 8) r = __dadd_rn(r, buf[i]);
    }
    double r0 = __shfl_sync(0xffffffffu, r, 0), r1 = __shfl_sync(0xffffffffu, r, 1);
    double r2 = __shfl_sync(0xffffffffu, r, 2), r3 = __shfl_sync(0xffffffffu, r, 3);
    double r4 = __shfl_sync(0xffffffffu, r, 4), r5 = __shfl_sync(0xffffffffu, r, 5);
    double r6 = __shfl_sync(0xffffffffu, r, 6), r7 = __shfl_sync(0xffffffffu, r, 7);
    if (lane == 0) {
        double res;
        int i;
        if (len < 8) {
            res = 0.0;
            i = 0;
        } else {
            res = __dadd_rn(__dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3)), __dadd_rn(__dadd_rn(r4, r5), __dadd_rn(r6, r7)));
            i = body;
        }
        for (; i < len; ++i) res = __dadd_rn(res, buf[i]);
        vals[l] = res;
    }
}

// Run r = blockIdx.y: assignments assign + r * astride, centroids cent + coff[r] * 8, leaf
// values vals + r * vstride.
struct RunOffsets {
    int coff[kMaxLossRuns];
};
__global__ void __launch_bounds__(kLeafWarps * 32) loss_leaf_kernel(const uint64_t* __restrict__ pts,
                                                                    const uint8_t* __restrict__ assign, int64_t astride,
                                                                    const double* __restrict__ cent, RunOffsets ro,
                                                                    int n, const RowFmt fmt, const int64_t* leaf_start,
                                                                    const int32_t* leaf_len, int L, double* vals,
                                                                    int64_t vstride) {
    __shared__ double s_buf[kLeafWarps][128];
    const int w = threadIdx.x >> 5;
    const int l = blockIdx.x * kLeafWarps + w;
    if (l >= L) return;
    const int r = blockIdx.y;
    const uint8_t* as = assign + r * astride;
    const double* cr = cent + size_t(ro.coff[r]) * kMaxKnobs;
    warp_leaf(l, leaf_start, leaf_len, vals + r * vstride, s_buf[w],
              [&](int64_t p) { return np_sq_dist(pts[p], cr + int(as[p]) * kMaxKnobs, n, fmt); });
}

__global__ void __launch_bounds__(kLeafWarps * 32) array_leaf_kernel(const double* __restrict__ x,
                                                                     const double* center, const int64_t* leaf_start,
                                                                     const int32_t* leaf_len, int L, double* vals) {
    __shared__ double s_buf[kLeafWarps][128];
    const int w = threadIdx.x >> 5;
    const int l = blockIdx.x * kLeafWarps + w;
    if (l >= L) return;
    const double c = center ? *center : 0.0;
    const bool sq = center != nullptr;
    warp_leaf(l, leaf_start, leaf_len, vals, s_buf[w], [&](int64_t p) {
        const double a = x[p];
        if (!sq) return a;
        const double d = __dsub_rn(a, c);
        return __dmul_rn(d, d);
    });
}

__global__ void __launch_bounds__(1024) combine_kernel(double* vals, int L, const int32_t* left, const int32_t* right,
                                                       const int32_t* level_start, int n_levels, int root,
                                                       double* out, int64_t vstride) {
    vals += blockIdx.x * vstride;  // one block per independent sum
    out += blockIdx.x;
    for (int lv = 0; lv < n_levels; ++lv) {
        const int a = level_start[lv], b = level_start[lv + 1];
        for (int i = a + threadIdx.x; i < b; i += blockDim.x) vals[L + i] = __dadd_rn(vals[left[i]], vals[right[i]]);
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = vals[root];
}

// Same combine with the node values and the tree in shared memory (one block): a level
// costs a block barrier instead of a global-memory round trip (14 levels at 1M points).
__global__ void __launch_bounds__(1024) combine_smem_kernel(const double* __restrict__ vals, int L, int I,
                                                            const int32_t* __restrict__ left,
                                                            const int32_t* __restrict__ right,
                                                            const int32_t* __restrict__ level_start, int n_levels,
                                                            int root, double* out, int64_t vstride) {
    extern __shared__ double sv[];  // [L + I] values, then [I] left, [I] right, [n_levels + 1] level starts
    vals += blockIdx.x * vstride;  // one block per independent sum
    out += blockIdx.x;
    int32_t* sl = reinterpret_cast<int32_t*>(sv + L + I);
    int32_t* sr = sl + I;
    int32_t* slv = sr + I;
    for (int i = threadIdx.x; i < L; i += blockDim.x) sv[i] = vals[i];
    for (int i = threadIdx.x; i < I; i += blockDim.x) {
        sl[i] = left[i];
        sr[i] = right[i];
    }
    for (int i = threadIdx.x; i <= n_levels; i += blockDim.x) slv[i] = level_start[i];
    __syncthreads();
    for (int lv = 0; lv < n_levels; ++lv) {
        const int a = slv[lv], b = slv[lv + 1];
        for (int i = a + threadIdx.x; i < b; i += blockDim.x) sv[L + i] = __dadd_rn(sv[sl[i]], sv[sr[i]]);
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sv[root];
}

static void combine(kt_engine* e, const PairwiseTree& t, double* vals, double* out_dev, int nsums = 1,
                    int64_t vstride = 0) {
    const int L = int(t.leaf_start.size());
    const int I = int(t.node_left.size());
    const size_t smem = size_t(L + I) * 8 + size_t(I) * 8 + size_t(t.n_levels + 1) * 4;
    const int optin = smem_optin(e->device);
    e->pre_launch("pairwise_combine");
    if (smem <= size_t(optin)) {
        allow_dynamic_smem((const void*)combine_smem_kernel);
        combine_smem_kernel<<<nsums, 1024, smem, e->stream>>>(vals, L, I, t.d_left, t.d_right, t.d_level,
                                                             t.n_levels, t.root, out_dev, vstride);
    } else {
        combine_kernel<<<nsums, 1024, 0, e->stream>>>(vals, L, t.d_left, t.d_right, t.d_level, t.n_levels, t.root,
                                                      out_dev, vstride);
    }
    e->check_launch("pairwise_combine");
}

void pairwise_loss(kt_engine* e, const uint64_t* pts, int64_t m, int n, const RowFmt& fmt, const uint8_t* assign,
                   const double* cent, double* out_dev) {
    const int zero = 0;
    pairwise_loss_runs(e, pts, m, n, fmt, assign, 0, cent, &zero, 1, out_dev);
}

void pairwise_loss_runs(kt_engine* e, const uint64_t* pts, int64_t m, int n, const RowFmt& fmt, const uint8_t* assign,
                        int64_t astride, const double* cent, const int* coff, int R, double* out_dev) {
    if (R < 1 || R > kMaxLossRuns) fail(KT_ERR_VALUE, "pairwise_loss_runs: 1..8 runs");
    const auto tree = pairwise_tree(e->device, m);
    const PairwiseTree& t = *tree;
    const int L = int(t.leaf_start.size());
    const int64_t vstride = int64_t(L) + int64_t(t.node_left.size());
    auto* vals = static_cast<double*>(e->scratch("loss.vals", size_t(vstride) * R * 8));
    RunOffsets ro{};
    for (int r = 0; r < R; ++r) ro.coff[r] = coff[r];
    e->pre_launch("loss_leaf");
    loss_leaf_kernel<<<dim3(unsigned(ceil_div(L, kLeafWarps)), unsigned(R)), kLeafWarps * 32, 0, e->stream>>>(
        pts, assign, astride, cent, ro, n, fmt, t.d_leaf_start, t.d_leaf_len, L, vals, vstride);
    e->check_launch("loss_leaf");
    combine(e, t, vals, out_dev, R, vstride);
}

void pairwise_sum(kt_engine* e, const double* x, int64_t m, const double* center, double* out_dev) {
    const auto tree = pairwise_tree(e->device, m);
    const PairwiseTree& t = *tree;
    const int L = int(t.leaf_start.size());
    auto* vals = static_cast<double*>(e->scratch("psum.vals", size_t(L + t.node_left.size()) * 8));
    e->pre_launch("psum_leaf");
    array_leaf_kernel<<<int(ceil_div(L, kLeafWarps)), kLeafWarps * 32, 0, e->stream>>>(x, center, t.d_leaf_start,
                                                                                     t.d_leaf_len, L, vals);
    e->check_launch("psum_leaf");
    combine(e, t, vals, out_dev);
}

}  // namespace kt
