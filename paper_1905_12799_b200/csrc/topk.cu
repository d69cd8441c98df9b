// topk.cu — the non-adaptive arms' batch choice on the device.
//
// Reference: knobtuner/driver.py:101-115 (_top_unvisited): walk the trajectory's entries,
// keep the first occurrence of every configuration that is not visited, stable-sort them by
// -score (np.argsort(-scores, kind="stable")) and return the first `cap`.
//
// Device formulation (exact):
//   1. K6's hash table gives every row's first-occurrence index (dedup_table);
//   2. a candidate is a first occurrence whose row is not in the (sorted) visited rows;
//      its key is (score descending, entry index ascending) — the stable order of -score,
//      with -0.0 folded onto +0.0 since numpy's sort compares them equal;
//   3. each block keeps a running top-`cap` list: candidates that beat its current worst
//      entry are compacted into shared memory, and a bitonic sort of list + survivors keeps
//      the best `cap`; one final block sorts the per-block lists.
#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace kt {
namespace {

constexpr int kTopMax = 64;         // GREEDY_BATCH (driver.py:28)
constexpr int kTopThreads = 512;
constexpr int kTopBuf = 2048;       // survivors + current list, one bitonic sort
constexpr int kTopBlocks = 128;     // final sort: 128 x 64 entries

__device__ __forceinline__ unsigned long long score_key(double s) {
    if (s != s) return 0ull;  // NaN: numpy sorts it last (ties among NaNs by index)
    if (s == 0.0) s = 0.0;  // -0.0 == 0.0 for numpy's sort
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(s));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// a precedes b in the batch order
__device__ __forceinline__ bool before(unsigned long long ka, uint32_t ia, unsigned long long kb, uint32_t ib) {
    return ka > kb || (ka == kb && ia < ib);
}

// Bitonic sort of n (power of two) entries into batch order; sentinel = (0, UINT32_MAX).
__device__ void bitonic_sort(unsigned long long* key, uint32_t* idx, int n) {
    for (int size = 2; size <= n; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            __syncthreads();
            for (int t = threadIdx.x; t < n / 2; t += blockDim.x) {
                const int lo = 2 * t - (t & (stride - 1));
                const int hi = lo + stride;
                const bool up = (lo & size) == 0;  // this sub-sequence ascends in batch order
                const unsigned long long kl = key[lo], kh = key[hi];
                const uint32_t il = idx[lo], ih = idx[hi];
                if (before(kh, ih, kl, il) == up) {
                    key[lo] = kh;
                    key[hi] = kl;
                    idx[lo] = ih;
                    idx[hi] = il;
                }
            }
        }
    }
    __syncthreads();
}

__device__ __forceinline__ bool is_visited(const uint64_t* vis, int nv, uint64_t row) {
    int lo = 0, hi = nv;  // vis ascending
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const uint64_t v = __ldg(vis + mid);
        if (v < row) lo = mid + 1;
        else hi = mid;
    }
    return lo < nv && __ldg(vis + lo) == row;
}

__global__ void __launch_bounds__(kTopThreads) top_block_kernel(const uint64_t* __restrict__ rows,
                                                                const double* __restrict__ scores, int64_t count,
                                                                const uint32_t* __restrict__ first,
                                                                const uint32_t* __restrict__ slot,
                                                                const uint64_t* __restrict__ vis, int nv, int cap,
                                                                unsigned long long* out_key, uint32_t* out_idx) {
    __shared__ unsigned long long s_key[kTopBuf];
    __shared__ uint32_t s_idx[kTopBuf];
    __shared__ int s_n;       // entries in the buffer (list first, then survivors)
    __shared__ unsigned long long s_wk;  // current worst kept entry (valid when the list is full)
    __shared__ uint32_t s_wi;
    if (threadIdx.x == 0) {
        s_n = 0;
        s_wk = 0ull;
        s_wi = 0xffffffffu;
    }
    __syncthreads();
    const int64_t per_round = int64_t(gridDim.x) * blockDim.x;
    for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < count; base += per_round) {
        const int64_t i = base + threadIdx.x;
        if (i < count && __ldg(first + slot[i]) == uint32_t(i)) {
            const uint64_t row = rows[i];
            const unsigned long long k = score_key(scores[i]);
            const bool full = s_wi != 0xffffffffu;  // set (between barriers) once the list holds cap entries
            if ((!full || before(k, uint32_t(i), s_wk, s_wi)) && !is_visited(vis, nv, row)) {
                const int p = atomicAdd(&s_n, 1);
                s_key[p] = k;
                s_idx[p] = uint32_t(i);
            }
        }
        __syncthreads();
        // compact when the next round could overflow the buffer (or at the end)
        const bool last = base + per_round >= count;
        const int n = s_n;
        __syncthreads();  // every thread has read s_n before the next round appends to it
        if (n > kTopBuf - kTopThreads || (last && n > 0)) {
            for (int t = n + threadIdx.x; t < kTopBuf; t += blockDim.x) {
                s_key[t] = 0ull;
                s_idx[t] = 0xffffffffu;
            }
            bitonic_sort(s_key, s_idx, kTopBuf);
            if (threadIdx.x == 0) {
                s_n = min(n, cap);
                if (s_n == cap) {
                    s_wk = s_key[cap - 1];
                    s_wi = s_idx[cap - 1];
                }
            }
            __syncthreads();
        }
    }
    for (int t = threadIdx.x; t < cap; t += blockDim.x) {
        const bool ok = t < s_n;
        out_key[blockIdx.x * kTopMax + t] = ok ? s_key[t] : 0ull;
        out_idx[blockIdx.x * kTopMax + t] = ok ? s_idx[t] : 0xffffffffu;
    }
}

// One block: sort the per-block lists (blocks * kTopMax entries, power of two) and gather the rows.
__global__ void __launch_bounds__(1024) top_final_kernel(const unsigned long long* in_key, const uint32_t* in_idx,
                                                          int n, int blocks, int cap, const uint64_t* __restrict__ rows,
                                                          uint64_t* out_rows, int* out_n) {
    extern __shared__ __align__(16) unsigned char s_dyn[];
    auto* key = reinterpret_cast<unsigned long long*>(s_dyn);
    auto* idx = reinterpret_cast<uint32_t*>(key + n);
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
        const int b = t / kTopMax, j = t % kTopMax;
        const bool ok = b < blocks && j < cap;
        key[t] = ok ? in_key[t] : 0ull;
        idx[t] = ok ? in_idx[t] : 0xffffffffu;
    }
    bitonic_sort(key, idx, n);
    __shared__ int s_cnt;
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    if (threadIdx.x < cap && idx[threadIdx.x] != 0xffffffffu) {
        out_rows[threadIdx.x] = rows[idx[threadIdx.x]];
        atomicMax(&s_cnt, int(threadIdx.x) + 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) *out_n = s_cnt;
}

}  // namespace
}  // namespace kt

extern "C" {

int kt_top_unvisited(kt_engine* e, const uint64_t* rows_dev, const double* scores_dev, int64_t count,
                     const uint64_t* visited, int64_t n_visited, int cap, uint64_t* batch_out, int32_t* batch_len) {
    KT_API_BEGIN
    using namespace kt;
    *batch_len = 0;
    if (cap < 0 || cap > kTopMax) fail(KT_ERR_UNSUPPORTED, "top_unvisited supports cap <= 64");
    if (count <= 0 || cap == 0) return KT_OK;
    if (n_visited >= (int64_t(1) << 31)) fail(KT_ERR_UNSUPPORTED, "visited set too large");
    std::vector<uint64_t> vis(visited, visited + n_visited);
    std::sort(vis.begin(), vis.end());
    auto* d_vis = static_cast<uint64_t*>(e->scratch("top.visited", std::max<size_t>(vis.size(), 1) * 8));
    if (!vis.empty()) KT_CUDA(cudaMemcpyAsync(d_vis, vis.data(), vis.size() * 8, cudaMemcpyHostToDevice, e->stream));
    const uint32_t *first, *slot;
    dedup_table(e, rows_dev, count, &first, &slot);
    const int blocks = int(std::min<int64_t>(kTopBlocks, std::max<int64_t>(1, ceil_div(count, kTopThreads))));
    auto* bkey = static_cast<unsigned long long*>(e->scratch("top.key", size_t(kTopBlocks) * kTopMax * 8));
    auto* bidx = static_cast<uint32_t*>(e->scratch("top.idx", size_t(kTopBlocks) * kTopMax * 4));
    e->pre_launch("top_block");
    top_block_kernel<<<blocks, kTopThreads, 0, e->stream>>>(rows_dev, scores_dev, count, first, slot, d_vis,
                                                             int(vis.size()), cap, bkey, bidx);
    e->check_launch("top_block");
    int n = 64;
    while (n < blocks * kTopMax) n <<= 1;
    const size_t smem = size_t(n) * 12;
    allow_dynamic_smem((const void*)top_final_kernel);
    auto* d_out = static_cast<uint64_t*>(e->scratch("top.out", kTopMax * 8 + 8));
    int* d_n = reinterpret_cast<int*>(d_out + kTopMax);
    KT_CUDA(cudaMemsetAsync(d_out, 0, kTopMax * 8 + 8, e->stream));  // read back whole (initcheck-clean)
    e->pre_launch("top_final");
    top_final_kernel<<<1, 1024, smem, e->stream>>>(bkey, bidx, n, blocks, cap, rows_dev, d_out, d_n);
    e->check_launch("top_final");
    auto* h = static_cast<uint64_t*>(e->staging("top.out", kTopMax * 8 + 8));
    KT_CUDA(cudaMemcpyAsync(h, d_out, kTopMax * 8 + 8, cudaMemcpyDeviceToHost, e->stream));
    e->sync();
    int len;
    std::memcpy(&len, h + kTopMax, 4);
    std::memcpy(batch_out, h, size_t(len) * 8);
    *batch_len = len;
    KT_API_END
}

}  // extern "C"
