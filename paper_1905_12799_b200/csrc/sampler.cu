// sampler.cu — adaptive sampling on the device: K6 dedup, K9 mode vote,
// K7 k-means++ init, K8 multi-k Lloyd, pairwise loss, knee scan, batch assembly.
//
// Reference: knobtuner/sampler.py (dedup :187-192, _plus_plus_init :56-69,
// kmeans :72-122, knee_scan :125-148, mode_config :151-158,
// round_to_config :161-170, adaptive_sample :173-215).
//
// Exactness strategy (the parity contract is bit-exact k, assignments, batch):
//   * dedup / mode vote are integer work;
//   * k-means++ weights are squared distances between lattice points, i.e.
//     integers, so cumsum / total / searchsorted are done exactly in int64;
//     the only float op is u * total, done in IEEE double like numpy;
//   * centroids are mean = (exact int64 sum) / count in IEEE double, which is
//     what numpy's mean of integer-valued float64 rows rounds to;
//   * assignment: a fast fp32 argmin with a proven error bound; any point whose
//     best/second-best gap is inside the bound is re-evaluated with the
//     reference's own float64 expression (numpy pairwise order, no FMA);
//   * the loss is numpy's pairwise sum over points, reproduced with the same
//     128-element blocks, 8 accumulators and split points.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <map>
#include <memory>
#include <unordered_set>
#include <vector>

#include "common.cuh"
#include "pairwise.cuh"
#include "rng.cuh"

namespace cg = cooperative_groups;

namespace kt {

// ============================================================== dedup (K6)
constexpr int kDedupRowsPerBlock = 1024;  // 256 threads x 4

__global__ void dedup_insert_kernel(const uint64_t* __restrict__ rows, int64_t count, uint64_t* keys,
                                    uint32_t* first, uint64_t mask, uint32_t* __restrict__ slot) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x) {
        const uint64_t key = rows[i];
        uint64_t h = mix64(key) & mask;
        while (true) {
            uint64_t cur = keys[h];
            if (cur == kEmptyRow) {
                cur = atomicCAS((unsigned long long*)&keys[h], (unsigned long long)kEmptyRow, (unsigned long long)key);
                if (cur == kEmptyRow) cur = key;
            }
            if (cur == key) {
                atomicMin(&first[h], uint32_t(i));
                slot[i] = uint32_t(h);  // the flag pass reads first[slot[i]] without probing again
                break;
            }
            h = (h + 1) & mask;
        }
    }
}

// One block = 1024 rows: ballot bitmask of first occurrences + block count.
__global__ void __launch_bounds__(256) dedup_flag_kernel(const uint32_t* __restrict__ slot, int64_t count,
                                                         const uint32_t* first, uint32_t* bits,
                                                         int64_t* block_counts) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t base = int64_t(blockIdx.x) * kDedupRowsPerBlock;
    int local = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int64_t w0 = base + j * 256 + warp * 32;
        const int64_t i = w0 + lane;
        bool is_first = false;
        if (i < count) is_first = __ldcg(first + slot[i]) == uint32_t(i);
        uint32_t b = __ballot_sync(0xffffffffu, is_first);
        if (lane == 0 && w0 < count) bits[w0 >> 5] = b;
        local += __popc(b);
    }
    __shared__ int s_cnt[8];
    if (lane == 0) s_cnt[warp] = local;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t t = 0;
        for (int w = 0; w < 8; ++w) t += s_cnt[w];
        block_counts[blockIdx.x] = t;
    }
}

// Exclusive scan of up to ~16M/1024 block counts in one block; total -> out[n].
__global__ void __launch_bounds__(1024) exclusive_scan_kernel(const int64_t* in, int64_t* out, int n) {
    __shared__ int64_t s_part[1024];
    const int per = (n + blockDim.x - 1) / blockDim.x;
    const int lo = min(n, int(threadIdx.x) * per), hi = min(n, lo + per);
    int64_t sum = 0;
    for (int i = lo; i < hi; ++i) sum += in[i];
    s_part[threadIdx.x] = sum;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
        int64_t v = threadIdx.x >= off ? s_part[threadIdx.x - off] : 0;
        __syncthreads();
        s_part[threadIdx.x] += v;
        __syncthreads();
    }
    int64_t run = s_part[threadIdx.x] - sum;
    for (int i = lo; i < hi; ++i) {
        int64_t v = in[i];
        out[i] = run;
        run += v;
    }
    if (threadIdx.x == blockDim.x - 1) out[n] = s_part[threadIdx.x];
}

__global__ void __launch_bounds__(256) dedup_scatter_kernel(const uint64_t* __restrict__ rows, int64_t count,
                                                            const uint32_t* bits, const int64_t* offsets,
                                                            uint64_t* __restrict__ out) {
    __shared__ int s_prefix[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t base = int64_t(blockIdx.x) * kDedupRowsPerBlock;
    const int64_t nwords = (count + 31) >> 5;
    if (warp == 0) {
        const int64_t w = (base >> 5) + lane;
        int c = w < nwords ? __popc(bits[w]) : 0;
        int incl = c;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            int v = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += v;
        }
        s_prefix[lane] = incl - c;
    }
    __syncthreads();
    const int64_t off0 = offsets[blockIdx.x];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int word_in_block = j * 8 + warp;
        const int64_t i = base + int64_t(word_in_block) * 32 + lane;
        if (i >= count) continue;
        const uint32_t b = bits[i >> 5];
        if ((b >> lane) & 1u) out[off0 + s_prefix[word_in_block] + __popc(b & ((1u << lane) - 1u))] = rows[i];
    }
}

void exclusive_scan(kt_engine* e, const int64_t* in, int64_t* out, int n) {
    e->pre_launch("exclusive_scan");
    exclusive_scan_kernel<<<1, 1024, 0, e->stream>>>(in, out, n);
    e->check_launch("exclusive_scan");
}

static uint64_t table_capacity(int64_t count) {
    uint64_t cap = 1024;
    while (cap < uint64_t(count) * 2) cap <<= 1;
    return cap;
}

void dedup_table(kt_engine* e, const uint64_t* rows, int64_t count, const uint32_t** first_out,
                 const uint32_t** slot_out) {
    if (count >= (int64_t(1) << 31)) fail(KT_ERR_UNSUPPORTED, "dedup supports < 2^31 rows per call");
    const uint64_t cap = table_capacity(count);
    auto* keys = static_cast<uint64_t*>(e->scratch("dedup.keys", cap * 8));
    auto* first = static_cast<uint32_t*>(e->scratch("dedup.first", cap * 4));
    KT_CUDA(cudaMemsetAsync(keys, 0xff, cap * 8, e->stream));
    KT_CUDA(cudaMemsetAsync(first, 0xff, cap * 4, e->stream));
    int grid = int(std::min<int64_t>(ceil_div(count, 256), int64_t(e->num_sms) * 8));
    e->pre_launch("dedup_insert");
    auto* slot = static_cast<uint32_t*>(e->scratch("dedup.slot", size_t(count) * 4));
    dedup_insert_kernel<<<grid, 256, 0, e->stream>>>(rows, count, keys, first, cap - 1, slot);
    e->check_launch("dedup_insert");
    *first_out = first;
    *slot_out = slot;
}

int64_t dedup(kt_engine* e, const uint64_t* rows, int64_t count, uint64_t* out) {
    if (count <= 0) return 0;
    const uint32_t *first, *slot;
    dedup_table(e, rows, count, &first, &slot);
    const int nb = int(ceil_div(count, kDedupRowsPerBlock));
    auto* bits = static_cast<uint32_t*>(e->scratch("dedup.bits", size_t(ceil_div(count, 32)) * 4 + 128));
    auto* counts = static_cast<int64_t*>(e->scratch("dedup.counts", size_t(nb) * 8));
    auto* offsets = static_cast<int64_t*>(e->scratch("dedup.offsets", size_t(nb + 1) * 8));
    e->pre_launch("dedup_flag");
    dedup_flag_kernel<<<nb, 256, 0, e->stream>>>(slot, count, first, bits, counts);
    e->check_launch("dedup_flag");
    exclusive_scan(e, counts, offsets, nb);
    e->pre_launch("dedup_scatter");
    dedup_scatter_kernel<<<nb, 256, 0, e->stream>>>(rows, count, bits, offsets, out);
    e->check_launch("dedup_scatter");
    auto* h_total = static_cast<int64_t*>(e->staging("dedup.total", 8));
    e->d2h(h_total, offsets + nb, 8);
    e->sync();
    return *h_total;
}

// ============================================================== mode vote (K9)
// Per-knob histograms back to back: knob d's bins start at off[d] (off[n] bins in all).
struct ModeArgs {
    RowFmt fmt;
    int n;
    int off[kMaxKnobs + 1];
};

// Knobs with <= 32 settings are counted with one warp ballot per setting (lane v keeps setting
// v's running count in a register, flushed once per launch); wider knobs (tile_f / tile_y /
// tile_x: 80-84 settings) use shared-memory atomics, whose conflicts across 32 random rows over
// ~80 bins are rare.  (Per-row __match_any_sync aggregation: 38 us per 1M rows.)
__global__ void __launch_bounds__(256) mode_hist_kernel(const uint64_t* __restrict__ rows, int64_t count,
                                                        const ModeArgs a, unsigned int* __restrict__ hist) {
    extern __shared__ unsigned int s_hist[];
    const int n = a.n, bins = a.off[a.n];
    for (int i = threadIdx.x; i < bins; i += blockDim.x) s_hist[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    unsigned int acc[kMaxKnobs];
#pragma unroll
    for (int d = 0; d < kMaxKnobs; ++d) acc[d] = 0;
    const int64_t warps_total = int64_t(gridDim.x) * (blockDim.x >> 5);
    const int64_t gw = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    for (int64_t base = gw * 32; base < count; base += warps_total * 32) {
        const int64_t i = base + lane;
        const bool valid = i < count;
        const uint64_t row = valid ? rows[i] : 0ull;
#pragma unroll
        for (int d = 0; d < kMaxKnobs; ++d) {
            if (d >= n) break;
            const int c = a.off[d + 1] - a.off[d];
            const int v = a.fmt.get(row, d);
            if (c <= 32) {
                for (int u = 0; u < c; ++u) {
                    const unsigned b = __ballot_sync(0xffffffffu, valid && v == u);
                    if (lane == u) acc[d] += __popc(b);
                }
            } else if (valid) {
                atomicAdd(&s_hist[a.off[d] + v], 1u);
            }
        }
    }
#pragma unroll
    for (int d = 0; d < kMaxKnobs; ++d)
        if (d < n && a.off[d + 1] - a.off[d] <= 32 && lane < a.off[d + 1] - a.off[d] && acc[d])
            atomicAdd(&s_hist[a.off[d] + lane], acc[d]);
    __syncthreads();
    for (int i = threadIdx.x; i < bins; i += blockDim.x)
        if (s_hist[i]) atomicAdd(&hist[i], s_hist[i]);
}

// Histograms of every knob on the device, copied back asynchronously into a pinned staging
// buffer (read after the caller's next synchronisation): adaptive_sample enqueues this before
// its knee scan, so the mode vote costs no synchronisation of its own.
static const unsigned int* mode_hist_async(kt_engine* e, const uint64_t* rows, int64_t count, int n,
                                           const RowFmt& fmt, const int32_t* cards) {
    if (count <= 0) fail(KT_ERR_VALUE, "mode vote needs at least one row");
    if (count >= (int64_t(1) << 32)) fail(KT_ERR_UNSUPPORTED, "mode vote supports < 2^32 rows");
    ModeArgs a{};
    a.fmt = fmt;
    a.n = n;
    for (int d = 0; d < n; ++d) a.off[d + 1] = a.off[d] + cards[d];
    const int bins = a.off[n];
    const size_t smem = size_t(bins) * 4;
    if (smem > 200 * 1024) fail(KT_ERR_UNSUPPORTED, "mode vote supports at most 51200 knob settings in all");
    auto* hist = static_cast<unsigned int*>(e->scratch("mode.hist", smem));
    KT_CUDA(cudaMemsetAsync(hist, 0, smem, e->stream));
    allow_dynamic_smem((const void*)mode_hist_kernel);
    int grid = int(std::min<int64_t>(ceil_div(count, 256), int64_t(e->num_sms) * 4));
    e->pre_launch("mode_hist");
    mode_hist_kernel<<<grid, 256, smem, e->stream>>>(rows, count, a, hist);
    e->check_launch("mode_hist");
    auto* h = static_cast<unsigned int*>(e->staging("mode.hist", smem));
    e->d2h(h, hist, smem);
    return h;
}

// mode_config's per-knob argmax (ties -> smallest index) from a copied-back histogram
static void mode_from_hist(const unsigned int* h, int n, const int32_t* cards, int32_t* mode_out) {
    int off = 0;
    for (int d = 0; d < n; ++d) {
        const unsigned int* hd = h + off;
        int best = 0;
        for (int v = 1; v < cards[d]; ++v)
            if (hd[v] > hd[best]) best = v;  // ties -> smallest index
        mode_out[d] = best;
        off += cards[d];
    }
}

void mode_vote(kt_engine* e, const uint64_t* rows, int64_t count, int n, const RowFmt& fmt, const int32_t* cards,
               int32_t* mode_out) {
    const unsigned int* h = mode_hist_async(e, rows, count, n, fmt, cards);
    e->sync();
    mode_from_hist(h, n, cards, mode_out);
}

// ====================================================== k-means++ init (K7)
// One cooperative launch produces centroids j0..j1-1.  Per centroid: every
// block redundantly selects it (scan of the per-chunk weight sums, then of
// the chosen chunk's weights), then all blocks update their chunks'
// weights d2[p] = min(d2[p], |p - c_j|^2) and chunk sums.  Weights and sums
// are double-buffered by centroid parity, so one grid barrier per centroid
// suffices.  Everything is exact int64 except u * total (IEEE double, as numpy).
constexpr int kInitChunk = 4096;  // points per chunk (one block-scan of 256 threads x 16)
constexpr int kInitThreads = 256;

struct InitArgs {
    const uint64_t* pts;
    int64_t m;
    int n;
    RowFmt fmt;
    int j0, j1;
    int64_t first_idx;
    const double* uniforms;  // u_1, u_2, ... (random() draws after integers(0, m))
    uint64_t* cent_rows;
    int* d2[2];
    long long* sums[2];
    int nchunks;
    unsigned int* barrier;  // grid-barrier counter, zeroed before the launch
    int64_t per_block;      // resident kernel: points per block (P); sums are per sub-chunk
    int nsub;               // resident kernel: sub-chunks per block
    int sub;                // resident kernel: points per sub-chunk (multiple of 32, <= kInitFinPer * threads)
};

// Block-wide inclusive scan of one int64 per thread with one barrier: warp scans, warp
// totals through shared memory, every warp adds the totals of the warps before it.
// Returns the thread's exclusive prefix; *total receives the block total.
template <int NT = kInitThreads>
__device__ __forceinline__ long long block_excl_scan1(long long v, long long* s_warp, long long* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    long long incl = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const long long t = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += t;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    long long before = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) {
        const long long x = s_warp[w];
        before += w < warp ? x : 0;
        tot += x;
    }
    *total = tot;
    return before + incl - v;
}

__device__ __forceinline__ void init_grid_barrier(unsigned int* ctr, unsigned int target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int cur;
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        do {
            asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(ctr) : "memory");
        } while (cur < target);
    }
    __syncthreads();
}

// Squared distance of two byte-layout rows: per-byte |a - b| (vabsdiffu4), then the
// byte dot products (dp4a) — exact, < 8 * 255^2.
__device__ __forceinline__ int byte_sq_dist(uint64_t a, uint64_t b) {
    const unsigned lo = __vabsdiffu4(unsigned(a), unsigned(b));
    const unsigned hi = __vabsdiffu4(unsigned(a >> 32), unsigned(b >> 32));
    return __dp4a(lo, lo, __dp4a(hi, hi, 0u));
}

template <bool BYTES>
__global__ void __launch_bounds__(kInitThreads) init_kernel(InitArgs a) {
    __shared__ long long s_warp[2][kInitThreads / 32];  // double-buffered: no barrier between scans
    __shared__ long long s_before;
    __shared__ int s_chunk;
    __shared__ unsigned long long s_found;
    const int tid = threadIdx.x, lane = tid & 31;
    constexpr int per = kInitChunk / kInitThreads;  // 16
    unsigned int n_bar = 0;
    for (int j = a.j0; j < a.j1; ++j) {
        // ---- centroid j (every block computes the same choice)
        uint64_t c;
        if (j == 0) {
            c = a.pts[a.first_idx];
        } else {
            const long long* cs = a.sums[(j - 1) & 1];
            const int* w = a.d2[(j - 1) & 1];
            // total and chunk prefix: each thread owns a contiguous slice of chunk sums
            const int cper = (a.nchunks + kInitThreads - 1) / kInitThreads;
            const int lo = min(a.nchunks, tid * cper), hi = min(a.nchunks, lo + cper);
            long long mine = 0;
            for (int i = lo; i < hi; ++i) mine += __ldcg(cs + i);
            if (tid == 0) s_found = ~0ull;
            long long total;
            const long long excl = block_excl_scan1(mine, s_warp[0], &total);
            const long long T = (long long)floor(__dmul_rn(a.uniforms[j - 1], double(total)));
            long long run = excl;
            for (int i = lo; i < hi; ++i) {
                const long long next = run + __ldcg(cs + i);
                if (run <= T && next > T) {
                    s_chunk = i;
                    s_before = run;
                }
                run = next;
            }
            if (tid == 0 && T >= total) s_chunk = -1;
            __syncthreads();
            const int ch = s_chunk;
            if (ch >= 0) {
                const int64_t p0 = int64_t(ch) * kInitChunk + tid * per;
                int v[per];
                long long tsum = 0;
                if (p0 + per <= a.m && (reinterpret_cast<uintptr_t>(w + p0) & 15) == 0) {
                    const int4* w4 = reinterpret_cast<const int4*>(w + p0);
#pragma unroll
                    for (int q = 0; q < per / 4; ++q) {
                        const int4 x = __ldcg(w4 + q);
                        v[4 * q] = x.x, v[4 * q + 1] = x.y, v[4 * q + 2] = x.z, v[4 * q + 3] = x.w;
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < per; ++q) v[q] = (p0 + q < a.m) ? __ldcg(w + p0 + q) : 0;
                }
#pragma unroll
                for (int q = 0; q < per; ++q) tsum += v[q];
                long long tot2;
                long long acc = s_before + block_excl_scan1(tsum, s_warp[1], &tot2);
                int first = -1;  // first point of the slice whose inclusive prefix passes T
#pragma unroll
                for (int q = 0; q < per; ++q) {
                    acc += v[q];
                    if (first < 0 && acc > T && p0 + q < a.m) first = q;
                }
                if (first >= 0) atomicMin(&s_found, (unsigned long long)(p0 + first));
            }
            __syncthreads();
            int64_t idx = s_found == ~0ull ? a.m - 1 : int64_t(s_found);
            if (idx > a.m - 1) idx = a.m - 1;
            c = a.pts[idx];  // same address in every thread: one broadcast load
        }
        if (blockIdx.x == 0 && tid == 0) a.cent_rows[j] = c;
        // ---- weights for the next centroid: d2 = min(d2, |p - c|^2), per-chunk sums
        const int* wold = a.d2[(j - 1) & 1];
        int* wnew = a.d2[j & 1];
        long long* snew = a.sums[j & 1];
        for (int ch = blockIdx.x; ch < a.nchunks; ch += gridDim.x) {
            const int64_t base = int64_t(ch) * kInitChunk;
            long long sum = 0;
#pragma unroll 4
            for (int q = 0; q < per; ++q) {
                const int64_t p = base + q * kInitThreads + tid;
                if (p < a.m) {
                    int v = BYTES ? byte_sq_dist(a.pts[p], c) : int(int_sq_dist(a.pts[p], c, a.n, a.fmt));  // < 2^31
                    if (j > 0) v = min(v, __ldcg(wold + p));
                    wnew[p] = v;
                    sum += v;
                }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
            __syncthreads();  // s_warp[0] reuse (previous chunk / selection scan)
            if (lane == 0) s_warp[0][tid >> 5] = sum;
            __syncthreads();
            if (tid == 0) {
                long long t = 0;
                for (int w = 0; w < kInitThreads / 32; ++w) t += s_warp[0][w];
                snew[ch] = t;
            }
        }
        init_grid_barrier(a.barrier, ++n_bar * gridDim.x);
    }
}

// Resident k-means++ (one block per SM): block b keeps its P points' rows and weights in
// shared memory for the whole launch, so a centroid's weight update reads no global
// memory; the weights are also written to global memory for the selection, which
// every block makes identically from per-sub-chunk sums (a.sub points each): a
// block scan over the sums finds the sub-chunk holding u * total, a second scan over
// its weights the point.  Same exact-integer arithmetic as init_kernel.
constexpr int kInitResThreads = 512;
constexpr int kInitSelPer = 8;   // sub-chunk sums per thread in the selection scan (independent loads)
constexpr int kInitFinPer = 4;   // weights per thread in the sub-chunk scan
constexpr int kInitMaxSub = 128; // sub-chunks per block

template <bool BYTES>
__global__ void __launch_bounds__(kInitResThreads, 1) init_res_kernel(InitArgs a) {
    extern __shared__ __align__(16) unsigned char s_dyn[];
    __shared__ long long s_warp[2][kInitResThreads / 32];
    __shared__ long long s_sub[kInitMaxSub];
    __shared__ long long s_before;
    __shared__ int s_chunk;
    __shared__ unsigned long long s_found;
    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t P = a.per_block, b0 = int64_t(blockIdx.x) * P;
    const int np = int(b0 < a.m ? (a.m - b0 < P ? a.m - b0 : P) : 0);
    uint64_t* s_rows = reinterpret_cast<uint64_t*>(s_dyn);
    int* s_d2 = reinterpret_cast<int*>(s_rows + P);
    const int* w_in = a.d2[(a.j0 - 1) & 1];
    for (int i = tid; i < np; i += kInitResThreads) {
        s_rows[i] = a.pts[b0 + i];
        if (a.j0 > 0) s_d2[i] = __ldcg(w_in + b0 + i);
    }
    for (int i = tid; i < a.nsub; i += kInitResThreads) s_sub[i] = 0;
    const int L = int(gridDim.x) * a.nsub;  // sub-chunks in point order: (block, sub)
    unsigned int n_bar = 0;
    __syncthreads();
    for (int j = a.j0; j < a.j1; ++j) {
        uint64_t c;
        if (j == 0) {
            c = a.pts[a.first_idx];
        } else {
            const long long* cs = a.sums[(j - 1) & 1];
            const int* w = a.d2[(j - 1) & 1];
            const int cper = (L + kInitResThreads - 1) / kInitResThreads;  // <= kInitSelPer (host)
            const int lo = min(L, tid * cper), hi = min(L, lo + cper);
            long long vals[kInitSelPer];
            long long mine = 0;
#pragma unroll
            for (int q = 0; q < kInitSelPer; ++q) {
                vals[q] = lo + q < hi ? __ldcg(cs + lo + q) : 0;
                mine += vals[q];
            }
            if (tid == 0) s_found = ~0ull;
            long long total;
            const long long excl = block_excl_scan1<kInitResThreads>(mine, s_warp[0], &total);
            const long long T = (long long)floor(__dmul_rn(a.uniforms[j - 1], double(total)));
            long long run = excl;
#pragma unroll
            for (int q = 0; q < kInitSelPer; ++q) {
                const long long next = run + vals[q];
                if (lo + q < hi && run <= T && next > T) {
                    s_chunk = lo + q;
                    s_before = run;
                }
                run = next;
            }
            if (tid == 0 && T >= total) s_chunk = -1;
            __syncthreads();
            const int ch = s_chunk;
            if (ch >= 0) {
                const int blk = ch / a.nsub, sb = ch % a.nsub;
                const int64_t pb = int64_t(blk) * P + int64_t(sb) * a.sub;  // first point of the sub-chunk
                const int64_t nb = blk * P + P < a.m ? blk * P + P : a.m;       // end of the block's points
                const int64_t len = pb < nb ? (nb - pb < a.sub ? nb - pb : a.sub) : 0;
                const int o0 = tid * kInitFinPer;
                int v[kInitFinPer];
                long long tsum = 0;
#pragma unroll
                for (int q = 0; q < kInitFinPer; ++q) {
                    v[q] = o0 + q < len ? __ldcg(w + pb + o0 + q) : 0;
                    tsum += v[q];
                }
                long long tot2;
                long long acc = s_before + block_excl_scan1<kInitResThreads>(tsum, s_warp[1], &tot2);
                int first = -1;
#pragma unroll
                for (int q = 0; q < kInitFinPer; ++q) {
                    acc += v[q];
                    if (first < 0 && acc > T && o0 + q < len) first = q;
                }
                if (first >= 0) atomicMin(&s_found, (unsigned long long)(pb + o0 + first));
            }
            __syncthreads();
            int64_t idx = s_found == ~0ull ? a.m - 1 : int64_t(s_found);
            if (idx > a.m - 1) idx = a.m - 1;
            c = a.pts[idx];
        }
        if (blockIdx.x == 0 && tid == 0) a.cent_rows[j] = c;
        // ---- weights for the next centroid, from shared memory
        int* wg = a.d2[j & 1];
        for (int i0 = 0; i0 < np; i0 += kInitResThreads) {  // warp-uniform trip count
            const int i = i0 + tid;
            int v = 0;
            if (i < np) {
                v = BYTES ? byte_sq_dist(s_rows[i], c) : int(int_sq_dist(s_rows[i], c, a.n, a.fmt));
                if (j > 0) v = min(v, s_d2[i]);
                s_d2[i] = v;
                wg[b0 + i] = v;
            }
            long long sum64;
            if (BYTES) {  // 32 weights < 2^19 each: one 32-bit warp reduction
                sum64 = (long long)__reduce_add_sync(0xffffffffu, unsigned(v));
            } else {  // int64: 32 weights < 2^31 each
                sum64 = v;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) sum64 += __shfl_xor_sync(0xffffffffu, sum64, off);
            }
            if (lane == 0 && i < np) {  // a warp's 32 points lie in one sub-chunk
                if (BYTES)  // sub-chunk sums < 2048 * 2^19 < 2^32: native 32-bit shared atomics
                    atomicAdd(reinterpret_cast<unsigned int*>(s_sub) + i / a.sub, unsigned(sum64));
                else  // (64-bit shared atomicAdd is a CAS loop)
                    atomicAdd(reinterpret_cast<unsigned long long*>(s_sub + i / a.sub), (unsigned long long)sum64);
            }
        }
        __syncthreads();
        long long* snew = a.sums[j & 1];
        for (int i = tid; i < a.nsub; i += kInitResThreads) {
            snew[int64_t(blockIdx.x) * a.nsub + i] =
                BYTES ? (long long)reinterpret_cast<const unsigned int*>(s_sub)[i] : s_sub[i];
            if (BYTES) reinterpret_cast<unsigned int*>(s_sub)[i] = 0;  // each thread clears what it read
            else s_sub[i] = 0;
        }
        init_grid_barrier(a.barrier, ++n_bar * gridDim.x);
    }
}

// ================================================================= Lloyd (K8)
// One cooperative launch runs Lloyd iterations for up to 8 values of k at once
// (speculative knee scan): every pass visits each point once under every
// active k.  Per point and k the kernel keeps ONE float, a Hamerly "budget":
// when the point was last evaluated (pass s) with bounds u >= |p - c_a| and
// l <= min_{j != a} |p - c_j|, it stores b = (l - u) + D_a(s), where D_a is a
// per-cluster running sum (directed rounding, every block computes the same
// table) of the amount pass t can shrink l - u: drift_a(t) + the largest drift
// of any other centroid.  At pass t the assignment provably cannot change while
// b - D_a(t) > margin, so a settled point costs a 1-byte assignment and a
// 4-byte budget read — no row, no distance, no write.  Points that are
// re-evaluated fetch their row and use fp32 distances with a proven error bound,
// and the reference's float64 expression whenever the bound cannot separate
// the two nearest centroids, so assignments equal numpy's argmin bit for bit.
// Cluster sums are exact integers, updated by the deltas of points that
// changed cluster; every block keeps an identical copy and derives the next
// centroids itself, so an iteration needs one grid barrier.
constexpr int kMaxRuns = 8;
constexpr int kMaxClusters = 256;  // sum of k over the runs of one launch
constexpr int kSumW = 9;           // 8 coordinate sums + count
// Per-block delta accumulators (int32 shared atomics): low bytes of the 8
// coordinates, count, then high bytes (nonzero only in wide row layouts), so
// every counter grows by at most 255 per point in any layout.
constexpr int kDeltaW = 17;
// Grid exchange slot spacing (uint64 units).  Packed (1) measured faster than one slot per
// 128-byte line (16: 1.21 -> 1.23 ms per 1M-point knee scan): the per-pass reads of all
// K x 9 sums are latency-, not L2-slice-bound.
#ifndef KT_DSTRIDE
#define KT_DSTRIDE 1
#endif
constexpr int kDStride = KT_DSTRIDE;          // uint64 per exchange slot
constexpr int kChgStride = 2 * KT_DSTRIDE;    // uint32 per changed flag
enum RunState : int {
    kActiveFromSums = 0,  // centroids = sums / counts of the previous pass (bounds valid)
    kActiveGiven = 1,     // centroids given in LloydArgs::cent (after a reseed)
    kConverged = 2,
    kMaxed = 3,
    kNeedsReseed = 4,
    kActiveFromRows = 5  // first pass: centroids = the k-means++ rows
};

__host__ __device__ __forceinline__ bool run_active(int st) {
    return st == kActiveFromSums || st == kActiveGiven || st == kActiveFromRows;
}

struct LloydArgs {
    const uint64_t* pts;
    int64_t m;
    int n;
    RowFmt fmt;
    float bk1;  // centroid-rounding coefficient of d2_bound (scales with the largest coordinate)
    int R;
    int k[kMaxRuns];
    int coff[kMaxRuns];
    int K;  // total clusters
    int it0, it_end, max_iters;
    int64_t stride;            // per-run row stride of assign/budget (m rounded up to 16)
    uint8_t* assign;           // [R][stride], 255 = unassigned
    float* budget;             // [R][stride] (l - u) + D_a(s) of the last evaluation
    float* dcum;               // [K] cumulative bound shrink D_j (carried across launches)
    int64_t per_block;         // resident kernel: points owned by each block (multiple of 16)
    int tile;                  // resident kernel: points per queue tile (multiple of 4)
    float spec_factor;         // speculative scan guard (kSpecFactor; KT_LLOYD_SPEC_FACTOR in tests)
    int rows_resident;         // resident kernel: the block's rows live in shared memory too
    int external;              // 1: one pass, deltas + changed counts -> ext, no in-kernel decisions
    int pack3;                 // resident kernel, P * largest knob index < 2^21: 3-word cluster deltas
    int cluster;               // resident kernel launched as one thread-block cluster: hardware barrier
    unsigned int* barrier;     // grid-barrier counter, zeroed before every launch
    unsigned long long* ext;   // external: [K][9] int64 deltas then [R] changed counts (all-reduced by the host)
    double* cent;              // [K][8] centroids of the latest pass
    const uint64_t* init_rows; // k-means++ rows (prefix shared by all runs)
    long long* S;              // [K][9] running sums
    unsigned long long* D;     // [3][K][9] per-pass deltas, kDStride apart
    unsigned int* chg;         // [3][kMaxRuns], kChgStride apart
    unsigned int* work;        // [3] per-pass chunk counters
    int* run_state;            // [R]
    int* run_iter;             // [R]
    int* ctrl;                 // [0] next iteration
    unsigned long long* stats; // optional [R][3]: point visits, unused, evaluations
    long long* timeline;       // optional [100][4] globaltimer stamps of block 0 per pass
    const int* freeze;         // optional (device-driven sharded loop): nonzero -> the launch is a no-op
    unsigned long long* slack; // optional probe [100][kMaxRuns][8]: points by budget slack b - D_a per pass
};

struct LloydLayout {
    size_t S, c64, c32, c2, delta, drift, dcum, cnext, total;
};

__host__ __device__ inline LloydLayout lloyd_layout(int K) {
    LloydLayout L;
    size_t o = 0;
    L.c64 = o;  // 64 B per cluster: keeps c32 16-byte aligned for float4 loads
    o += size_t(K) * kMaxKnobs * 8;
    L.c32 = o;
    o += size_t(K) * kMaxKnobs * 4;
    L.c2 = o;  // centroid pairs of each run, knob-interleaved (f32x2 distances); odd k padded with NaN
    o += size_t(K + kMaxRuns) * kMaxKnobs * 4;
    L.S = o;
    o += size_t(K) * kSumW * 8;
    L.delta = o;
    o += size_t(K) * kDeltaW * 4;
    L.drift = o;
    o += size_t(K) * 4;
    L.dcum = o;
    o += size_t(K) * 4;
    o = (o + 7) & ~size_t(7);
    L.cnext = o;  // next pass's centroids, computed right after the grid barrier
    o += size_t(K) * kMaxKnobs * 8;
    L.total = (o + 15) & ~size_t(15);
    return L;
}

struct LloydQueueEntry {
    uint32_t point;
    int32_t old;
};
constexpr int kLloydThreads = 256;

struct RunShared {
    unsigned int cnt[kMaxRuns][3];
    int state[kMaxRuns];
    int changed[kMaxRuns];
    float m1[kMaxRuns], m2[kMaxRuns];  // largest / second largest drift
    int amax[kMaxRuns];
    int exit_flag[2], n_active[2];  // by pass parity: reset two passes before they are read again
    unsigned int chg_g[kMaxRuns];  // changed flags of the whole grid (after the barrier)
    int empty[kMaxRuns];           // a cluster of the run ended the pass empty
    float dmax[kMaxRuns];          // largest shrink D_j of the run's clusters (scan prefilter)
    int spec_bad[2];               // by pass parity: a run's shrink outgrew the speculative scan's table
};

// Speculative scan (resident kernel, one tile per block): while a block waits at the grid
// barrier of pass t it already scans its points for pass t+1 against s_dspec[g] = D_a(t+1)
// estimate = D_a(t) + G (G = kSpecFactor x the run's largest shrink step of the last pass).
// The decision phase checks the real D_a(t+1) <= s_dspec for every cluster of every run
// that goes on; then every point the scan settled has b - D_a(t+1) >= b - s_dspec > margin
// (rounded down), so the speculative queue holds every unsettled point (and a few settled
// ones, which an evaluation leaves unchanged: evaluations are exact).  Otherwise the queue
// is dropped and the pass scans as before.
#ifndef KT_LLOYD_SPEC
#define KT_LLOYD_SPEC 1
#endif
#ifndef KT_SPEC_FACTOR
#define KT_SPEC_FACTOR 1.25f
#endif
constexpr float kSpecFactor = KT_SPEC_FACTOR;
// Only where the scan is long enough to hide: blocks of >= 1536 points (1M points, 7,056 per
// block: 1.19 -> 1.13 ms per knee scan; 262K, 1,772 per block: 0.83 -> 0.78).  With fewer points
// per block the scan is short and the extra evaluations cost more than the overlap saves
// (AlexNet RL tasks, ~900 points per block: Lloyd 4.51 -> 4.81 ms per RL step with speculation).
#ifndef KT_SPEC_MIN_POINTS
#define KT_SPEC_MIN_POINTS 1536
#endif
constexpr int kSpecMinPoints = KT_SPEC_MIN_POINTS;
#ifndef KT_SPEC_RETEST
#define KT_SPEC_RETEST 0
#endif
#ifndef KT_SPEC_PERCLUSTER
#define KT_SPEC_PERCLUSTER 1
#endif

// Conservative |fp32 - exact| bound for sum_i (p_i - c_i)^2 with p_i, |c_i| <= 255
// (derivation in DESIGN.md §K8).
// k1 = 6.5e-5 for coordinates <= 255 and grows linearly with the largest coordinate.
// Square roots of the bounds use the MUFU approximation widened by kSqrtSlack (relative):
// sqrt.approx.f32's relative error is below 2^-22 on normal inputs (measured exhaustively
// over [2^-30, 2^30] by tools/sqrt_approx_check.cu: 1.7e-7), so the widened values stay
// on the safe side of the directed-rounding ones they replace (__fsqrt_ru / __fsqrt_rd
// are multi-instruction sequences; this is one MUFU + one FMUL).
#ifndef KT_FAST_SQRT
#define KT_FAST_SQRT 1
#endif
constexpr float kSqrtSlack = 1.0f / (1 << 20);
__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float d2_bound(float d, float k1) {
    if (KT_FAST_SQRT) return (k1 * (1.0f + 4.0f * kSqrtSlack)) * sqrt_approx(8.0f * d + 8.0f) + 5.5e-7f * d + 1e-6f;
    return k1 * sqrtf(8.0f * d + 8.0f) + 5.5e-7f * d + 1e-6f;
}
__device__ __forceinline__ float dist_up(float d2, float k1) {
    const float x = __fadd_ru(d2, d2_bound(d2, k1));
    if (KT_FAST_SQRT) return __fmul_ru(sqrt_approx(x), 1.0f + kSqrtSlack);
    return __fsqrt_ru(x);
}
__device__ __forceinline__ float dist_dn(float d2, float k1) {
    const float lo = __fsub_rd(d2, d2_bound(d2, k1));
    if (KT_FAST_SQRT) return lo > 1e-30f ? __fmul_rd(sqrt_approx(lo), 1.0f - kSqrtSlack) : 0.0f;
    return lo > 0.0f ? __fsqrt_rd(lo) : 0.0f;
}
// Settled iff (l - u) > margin: distances are <= 255*sqrt(8) ~ 721, so float64
// rounding of the reference's squared distances (< 1e-10) cannot reorder two
// centroids whose true distances differ by this much.
constexpr float kSettleMargin = 1e-3f;
#ifndef KT_ASSIGN_UNROLL
#define KT_ASSIGN_UNROLL 4
#endif
constexpr int kAssignUnroll = KT_ASSIGN_UNROLL;  // centroid loop of the f32 assignment (4: 1.30 ms, 2: 1.33, 1: 1.35)

__device__ __forceinline__ void unpack_row(uint64_t row, float p[kMaxKnobs], const RowFmt& f) {
    if (!f.bytes) {
#pragma unroll
        for (int i = 0; i < kMaxKnobs; ++i) p[i] = float(f.get(row, i));  // unused knobs: width 0 -> 0
        return;
    }
    const uint32_t lo = uint32_t(row), hi = uint32_t(row >> 32);
    p[0] = float(lo & 0xff);
    p[1] = float((lo >> 8) & 0xff);
    p[2] = float((lo >> 16) & 0xff);
    p[3] = float(lo >> 24);
    p[4] = float(hi & 0xff);
    p[5] = float((hi >> 8) & 0xff);
    p[6] = float((hi >> 16) & 0xff);
    p[7] = float(hi >> 24);
}

__device__ __forceinline__ float f32_d2(const float p[kMaxKnobs], const float* c) {
    const float4 c0 = *reinterpret_cast<const float4*>(c);
    const float4 c1 = *reinterpret_cast<const float4*>(c + 4);
    float t, d = 0.0f;
    t = p[0] - c0.x; d = fmaf(t, t, d);
    t = p[1] - c0.y; d = fmaf(t, t, d);
    t = p[2] - c0.z; d = fmaf(t, t, d);
    t = p[3] - c0.w; d = fmaf(t, t, d);
    t = p[4] - c1.x; d = fmaf(t, t, d);
    t = p[5] - c1.y; d = fmaf(t, t, d);
    t = p[6] - c1.z; d = fmaf(t, t, d);
    t = p[7] - c1.w; d = fmaf(t, t, d);
    return d;
}

// Upper bound of sqrt(d2) in float (centroid drift): d2 rounded up to float, the MUFU
// square root widened by kSqrtSlack (one MUFU instead of a float64 square root).
__device__ __forceinline__ float drift_up(double d2) {
    const float x = __double2float_ru(d2 * (1.0 + 1e-12));
    return x > 1e-30f ? __fmul_ru(sqrt_approx(x), 1.0f + kSqrtSlack) : 1e-15f;
}

// Centroid pairs: run r's clusters (2q, 2q+1) share 16 floats {c_2q[i], c_2q+1[i]} for
// i = 0..7 at c2 + (pair offset of r + q) * 16, so one packed f32x2 subtract and one
// f32x2 FMA per knob advance two distances (Blackwell FADD2 / FFMA2): per lane the
// same rn operations in the same order as f32_d2, so the distances are bit-identical.
__device__ __forceinline__ int pair_base(const int* k, int r) {
    int o = 0;
    for (int q = 0; q < r; ++q) o += (k[q] + 1) >> 1;
    return o;
}
__device__ __forceinline__ unsigned long long f2_pack(float x) {
    unsigned long long v;
    asm("mov.b64 %0, {%1,%1};" : "=l"(v) : "f"(x));
    return v;
}
__device__ __forceinline__ void f32x2_d2(const float p[kMaxKnobs], const float* c, float& d0, float& d1) {
    const ulonglong2* c4 = reinterpret_cast<const ulonglong2*>(c);
    unsigned long long d = 0ull, t;
#pragma unroll
    for (int h = 0; h < 4; ++h) {
        const ulonglong2 cc = c4[h];
        asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(f2_pack(p[2 * h])), "l"(cc.x));
        asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(d) : "l"(t));
        asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(f2_pack(p[2 * h + 1])), "l"(cc.y));
        asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(d) : "l"(t));
    }
    asm("mov.b64 {%0,%1}, %2;" : "=f"(d0), "=f"(d1) : "l"(d));
}

// Full assignment of one point under one k; returns the cluster and fresh bounds.
__device__ __forceinline__ int full_assign(const float* c32, const float* c2, const double* c64, uint64_t row,
                                           const float p[kMaxKnobs],
                                           int k, int n, const RowFmt& fmt, float k1, float& u, float& l) {
    float best = INFINITY, second = INFINITY;
    int bj = 0;
#pragma unroll (kAssignUnroll)
    for (int j = 0; j < k; j += 2) {
        float dd[2];
        f32x2_d2(p, c2 + j * kMaxKnobs, dd[0], dd[1]);  // odd k: the pad lane is NaN, never below
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float d = dd[h];
            if (d < best) {
                second = best;
                best = d;
                bj = j + h;
            } else if (d < second) {
                second = d;
            }
        }
    }
    if (k > 1 && !(second - best > d2_bound(best, k1) + d2_bound(second, k1))) {
        // ambiguous: the reference's own float64 expression decides (ties -> lowest j)
        // (rare: rolled loops keep the resident kernel's loop body small; an out-of-line
        // __noinline__ version and a compile-time delta variant both measured slower:
        // 1.18 -> 1.33 / 1.26 ms per 1M-point knee scan)
        double bd = INFINITY;
#pragma unroll 1
        for (int j = 0; j < k; ++j) {
            const double d = np_sq_dist(row, c64 + j * kMaxKnobs, n, fmt);
            if (d < bd) {
                bd = d;
                bj = j;
            }
        }
        second = INFINITY;
#pragma unroll 1
        for (int j = 0; j < k; ++j) {
            const float d = f32_d2(p, c32 + j * kMaxKnobs);
            if (j == bj) best = d;
            else second = fminf(second, d);
        }
    }
    u = dist_up(best, k1);
    l = k > 1 ? dist_dn(second, k1) : INFINITY;
    return bj;
}

// Grid barrier for the Lloyd launches: one release-add per block on a monotonic
// counter (zeroed by the host before the launch) and an acquire spin by thread 0;
// bar.sync on both sides makes it cumulative for the whole block.  Cheaper than
// cooperative_groups' grid.sync (no separate fences, no generation flip).
constexpr bool kCustomGridBarrier = true;
__device__ __forceinline__ void lloyd_grid_barrier(unsigned int* ctr, unsigned int target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int cur;
        asm volatile("atom.add.release.gpu.u32 _, [%0], 1;" ::"l"(ctr) : "memory");  // (red.release: same speed)
        // spin relaxed (an acquire load invalidates L1 on every poll), then acquire once
        do {
            asm volatile("ld.relaxed.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(ctr) : "memory");
        } while (cur < target);
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(ctr) : "memory");
    }
    __syncthreads();
}

// Per-run decision after a pass whose summed deltas are already in S (sampler.py:99-116):
// unchanged -> converged; last iteration -> maxed; an empty cluster -> reseed (host);
// else active with centroids = sums / counts.  Returns the new state.
__device__ __forceinline__ int lloyd_decide(const LloydArgs& a, const long long* S, int r, int st, bool changed, int it) {
    if (!changed) return kConverged;
    if (it == a.max_iters - 1) return kMaxed;
    for (int j = 0; j < a.k[r]; ++j)
        if (S[(a.coff[r] + j) * kSumW + 8] == 0) return kNeedsReseed;
    return kActiveFromSums;
}

// Resident variant: block b owns points [b*P, (b+1)*P) for the whole launch and
// keeps their assignments and budgets in shared memory, so a settled point costs
// two shared-memory reads per pass and no global traffic at all; the points the
// budgets cannot settle go through a block-wide queue (tiles of `tile` points,
// so the queue never overflows) and only they fetch their rows from L2.
constexpr int kLloydResThreads = 640;  // 20 warps (A/B at 1M points: 640 1.285 ms, 768 1.295, 896 1.287; 512 and 1024 slower)
constexpr int kEvalUnroll = 1;  // queue entries per thread per iteration (1 measured best: smaller code, 1.45 -> 1.41 ms)
constexpr int kScanQuads = 4;   // quads per thread per scan round
// Resident-kernel cluster-sum deltas: 0 = packed 64-bit shared words (5 CAS atomics per
// move), 1 = 17-wide int32 shared counters (9 native atomics), 2 = a private int32
// copy per warp (9 native atomics, contention only within a warp).  Measured on B200
// (1M-point knee scan, 100 passes): 1.61 / 1.79 / 1.97 ms -> mode 0.
constexpr int kDeltaMode = 0;
constexpr int kLloydQueueMax = 16384;  // block queue entries (point | run << 16 | old << 24)
constexpr int kLloydQueueMin = 2048;

// Shared-memory bytes of the resident kernel before the queue: tables, [R][P]
// assignments, [R][P] budgets and (optionally) the block's P rows.
__host__ __device__ inline size_t lloyd_resident_bytes(int K, int R, int64_t P, bool rows) {
    return lloyd_layout(K).total + ((size_t(R) * P + 15) & ~size_t(15)) + size_t(R) * P * 4 + (rows ? size_t(P) * 8 : 0);
}

// Evaluate one point under run r: full assignment and its new budget.
__device__ __forceinline__ int lloyd_assign(const LloydArgs& a, const RowFmt& fmt, const float* c32, const float* c2,
                                            const int* pcoff, const double* c64, const float* dcum, int r, uint64_t row,
                                            float& budget) {
    const int co = a.coff[r];
    float p[kMaxKnobs];
    unpack_row(row, p, fmt);
    float u, l;
    const int j = full_assign(c32 + co * kMaxKnobs, c2 + pcoff[r] * 2 * kMaxKnobs, c64 + co * kMaxKnobs, row, p, a.k[r],
                              a.n, fmt, a.bk1, u, l);
    budget = __fadd_rd(__fsub_rd(l, u), dcum[co + j]);
    return j;
}

// Resident kernel deltas: two coordinates per 64-bit shared atomic (32-bit fields,
// two's complement across the pair: every field's true per-pass block total stays
// within +-2^31 since P <= 32767 points of value < 2^16), the count in a fifth
// word — 5 atomics per point move instead of 9.
constexpr int kPackedW = 5;
__device__ __forceinline__ void packed_delta(unsigned long long* d, uint64_t row, int sign, int n, const RowFmt& fmt) {
#pragma unroll
    for (int c = 0; c < kMaxKnobs; c += 2) {
        if (c >= n) break;
        const unsigned long long lo = unsigned(fmt.get(row, c));
        const unsigned long long hi = c + 1 < n ? unsigned(fmt.get(row, c + 1)) : 0u;
        const unsigned long long v = lo | (hi << 32);
        atomicAdd(d + (c >> 1), sign > 0 ? v : 0ull - v);
    }
    atomicAdd(d + 4, sign > 0 ? 1ull : ~0ull);
}
// P * (largest knob index) < 2^21: three 21-bit unsigned fields per 64-bit word, points
// joining a cluster added to its words 0-2 and points leaving it to words 3-5 (each field's
// per-pass block total < 2^21, no carries between fields): 3 atomics per side instead of 5.
constexpr int kPack3W = 6;
__device__ __forceinline__ void pack3_delta(unsigned long long* d, uint64_t row, int sign) {
    const unsigned long long m = 0xffull;
    const unsigned long long v0 = (row & m) | (((row >> 8) & m) << 21) | (((row >> 16) & m) << 42);
    const unsigned long long v1 = ((row >> 24) & m) | (((row >> 32) & m) << 21) | (((row >> 40) & m) << 42);
    const unsigned long long v2 = ((row >> 48) & m) | (((row >> 56) & m) << 21) | (1ull << 42);
    unsigned long long* w = d + (sign > 0 ? 0 : 3);
    atomicAdd(w, v0);
    atomicAdd(w + 1, v1);
    atomicAdd(w + 2, v2);
}
__device__ __forceinline__ void pack3_delta_fmt(unsigned long long* d, uint64_t row, int sign, int n,
                                                const RowFmt& fmt) {
    unsigned long long v[3] = {0ull, 0ull, 0ull};
#pragma unroll
    for (int c = 0; c < kMaxKnobs; ++c)
        if (c < n) v[c / 3] |= (unsigned long long)fmt.get(row, c) << (21 * (c % 3));
    v[2] |= 1ull << 42;
    unsigned long long* w = d + (sign > 0 ? 0 : 3);
    atomicAdd(w, v[0]);
    atomicAdd(w + 1, v[1]);
    atomicAdd(w + 2, v[2]);
}
__device__ __forceinline__ long long pack3_field(const unsigned long long* d, int c) {
    const int q = c / 3, sh = 21 * (c % 3);
    const long long plus = (long long)((d[q] >> sh) & 0x1fffffull);
    const long long minus = (long long)((d[3 + q] >> sh) & 0x1fffffull);
    return plus - minus;
}
__device__ __forceinline__ long long packed_field(const unsigned long long* d, int c) {
    const unsigned long long v = d[c < 8 ? c >> 1 : 4];
    const long long lo = (long long)(int)(unsigned)(v & 0xffffffffull);
    if (c == 8 || !(c & 1)) return lo;
    return (long long)(v - (unsigned long long)lo) >> 32;
}

__device__ __forceinline__ void lane_delta(int* d, uint64_t row, int sign, int n, const RowFmt& fmt) {
    for (int c = 0; c < n; ++c) {
        const int v = fmt.get(row, c);
        atomicAdd(d + c, sign * (v & 0xff));
        if (v >> 8) atomicAdd(d + 9 + c, sign * (v >> 8));
    }
    atomicAdd(d + 8, sign);
}

// Warp-aggregated cluster-sum deltas (all 32 lanes call it): lanes passing the same
// cluster g >= 0 are reduced with __reduce_add_sync and one leader per group
// updates the block's shared counters — no same-address atomic storms when many
// points move (the first passes move every point).
__device__ __forceinline__ void warp_delta(int* delta, int g, uint64_t row, int sign, int n, const RowFmt& fmt) {
    unsigned pending = __ballot_sync(0xffffffffu, g >= 0);
    const int lane = threadIdx.x & 31;
    while (pending) {
        const int leader = __ffs(pending) - 1;
        const int gl = __shfl_sync(0xffffffffu, g, leader);
        const bool mine = g == gl;
        const unsigned grp = __ballot_sync(0xffffffffu, mine);
        int* d = delta + gl * kDeltaW;
        for (int c = 0; c < n; ++c) {
            const int v = mine ? fmt.get(row, c) : 0;
            const int lo = int(__reduce_add_sync(0xffffffffu, unsigned(v & 0xff)));
            if (lane == leader && lo) atomicAdd(d + c, sign * lo);
            if (!fmt.bytes) {
                const int hi = int(__reduce_add_sync(0xffffffffu, unsigned(v >> 8)));
                if (lane == leader && hi) atomicAdd(d + 9 + c, sign * hi);
            }
        }
        if (lane == leader) atomicAdd(d + 8, sign * __popc(grp));
        pending &= ~grp;
    }
}

// Evaluate one point under run r (one lane, no warp cooperation): assignment,
// budget, and the shared-counter deltas of a move.
__device__ __forceinline__ int lloyd_eval(const LloydArgs& a, const RowFmt& fmt, const float* c32, const float* c2,
                                          const int* pcoff, const double* c64, const float* dcum, int* delta, int r,
                                          uint64_t row, int old, float& budget) {
    const int co = a.coff[r];
    const int j = lloyd_assign(a, fmt, c32, c2, pcoff, c64, dcum, r, row, budget);
    if (j != old) {
        int* dn = delta + (co + j) * kDeltaW;
        for (int c = 0; c < a.n; ++c) {
            const int v = fmt.get(row, c);
            atomicAdd(dn + c, v & 0xff);
            if (v >> 8) atomicAdd(dn + 9 + c, v >> 8);
        }
        atomicAdd(dn + 8, 1);
        if (old != 255) {
            int* dold = delta + (co + old) * kDeltaW;
            for (int c = 0; c < a.n; ++c) {
                const int v = fmt.get(row, c);
                atomicSub(dold + c, v & 0xff);
                if (v >> 8) atomicSub(dold + 9 + c, v >> 8);
            }
            atomicSub(dold + 8, 1);
        }
    }
    return j;
}

// BYTES: the byte-per-knob row layout as a compile-time RowFmt (constant shifts, no
// generic-width code in the loop bodies); the bit-field layout reads a.fmt.
// Probe builds (-DKT_LLOYD_PROBES=1) compile in the per-run visit counters and the
// per-pass timeline that KT_LLOYD_STATS / KT_LLOYD_TIMELINE read; the default build
// leaves them out of the kernel (a smaller loop body measured faster).
#ifndef KT_LLOYD_PROBES
#define KT_LLOYD_PROBES 0
#endif
constexpr bool kLloydProbes = KT_LLOYD_PROBES != 0;

template <bool RESIDENT, bool BYTES>
__global__ void __launch_bounds__(RESIDENT ? kLloydResThreads : kLloydThreads, RESIDENT ? 1 : 3)
    lloyd_kernel(LloydArgs a) {
    extern __shared__ __align__(16) unsigned char s_dyn[];
    if (a.freeze && *a.freeze) return;  // every block reads the same flag: uniform exit
    __shared__ RunShared rs;
    __shared__ uint8_t run_of[kMaxClusters];
    __shared__ LloydQueueEntry wqueue[RESIDENT ? 1 : kLloydThreads / 32 * 128];
    __shared__ int s_qn[2];  // resident kernel: queue counters (alternating tiles)
    __shared__ float s_dspec[RESIDENT && KT_LLOYD_SPEC ? kMaxClusters : 1];  // speculative shrink table
    // the dynamic window is only guaranteed 8-byte aligned after static smem (tools add their
    // own static smem): align explicitly for the float4 centroid loads (16 spare bytes allocated)
    // generic pointer arithmetic measured faster here than align_shared<16> (1.60 vs 1.95 ms per 1M-point knee scan)
#ifndef KT_SMEM_PROVENANCE
#define KT_SMEM_PROVENANCE 0
#endif
    // KT_SMEM_PROVENANCE 1 offsets from s_dyn itself so every derived pointer keeps the shared
    // address space (LDS / STS instead of generic LD / ST): measured SLOWER on B200 (1M-point
    // knee scan 1.20 -> 1.59 ms; heavy-pass evaluation 33 -> 45 us, grid-barrier wait 2 -> 5 us)
    unsigned char* s_raw = KT_SMEM_PROVENANCE
        ? s_dyn + ((16u - (unsigned(__cvta_generic_to_shared(s_dyn)) & 15u)) & 15u)
        : reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(s_dyn) + 15) & ~uintptr_t(15));
    const LloydLayout L = lloyd_layout(a.K);
    double* c64 = reinterpret_cast<double*>(s_raw + L.c64);
    long long* S = reinterpret_cast<long long*>(s_raw + L.S);
    float* c32 = reinterpret_cast<float*>(s_raw + L.c32);
    float* c2 = reinterpret_cast<float*>(s_raw + L.c2);
    __shared__ int s_pcoff[kMaxRuns];
    __shared__ uint8_t s_pslot[kMaxClusters];  // in-run index j of cluster g (its pair slot: pcoff[r] * 2 + j)
    int* delta = reinterpret_cast<int*>(s_raw + L.delta);
    unsigned long long* delta64 = reinterpret_cast<unsigned long long*>(s_raw + L.delta);  // resident layout
    float* drift = reinterpret_cast<float*>(s_raw + L.drift);
    float* dcum = reinterpret_cast<float*>(s_raw + L.dcum);
    double* cnext = reinterpret_cast<double*>(s_raw + L.cnext);
    cg::grid_group grid = cg::this_grid();
    const int tid = threadIdx.x;
    const int K = a.K, R = a.R, n = a.n;
    const int64_t m = a.m;
    const int lane = tid & 31;
    RowFmt fmt;
    if constexpr (BYTES) {
#pragma unroll
        for (int i = 0; i < kMaxKnobs; ++i) {
            fmt.shift[i] = uint8_t(8 * i);
            fmt.width[i] = 8;
        }
        fmt.cmax = 255;
        fmt.bytes = 1;
    } else {
        fmt = a.fmt;
    }

    // resident state of this block's points
    const int64_t P = a.per_block;
    const int64_t b0 = RESIDENT ? int64_t(blockIdx.x) * P : 0;
    const int np = RESIDENT ? int(b0 < m ? (m - b0 < P ? m - b0 : P) : 0) : 0;
    uint8_t* s_asg = s_raw + L.total;                                          // [R][P]
    float* s_bud = reinterpret_cast<float*>(s_asg + ((size_t(R) * P + 15) & ~size_t(15)));  // [R][P]
    uint64_t* s_rows = reinterpret_cast<uint64_t*>(s_bud + size_t(R) * P);   // [P] if rows_resident
    uint32_t* s_queue = reinterpret_cast<uint32_t*>(s_rows + (a.rows_resident ? P : 0));  // [tile * R]
    int* delta_w = reinterpret_cast<int*>(s_queue + size_t(a.tile) * R);    // kDeltaMode 2: [warps][K][17]
    const int nwarps_blk = blockDim.x >> 5;

    for (int i = tid; i < K * kSumW; i += blockDim.x) S[i] = a.S[i];
    for (int i = tid; i < K * kMaxKnobs; i += blockDim.x) c64[i] = a.cent[i];  // centroids of the previous pass
    for (int i = tid; i < K; i += blockDim.x) dcum[i] = a.dcum[i];
    if (tid < R) rs.state[tid] = a.run_state[tid];
    if (tid < kMaxRuns) rs.empty[tid] = 0;
    if (tid < kMaxRuns * 3) rs.cnt[tid / 3][tid % 3] = 0;
    if (tid < 2) s_qn[tid] = 0;
    for (int r = 0; r < R; ++r)
        for (int j = tid; j < a.k[r]; j += blockDim.x) {
            run_of[a.coff[r] + j] = uint8_t(r);
            s_pslot[a.coff[r] + j] = uint8_t(j);
        }
    if (tid < R) s_pcoff[tid] = pair_base(a.k, tid);
    for (int i = tid; i < (K + kMaxRuns) * kMaxKnobs; i += blockDim.x) c2[i] = __int_as_float(0x7fc00000);  // NaN pads
    if (RESIDENT) {
        for (int r = 0; r < R; ++r) {
            // budgets are only meaningful (and only written) once a run has bounds
            const bool bounds = a.run_state[r] == kActiveFromSums;
            for (int i = tid; i < np; i += blockDim.x) {
                s_asg[r * P + i] = a.assign[int64_t(r) * a.stride + b0 + i];
                s_bud[r * P + i] = bounds ? a.budget[int64_t(r) * a.stride + b0 + i] : 0.0f;
            }
            for (int i = np + tid; i < ((np + 3) & ~3); i += blockDim.x) s_asg[r * P + i] = 255;  // quad padding
        }
        if (a.rows_resident)
            for (int i = tid; i < np; i += blockDim.x) s_rows[i] = a.pts[b0 + i];
    }
    auto c2_slot = [&](int g, int i) {
        const int j = s_pslot[g];
        return (s_pcoff[run_of[g]] * 2 + (j & ~1)) * kMaxKnobs + 2 * i + (j & 1);
    };
    unsigned int n_bar = 0;  // grid barriers passed (custom barrier target = n_bar * gridDim.x)
    auto grid_barrier = [&]() {
        if (RESIDENT && a.cluster) {  // the whole grid is one cluster: barrier.cluster (release / acquire)
            asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
            asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
        } else if (kCustomGridBarrier) {
            lloyd_grid_barrier(a.barrier, ++n_bar * gridDim.x);
        } else {
            grid.sync();
        }
    };
    // the same barrier split in two, so a block can work between its arrival and its wait
    auto grid_arrive = [&]() {
        if (RESIDENT && a.cluster) {
            asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        } else {
            __syncthreads();
            if (threadIdx.x == 0) asm volatile("atom.add.release.gpu.u32 _, [%0], 1;" ::"l"(a.barrier) : "memory");
        }
    };
    auto grid_wait = [&]() {
        if (RESIDENT && a.cluster) {
            asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
        } else {
            const unsigned int target = ++n_bar * gridDim.x;
            if (threadIdx.x == 0) {
                unsigned int cur;
                do {
                    asm volatile("ld.relaxed.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(a.barrier) : "memory");
                } while (cur < target);
                asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(a.barrier) : "memory");
            }
            __syncthreads();
        }
    };
    grid_barrier();  // every block has read a.cent / a.dcum before block 0 overwrites them

    int it = a.it0;
    auto stamp = [&](int phase) {
        if (kLloydProbes && a.timeline && blockIdx.x == 0 && tid == 0 && it < 100) {
            long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            a.timeline[it * 16 + phase] = t;
        }
    };
    // scan of points [t0, t1): kScanQuads quads per thread and round (independent loads, one
    // warp scan + one queue atomic per warp and round); unsettled (point, run, old) -> queue.
    // dtab: the shrink table the budgets are tested against (dcum, or the speculative s_dspec)
    auto scan_tile = [&](int t0, int t1, int* qn, const float* dtab) {
        const int tq1 = (t1 + 3) >> 2;
        for (int qd0 = t0 >> 2; qd0 < tq1; qd0 += kScanQuads * blockDim.x) {
            for (int r = 0; r < R; ++r) {
                const int st = rs.state[r];
                if (!run_active(st)) continue;
                const int co = a.coff[r];
                unsigned todo = 0;  // bit 4q + e: point e of quad q
                uint32_t as4[kScanQuads];
#pragma unroll
                for (int q = 0; q < kScanQuads; ++q) {
                    const int qd = qd0 + q * blockDim.x + tid;
                    const int p0 = qd << 2;
                    const int cnt = qd < tq1 ? (t1 - p0 < 4 ? t1 - p0 : 4) : 0;
                    as4[q] = 0xffffffffu;
                    if (cnt > 0) {
                        as4[q] = *reinterpret_cast<const uint32_t*>(s_asg + r * P + p0);
                        if (st == kActiveFromSums) {
                            const float4 b4 = *reinterpret_cast<const float4*>(s_bud + r * P + p0);
                            const float bb[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const int old = (as4[q] >> (8 * e)) & 0xff;
                                if (e >= cnt) continue;
                                if (old == 255 || !(__fsub_rd(bb[e], dtab[co + old]) > kSettleMargin))
                                    todo |= 1u << (4 * q + e);
                            }
                        } else {
                            todo |= ((1u << cnt) - 1u) << (4 * q);
                        }
                    }
                }
                // warp-aggregated append
                const int c = __popc(todo);
                int incl = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                int wbase = 0;
                if (lane == 31 && incl) wbase = atomicAdd(qn, incl);
                wbase = __shfl_sync(0xffffffffu, wbase, 31);
                int pos = wbase + incl - c;
                while (todo) {
                    const int bit = __ffs(todo) - 1;
                    todo &= todo - 1;
                    const int q = bit >> 2, e = bit & 3;
                    const int p0 = (qd0 + q * int(blockDim.x) + tid) << 2;
                    uint32_t aq = as4[0];  // select without dynamic register indexing
#pragma unroll
                    for (int qq = 1; qq < kScanQuads; ++qq) aq = q == qq ? as4[qq] : aq;
                    s_queue[pos++] = uint32_t(p0 + e) | (uint32_t(r) << 16) | (((aq >> (8 * e)) & 0xffu) << 24);
                }
            }
        }
    };
    int tile_parity = 0;  // queue counter in use (alternates per tile, across passes too)
    bool entry = true;
    bool spec_hit = false;    // this pass's queue was built by the previous pass's speculative scan
    bool spec_ready = false;  // s_dspec holds the next pass's table (after a decision phase)
    while (it < a.it_end) {
        stamp(0);
        if (tid == 0) {  // written by this pass's update, read after its final barrier
            rs.exit_flag[it & 1] = 0;
            rs.n_active[it & 1] = 0;
            rs.spec_bad[it & 1] = 0;
        }
        if (tid < kMaxRuns) rs.empty[tid] = 0;  // likewise (ordered by the tile / grid barriers)
        if (entry) {  // launch entry; later passes get their centroids from the fused update below
        entry = false;
        // ---- this pass's centroids and each centroid's drift from the previous pass:
        // one thread per (cluster, coordinate); 8 consecutive lanes reduce a drift
        for (int x0 = 0; x0 < K * kMaxKnobs; x0 += blockDim.x) {
            const int x = x0 + tid;
            const int g = x >> 3, i = x & 7;
            const int r = x < K * kMaxKnobs ? run_of[g] : 0;
            const int st = rs.state[r];
            const bool live = x < K * kMaxKnobs && run_active(st);
            double dlt2 = 0.0;
            if (live) {
                double c;
                if (i >= n) c = 0.0;
                else if (st == kActiveFromSums) c = __ddiv_rn(double(S[g * kSumW + i]), double(S[g * kSumW + 8]));
                else if (st == kActiveGiven) c = a.cent[g * kMaxKnobs + i];
                else c = double(a.fmt.get(a.init_rows[g - a.coff[r]], i));
                const double dlt = c - c64[g * kMaxKnobs + i];
                dlt2 = dlt * dlt;
                c64[g * kMaxKnobs + i] = c;
                c32[g * kMaxKnobs + i] = float(c);
                c2[c2_slot(g, i)] = float(c);
                if (blockIdx.x == 0) a.cent[g * kMaxKnobs + i] = c;
            }
            dlt2 += __shfl_xor_sync(0xffffffffu, dlt2, 1);
            dlt2 += __shfl_xor_sync(0xffffffffu, dlt2, 2);
            dlt2 += __shfl_xor_sync(0xffffffffu, dlt2, 4);
            if (live && i == 0) drift[g] = drift_up(dlt2);
        }
        for (int i = tid; i < K * kDeltaW; i += blockDim.x) delta[i] = 0;  // also clears delta64 (K*5*8 <= K*17*4)
        if (RESIDENT && kDeltaMode == 2)
            for (int i = tid; i < nwarps_blk * K * kDeltaW; i += blockDim.x) delta_w[i] = 0;
        if (tid < kMaxRuns) rs.changed[tid] = 0;
        __syncthreads();
        if (tid < R && run_active(rs.state[tid])) {
            float m1 = 0.0f, m2 = 0.0f;
            int am = -1;
            for (int j = 0; j < a.k[tid]; ++j) {
                const float d = drift[a.coff[tid] + j];
                if (d > m1) {
                    m2 = m1;
                    m1 = d;
                    am = j;
                } else if (d > m2) {
                    m2 = d;
                }
            }
            // ---- cumulative shrink of (l - u): own drift + largest drift among the other centroids
            const int st = rs.state[tid];
            float dm = 0.0f;
            for (int j = 0; j < a.k[tid]; ++j) {
                const int g = a.coff[tid] + j;
                if (st != kActiveFromSums) dcum[g] = 0.0f;  // every point is evaluated afresh this pass
                else dcum[g] = __fadd_ru(dcum[g], __fadd_ru(drift[g], j == am ? m2 : m1));
                dm = fmaxf(dm, dcum[g]);
            }
            rs.dmax[tid] = dm;
        }
        __syncthreads();
        }

        stamp(1);
        if (kLloydProbes && RESIDENT && a.slack && it < 100) {
            // slack histogram of this block's points (run r, bucket: < margin, 0.25, 0.5, 1, 2, 4, 8, more)
            for (int r = 0; r < R; ++r) {
                if (rs.state[r] != kActiveFromSums) continue;
                unsigned cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                for (int i = tid; i < np; i += blockDim.x) {
                    const int old = s_asg[r * P + i];
                    const float sl = old == 255 ? -1.0f : __fsub_rd(s_bud[r * P + i], dcum[a.coff[r] + old]);
                    const int bkt = sl <= kSettleMargin ? 0 : sl < 0.25f ? 1 : sl < 0.5f ? 2 : sl < 1.0f ? 3
                                  : sl < 2.0f ? 4 : sl < 4.0f ? 5 : sl < 8.0f ? 6 : 7;
                    ++cnt[bkt];
                }
                for (int b = 0; b < 8; ++b) {
                    const unsigned v = __reduce_add_sync(0xffffffffu, cnt[b]);
                    if (lane == 0 && v) atomicAdd(a.slack + (size_t(it) * kMaxRuns + r) * 8 + b, (unsigned long long)v);
                }
            }
        }
        if constexpr (RESIDENT) {
            // ---- assignment pass over this block's resident points, one tile at a time
            for (int t0 = 0; t0 < np; t0 += a.tile) {
                const int t1 = t0 + a.tile < np ? t0 + a.tile : np;
                int* qn = s_qn + tile_parity;
                const bool spec_pass = spec_hit;  // the queue holds candidates tested against s_dspec
                if (!spec_hit) scan_tile(t0, t1, qn, dcum);
                spec_hit = false;
                if (t0 == 0) stamp(10);
                __syncthreads();
                if (t0 == 0) stamp(2);
                if (tid == 0) s_qn[tile_parity ^ 1] = 0;
                const int nqueued = *qn;
                if (kLloydProbes && a.stats && tid == 0)
                    for (int r = 0; r < R; ++r)
                        if (run_active(rs.state[r])) rs.cnt[r][0] += unsigned(t1 - t0);
                // evaluate: rows from shared memory (or L2), kEvalUnroll per thread at a time
                for (int i0 = 0; i0 < nqueued; i0 += kEvalUnroll * blockDim.x) {
                    uint32_t ent[kEvalUnroll];
                    uint64_t row[kEvalUnroll];
#pragma unroll
                    for (int u = 0; u < kEvalUnroll; ++u) {
                        const int i = i0 + u * blockDim.x + tid;
                        ent[u] = i < nqueued ? s_queue[i] : 0xffffffffu;
                        if (ent[u] == 0xffffffffu) row[u] = 0ull;
                        else if (a.rows_resident) row[u] = s_rows[ent[u] & 0xffffu];
                        else row[u] = __ldg(a.pts + b0 + (ent[u] & 0xffffu));
                    }
#pragma unroll
                    for (int u = 0; u < kEvalUnroll; ++u) {
                        if (ent[u] == 0xffffffffu) continue;
                        const int pl = int(ent[u] & 0xffffu), r = int((ent[u] >> 16) & 0xff), old = int(ent[u] >> 24);
                        if (KT_LLOYD_SPEC && spec_pass) {
                            if (!run_active(rs.state[r])) continue;  // a speculative entry of a run that stopped
                            // re-test against the real shrink table: the scan's guard let it through
                            if (KT_SPEC_RETEST && old != 255 &&
                                __fsub_rd(s_bud[r * P + pl], dcum[a.coff[r] + old]) > kSettleMargin)
                                continue;
                        }
                        float bud;
                        const int j = lloyd_assign(a, fmt, c32, c2, s_pcoff, c64, dcum, r, row[u], bud);
                        s_bud[r * P + pl] = bud;
                        if (kLloydProbes && a.stats) atomicAdd(&rs.cnt[r][2], 1u);
                        if (j != old) {
                            s_asg[r * P + pl] = uint8_t(j);
                            rs.changed[r] = 1;
                            const int gn = a.coff[r] + j, go = a.coff[r] + old;
                            if (kDeltaMode == 0) {
                                if (BYTES && a.pack3) {
                                    pack3_delta(delta64 + gn * kPack3W, row[u], 1);
                                    if (old != 255) pack3_delta(delta64 + go * kPack3W, row[u], -1);
                                } else if (!BYTES && a.pack3) {
                                    pack3_delta_fmt(delta64 + gn * kPack3W, row[u], 1, n, fmt);
                                    if (old != 255) pack3_delta_fmt(delta64 + go * kPack3W, row[u], -1, n, fmt);
                                } else {
                                    packed_delta(delta64 + gn * kPackedW, row[u], 1, n, fmt);
                                    if (old != 255) packed_delta(delta64 + go * kPackedW, row[u], -1, n, fmt);
                                }
                            } else {
                                int* dw = kDeltaMode == 2 ? delta_w + (tid >> 5) * K * kDeltaW : delta;
                                lane_delta(dw + gn * kDeltaW, row[u], 1, n, fmt);
                                if (old != 255) lane_delta(dw + go * kDeltaW, row[u], -1, n, fmt);
                            }
                        }
                    }
                }
                tile_parity ^= 1;
                if (t0 == 0) stamp(11);
                __syncthreads();
                if (t0 == 0) stamp(3);
            }
        } else {
            // ---- assignment pass.  Per warp and round: each lane tests 4 consecutive
            // points against their budgets; the points the budgets cannot settle are
            // queued in shared memory and then evaluated by all 32 lanes together.
            const int64_t nq = (m + 3) >> 2;
            LloydQueueEntry* queue = wqueue + (tid >> 5) * 128;
            // warps grab 32-quad chunks from a per-pass counter (claimed one chunk ahead)
            unsigned int* work = a.work + (it % 3);
            unsigned int next = 0, ahead = 0;
            if (lane == 0) next = atomicAdd(work, 32u);
            next = __shfl_sync(0xffffffffu, next, 0);
            while (int64_t(next) < nq) {
                const unsigned int chunk = next;
                if (lane == 0) ahead = atomicAdd(work, 32u);
                const int64_t q = int64_t(chunk) + lane;
                const int64_t p0 = q << 2;
                const int cnt = q < nq ? int(m - p0 < 4 ? m - p0 : 4) : 0;
                for (int r = 0; r < R; ++r) {
                    const int st = rs.state[r];
                    if (!run_active(st)) continue;
                    const int co = a.coff[r];
                    uint8_t* as_r = a.assign + int64_t(r) * a.stride;
                    float* bg_r = a.budget + int64_t(r) * a.stride;
                    unsigned todo = 0;  // bit e: point e needs distance work
                    uint32_t as4 = 0xffffffffu;
                    if (cnt > 0) {
                        as4 = *reinterpret_cast<const uint32_t*>(as_r + p0);
                        if (st == kActiveFromSums) {
                            const float4 b4 = reinterpret_cast<const float4*>(bg_r)[q];
                            const float bb[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const int old = (as4 >> (8 * e)) & 0xff;
                                if (e >= cnt) continue;
                                if (old == 255 || !(__fsub_rd(bb[e], dcum[co + old]) > kSettleMargin)) todo |= 1u << e;
                            }
                        } else {
                            todo = (1u << cnt) - 1u;
                        }
                    }
                    // warp-level compaction of the unsettled points
                    int base = 0;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const bool mine = (todo >> e) & 1u;
                        const unsigned bal = __ballot_sync(0xffffffffu, mine);
                        if (mine) {
                            LloydQueueEntry& qe = queue[base + __popc(bal & ((1u << lane) - 1u))];
                            qe.point = uint32_t(p0 + e);
                            qe.old = (as4 >> (8 * e)) & 0xff;
                        }
                        base += __popc(bal);
                    }
                    __syncwarp();
                    for (int i = lane; i < base; i += 32) {
                        const LloydQueueEntry qe = queue[i];
                        const uint64_t row = __ldg(a.pts + qe.point);
                        float bud;
                        const int j = lloyd_eval(a, fmt, c32, c2, s_pcoff, c64, dcum, delta, r, row, qe.old, bud);
                        bg_r[qe.point] = bud;
                        if (j != qe.old) {
                            as_r[qe.point] = uint8_t(j);
                            rs.changed[r] = 1;
                        }
                    }
                    if (kLloydProbes && a.stats) {
                        const unsigned valid = __reduce_add_sync(0xffffffffu, unsigned(cnt));
                        if (lane == 0) {
                            atomicAdd(&rs.cnt[r][0], valid);
                            atomicAdd(&rs.cnt[r][2], unsigned(base));
                        }
                    }
                    __syncwarp();
                }
                next = __shfl_sync(0xffffffffu, ahead, 0);
            }
        }
        if (!RESIDENT) __syncthreads();  // the resident tile loop ends with one
        const int buf = it % 3;
        unsigned long long* Dcur = a.external ? a.ext : a.D + size_t(buf) * K * kSumW * kDStride;
        const int ds = a.external ? 1 : kDStride;
        for (int i = tid; i < K * kSumW; i += blockDim.x) {
            const int g = i / kSumW, c = i % kSumW;
            long long vw = 0;
            if (RESIDENT && kDeltaMode == 2)
                for (int w = 0; w < nwarps_blk; ++w) {
                    const int* dw = delta_w + (w * K + g) * kDeltaW;
                    vw += (long long)dw[c] + (c < 8 ? 256ll * dw[9 + c] : 0ll);
                }
            const long long v = (RESIDENT && kDeltaMode == 2) ? vw
                              : (RESIDENT && kDeltaMode == 0)
                                  ? (a.pack3 ? pack3_field(delta64 + g * kPack3W, c) : packed_field(delta64 + g * kPackedW, c))
                                         : (long long)delta[g * kDeltaW + c] + (c < 8 ? 256ll * delta[g * kDeltaW + 9 + c] : 0ll);
            if (v) atomicAdd(Dcur + size_t(i) * ds, (unsigned long long)v);
        }
        if (a.external) {  // sharded k-means: the host all-reduces ext, then kt_lloyd_apply decides
            if (tid < R && rs.changed[tid]) atomicAdd(a.ext + size_t(K) * kSumW + tid, 1ull);
            stamp(4);
            ++it;
            break;
        }
        if (tid < R && rs.changed[tid]) atomicOr(a.chg + (buf * kMaxRuns + tid) * kChgStride, 1u);
        if (blockIdx.x == 0) {
            const int nb = (it + 1) % 3;
            for (int i = tid; i < K * kSumW; i += blockDim.x) a.D[(size_t(nb) * K * kSumW + i) * kDStride] = 0ull;
            if (tid < kMaxRuns) a.chg[(nb * kMaxRuns + tid) * kChgStride] = 0u;
            if (tid == 0) a.work[nb] = 0u;
        }
        stamp(4);
        bool spec_scanned = false;
        if (RESIDENT && KT_LLOYD_SPEC && P >= kSpecMinPoints) {
            grid_arrive();
            // speculative scan for the next pass (every active run must continue from sums)
            bool ok = spec_ready && np <= a.tile && it + 1 < a.it_end && it + 1 < a.max_iters;
            for (int r = 0; r < R && ok; ++r) ok = !run_active(rs.state[r]) || rs.state[r] == kActiveFromSums;
            if (ok) {
                scan_tile(0, np, s_qn + tile_parity, s_dspec);
                spec_scanned = true;
            }
            grid_wait();
        } else {
            grid_barrier();
        }
        stamp(5);

        // ---- fused update (identical in every block): sums += grid deltas, the next pass's
        // centroids and drifts (one thread per (cluster, coordinate)), then one warp per run
        // decides (sampler.py:99-116), reduces its drifts, advances its shrink table, and
        // every thread commits the centroids of the runs that go on.
        if (tid < R) rs.chg_g[tid] = __ldcg(a.chg + (buf * kMaxRuns + tid) * kChgStride);
        for (int x0 = 0; x0 < K * kMaxKnobs; x0 += blockDim.x) {
            const int x = x0 + tid;
            const int g = x >> 3, i = x & 7;
            const int r = x < K * kMaxKnobs ? run_of[g] : 0;
            const bool live = x < K * kMaxKnobs && run_active(rs.state[r]);
            double dlt2 = 0.0;
            long long cnt_new = 0;
            if (live) {
                const long long cnt = S[g * kSumW + 8] + (long long)__ldcg(Dcur + size_t(g * kSumW + 8) * ds);
                cnt_new = cnt;
                double c = 0.0;
                if (i < n) {
                    const long long sv = S[g * kSumW + i] + (long long)__ldcg(Dcur + size_t(g * kSumW + i) * ds);
                    S[g * kSumW + i] = sv;
                    if (cnt > 0) c = __ddiv_rn(double(sv), double(cnt));
                }
                cnext[g * kMaxKnobs + i] = c;
                const double dlt = c - c64[g * kMaxKnobs + i];
                dlt2 = dlt * dlt;
                if (i == 7 && cnt == 0) rs.empty[r] = 1;
            }
            __syncwarp();  // every lane of the cluster has read the old count
            if (live && i == 7) S[g * kSumW + 8] = cnt_new;
            dlt2 += __shfl_xor_sync(0xffffffffu, dlt2, 1);
            dlt2 += __shfl_xor_sync(0xffffffffu, dlt2, 2);
            dlt2 += __shfl_xor_sync(0xffffffffu, dlt2, 4);
            if (live && i == 0) drift[g] = drift_up(dlt2);
        }
        for (int i = tid; i < K * kDeltaW; i += blockDim.x) delta[i] = 0;  // also clears delta64
        if (RESIDENT && kDeltaMode == 2)
            for (int i = tid; i < nwarps_blk * K * kDeltaW; i += blockDim.x) delta_w[i] = 0;
        stamp(6);
        __syncthreads();
        stamp(7);
        {
            const int w = tid >> 5;
            if (w < R) {
                const int r = w;
                int st = rs.state[r];
                if (run_active(st)) {
                    if (!rs.chg_g[r]) st = kConverged;
                    else if (it == a.max_iters - 1) st = kMaxed;
                    else if (rs.empty[r]) st = kNeedsReseed;
                    else st = kActiveFromSums;
                    if (lane == 0) {
                        if (st != kActiveFromSums && blockIdx.x == 0) a.run_iter[r] = it;
                        if (st == kNeedsReseed) rs.exit_flag[it & 1] = 1;
                        if (st == kActiveFromSums) atomicAdd(&rs.n_active[it & 1], 1);
                    }
                    if (st == kActiveFromSums && it + 1 < a.it_end) {
                        // m1 = largest drift, amax = its first index, m2 = largest of the others
                        // (at the launch's last pass the next launch's entry phase does this)
                        const int k = a.k[r], co = a.coff[r];
                        const float d0 = lane < k ? drift[co + lane] : 0.0f;
                        const float d1 = lane + 32 < k ? drift[co + lane + 32] : 0.0f;
                        const unsigned b0 = __float_as_uint(d0), b1 = __float_as_uint(d1);
                        const unsigned mx = __reduce_max_sync(0xffffffffu, b0 > b1 ? b0 : b1);
                        const unsigned h0 = __ballot_sync(0xffffffffu, lane < k && b0 == mx);
                        const unsigned h1 = __ballot_sync(0xffffffffu, lane + 32 < k && b1 == mx);
                        const int am = h0 ? __ffs(h0) - 1 : 32 + __ffs(h1) - 1;
                        const unsigned o0 = (lane < k && lane != am) ? b0 : 0u;
                        const unsigned o1 = (lane + 32 < k && lane + 32 != am) ? b1 : 0u;
                        const float m1 = __uint_as_float(mx);
                        const float m2 = __uint_as_float(__reduce_max_sync(0xffffffffu, o0 > o1 ? o0 : o1));
                        const float s0 = __fadd_ru(d0, lane == am ? m2 : m1), s1 = __fadd_ru(d1, lane + 32 == am ? m2 : m1);
                        const float n0 = lane < k ? __fadd_ru(dcum[co + lane], s0) : 0.0f;
                        const float n1 = lane + 32 < k ? __fadd_ru(dcum[co + lane + 32], s1) : 0.0f;
                        if (lane < k) dcum[co + lane] = n0;
                        if (lane + 32 < k) dcum[co + lane + 32] = n1;
                        if (KT_LLOYD_SPEC && RESIDENT && P >= kSpecMinPoints) {
                            // check the speculative table this pass's scan used, then the next one:
                            // D_a(t+2) estimate = D_a(t+1) + kSpecFactor x this pass's largest step
                            const bool bad = (lane < k && !(n0 <= s_dspec[co + lane])) ||
                                             (lane + 32 < k && !(n1 <= s_dspec[co + lane + 32]));
                            if (__any_sync(0xffffffffu, bad) && lane == 0) {
                                rs.spec_bad[it & 1] = 1;
                                s_qn[tile_parity] = 0;  // drop the speculative queue (its scan ended before the wait)
                            }
                            float G0, G1;
                            if (KT_SPEC_PERCLUSTER) {  // each cluster's own last step
                                G0 = __fmul_ru(s0, a.spec_factor);
                                G1 = __fmul_ru(s1, a.spec_factor);
                            } else {  // the run's largest last step
                                const float stepmax = __uint_as_float(__reduce_max_sync(
                                    0xffffffffu, __float_as_uint(fmaxf(lane < k ? s0 : 0.0f, lane + 32 < k ? s1 : 0.0f))));
                                G0 = G1 = __fmul_ru(stepmax, a.spec_factor);
                            }
                            if (lane < k) s_dspec[co + lane] = __fadd_ru(n0, G0);
                            if (lane + 32 < k) s_dspec[co + lane + 32] = __fadd_ru(n1, G1);
                        }
                    }
                    __syncwarp();  // every lane has read rs.state[r]
                    if (lane == 0) {
                        rs.state[r] = st;
                        rs.changed[r] = 0;
                    }
                }
            }
        }
        stamp(8);
        // same phase: commit the next pass's centroids of the runs that go on (converged /
        // maxed runs keep the centroids of their last pass: the reference's result; reseeds
        // are set by the host).  "Goes on" is decided from inputs this phase does not write
        // (a run that was inactive never sets its changed flag), so no barrier in between.
        for (int x = tid; x < K * kMaxKnobs && it + 1 < a.it_end; x += blockDim.x) {
            const int g = x >> 3, r = run_of[g];
            if (rs.chg_g[r] && it != a.max_iters - 1 && !rs.empty[r]) {
                const double c = cnext[x];
                c64[x] = c;
                c32[x] = float(c);
                c2[c2_slot(g, x & 7)] = float(c);
                if (blockIdx.x == 0) a.cent[x] = c;
            }
        }
        stamp(9);
        __syncthreads();
        const bool stop = rs.exit_flag[it & 1] || rs.n_active[it & 1] == 0;
        spec_hit = spec_scanned && !rs.spec_bad[it & 1];
        if (kLloydProbes && a.stats && tid == 0 && spec_scanned) rs.cnt[0][1] += spec_hit ? 1u : 1000u;  // hits + 1000 x misses
        spec_ready = true;
        ++it;
        if (stop) break;
    }
    if (RESIDENT) {
        for (int r = 0; r < R; ++r)
            for (int i = tid; i < np; i += blockDim.x) {
                a.assign[int64_t(r) * a.stride + b0 + i] = s_asg[r * P + i];
                a.budget[int64_t(r) * a.stride + b0 + i] = s_bud[r * P + i];
            }
    }
    if (kLloydProbes && a.stats && tid < R * 3) atomicAdd(a.stats + tid, (unsigned long long)rs.cnt[tid / 3][tid % 3]);
    if (blockIdx.x == 0) {
        for (int i = tid; i < K * kSumW; i += blockDim.x) a.S[i] = S[i];
        for (int i = tid; i < K; i += blockDim.x) a.dcum[i] = dcum[i];
        if (tid < R) a.run_state[tid] = rs.state[tid];
        if (tid == 0) a.ctrl[0] = it;
    }
}

// Sharded k-means: S += all-reduced deltas, then every run's decision (one block).
__global__ void lloyd_apply_kernel(LloydArgs a, const long long* __restrict__ ext, int it) {
    __shared__ long long S[kMaxClusters * kSumW];
    const int K = a.K;
    for (int i = threadIdx.x; i < K * kSumW; i += blockDim.x) S[i] = a.S[i] + ext[i];
    __syncthreads();
    for (int i = threadIdx.x; i < K * kSumW; i += blockDim.x) a.S[i] = S[i];
    if (threadIdx.x < a.R) {
        const int r = threadIdx.x;
        const int st = a.run_state[r];
        if (run_active(st)) {
            const int ns = lloyd_decide(a, S, r, st, ext[size_t(K) * kSumW + r] != 0, it);
            if (ns != kActiveFromSums) a.run_iter[r] = it;
            a.run_state[r] = ns;
        }
    }
}

// Device-driven variant for kt_lloyd_run: the iteration counter and a freeze flag live in
// device memory, so the host can enqueue several pass -> all-reduce -> apply rounds ahead:
// once a run needs a reseed (host work) every later enqueued pass and apply is a no-op.
__global__ void lloyd_apply_dev_kernel(LloydArgs a, const long long* __restrict__ ext, int* it_dev, int* freeze) {
    __shared__ long long S[kMaxClusters * kSumW];
    __shared__ int any_reseed;
    if (*freeze) return;
    const int K = a.K;
    const int it = *it_dev;
    if (threadIdx.x == 0) any_reseed = 0;
    for (int i = threadIdx.x; i < K * kSumW; i += blockDim.x) S[i] = a.S[i] + ext[i];
    __syncthreads();
    for (int i = threadIdx.x; i < K * kSumW; i += blockDim.x) a.S[i] = S[i];
    if (threadIdx.x < a.R) {
        const int r = threadIdx.x;
        const int st = a.run_state[r];
        if (run_active(st)) {
            const int ns = lloyd_decide(a, S, r, st, ext[size_t(K) * kSumW + r] != 0, it);
            if (ns != kActiveFromSums) a.run_iter[r] = it;
            if (ns == kNeedsReseed) atomicOr(&any_reseed, 1);
            a.run_state[r] = ns;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        *it_dev = it + 1;
        if (any_reseed) *freeze = 1;
    }
}

// ============================================================ reseed helpers
__global__ void point_d2_kernel(const uint64_t* __restrict__ pts, int64_t m, int n, const RowFmt fmt,
                                const uint8_t* __restrict__ assign, const double* __restrict__ cent,
                                double* __restrict__ out) {
    for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < m; p += int64_t(gridDim.x) * blockDim.x)
        out[p] = np_sq_dist(pts[p], cent + int(assign[p]) * kMaxKnobs, n, fmt);
}

// argmax of d2 over points not in `blocked` (ties -> lowest index); per-block partials.
__global__ void __launch_bounds__(256) argmax_kernel(const double* __restrict__ d2, int64_t m,
                                                     const int64_t* blocked, int n_blocked, double* part_v,
                                                     int64_t* part_i) {
    double bv = -1.0;
    int64_t bi = -1;
    for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < m; p += int64_t(gridDim.x) * blockDim.x) {
        bool skip = false;
        for (int q = 0; q < n_blocked; ++q) skip |= blocked[q] == p;
        if (skip) continue;
        const double v = d2[p];
        if (v > bv) {
            bv = v;
            bi = p;
        }
    }
    __shared__ double s_v[256];
    __shared__ int64_t s_i[256];
    s_v[threadIdx.x] = bv;
    s_i[threadIdx.x] = bi;
    __syncthreads();
    for (int off = 128; off; off >>= 1) {
        if (threadIdx.x < off) {
            const double ov = s_v[threadIdx.x + off];
            const int64_t oi = s_i[threadIdx.x + off];
            const double mv = s_v[threadIdx.x];
            const int64_t mi = s_i[threadIdx.x];
            if (oi >= 0 && (mi < 0 || ov > mv || (ov == mv && oi < mi))) {
                s_v[threadIdx.x] = ov;
                s_i[threadIdx.x] = oi;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part_v[blockIdx.x] = s_v[0];
        part_i[blockIdx.x] = s_i[0];
    }
}


// ============================================================ orchestration
constexpr int64_t kLloydMinPerBlock = 1;  // resident kernel: fewest points per block before shrinking the grid
// up to this many points: one 16-block cluster (cluster barrier) instead of the cooperative grid
// (B200, resident kernel per launch: 1K points 0.296 -> 0.277 ms, 5K 0.344 -> 0.332, 20K 0.283 -> 0.297)
constexpr int64_t kLloydClusterMaxPoints = 8192;
constexpr int kLloydClusterBlocks = 16;

// Launch plan of one Lloyd launch over m points and K clusters in R runs: the resident
// kernel whenever the state fits shared memory, else the streaming kernel.
struct LloydPlan {
    const void* kern;
    int grid, threads;
    size_t smem;
};

static LloydPlan plan_lloyd(kt_engine* e, int64_t m, int K, int R, LloydArgs& a, bool allow_cluster = true) {
    // Resident kernel (one block per SM keeps its points' assignments and budgets
    // in shared memory for the whole launch) whenever they fit; else the
    // streaming kernel (state in global memory, dynamic chunk scheduling).
    const char* mode = std::getenv("KT_LLOYD_MODE");
    const bool force_stream = mode && std::strcmp(mode, "stream") == 0;
    // blocks of the resident kernel: one per SM, fewer for small point sets (a pass is then
    // latency-bound and its grid barrier gets cheaper with fewer arrivals)
    int blocks = int(std::max<int64_t>(1, std::min<int64_t>(e->num_sms, ceil_div(m, kLloydMinPerBlock))));
    if (const char* b = std::getenv("KT_LLOYD_BLOCKS")) blocks = std::max(1, std::min(e->num_sms, std::atoi(b)));
    // small point sets: one cluster of up to 16 blocks, synchronised by the cluster barrier
    int cluster = m <= kLloydClusterMaxPoints ? kLloydClusterBlocks : 0;
    if (const char* c = std::getenv("KT_LLOYD_CLUSTER")) cluster = std::max(0, std::min(16, std::atoi(c)));
    if (a.external || !allow_cluster) cluster = 0;
    if (cluster) blocks = cluster;
    const int64_t P = ((ceil_div(m, int64_t(blocks)) + 15) & ~int64_t(15));
    const bool bytes = a.fmt.bytes != 0;
    // byte rows: the byte kernel packs all 8 bytes (unused knobs are 0), field bound 255
    const int64_t field_max = bytes ? 255 : std::max<int64_t>(1, a.fmt.cmax);
    const bool pack3 = P * field_max < (int64_t(1) << 21) && !std::getenv("KT_LLOYD_PACK5");
    const void* kres = bytes ? (const void*)lloyd_kernel<true, true> : (const void*)lloyd_kernel<true, false>;
    const void* kstr = bytes ? (const void*)lloyd_kernel<false, true> : (const void*)lloyd_kernel<false, false>;
    cudaFuncAttributes fa{};
    fa.sharedSizeBytes = static_smem(kres);
    const int optin = smem_optin(e->device);
    // smem plan: state (+ rows when they fit) + a queue of >= kLloydQueueMin entries
    const int64_t dw_bytes = kDeltaMode == 2 ? int64_t(kLloydResThreads / 32) * K * kDeltaW * 4 : 0;
    const int64_t avail = int64_t(optin) - int64_t(fa.sharedSizeBytes) - 16 - dw_bytes;
    const char* rows_env = std::getenv("KT_LLOYD_ROWS");  // tests: "global" = rows gathered from L2
    bool rows_res = int64_t(lloyd_resident_bytes(K, R, P, true)) + 4 * kLloydQueueMin <= avail &&
                    !(rows_env && std::strcmp(rows_env, "global") == 0);
    const int64_t base_bytes = int64_t(lloyd_resident_bytes(K, R, P, rows_res));
    const int64_t qcap = std::min<int64_t>(kLloydQueueMax, (avail - base_bytes) / 4);
    const int64_t tile = std::min<int64_t>(P, (qcap / R) & ~int64_t(3));
    const size_t res_smem = size_t(base_bytes + tile * R * 4 + 16 + dw_bytes);
    bool resident = !force_stream && P < 32768 && qcap >= kLloydQueueMin && tile >= 4;
    LloydPlan pl;
    size_t& smem = pl.smem;
    int& grid = pl.grid;
    int& threads = pl.threads;
    const void*& kern = pl.kern;
    if (resident) {
        allow_dynamic_smem((const void*)kres);
        resident = occupancy_blocks(kres, kLloydResThreads, res_smem) >= 1;
    }
    if (resident && cluster) {
        // a cluster this size must be schedulable with this shared-memory footprint (one GPC)
        if (cluster > 8 &&
            cudaFuncSetAttribute(kres, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
            cudaGetLastError();
            return plan_lloyd(e, m, K, R, a, false);
        }
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(unsigned(cluster));
        cfg.blockDim = dim3(unsigned(kLloydResThreads));
        cfg.dynamicSmemBytes = res_smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = unsigned(cluster);
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n_clusters = 0;
        if (cudaOccupancyMaxActiveClusters(&n_clusters, kres, &cfg) != cudaSuccess || n_clusters < 1) {
            cudaGetLastError();
            return plan_lloyd(e, m, K, R, a, false);  // the grid (and P) planned without a cluster
        }
    } else if (cluster) {
        return plan_lloyd(e, m, K, R, a, false);
    }
    if (resident) {
        smem = res_smem;
        grid = blocks;
        threads = kLloydResThreads;
        kern = kres;
        a.per_block = P;
        a.tile = int(tile);
        a.rows_resident = rows_res ? 1 : 0;
        a.pack3 = pack3 ? 1 : 0;
        a.spec_factor = kSpecFactor;
        // tests: 0 makes nearly every speculative scan miss (rescan path), a large factor makes
        // every one hit with many extra evaluations — both must stay bit-exact
        if (const char* f = std::getenv("KT_LLOYD_SPEC_FACTOR")) a.spec_factor = std::max(0.0f, float(std::atof(f)));
        a.cluster = cluster;
        if (const char* t = std::getenv("KT_LLOYD_TILE"))  // tests: force many tiles per block
            a.tile = std::max(4, std::min(a.tile, std::atoi(t) & ~3));
    } else {
        smem = lloyd_layout(K).total + 16;
        allow_dynamic_smem((const void*)kstr);
        const int occ = std::max(1, occupancy_blocks(kstr, kLloydThreads, smem));
        // Passes are latency-bound: small point sets run fastest with one block per SM
        // (cheaper grid barrier), large ones with every resident block (measured on
        // B200: m = 134K -> 148 blocks, m = 1M -> 444); ~900 points per block between.
        const int64_t per_sm = std::max<int64_t>(1, std::min<int64_t>(occ, ceil_div(m, int64_t(900) * e->num_sms)));
        grid = int(std::max<int64_t>(1, std::min<int64_t>(per_sm * e->num_sms, ceil_div(m, 256))));
        threads = kLloydThreads;
        kern = kstr;
        a.per_block = 0;
        a.tile = 0;
        a.rows_resident = 0;
        a.pack3 = 0;
        a.spec_factor = kSpecFactor;
        a.cluster = 0;
    }
    return pl;
}

// One Lloyd launch: cooperative (grid barrier), or as a single cluster (cluster barrier).
static void launch_lloyd(kt_engine* e, const LloydPlan& pl, LloydArgs& a) {
    void* params[] = {&a};
    if (a.cluster) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(unsigned(pl.grid));
        cfg.blockDim = dim3(unsigned(pl.threads));
        cfg.dynamicSmemBytes = pl.smem;
        cfg.stream = e->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = unsigned(pl.grid);
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        KT_CUDA(cudaLaunchKernelExC(&cfg, pl.kern, params));
    } else {
        KT_CUDA(cudaLaunchCooperativeKernel(pl.kern, pl.grid, pl.threads, params, pl.smem, e->stream));
    }
}

struct KmeansSession {
    kt_engine* e;
    const uint64_t* pts;
    int64_t m;
    int n;
    RowFmt fmt;
    uint64_t seed;
    // incremental k-means++ state
    int chosen = 0;  // centroids chosen so far
    int64_t first_idx = 0;
    std::vector<double> uniforms;  // u_1..u_62
    uint64_t* cent_rows = nullptr;
    int* d2 = nullptr;
    long long* chunk_sums = nullptr;
    double* d_uniforms = nullptr;
    int nchunks = 0;
    // resident init (init_res_kernel) when a block's rows + weights fit in shared memory
    bool init_res = false;
    int64_t init_P = 0;
    int init_nsub = 0;
    int init_sub = 0;
    size_t init_smem = 0;
    const void* init_kern = nullptr;
    long long* sub_sums = nullptr;

    KmeansSession(kt_engine* e_, const uint64_t* p, int64_t m_, int n_, const RowFmt& f, uint64_t s)
        : e(e_), pts(p), m(m_), n(n_), fmt(f), seed(s) {
        // k-means++ weights are exact integers: int32 per point, and every prefix
        // sum below 2^53 so that numpy's float64 cumsum is exact too
        double max_d2 = 0.0;
        for (int i = 0; i < n; ++i) {
            const double c = f.bytes ? 254.0 : double((1ll << f.width[i]) - 1);
            max_d2 += c * c;
        }
        if (max_d2 >= 2147483648.0 || max_d2 * double(m) >= 9007199254740992.0)
            fail(KT_ERR_UNSUPPORTED, "k-means++ weights of this space exceed the exact-integer range");
        uint32_t w[2];
        int nw = u64_words(seed, w);
        Pcg64 g = pcg64_from_seed_sequence(w, nw, nullptr, 0);
        if (m > 0xffffffffll) fail(KT_ERR_UNSUPPORTED, "k-means supports < 2^32 points");
        first_idx = int64_t(g.bounded32(uint32_t(m - 1)));
        uniforms.resize(64);
        for (auto& u : uniforms) u = g.random();
        cent_rows = static_cast<uint64_t*>(e->scratch("km.cent_rows", 64 * 8));
        d2 = static_cast<int*>(e->scratch("km.d2", size_t((m + 3) & ~int64_t(3)) * 8));  // two 16 B-aligned buffers
        nchunks = int(ceil_div(m, kInitChunk));
        chunk_sums = static_cast<long long*>(e->scratch("km.chunk_sums", size_t(nchunks) * 16));
        d_uniforms = static_cast<double*>(e->scratch("km.uniforms", 64 * 8));
        {
            const char* mode = std::getenv("KT_INIT_MODE");  // tests: "chunked" = init_kernel
            // sub-chunks: at most kInitSelPer sums per thread in the selection scan, at most
            // kInitFinPer weights per thread in the sub-chunk scan, warp-aligned
            init_P = (ceil_div(m, int64_t(e->num_sms)) + 31) & ~int64_t(31);
            const int64_t max_sub_blocks = int64_t(kInitSelPer) * kInitResThreads / e->num_sms;
            init_sub = int((ceil_div(init_P, std::max<int64_t>(1, std::min<int64_t>(max_sub_blocks, kInitMaxSub))) + 31) &
                           ~int64_t(31));
            init_nsub = int(ceil_div(init_P, int64_t(init_sub)));
            init_smem = size_t(init_P) * 12;
            const int optin = smem_optin(e->device);
            cudaFuncAttributes fa{};
            init_kern = f.bytes ? (const void*)init_res_kernel<true> : (const void*)init_res_kernel<false>;
            fa.sharedSizeBytes = static_smem(init_kern);
            init_res = !(mode && std::strcmp(mode, "chunked") == 0) && init_nsub <= kInitMaxSub &&
                       int64_t(init_nsub) * e->num_sms <= int64_t(kInitSelPer) * kInitResThreads &&
                       init_sub <= kInitFinPer * kInitResThreads &&
                       init_smem + fa.sharedSizeBytes <= size_t(optin);
            if (init_res) {
                allow_dynamic_smem(init_kern);
                init_res = occupancy_blocks(init_kern, kInitResThreads, init_smem) >= 1;
            }
            if (init_res)
                sub_sums = static_cast<long long*>(
                    e->scratch("km.init_sub", size_t(e->num_sms) * size_t(init_nsub) * 16));
        }
        auto* h = static_cast<double*>(e->staging("km.uniforms", 64 * 8));
        std::copy(uniforms.begin(), uniforms.end(), h);
        KT_CUDA(cudaMemcpyAsync(d_uniforms, h, 64 * 8, cudaMemcpyHostToDevice, e->stream));
    }

    void ensure_init(int k) {
        k = std::min<int64_t>(std::max(k, 1), 63);
        if (chosen >= k) return;
        InitArgs ia{};
        ia.pts = pts;
        ia.m = m;
        ia.n = n;
        ia.fmt = fmt;
        ia.j0 = chosen;
        ia.j1 = k;
        ia.first_idx = first_idx;
        ia.uniforms = d_uniforms;
        ia.cent_rows = cent_rows;
        ia.d2[0] = d2;
        ia.d2[1] = d2 + ((m + 3) & ~int64_t(3));
        ia.sums[0] = chunk_sums;
        ia.sums[1] = chunk_sums + nchunks;
        ia.nchunks = nchunks;
        ia.barrier = static_cast<unsigned int*>(e->scratch("km.init_barrier", 16));
        KT_CUDA(cudaMemsetAsync(ia.barrier, 0, 16, e->stream));
        if (init_res) {
            ia.per_block = init_P;
            ia.nsub = init_nsub;
            ia.sub = init_sub;
            ia.sums[0] = sub_sums;
            ia.sums[1] = sub_sums + size_t(e->num_sms) * init_nsub;
            void* params[] = {&ia};
            e->pre_launch("kmeanspp_init");
            KT_CUDA(cudaLaunchCooperativeKernel(init_kern, e->num_sms, kInitResThreads, params,
                                                init_smem, e->stream));
            e->check_launch("kmeanspp_init");
            chosen = k;
            return;
        }
        const void* kchunk = fmt.bytes ? (const void*)init_kernel<true> : (const void*)init_kernel<false>;
        const int occ = std::max(1, occupancy_blocks(kchunk, kInitThreads, 0));
        const int grid = int(std::max<int64_t>(1, std::min<int64_t>(int64_t(occ) * e->num_sms, nchunks)));
        void* params[] = {&ia};
        e->pre_launch("kmeanspp_init");
        KT_CUDA(cudaLaunchCooperativeKernel(kchunk, grid, kInitThreads, params, 0, e->stream));
        e->check_launch("kmeanspp_init");
        chosen = k;
    }

    struct RunResult {
        int k;
        int passes;
        double loss;
    };

    // Lloyd for the given ks (ascending); results in cent (device, [K][8]) and assign ([R][m]).
    std::vector<RunResult> run(const std::vector<int>& ks, std::vector<double>* history /* R==1 only */) {
        const int R = int(ks.size());
        if (R < 1 || R > kMaxRuns) fail(KT_ERR_INTERNAL, "bad run count");
        LloydArgs a{};
        a.pts = pts;
        a.m = m;
        a.n = n;
        a.fmt = fmt;
        a.bk1 = float(6.5e-5 * std::max(1.0, double(fmt.cmax) / 255.0));
        a.R = R;
        int K = 0;
        for (int r = 0; r < R; ++r) {
            a.k[r] = ks[r];
            a.coff[r] = K;
            K += ks[r];
        }
        if (K > kMaxClusters) fail(KT_ERR_INTERNAL, "too many clusters in one launch");
        a.K = K;
        a.max_iters = 100;
        ensure_init(ks.back());
        a.stride = (m + 15) & ~int64_t(15);
        a.assign = static_cast<uint8_t*>(e->scratch("km.assign", size_t(R) * a.stride));
        a.cent = static_cast<double*>(e->scratch("km.cent", size_t(K) * kMaxKnobs * 8));
        a.S = static_cast<long long*>(e->scratch("km.S", size_t(K) * kSumW * 8));
        a.D = static_cast<unsigned long long*>(e->scratch("km.D", size_t(3) * K * kSumW * kDStride * 8));
        a.chg = static_cast<unsigned int*>(e->scratch("km.chg", 3 * kMaxRuns * kChgStride * 4));
        a.work = static_cast<unsigned int*>(e->scratch("km.work", 16));
        a.run_state = static_cast<int*>(e->scratch("km.state", kMaxRuns * 4));
        a.run_iter = static_cast<int*>(e->scratch("km.iter", kMaxRuns * 4));
        a.ctrl = static_cast<int*>(e->scratch("km.ctrl", 16));
        a.barrier = static_cast<unsigned int*>(e->scratch("km.barrier", 16));
        static const bool want_stats = kLloydProbes && std::getenv("KT_LLOYD_STATS") != nullptr;
        static const bool want_slack = kLloydProbes && std::getenv("KT_LLOYD_SLACK") != nullptr;
        a.slack = nullptr;
        if (want_slack) {
            a.slack = static_cast<unsigned long long*>(e->scratch("km.slack", size_t(100) * kMaxRuns * 8 * 8));
            KT_CUDA(cudaMemsetAsync(a.slack, 0, size_t(100) * kMaxRuns * 8 * 8, e->stream));
        }
        a.stats = nullptr;
        if (want_stats) {
            a.stats = static_cast<unsigned long long*>(e->scratch("km.stats", kMaxRuns * 3 * 8));
            KT_CUDA(cudaMemsetAsync(a.stats, 0, kMaxRuns * 3 * 8, e->stream));
        }
        static const bool want_timeline = kLloydProbes && std::getenv("KT_LLOYD_TIMELINE") != nullptr;
        a.timeline = want_timeline ? static_cast<long long*>(e->scratch("km.timeline", 1600 * 8)) : nullptr;
        double* d_loss = static_cast<double*>(e->scratch("km.loss", kMaxRuns * 8));
        a.budget = static_cast<float*>(e->scratch("km.budget", size_t(R) * a.stride * sizeof(float)));
        a.dcum = static_cast<float*>(e->scratch("km.dcum", size_t(K) * sizeof(float)));
        a.init_rows = cent_rows;
        KT_CUDA(cudaMemsetAsync(a.assign, 0xff, size_t(R) * a.stride, e->stream));
        KT_CUDA(cudaMemsetAsync(a.S, 0, size_t(K) * kSumW * 8, e->stream));
        KT_CUDA(cudaMemsetAsync(a.cent, 0, size_t(K) * kMaxKnobs * 8, e->stream));
        KT_CUDA(cudaMemsetAsync(a.dcum, 0, size_t(K) * sizeof(float), e->stream));
        auto* h_state = static_cast<int*>(e->staging("km.state", 64));
        for (int r = 0; r < R; ++r) h_state[r] = kActiveFromRows;
        KT_CUDA(cudaMemcpyAsync(a.run_state, h_state, R * 4, cudaMemcpyHostToDevice, e->stream));

        const LloydPlan plan = plan_lloyd(e, m, K, R, a);
        const void* kern = plan.kern;
        const int grid = plan.grid, threads = plan.threads;
        const size_t smem = plan.smem;
        int it = 0;
        auto* h_ctrl = static_cast<int*>(e->staging("km.ctrl", 64));
        auto* h_iter = static_cast<int*>(e->staging("km.iter", 64));
        auto* h_S = static_cast<long long*>(e->staging("km.S", size_t(kMaxClusters) * kSumW * 8));
        auto* h_loss = static_cast<double*>(e->staging("km.loss", 64 * 8));
        h_cent = static_cast<double*>(e->staging("km.cent", size_t(kMaxClusters) * kMaxKnobs * 8));
        while (true) {
            KT_CUDA(cudaMemsetAsync(a.D, 0, size_t(3) * K * kSumW * kDStride * 8, e->stream));
            KT_CUDA(cudaMemsetAsync(a.chg, 0, 3 * kMaxRuns * kChgStride * 4, e->stream));
            KT_CUDA(cudaMemsetAsync(a.work, 0, 16, e->stream));
            KT_CUDA(cudaMemsetAsync(a.barrier, 0, 16, e->stream));
            a.it0 = it;
            a.it_end = history ? it + 1 : a.max_iters;
            e->pre_launch("lloyd");
            launch_lloyd(e, plan, a);
            e->check_launch("lloyd");
            ++lloyd_launches;
            if (history) {
                pairwise_loss(e, pts, m, n, fmt, a.assign, a.cent, d_loss);
                e->d2h({{h_ctrl, a.ctrl, 4}, {h_state, a.run_state, size_t(R) * 4}, {h_loss, d_loss, 8}});
            } else {
                // speculatively finish (no reseed is the common case): losses, pass counts and
                // centroids come back with the launch state in one read-back and one synchronisation
                pairwise_loss_runs(e, pts, m, n, fmt, a.assign, a.stride, a.cent, a.coff, R, d_loss);
                e->d2h({{h_ctrl, a.ctrl, 4}, {h_state, a.run_state, size_t(R) * 4}, {h_loss, d_loss, size_t(R) * 8},
                        {h_iter, a.run_iter, size_t(R) * 4}, {h_cent, a.cent, size_t(K) * kMaxKnobs * 8}});
            }
            e->sync();
            it = h_ctrl[0];
            if (history) history->push_back(h_loss[0]);
            bool reseed = false, active = false;
            for (int r = 0; r < R; ++r) {
                reseed |= h_state[r] == kNeedsReseed;
                active |= run_active(h_state[r]);
            }
            if (reseed) {
                e->d2h(h_S, a.S, size_t(K) * kSumW * 8);
                e->sync();
                for (int r = 0; r < R; ++r)
                    if (h_state[r] == kNeedsReseed) reseed_run(a, r, h_S);
                for (int r = 0; r < R; ++r)
                    if (h_state[r] == kNeedsReseed) h_state[r] = kActiveGiven;
                KT_CUDA(cudaMemcpyAsync(a.run_state, h_state, R * 4, cudaMemcpyHostToDevice, e->stream));
                continue;
            }
            if (!active) break;
        }
        std::vector<RunResult> out(R);
        if (history) {
            pairwise_loss_runs(e, pts, m, n, fmt, a.assign, a.stride, a.cent, a.coff, R, d_loss);
            e->d2h({{h_loss, d_loss, size_t(R) * 8}, {h_iter, a.run_iter, size_t(R) * 4},
                    {h_cent, a.cent, size_t(K) * kMaxKnobs * 8}});
            e->sync();
        }
        if (a.slack) {
            std::vector<unsigned long long> hsl(size_t(100) * kMaxRuns * 8);
            KT_CUDA(cudaMemcpy(hsl.data(), a.slack, hsl.size() * 8, cudaMemcpyDeviceToHost));
            for (int it2 = 0; it2 < 100; ++it2)
                for (int r = 0; r < R; ++r) {
                    const unsigned long long* c = hsl.data() + (size_t(it2) * kMaxRuns + r) * 8;
                    unsigned long long t = 0;
                    for (int b = 0; b < 8; ++b) t += c[b];
                    if (!t) continue;
                    std::fprintf(stderr, "[slack] k=%d pass %d: <=margin %llu <0.25 %llu <0.5 %llu <1 %llu <2 %llu <4 %llu <8 %llu more %llu\n",
                                 ks[r], it2, c[0], c[1], c[2], c[3], c[4], c[5], c[6], c[7]);
                }
        }
        if (a.stats) {
            unsigned long long hs[kMaxRuns * 3];
            KT_CUDA(cudaMemcpy(hs, a.stats, R * 3 * 8, cudaMemcpyDeviceToHost));
            for (int r = 0; r < R; ++r)
                std::fprintf(stderr, "[lloyd] k=%d passes=%d visits=%llu unused=%llu evaluated=%llu\n", ks[r], h_iter[r] + 1,
                             hs[r * 3], hs[r * 3 + 1], hs[r * 3 + 2]);
        }
        if (a.timeline) {
            long long tl[1600];
            KT_CUDA(cudaMemcpy(tl, a.timeline, sizeof(tl), cudaMemcpyDeviceToHost));
            int mp = 0;
            for (int r = 0; r < R; ++r) mp = std::max(mp, h_iter[r] + 1);
            for (int it = 0; it + 1 < std::min(100, mp); ++it) {
                const long long* t = tl + it * 16;
                std::fprintf(stderr, "[lloyd] pass %d: centroids %.1f us, scan %.1f us, eval %.1f us, flush %.1f us, "
                             "barrier %.1f us, rest %.1f us (update %.1f us, sync %.1f us, decide %.1f us, commit %.1f us, "
                             "final sync %.1f us; own scan %.1f us, own eval %.1f us)\n",
                             it, (t[1] - t[0]) * 1e-3, (t[2] - t[1]) * 1e-3, (t[3] - t[2]) * 1e-3, (t[4] - t[3]) * 1e-3,
                             (t[5] - t[4]) * 1e-3, (t[16] - t[5]) * 1e-3, (t[6] - t[5]) * 1e-3, (t[7] - t[6]) * 1e-3,
                             (t[8] - t[7]) * 1e-3, (t[9] - t[8]) * 1e-3, (t[16] - t[9]) * 1e-3, (t[10] - t[1]) * 1e-3,
                             (t[11] - t[2]) * 1e-3);
            }
        }
        int max_passes = 0;
        for (int r = 0; r < R; ++r) {
            out[r] = {ks[r], h_iter[r] + 1, h_loss[r]};
            max_passes = std::max(max_passes, h_iter[r] + 1);
        }
        for (int it = 0; it < max_passes; ++it) {  // algorithmic bytes of the fused passes
            int active = 0;
            for (int r = 0; r < R; ++r) active += out[r].passes > it;
            lloyd_bytes += m * (n + 1) * active;  // (n + 1) B per point per pass per k
        }
        last_args = a;
        return out;
    }

    // Empty clusters after pass `it`: non-empty -> mean, empty -> farthest
    // unblocked points by the pass's own point distances (sampler.py:104-115).
    void reseed_run(LloydArgs& a, int r, const long long* h_S) {
        const int k = a.k[r], co = a.coff[r];
        const uint8_t* asg = a.assign + size_t(r) * a.stride;
        double* cent = a.cent + size_t(co) * kMaxKnobs;  // centroids used by the pass
        auto* pd2 = static_cast<double*>(e->scratch("km.pd2", size_t(m) * 8));
        const int grid = int(std::min<int64_t>(ceil_div(m, 256), int64_t(e->num_sms) * 4));
        e->pre_launch("point_d2");
        point_d2_kernel<<<grid, 256, 0, e->stream>>>(pts, m, n, fmt, asg, cent, pd2);
        e->check_launch("point_d2");
        std::vector<int64_t> blocked;
        auto* d_blocked = static_cast<int64_t*>(e->scratch("km.blocked", 64 * 8));
        auto* pv = static_cast<double*>(e->scratch("km.part_v", size_t(grid) * 8));
        auto* pi = static_cast<int64_t*>(e->scratch("km.part_i", size_t(grid) * 8));
        auto* h_pv = static_cast<double*>(e->staging("km.part_v", size_t(grid) * 8));
        auto* h_pi = static_cast<int64_t*>(e->staging("km.part_i", size_t(grid) * 8));
        auto* h_rows = static_cast<uint64_t*>(e->staging("km.reseed_rows", 64 * 8));
        std::vector<double> newc(size_t(k) * kMaxKnobs, 0.0);
        std::vector<int> empties;
        for (int j = 0; j < k; ++j) {
            const long long* s = h_S + size_t(co + j) * kSumW;
            if (s[8] == 0) {
                empties.push_back(j);
                continue;
            }
            for (int i = 0; i < n; ++i) newc[size_t(j) * kMaxKnobs + i] = double(s[i]) / double(s[8]);
        }
        for (size_t q = 0; q < empties.size(); ++q) {
            if (!blocked.empty())
                KT_CUDA(cudaMemcpyAsync(d_blocked, blocked.data(), blocked.size() * 8, cudaMemcpyHostToDevice, e->stream));
            e->pre_launch("argmax");
            argmax_kernel<<<grid, 256, 0, e->stream>>>(pd2, m, d_blocked, int(blocked.size()), pv, pi);
            e->check_launch("argmax");
            e->d2h(h_pv, pv, size_t(grid) * 8);
            e->d2h(h_pi, pi, size_t(grid) * 8);
            e->sync();
            double bv = -1.0;
            int64_t bi = -1;
            for (int b = 0; b < grid; ++b)
                if (h_pi[b] >= 0 && (bi < 0 || h_pv[b] > bv || (h_pv[b] == bv && h_pi[b] < bi))) {
                    bv = h_pv[b];
                    bi = h_pi[b];
                }
            if (bi < 0) fail(KT_ERR_INTERNAL, "no point left to reseed an empty cluster");
            blocked.push_back(bi);
        }
        // fetch the chosen points' rows
        for (size_t q = 0; q < blocked.size(); ++q)
            e->d2h(h_rows + q, pts + blocked[q], 8);
        e->sync();
        for (size_t q = 0; q < empties.size(); ++q)
            for (int i = 0; i < n; ++i) newc[size_t(empties[q]) * kMaxKnobs + i] = double(fmt.get(h_rows[q], i));
        auto* h_c = static_cast<double*>(e->staging("km.newc", size_t(kMaxClusters) * kMaxKnobs * 8));
        std::copy(newc.begin(), newc.end(), h_c);
        KT_CUDA(cudaMemcpyAsync(cent, h_c, newc.size() * 8, cudaMemcpyHostToDevice, e->stream));
    }

    LloydArgs last_args{};
    double* h_cent = nullptr;  // host copy of the last run's centroids [K][8] (pinned staging)
    int64_t lloyd_bytes = 0;
    int lloyd_launches = 0;
};

// Batches of consecutive ks run speculatively in one Lloyd launch.
static std::vector<int> next_batch(int k0, int upper, int round) {
    static const int widths[] = {2, 2, 4, 8};
    int want = round < 4 ? widths[round] : 8;
    std::vector<int> ks;
    int total = 0;
    for (int k = k0; k <= upper && int(ks.size()) < want; ++k) {
        if (total + k > kMaxClusters) break;
        ks.push_back(k);
        total += k;
    }
    return ks;
}

struct KneeResult {
    std::vector<int> ks;
    std::vector<double> losses;
    int chosen_k = 0;
    int passes = 0;
    int64_t lloyd_bytes = 0;
    int lloyd_launches = 0;
    std::vector<double> centroids;  // chosen_k * n
    const uint8_t* assign_dev = nullptr;  // chosen run's assignment (device), valid until next engine call
};

static KneeResult knee_scan(kt_engine* e, const uint64_t* pts, int64_t m, int n, const RowFmt& fmt, uint64_t seed,
                            double knee_c, int k_max) {
    const int upper = int(std::min<int64_t>(k_max, m));
    if (upper < 8) fail(KT_ERR_VALUE, "knee scan needs at least 8 distinct points");
    KmeansSession ses(e, pts, m, n, fmt, seed);
    KneeResult res;
    double previous = INFINITY;
    int k0 = 8;
    for (int round = 0; k0 <= upper; ++round) {
        std::vector<int> ks = next_batch(k0, upper, round);
        auto out = ses.run(ks, nullptr);
        int stop = -1;
        for (size_t r = 0; r < out.size(); ++r) {
            res.ks.push_back(out[r].k);
            res.losses.push_back(out[r].loss);
            res.passes += out[r].passes;
            if (knee_c * out[r].loss > previous) {
                stop = int(r);
                break;
            }
            previous = out[r].loss;
        }
        const int pick = stop >= 0 ? stop : int(out.size()) - 1;
        const bool done = stop >= 0 || ks.back() >= upper;
        if (done) {
            res.chosen_k = ks[pick];
            const LloydArgs& a = ses.last_args;
            const double* c = ses.h_cent + size_t(a.coff[pick]) * kMaxKnobs;  // copied with the losses
            res.centroids.resize(size_t(ks[pick]) * n);
            for (int j = 0; j < ks[pick]; ++j)
                for (int i = 0; i < n; ++i) res.centroids[size_t(j) * n + i] = c[size_t(j) * kMaxKnobs + i];
            res.assign_dev = a.assign + size_t(pick) * a.stride;
            res.lloyd_bytes = ses.lloyd_bytes;
            res.lloyd_launches = ses.lloyd_launches;
            return res;
        }
        k0 = ks.back() + 1;
    }
    fail(KT_ERR_INTERNAL, "knee scan ended without a result");
}

}  // namespace kt

using namespace kt;

extern "C" {

int kt_dedup(kt_engine* e, const uint64_t* rows_dev, int64_t count, uint64_t* distinct_dev, int64_t* n_distinct) {
    KT_API_BEGIN
    *n_distinct = dedup(e, rows_dev, count, distinct_dev);
    KT_API_END
}

int kt_mode_vote(kt_engine* e, const uint64_t* rows_dev, int64_t count, int n_knobs, const int32_t* cards,
                 int32_t* mode_out) {
    KT_API_BEGIN
    const RowFmt fmt = row_fmt(cards, n_knobs);
    mode_vote(e, rows_dev, count, n_knobs, fmt, cards, mode_out);
    KT_API_END
}

int kt_kmeans(kt_engine* e, const uint64_t* points_dev, int64_t m, int n_knobs, const int32_t* cards, int k,
              uint64_t seed,
              double* centroids_out, int64_t* assignment_out, double* loss_out, double* history_out,
              int32_t* n_passes) {
    KT_API_BEGIN
    if (m < 1) fail(KT_ERR_VALUE, "kmeans needs at least one point");
    if (n_knobs < 1 || n_knobs > kMaxKnobs) fail(KT_ERR_UNSUPPORTED, "1..8 knobs supported");
    if (k < 1 || k > 63) fail(KT_ERR_UNSUPPORTED, "engine k-means supports 1 <= k <= 63");
    // n_distinct check (sampler.py:84-87) is done by the caller with kt_dedup.
    KmeansSession ses(e, points_dev, m, n_knobs, row_fmt(cards, n_knobs), seed);
    std::vector<double> hist;
    auto out = ses.run({k}, history_out ? &hist : nullptr);
    const LloydArgs& a = ses.last_args;
    std::vector<double> c(size_t(k) * kMaxKnobs);
    KT_CUDA(cudaMemcpyAsync(c.data(), a.cent, c.size() * 8, cudaMemcpyDeviceToHost, e->stream));
    std::vector<uint8_t> asg;
    if (assignment_out) {
        asg.resize(size_t(m));
        KT_CUDA(cudaMemcpyAsync(asg.data(), a.assign, size_t(m), cudaMemcpyDeviceToHost, e->stream));
    }
    e->sync();
    for (int j = 0; j < k; ++j)
        for (int i = 0; i < n_knobs; ++i) centroids_out[size_t(j) * n_knobs + i] = c[size_t(j) * kMaxKnobs + i];
    if (assignment_out)
        for (int64_t p = 0; p < m; ++p) assignment_out[p] = asg[size_t(p)];
    *loss_out = out[0].loss;
    *n_passes = out[0].passes;
    if (history_out) {
        if (int(hist.size()) != out[0].passes) fail(KT_ERR_INTERNAL, "history length mismatch");
        std::copy(hist.begin(), hist.end(), history_out);
    }
    KT_API_END
}

int kt_knee_scan(kt_engine* e, const uint64_t* points_dev, int64_t m, int n_knobs, const int32_t* cards, uint64_t seed,
                 double knee_constant, int k_max, int32_t* scanned_k, double* scanned_loss, int32_t* n_scanned,
                 double* centroids_out, int64_t* assignment_out) {
    KT_API_BEGIN
    if (n_knobs < 1 || n_knobs > kMaxKnobs) fail(KT_ERR_UNSUPPORTED, "1..8 knobs supported");
    if (k_max > 63) fail(KT_ERR_UNSUPPORTED, "engine knee scan supports k_max <= 63");
    KneeResult r = knee_scan(e, points_dev, m, n_knobs, row_fmt(cards, n_knobs), seed, knee_constant, k_max);
    *n_scanned = int32_t(r.ks.size());
    for (size_t i = 0; i < r.ks.size(); ++i) {
        scanned_k[i] = r.ks[i];
        scanned_loss[i] = r.losses[i];
    }
    std::copy(r.centroids.begin(), r.centroids.end(), centroids_out);
    if (assignment_out) {
        std::vector<uint8_t> asg(static_cast<size_t>(m));
        KT_CUDA(cudaMemcpyAsync(asg.data(), r.assign_dev, size_t(m), cudaMemcpyDeviceToHost, e->stream));
        e->sync();
        for (int64_t p = 0; p < m; ++p) assignment_out[p] = asg[size_t(p)];
    }
    KT_API_END
}

int kt_adaptive_sample(kt_engine* e, const uint64_t* rows_dev, int64_t count, int n_knobs, const int32_t* cards,
                       const uint64_t* visited_rows, int64_t n_visited, uint64_t seed, double knee_constant,
                       uint64_t* batch_out, int32_t* batch_len, kt_sample_info* info) {
    KT_API_BEGIN
    if (count < 1) fail(KT_ERR_VALUE, "trajectory is empty");
    const RowFmt fmt = row_fmt(cards, n_knobs);
    kt_sample_info local{};
    kt_sample_info& inf = info ? *info : local;
    std::memset(&inf, 0, sizeof(inf));
    std::unordered_set<uint64_t> visited(visited_rows, visited_rows + n_visited);
    auto* distinct = static_cast<uint64_t*>(e->scratch("as.distinct", size_t(count) * 8));
    const int64_t m = dedup(e, rows_dev, count, distinct);
    inf.n_distinct = m;
    int len = 0;
    if (m <= 8) {  // sampler.py:194-195
        uint64_t h[8];
        KT_CUDA(cudaMemcpyAsync(h, distinct, size_t(m) * 8, cudaMemcpyDeviceToHost, e->stream));
        e->sync();
        for (int64_t i = 0; i < m; ++i)
            if (!visited.count(h[i])) batch_out[len++] = h[i];
        *batch_len = len;
        return KT_OK;
    }
    // the mode is needed only if a centroid rounds onto a visited config: with a visited set,
    // enqueue the vote now (its histograms ride back with the knee scan's synchronisations)
    const unsigned int* mode_h = n_visited > 0 ? mode_hist_async(e, rows_dev, count, n_knobs, fmt, cards) : nullptr;
    KneeResult r = knee_scan(e, distinct, m, n_knobs, fmt, seed, knee_constant, 63);
    inf.chosen_k = r.chosen_k;
    inf.n_scanned = int32_t(r.ks.size());
    for (size_t i = 0; i < r.ks.size() && i < 56; ++i) {
        inf.scanned_k[i] = r.ks[i];
        inf.scanned_loss[i] = r.losses[i];
    }
    inf.lloyd_passes = r.passes;
    inf.lloyd_bytes = r.lloyd_bytes;
    inf.lloyd_launches = r.lloyd_launches;
    // batch assembly (sampler.py:200-215)
    bool have_mode = false;
    uint64_t mode_row = 0;
    std::unordered_set<uint64_t> taken;
    for (int j = 0; j < r.chosen_k; ++j) {
        uint64_t row = 0;
        for (int i = 0; i < n_knobs; ++i) {
            const double x = r.centroids[size_t(j) * n_knobs + i];
            const double f = std::floor(x + 0.5);
            long long idx = f < 0.0 ? 0 : (f > double(cards[i] - 1) ? cards[i] - 1 : (long long)f);
            row = fmt.set(row, i, int(idx));
        }
        if (visited.count(row)) {
            if (!have_mode) {
                int32_t md[kMaxKnobs];
                e->sync();  // (already idle: the knee scan ended with one)
                mode_from_hist(mode_h, n_knobs, cards, md);
                mode_row = 0;
                for (int i = 0; i < n_knobs; ++i) mode_row = fmt.set(mode_row, i, md[i]);
                have_mode = true;
            }
            inf.used_mode = 1;
            row = mode_row;
            if (visited.count(row)) continue;
        }
        if (taken.count(row)) continue;
        taken.insert(row);
        batch_out[len++] = row;
    }
    *batch_len = len;
    KT_API_END
}

}  // extern "C"

// ====================================================== sharded k-means
// One rank's contiguous shard of the distinct points.  The host drives the passes
// and all-reduces (sum) the int64 buffer [K][9] cluster deltas + [R] changed counts
// between kt_lloyd_pass and kt_lloyd_apply; every rank then holds the same global
// sums, so decisions and centroids are identical everywhere (exact integers).
struct kt_comm;
namespace kt {
void comm_all_reduce_i64(kt_comm* c, int64_t* buf, int64_t count);  // comm.cu
}

struct kt_lloyd {
    kt_engine* e = nullptr;
    const uint64_t* pts = nullptr;
    int64_t m = 0;
    int n = 0;
    RowFmt fmt{};
    kt::LloydArgs a{};
    kt::LloydPlan plan{};
    int it = 0;
    std::vector<void*> bufs;
    double* pd2 = nullptr;
    int* it_dev = nullptr;     // device-driven loop: [0] iteration, [1] freeze flag
    uint64_t* ext_dev = nullptr;

    void* alloc(size_t bytes) {
        void* p = nullptr;
        KT_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
        bufs.push_back(p);
        return p;
    }
    ~kt_lloyd() {
        for (void* p : bufs) cudaFree(p);
    }
};

extern "C" {

int kt_lloyd_create(kt_engine* e, const uint64_t* shard_pts_dev, int64_t shard_m, int n_knobs, const int32_t* cards,
                    int n_runs, const int32_t* ks, const uint64_t* init_rows, kt_lloyd** out) {
    KT_API_BEGIN
    if (shard_m < 1) fail(KT_ERR_VALUE, "a k-means shard needs at least one point");
    if (n_knobs < 1 || n_knobs > kMaxKnobs) fail(KT_ERR_UNSUPPORTED, "1..8 knobs supported");
    if (n_runs < 1 || n_runs > kMaxRuns) fail(KT_ERR_VALUE, "1..8 runs per launch");
    auto l = std::make_unique<kt_lloyd>();
    l->e = e;
    l->pts = shard_pts_dev;
    l->m = shard_m;
    l->n = n_knobs;
    l->fmt = row_fmt(cards, n_knobs);
    LloydArgs& a = l->a;
    a.pts = shard_pts_dev;
    a.m = shard_m;
    a.n = n_knobs;
    a.fmt = l->fmt;
    a.bk1 = float(6.5e-5 * std::max(1.0, double(l->fmt.cmax) / 255.0));
    a.R = n_runs;
    int K = 0, kmax = 0;
    for (int r = 0; r < n_runs; ++r) {
        if (ks[r] < 1 || ks[r] > 63) fail(KT_ERR_VALUE, "1 <= k <= 63");
        a.k[r] = ks[r];
        a.coff[r] = K;
        K += ks[r];
        kmax = std::max(kmax, ks[r]);
    }
    if (K > kMaxClusters) fail(KT_ERR_VALUE, "too many clusters in one launch");
    a.K = K;
    a.max_iters = 100;
    a.stride = (shard_m + 15) & ~int64_t(15);
    a.assign = static_cast<uint8_t*>(l->alloc(size_t(n_runs) * a.stride));
    a.budget = static_cast<float*>(l->alloc(size_t(n_runs) * a.stride * 4));
    a.dcum = static_cast<float*>(l->alloc(size_t(K) * 4));
    a.cent = static_cast<double*>(l->alloc(size_t(K) * kMaxKnobs * 8));
    a.S = static_cast<long long*>(l->alloc(size_t(K) * kSumW * 8));
    a.D = static_cast<unsigned long long*>(l->alloc(size_t(3) * K * kSumW * kDStride * 8));
    a.chg = static_cast<unsigned int*>(l->alloc(3 * kMaxRuns * kChgStride * 4));
    a.work = static_cast<unsigned int*>(l->alloc(16));
    a.run_state = static_cast<int*>(l->alloc(kMaxRuns * 4));
    a.run_iter = static_cast<int*>(l->alloc(kMaxRuns * 4));
    a.ctrl = static_cast<int*>(l->alloc(16));
    a.barrier = static_cast<unsigned int*>(l->alloc(16));
    auto* rows = static_cast<uint64_t*>(l->alloc(size_t(kmax) * 8));
    a.init_rows = rows;
    a.external = 1;
    cudaStream_t st = e->stream;
    KT_CUDA(cudaMemcpyAsync(rows, init_rows, size_t(kmax) * 8, cudaMemcpyHostToDevice, st));
    KT_CUDA(cudaMemsetAsync(a.assign, 0xff, size_t(n_runs) * a.stride, st));
    KT_CUDA(cudaMemsetAsync(a.S, 0, size_t(K) * kSumW * 8, st));
    KT_CUDA(cudaMemsetAsync(a.cent, 0, size_t(K) * kMaxKnobs * 8, st));
    KT_CUDA(cudaMemsetAsync(a.dcum, 0, size_t(K) * 4, st));
    std::vector<int> h(kMaxRuns, kActiveFromRows), zero(kMaxRuns, 0);
    KT_CUDA(cudaMemcpyAsync(a.run_state, h.data(), kMaxRuns * 4, cudaMemcpyHostToDevice, st));
    KT_CUDA(cudaMemsetAsync(a.run_iter, 0, kMaxRuns * 4, st));
    l->plan = plan_lloyd(e, shard_m, K, n_runs, a);
    e->sync();  // host vectors above go out of scope
    *out = l.release();
    KT_API_END
}

int kt_lloyd_destroy(kt_lloyd* l) {
    KT_API_BEGIN
    delete l;
    KT_API_END
}

int kt_lloyd_clusters(const kt_lloyd* l, int32_t* n_clusters) {
    KT_API_BEGIN
    *n_clusters = l->a.K;
    KT_API_END
}

int kt_lloyd_pass(kt_engine* e, kt_lloyd* l, uint64_t* ext_dev) {
    KT_API_BEGIN
    LloydArgs& a = l->a;
    KT_CUDA(cudaMemsetAsync(ext_dev, 0, (size_t(a.K) * kSumW + a.R) * 8, e->stream));
    KT_CUDA(cudaMemsetAsync(a.work, 0, 16, e->stream));
    KT_CUDA(cudaMemsetAsync(a.barrier, 0, 16, e->stream));
    a.ext = reinterpret_cast<unsigned long long*>(ext_dev);
    a.it0 = l->it;
    a.it_end = l->it + 1;
    a.stats = nullptr;
    a.timeline = nullptr;
    void* params[] = {&a};
    // the dynamic-smem limit is a per-function attribute: other shards / sessions may have lowered it
    allow_dynamic_smem((const void*)l->plan.kern);
    e->pre_launch("lloyd");
    KT_CUDA(cudaLaunchCooperativeKernel(l->plan.kern, l->plan.grid, l->plan.threads, params, l->plan.smem, e->stream));
    e->check_launch("lloyd");
    KT_API_END
}

int kt_lloyd_run(kt_engine* e, kt_lloyd* l, kt_comm* comm, int batch, int32_t* states_out, int32_t* passes_out,
                 int32_t* reseed_out) {
    KT_API_BEGIN
    LloydArgs& a = l->a;
    if (batch < 1) fail(KT_ERR_VALUE, "batch must be >= 1");
    const int64_t next = int64_t(a.K) * kSumW + a.R;
    if (!l->it_dev) l->it_dev = static_cast<int*>(l->alloc(16));
    if (!l->ext_dev) l->ext_dev = static_cast<uint64_t*>(l->alloc(size_t(next) * 8));
    auto* hs = static_cast<int*>(e->staging("lloyd.run", (2 * kMaxRuns + 4) * 4));
    hs[0] = l->it;
    hs[1] = 0;
    KT_CUDA(cudaMemcpyAsync(l->it_dev, hs, 8, cudaMemcpyHostToDevice, e->stream));
    a.ext = reinterpret_cast<unsigned long long*>(l->ext_dev);
    a.freeze = l->it_dev + 1;
    a.stats = nullptr;
    a.timeline = nullptr;
    allow_dynamic_smem((const void*)l->plan.kern);
    *reseed_out = 0;
    for (;;) {
        for (int c = 0; c < batch; ++c) {  // enqueued ahead: no host synchronisation inside a batch
            KT_CUDA(cudaMemsetAsync(l->ext_dev, 0, size_t(next) * 8, e->stream));
            KT_CUDA(cudaMemsetAsync(a.work, 0, 16, e->stream));
            KT_CUDA(cudaMemsetAsync(a.barrier, 0, 16, e->stream));
            a.it0 = l->it + c;  // only indexes scratch in the external pass; the decision reads it_dev
            a.it_end = a.it0 + 1;
            void* params[] = {&a};
            e->pre_launch("lloyd");
            KT_CUDA(cudaLaunchCooperativeKernel(l->plan.kern, l->plan.grid, l->plan.threads, params, l->plan.smem,
                                                e->stream));
            e->check_launch("lloyd");
            if (comm) comm_all_reduce_i64(comm, reinterpret_cast<int64_t*>(l->ext_dev), next);
            e->pre_launch("lloyd_apply_dev");
            lloyd_apply_dev_kernel<<<1, 256, 0, e->stream>>>(a, reinterpret_cast<const long long*>(l->ext_dev),
                                                             l->it_dev, l->it_dev + 1);
            e->check_launch("lloyd_apply_dev");
        }
        e->d2h(hs, l->it_dev, 8);
        e->d2h(hs + 2, a.run_state, a.R * 4);
        e->d2h(hs + 2 + kMaxRuns, a.run_iter, a.R * 4);
        e->sync();
        l->it = hs[0];
        bool active = false;
        for (int r = 0; r < a.R; ++r) active |= run_active(hs[2 + r]);
        if (hs[1] || !active) break;
    }
    a.freeze = nullptr;
    for (int r = 0; r < a.R; ++r) {
        states_out[r] = hs[2 + r];
        if (passes_out) passes_out[r] = run_active(hs[2 + r]) ? l->it : hs[2 + kMaxRuns + r] + 1;
    }
    *reseed_out = hs[1];
    KT_API_END
}

int kt_lloyd_apply(kt_engine* e, kt_lloyd* l, const uint64_t* ext_dev, int32_t* states_out, int32_t* passes_out) {
    KT_API_BEGIN
    LloydArgs& a = l->a;
    e->pre_launch("lloyd_apply");
    lloyd_apply_kernel<<<1, 256, 0, e->stream>>>(a, reinterpret_cast<const long long*>(ext_dev), l->it);
    e->check_launch("lloyd_apply");
    ++l->it;
    auto* hs = static_cast<int*>(e->staging("lloyd.state", 2 * kMaxRuns * 4));
    e->d2h(hs, a.run_state, a.R * 4);
    e->d2h(hs + kMaxRuns, a.run_iter, a.R * 4);
    e->sync();
    for (int r = 0; r < a.R; ++r) {
        states_out[r] = hs[r];
        if (passes_out) passes_out[r] = run_active(hs[r]) ? l->it : hs[kMaxRuns + r] + 1;
    }
    KT_API_END
}

int kt_lloyd_sums(kt_engine* e, kt_lloyd* l, int64_t* sums_out) {
    KT_API_BEGIN
    KT_CUDA(cudaMemcpyAsync(sums_out, l->a.S, size_t(l->a.K) * kSumW * 8, cudaMemcpyDeviceToHost, e->stream));
    e->sync();
    KT_API_END
}

int kt_lloyd_farthest(kt_engine* e, kt_lloyd* l, int run, const int64_t* blocked, int n_blocked, double* d2_out,
                      int64_t* idx_out) {
    KT_API_BEGIN
    LloydArgs& a = l->a;
    if (run < 0 || run >= a.R) fail(KT_ERR_VALUE, "bad run");
    const int64_t m = l->m;
    if (!l->pd2) l->pd2 = static_cast<double*>(l->alloc(size_t(m) * 8));
    const int grid = int(std::min<int64_t>(ceil_div(m, 256), int64_t(e->num_sms) * 4));
    e->pre_launch("point_d2");
    point_d2_kernel<<<grid, 256, 0, e->stream>>>(l->pts, m, l->n, l->fmt, a.assign + size_t(run) * a.stride,
                                                 a.cent + size_t(a.coff[run]) * kMaxKnobs, l->pd2);
    e->check_launch("point_d2");
    auto* d_blocked = static_cast<int64_t*>(e->scratch("lloyd.blocked", 64 * 8));
    if (n_blocked > 64) fail(KT_ERR_VALUE, "at most 64 blocked points");
    if (n_blocked)
        KT_CUDA(cudaMemcpyAsync(d_blocked, blocked, size_t(n_blocked) * 8, cudaMemcpyHostToDevice, e->stream));
    auto* pv = static_cast<double*>(e->scratch("lloyd.part_v", size_t(grid) * 8));
    auto* pi = static_cast<int64_t*>(e->scratch("lloyd.part_i", size_t(grid) * 8));
    e->pre_launch("argmax");
    argmax_kernel<<<grid, 256, 0, e->stream>>>(l->pd2, m, d_blocked, n_blocked, pv, pi);
    e->check_launch("argmax");
    std::vector<double> hv(grid);
    std::vector<int64_t> hi(grid);
    KT_CUDA(cudaMemcpyAsync(hv.data(), pv, size_t(grid) * 8, cudaMemcpyDeviceToHost, e->stream));
    KT_CUDA(cudaMemcpyAsync(hi.data(), pi, size_t(grid) * 8, cudaMemcpyDeviceToHost, e->stream));
    e->sync();
    double bv = -1.0;
    int64_t bi = -1;
    for (int b = 0; b < grid; ++b)
        if (hi[b] >= 0 && (bi < 0 || hv[b] > bv || (hv[b] == bv && hi[b] < bi))) {
            bv = hv[b];
            bi = hi[b];
        }
    *d2_out = bv;
    *idx_out = bi;
    KT_API_END
}

int kt_lloyd_set_centroids(kt_engine* e, kt_lloyd* l, int run, const double* centroids) {
    KT_API_BEGIN
    LloydArgs& a = l->a;
    if (run < 0 || run >= a.R) fail(KT_ERR_VALUE, "bad run");
    const int k = a.k[run];
    std::vector<double> c(size_t(k) * kMaxKnobs, 0.0);
    for (int j = 0; j < k; ++j)
        for (int i = 0; i < l->n; ++i) c[size_t(j) * kMaxKnobs + i] = centroids[size_t(j) * l->n + i];
    const int given = kActiveGiven;
    KT_CUDA(cudaMemcpyAsync(a.cent + size_t(a.coff[run]) * kMaxKnobs, c.data(), c.size() * 8, cudaMemcpyHostToDevice,
                            e->stream));
    KT_CUDA(cudaMemcpyAsync(a.run_state + run, &given, 4, cudaMemcpyHostToDevice, e->stream));
    e->sync();
    KT_API_END
}

int kt_lloyd_centroids(kt_engine* e, kt_lloyd* l, int run, double* centroids_out) {
    KT_API_BEGIN
    LloydArgs& a = l->a;
    if (run < 0 || run >= a.R) fail(KT_ERR_VALUE, "bad run");
    const int k = a.k[run];
    std::vector<double> c(size_t(k) * kMaxKnobs);
    KT_CUDA(cudaMemcpyAsync(c.data(), a.cent + size_t(a.coff[run]) * kMaxKnobs, c.size() * 8, cudaMemcpyDeviceToHost,
                            e->stream));
    e->sync();
    for (int j = 0; j < k; ++j)
        for (int i = 0; i < l->n; ++i) centroids_out[size_t(j) * l->n + i] = c[size_t(j) * kMaxKnobs + i];
    KT_API_END
}

int kt_lloyd_assignment(kt_engine* e, kt_lloyd* l, int run, int64_t* assignment_out) {
    KT_API_BEGIN
    LloydArgs& a = l->a;
    if (run < 0 || run >= a.R) fail(KT_ERR_VALUE, "bad run");
    std::vector<uint8_t> h(size_t(l->m));
    KT_CUDA(cudaMemcpyAsync(h.data(), a.assign + size_t(run) * a.stride, size_t(l->m), cudaMemcpyDeviceToHost,
                            e->stream));
    e->sync();
    for (int64_t p = 0; p < l->m; ++p) assignment_out[p] = h[size_t(p)];
    KT_API_END
}

int kt_lloyd_leaf_losses(kt_engine* e, kt_lloyd* l, int run, const int64_t* bounds, int n_leaves, double* out) {
    KT_API_BEGIN
    LloydArgs& a = l->a;
    if (run < 0 || run >= a.R) fail(KT_ERR_VALUE, "bad run");
    auto* d = static_cast<double*>(e->scratch("lloyd.leaf", size_t(std::max(n_leaves, 1)) * 8));
    for (int i = 0; i < n_leaves; ++i) {
        const int64_t lo = bounds[i], hi = bounds[i + 1];
        if (lo < 0 || hi > l->m || hi <= lo) fail(KT_ERR_VALUE, "bad leaf bounds");
        pairwise_loss(e, l->pts + lo, hi - lo, l->n, l->fmt, a.assign + size_t(run) * a.stride + lo,
                      a.cent + size_t(a.coff[run]) * kMaxKnobs, d + i);
    }
    KT_CUDA(cudaMemcpyAsync(out, d, size_t(n_leaves) * 8, cudaMemcpyDeviceToHost, e->stream));
    e->sync();
    KT_API_END
}

int kt_kmeanspp_rows(kt_engine* e, const uint64_t* points_dev, int64_t m, int n_knobs, const int32_t* cards,
                     uint64_t seed, int k, uint64_t* rows_out) {
    KT_API_BEGIN
    if (k < 1 || k > 63) fail(KT_ERR_VALUE, "1 <= k <= 63");
    if (m < 1) fail(KT_ERR_VALUE, "k-means++ needs at least one point");
    KmeansSession ses(e, points_dev, m, n_knobs, row_fmt(cards, n_knobs), seed);
    ses.ensure_init(k);
    KT_CUDA(cudaMemcpyAsync(rows_out, ses.cent_rows, size_t(k) * 8, cudaMemcpyDeviceToHost, e->stream));
    e->sync();
    KT_API_END
}

}  // extern "C"
