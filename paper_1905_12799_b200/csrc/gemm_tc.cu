// gemm_tc.cu — fp32 GEMMs on the 5th-generation tensor cores (tcgen05, kind::tf32, "3xTF32").
//
// C[m][n] = epi( sum_k A(m,k) * B(k,n) ) with the same operand conventions as
// the CUDA-core gemm in ppo.cu:
//   A(m,k) = TA ? A[k*lda + m] (MN-major) : A[m*lda + k] (K-major)
//   B(k,n) = TB ? B[n*ldb + k] (K-major)  : B[k*ldb + n] (MN-major)
// One CTA (256 threads) owns a 128 x BN output tile whose fp32 accumulator
// lives in TMEM.  K is consumed in chunks of 16: all threads stage the chunk
// into shared memory in the canonical no-swizzle UMMA layout (umma.cuh), split
// into tf32 hi and lo parts (MN-major global operands are transposed while
// staging, so the tensor core always reads K-major tiles); one thread issues
// hi*hi + hi*lo + lo*hi for each of the 2 k-groups (6 tcgen05.mma), committing
// to an mbarrier.  Two stage
// buffers let the next chunk's loads overlap the tensor core.  The dropped
// lo*lo term is 2^-22 relative, so products are fp32-accurate; accumulation is
// fp32 in TMEM.  The epilogue (bias + tanh, tanh derivative, or split-K
// partial store) reads TMEM with tcgen05.ld, one row per thread.
#include <algorithm>
#include <type_traits>

#include "common.cuh"
#include "umma.cuh"

namespace kt {

#ifndef KT_TC_THREADS
#define KT_TC_THREADS 256  // A/B on the RL step (GEMM ms per step): 128 threads x 3 CTAs 9.14, 256 x 3 8.29, 256 x 2 10.2; + specialised epilogue loops 7.78
#endif
#ifndef KT_TC_MINB
#define KT_TC_MINB 3
#endif
// 128 threads: one warp per TMEM lane quadrant.  256: two warps per quadrant (they split the
// tile's columns in the epilogue; MN-major operands are staged by one half each).
constexpr int kTcBM = 128, kTcBK = 16, kTcThreads = KT_TC_THREADS;
static_assert(kTcThreads == 128 || kTcThreads == 256, "one or two warps per TMEM lane quadrant");
#ifndef KT_TC_LOOKAHEAD
#define KT_TC_LOOKAHEAD 1  // chunks of global loads in flight ahead of the MMA issue (2 measured slower: fwd 3.55 -> 3.70 ms per RL step)
#endif

struct TcGemmArgs {
    int M, N, K;
    const float* A;
    int lda;
    const float* B;
    int ldb;
    float* C;
    int ldc;
    int epi;  // 0 none, 1 bias+tanh, 2 * (1 - aux^2), 3 bias
    const float* bias;
    const float* aux;
    int ldaux;
    int kchunk;  // K range per blockIdx.z (multiple of kTcBK)
    int BN;      // tile N (multiple of 16, <= 128)
    double* colpart;  // optional: per-(row tile, warp) float64 column sums of C, [gridDim.y * 4][N]
};

// Staging is split in two so the next chunk's global loads are in flight while the
// current chunk is converted and handed to the tensor core: load_tile fills a
// per-thread register fragment, store_tile splits it into tf32 hi/lo and writes
// the canonical K-major layout.  A thread owns `kPer` 4-element vectors per tile.
template <int ROWS_MAX, bool MN = false>
struct Frag {
    // K-major: every thread holds kPer 4-vectors; MN-major: a 4 x 4 block (threads of one half)
    static constexpr int kPer = MN ? 4 : ROWS_MAX * (kTcBK / 4) / kTcThreads;
    float4 v[kPer];
};
// MN-major staging: the thread half that stages operand `b_op` (both halves of a 128-thread CTA)
__device__ __forceinline__ int mn_thread(bool b_op) {
    return kTcThreads == 256 && b_op ? int(threadIdx.x) - 128 : int(threadIdx.x);
}

template <bool MN_MAJOR, int ROWS_MAX>
__device__ __forceinline__ void load_tile(Frag<ROWS_MAX, MN_MAJOR>& fr, const float* __restrict__ G, int ld, int rows,
                                          int r0, int rlimit, int k0, int klimit, bool vec_ok, bool b_op) {
    if constexpr (MN_MAJOR) {
        // MN-major G[k * ld + r]: a thread owns a 4-row x 4-k block — four 16-byte loads along r
        // (coalesced across lanes), transposed to K-major in store_tile
        const int b = mn_thread(b_op), rgn = rows >> 2;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) fr.v[kk] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (b >= 0 && b < rows) {
            const int rb = b % rgn, kb = b / rgn;
            const int gr = r0 + 4 * rb;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const int gk = k0 + 4 * kb + kk;
                if (gk >= klimit) continue;
                const float* src = G + size_t(gk) * ld + gr;
                if (vec_ok && gr + 3 < rlimit) {
                    fr.v[kk] = __ldg(reinterpret_cast<const float4*>(src));
                } else {
                    float v[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        if (gr + e < rlimit) v[e] = __ldg(src + e);
                    fr.v[kk] = make_float4(v[0], v[1], v[2], v[3]);
                }
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < Frag<ROWS_MAX>::kPer; ++i) {
            const int f = threadIdx.x + i * kTcThreads;
            float v[4] = {0.f, 0.f, 0.f, 0.f};
            if (f < rows * (kTcBK / 4)) {
                // K-major: G[(r0 + r) * ld + k0 + k]
                const int r = f / (kTcBK / 4), kq = f % (kTcBK / 4);
                const int gr = r0 + r, gk = k0 + 4 * kq;
                if (gr < rlimit) {
                    const float* src = G + size_t(gr) * ld + gk;
                    if (vec_ok && gk + 3 < klimit) {
                        const float4 q = __ldg(reinterpret_cast<const float4*>(src));
                        v[0] = q.x, v[1] = q.y, v[2] = q.z, v[3] = q.w;
                    } else {
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            if (gk + e < klimit) v[e] = __ldg(src + e);
                    }
                }
            }
            fr.v[i] = make_float4(v[0], v[1], v[2], v[3]);
        }
    }
}

template <bool MN_MAJOR, int ROWS_MAX>
__device__ __forceinline__ void store_tile(const Frag<ROWS_MAX, MN_MAJOR>& fr, float* hi, float* lo, int rows,
                                           bool b_op) {
    if constexpr (MN_MAJOR) {
        const int b = mn_thread(b_op), rgn = rows >> 2;
        if (b < 0 || b >= rows) return;
        const int rb = b % rgn, kb = b / rgn;
        const float* f0 = reinterpret_cast<const float*>(&fr.v[0]);
        const float* f1 = reinterpret_cast<const float*>(&fr.v[1]);
        const float* f2 = reinterpret_cast<const float*>(&fr.v[2]);
        const float* f3 = reinterpret_cast<const float*>(&fr.v[3]);
#pragma unroll
        for (int j = 0; j < 4; ++j) {  // row 4rb + j: its four k values of k-quad kb
            const int r = 4 * rb + j;
            const int off = kb * rows * 4 + (r >> 3) * 32 + (r & 7) * 4;
            float4 h, l;
            umma::split_tf32(f0[j], h.x, l.x);
            umma::split_tf32(f1[j], h.y, l.y);
            umma::split_tf32(f2[j], h.z, l.z);
            umma::split_tf32(f3[j], h.w, l.w);
            *reinterpret_cast<float4*>(hi + off) = h;
            *reinterpret_cast<float4*>(lo + off) = l;
        }
    } else {
#pragma unroll
        for (int i = 0; i < Frag<ROWS_MAX>::kPer; ++i) {
            const int f = threadIdx.x + i * kTcThreads;
            if (f >= rows * (kTcBK / 4)) break;
            const int r = f / (kTcBK / 4), kq = f % (kTcBK / 4);
            const int off = kq * rows * 4 + (r >> 3) * 32 + (r & 7) * 4;
            float4 h, l;
            umma::split_tf32(fr.v[i].x, h.x, l.x);
            umma::split_tf32(fr.v[i].y, h.y, l.y);
            umma::split_tf32(fr.v[i].z, h.z, l.z);
            umma::split_tf32(fr.v[i].w, h.w, l.w);
            *reinterpret_cast<float4*>(hi + off) = h;
            *reinterpret_cast<float4*>(lo + off) = l;
        }
    }
}

// Shared tiles are always K-major (canonical no-swizzle layout, umma.cuh).
__device__ __forceinline__ uint64_t tile_desc(uint32_t base, int rows, int j) {
    return umma::smem_desc(base + uint32_t(2 * j * rows * 16), uint32_t(rows * 16), 128u);
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(kTcThreads, KT_TC_MINB) tc_gemm_kernel(TcGemmArgs g) {
    extern __shared__ __align__(1024) unsigned char s_dyn[];
    __shared__ uint64_t mma_bar[2];
    __shared__ uint32_t tmem_slot;
    constexpr bool A_MN = TA, B_MN = !TB;  // global-memory majorness (staging transposes MN-major)
    const int BN = g.BN;
    float* base = reinterpret_cast<float*>(align_shared<1024>(s_dyn));
    const int a_floats = kTcBM * kTcBK, b_floats = BN * kTcBK;
    const int stage_floats = 2 * a_floats + 2 * b_floats;  // A hi, A lo, B hi, B lo
    const int tid = threadIdx.x, warp = tid >> 5;
    const int m0 = blockIdx.y * kTcBM, n0 = blockIdx.x * BN;
    const int kbeg = blockIdx.z * g.kchunk, kend = min(g.K, kbeg + g.kchunk);
    const int nchunks = kend > kbeg ? (kend - kbeg + kTcBK - 1) / kTcBK : 0;
    const uint32_t ncols = BN <= 32 ? 32u : (BN <= 64 ? 64u : 128u);

    if (tid == 0) {
        umma::mbar_init(umma::smem_addr(&mma_bar[0]), 1);
        umma::mbar_init(umma::smem_addr(&mma_bar[1]), 1);
        umma::mbar_fence_init();
    }
    if (warp == 0) umma::tmem_alloc(umma::smem_addr(&tmem_slot), ncols);
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tmem = tmem_slot;
    const uint32_t idesc = umma::idesc_tf32(BN, false, false);
    const bool a_vec = (g.lda % 4) == 0 && (reinterpret_cast<uintptr_t>(g.A) % 16) == 0;
    const bool b_vec = (g.ldb % 4) == 0 && (reinterpret_cast<uintptr_t>(g.B) % 16) == 0;

    // one chunk's MMAs: split into tf32 hi/lo in stage s, then one thread issues them
    // `prefetch` runs between the proxy fence and the block barrier: the fence waits for every
    // outstanding memory operation of the thread, so loads issued before it would be drained
    // there (the next chunk's global loads are only in flight across the MMA if issued after)
    using FragA = Frag<kTcBM, A_MN>;
    using FragB = Frag<128, B_MN>;
    auto stage_and_issue = [&](const FragA& A, const FragB& B, int cc, auto&& prefetch) {
        const int s = cc & 1;
        if (cc >= 2) umma::mbar_wait(umma::smem_addr(&mma_bar[s]), uint32_t((cc - 2) >> 1) & 1u);
        float* st = base + s * stage_floats;
        float *a_hi = st, *a_lo = st + a_floats, *b_hi = st + 2 * a_floats, *b_lo = b_hi + b_floats;
        store_tile<A_MN, kTcBM>(A, a_hi, a_lo, kTcBM, false);
        store_tile<B_MN, 128>(B, b_hi, b_lo, BN, true);
        umma::fence_async_smem();
        prefetch();
        __syncthreads();
        if (tid == 0) {
            umma::fence_after();
            const uint32_t ah = umma::smem_addr(a_hi), al = umma::smem_addr(a_lo);
            const uint32_t bh = umma::smem_addr(b_hi), bl = umma::smem_addr(b_lo);
#pragma unroll
            for (int j = 0; j < kTcBK / 8; ++j) {
                const uint64_t dah = tile_desc(ah, kTcBM, j), dal = tile_desc(al, kTcBM, j);
                const uint64_t dbh = tile_desc(bh, BN, j), dbl = tile_desc(bl, BN, j);
                umma::mma_tf32(tmem, dah, dbh, idesc, (cc | j) != 0);
                umma::mma_tf32(tmem, dah, dbl, idesc, 1u);
                umma::mma_tf32(tmem, dal, dbh, idesc, 1u);
            }
            umma::commit(umma::smem_addr(&mma_bar[s]));
        }
        __syncwarp();
    };
    auto load_chunk = [&](FragA& A, FragB& B, int cc) {
        const int k1 = kbeg + cc * kTcBK;
        load_tile<A_MN, kTcBM>(A, g.A, g.lda, kTcBM, m0, g.M, k1, kend, a_vec, false);
        load_tile<B_MN, 128>(B, g.B, g.ldb, BN, n0, g.N, k1, kend, b_vec, true);
    };
#if KT_TC_LOOKAHEAD == 2
    // global loads run two chunks ahead of the split + MMA issue (three register fragments,
    // statically indexed by unrolling the chunk loop by three)
    FragA fa[3];
    FragB fb[3];
    if (nchunks > 0) load_chunk(fa[0], fb[0], 0);
    if (nchunks > 1) load_chunk(fa[1], fb[1], 1);
#pragma unroll 1
    for (int c = 0; c < nchunks; c += 3) {
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            const int cc = c + t;
            if (cc >= nchunks) break;
            stage_and_issue(fa[t], fb[t], cc, [&] {
                if (cc + 2 < nchunks) load_chunk(fa[(t + 2) % 3], fb[(t + 2) % 3], cc + 2);
            });
        }
    }
#else
    FragA fa[2];
    FragB fb[2];
    if (nchunks > 0) load_chunk(fa[0], fb[0], 0);
#pragma unroll 1
    for (int c = 0; c < nchunks; c += 2) {
        // two chunks per trip so the register fragments stay statically indexed
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const int cc = c + half;
            if (cc >= nchunks) break;
            stage_and_issue(fa[half], fb[half], cc, [&] {  // overlaps this chunk's MMA
                if (cc + 1 < nchunks) load_chunk(fa[half ^ 1], fb[half ^ 1], cc + 1);
            });
        }
    }
#endif
    if (nchunks > 0) umma::mbar_wait(umma::smem_addr(&mma_bar[(nchunks - 1) & 1]), uint32_t((nchunks - 1) >> 1) & 1u);
    umma::fence_after();

    // ---- epilogue: each warp drains its 32 TMEM lanes (rows) 32 columns at a time,
    // transposes through shared memory (the stage buffers are free now) and writes
    // full 128-byte row segments, applying bias / tanh / tanh' per element.
    const int lane = tid & 31;
    const int quad = warp & 3;                      // TMEM lane quadrant = the tile's rows 32q..32q+31
    constexpr int kHalves = kTcThreads / 128;       // warps per quadrant, interleaved over 32-column groups
    float* scratch = base + warp * (32 * 33);
    float* Cz = g.C + size_t(blockIdx.z) * size_t(g.M) * g.ldc;
    for (int c0 = 32 * (warp >> 2); c0 < BN; c0 += 32 * kHalves) {
        float v[32];
        if (nchunks > 0) {
            umma::tmem_ld32(tmem + (uint32_t(quad * 32) << 16) + uint32_t(c0), v);
        } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.f;
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) scratch[lane * 33 + i] = v[i];
        __syncwarp();
        const int n = n0 + c0 + lane;
        const bool col_ok = c0 + lane < BN && n < g.N;
        const float bias = col_ok && (g.epi == 1 || g.epi == 3) ? g.bias[n] : 0.f;
        const int mbase = m0 + quad * 32;
        float hv[32];
        if (g.epi == 2) {  // all 32 aux loads in flight before any store
#pragma unroll
            for (int r = 0; r < 32; ++r)
                hv[r] = (col_ok && mbase + r < g.M) ? __ldg(g.aux + size_t(mbase + r) * g.ldaux + n) : 0.f;
        }
        // one specialised store loop per epilogue (uniform branch outside the 32-row loop);
        // csum = this warp's 32 rows of column n in row order (bias gradients), only if wanted
        auto store_rows = [&](auto op, auto want_csum) {
            double csum = 0.0;
#pragma unroll
            for (int r = 0; r < 32; ++r) {
                const int mm = mbase + r;
                if (mm >= g.M || !col_ok) continue;
                const float x = op(scratch[r * 33 + lane], r);
                Cz[size_t(mm) * g.ldc + n] = x;
                if constexpr (decltype(want_csum)::value) csum += double(x);
            }
            return csum;
        };
        auto store = [&](auto op) {
            if (g.colpart) {
                const double cs = store_rows(op, std::true_type{});
                if (col_ok) g.colpart[size_t(blockIdx.y * 4 + quad) * g.N + n] = cs;
            } else {
                store_rows(op, std::false_type{});
            }
        };
        if (g.epi == 1) store([&](float x, int) { return tanhf(x + bias); });
        else if (g.epi == 3) store([&](float x, int) { return x + bias; });
        else if (g.epi == 2) store([&](float x, int r) { return x * (1.0f - hv[r] * hv[r]); });
        else store([](float x, int) { return x; });
        __syncwarp();
    }
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc(tmem, ncols);
}

template <bool TA, bool TB>
static void launch_tc(kt_engine* e, const TcGemmArgs& a, dim3 grid, size_t smem) {
    auto kern = tc_gemm_kernel<TA, TB>;
    allow_dynamic_smem((const void*)kern);
    // per-role names so kernel_stats separates the PPO GEMM shapes
    const char* name = TA ? "tc_gemm_wgrad" : (a.epi == 2 ? "tc_gemm_dgrad" : "tc_gemm_fwd");
    e->pre_launch(name);
    kern<<<grid, kTcThreads, smem, e->stream>>>(a);
    e->check_launch(name);
}

// Public helper used by ppo.cu and kt_gemm_f32.
void tc_gemm(kt_engine* e, bool TA, bool TB, int M, int N, int K, const float* A, int lda, const float* B, int ldb,
             float* C, int ldc, int epi, const float* bias, const float* aux, int ldaux, int splits,
             double* colpart) {
    TcGemmArgs a{M, N, K, A, lda, B, ldb, C, ldc, epi, bias, aux, ldaux, 0, 0, colpart};
    if (colpart && (splits != 1 || N > 128)) fail(KT_ERR_VALUE, "tc_gemm column sums need one N tile, no split-K");
    const int n_tiles = int(ceil_div(N, 128));
    int bn = int(ceil_div(ceil_div(N, n_tiles), 16) * 16);
    bn = std::max(16, std::min(128, bn));
    a.BN = bn;
    a.kchunk = int(ceil_div(ceil_div(K, splits), kTcBK) * kTcBK);
    dim3 grid(unsigned(ceil_div(N, bn)), unsigned(ceil_div(M, kTcBM)), unsigned(splits));
    const size_t smem = size_t(2) * (2 * kTcBM * kTcBK + 2 * bn * kTcBK) * 4 + 1024;
    if (TA && TB) launch_tc<true, true>(e, a, grid, smem);
    else if (TA) launch_tc<true, false>(e, a, grid, smem);
    else if (TB) launch_tc<false, true>(e, a, grid, smem);
    else launch_tc<false, false>(e, a, grid, smem);
}

}  // namespace kt

extern "C" int kt_gemm_f32(kt_engine* e, int trans_a, int trans_b, int M, int N, int K, const float* A, int lda,
                           const float* B, int ldb, float* C, int ldc) {
    KT_API_BEGIN
    if (M < 1 || N < 1 || K < 0) kt::fail(KT_ERR_VALUE, "bad GEMM shape");
    kt::tc_gemm(e, trans_a != 0, trans_b != 0, M, N, K, A, lda, B, ldb, C, ldc, 0, nullptr, nullptr, 0, 1, nullptr);
    KT_API_END
}
