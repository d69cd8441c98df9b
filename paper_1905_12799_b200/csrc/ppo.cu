// ppo.cu — K4 rewards / GAE / normalisation and K5 PPO update, plus the
// run_search_round orchestration (agent.py:267-366) around K1 (rollout.cu).
//
// Reference: run_search_round reward shaping (agent.py:331-349), compute_gae
// (agent.py:191-210), ppo_update (agent.py:218-258), ppo_loss_and_grads and
// _backward (nets.py:94-171), adam_step (nets.py:189-200).
//
// Numerics.  Statistics that gate control flow or normalise data (reward and
// advantage mean / std) use numpy's pairwise float64 order (pairwise.cu); GAE
// runs in float64, one thread per episode, in the reference's reverse order;
// the master parameters and Adam moments are float64 with the reference's
// update expression.  The PPO forward/backward GEMMs run on the tensor cores
// (tcgen05 kind::tf32 with a 3xTF32 hi/lo split = fp32-accurate products, fp32
// accumulation in TMEM) with float64 split-K reduction of the weight gradients
// in a fixed order, so results are deterministic run to run and within the
// north star's fp32 tolerance of the float64 reference.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "agent.cuh"
#include "forest.cuh"
#include "pairwise.cuh"
#include "rng.cuh"

namespace kt {

// GEMMs run on the tensor cores (gemm_tc.cu, 3xTF32 tcgen05); epilogue codes:
enum Epi : int { kEpiNone = 0, kEpiBiasTanh = 1, kEpiTanhDeriv = 2, kEpiBias = 3 };

// out[i] (float64) = sum_z part[z][i] in z order
// out[i] = sum over split-K partials, fixed order: warp w sums splits z = w (mod 8)
// for the block's 32 elements (lanes), then the 8 warp sums combine in warp order.
__global__ void __launch_bounds__(256) reduce_splits_kernel(const float* __restrict__ part, int splits, int64_t count,
                                                            double* __restrict__ out) {
    __shared__ double red[8][33];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t i = int64_t(blockIdx.x) * 32 + lane;
    double s = 0.0;
    if (i < count) {
        int z = warp;
        for (; z + 24 < splits; z += 32) {
            const double x0 = part[size_t(z) * count + i], x1 = part[size_t(z + 8) * count + i];
            const double x2 = part[size_t(z + 16) * count + i], x3 = part[size_t(z + 24) * count + i];
            s += x0;
            s += x1;
            s += x2;
            s += x3;
        }
        for (; z < splits; z += 8) s += double(part[size_t(z) * count + i]);
    }
    red[warp][lane] = s;
    __syncthreads();
    if (warp == 0 && i < count) {
        double t = red[0][lane];
        for (int w = 1; w < 8; ++w) t += red[w][lane];
        out[i] = t;
    }
}

// Column sums of X[rows][cols] -> out (float64), deterministic two-level order:
// block b sums rows [b*R, (b+1)*R) — warp w takes rows r = w (mod 8), lanes take
// columns — then the 8 warp sums combine in warp order; the final kernel sums the
// block partials of one column by a fixed strided split and a fixed smem tree.
constexpr int kColsumRows = 512;

template <class Tv>
__global__ void __launch_bounds__(256) colsum_partial_kernel(const Tv* __restrict__ X, int64_t rows, int cols, int ld,
                                                             double* __restrict__ part) {
    __shared__ double red[8][33];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t r0 = int64_t(blockIdx.x) * kColsumRows, r1 = min(rows, r0 + kColsumRows);
    for (int c0 = 0; c0 < cols; c0 += 32) {
        const int c = c0 + lane;
        double s = 0.0;
        if (c < cols) {
            int64_t r = r0 + warp;
            for (; r + 24 < r1; r += 32) {  // four independent loads in flight
                const double x0 = double(X[size_t(r) * ld + c]), x1 = double(X[size_t(r + 8) * ld + c]);
                const double x2 = double(X[size_t(r + 16) * ld + c]), x3 = double(X[size_t(r + 24) * ld + c]);
                s += x0;
                s += x1;
                s += x2;
                s += x3;
            }
            for (; r < r1; r += 8) s += double(X[size_t(r) * ld + c]);
        }
        red[warp][lane] = s;
        __syncthreads();
        if (warp == 0 && c < cols) {
            double t = red[0][lane];
            for (int w = 1; w < 8; ++w) t += red[w][lane];
            part[size_t(blockIdx.x) * cols + c] = t;
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(256) colsum_final_kernel(const double* __restrict__ part, int blocks, int cols,
                                                           double* __restrict__ out) {
    __shared__ double red[256];
    const int c = blockIdx.x;
    double s = 0.0;
    for (int b = threadIdx.x; b < blocks; b += 256) s += part[size_t(b) * cols + c];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[c] = red[0];
}

// ============================================================ weights
// Dense fp32 matrices for the PPO GEMMs (row-major [out][in]), from float64 params.
struct DenseWeights {
    float* w1;   // [h][n]
    float* b1;   // [h]
    float* w2;   // [2g][h]  rows 0..g-1 = w2p, g..2g-1 = w2v
    float* b2;   // [2g]
    float* w3;   // [3n+1][2g] block diagonal: logits from hp, value from hv
    float* b3;   // [3n+1]
};

__global__ void dense_weights_kernel(const double* p, int n, int h, int g, DenseWeights d) {
    const ParamLayout L = param_layout(n, h, g);
    const int t = blockIdx.x * blockDim.x + threadIdx.x, T = gridDim.x * blockDim.x;
    for (int i = t; i < h * n; i += T) d.w1[i] = float(p[L.w1 + i]);
    for (int i = t; i < h; i += T) d.b1[i] = float(p[L.b1 + i]);
    for (int i = t; i < g * h; i += T) {
        d.w2[i] = float(p[L.w2p + i]);
        d.w2[g * h + i] = float(p[L.w2v + i]);
    }
    for (int i = t; i < g; i += T) {
        d.b2[i] = float(p[L.b2p + i]);
        d.b2[g + i] = float(p[L.b2v + i]);
    }
    const int n3 = 3 * n;
    for (int i = t; i < (n3 + 1) * 2 * g; i += T) {
        const int o = i / (2 * g), k = i % (2 * g);
        float v = 0.f;
        if (o < n3 && k < g) v = float(p[L.w3p + o * g + k]);
        if (o == n3 && k >= g) v = float(p[L.w3v + k - g]);
        d.w3[i] = v;
    }
    for (int i = t; i < n3; i += T) d.b3[i] = float(p[L.b3p + i]);
    if (t == 0) d.b3[n3] = float(p[L.b3v]);
}

// ============================================================ reward shaping / GAE
// rewards[t] = score of the configuration step t landed on (agent.py:339-342)
__global__ void gather_rewards_kernel(const double* scores, const int32_t* lengths, const int64_t* step_off,
                                      const int64_t* visit_off, int E, double* rewards) {
    const int ep = blockIdx.x;
    if (ep >= E) return;
    const int len = lengths[ep];
    for (int s = threadIdx.x; s < len; s += blockDim.x) rewards[step_off[ep] + s] = scores[visit_off[ep] + 1 + s];
}

// count: local rows; n_stat: rows of the whole round (all shards) the statistics are over
__global__ void normalize_kernel(double* x, int64_t count, int64_t n_stat, const double* sum, const double* sumsq,
                                 double floor_std, int center_only_returns, double* returns, const double* values) {
    const double mean = __ddiv_rn(*sum, double(n_stat));
    const double sd = __dsqrt_rn(__ddiv_rn(*sumsq, double(n_stat)));
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x) {
        const double v = x[i];
        if (sd < floor_std) {
            x[i] = 0.0;
            if (returns) returns[i] = values[i];
        } else {
            if (returns) returns[i] = v + values[i];
            x[i] = center_only_returns ? v : __ddiv_rn(__dsub_rn(v, mean), sd);
        }
    }
}

__global__ void mean_kernel(const double* sum, int64_t count, double* mean) { *mean = __ddiv_rn(*sum, double(count)); }

// per-episode GAE, terminal value 0 (agent.py:191-210, :230-233)
__global__ void gae_kernel(const double* rewards, const double* values, const int32_t* lengths, const int64_t* step_off,
                           int E, double gamma, double lam, double* adv) {
    const int ep = blockIdx.x * blockDim.x + threadIdx.x;
    if (ep >= E) return;
    const int64_t o = step_off[ep];
    const int len = lengths[ep];
    double acc = 0.0;
    const double gl = gamma * lam;
    for (int t = len - 1; t >= 0; --t) {
        const double next = t + 1 < len ? values[o + t + 1] : 0.0;
        const double delta = __dsub_rn(__dadd_rn(rewards[o + t], __dmul_rn(gamma, next)), values[o + t]);
        acc = __dadd_rn(delta, __dmul_rn(gl, acc));
        adv[o + t] = acc;
    }
}

// ============================================================ PPO row-wise part
// Inputs per row: logits+value z[row][3n+1], actions, old logp, advantages, returns.
// Outputs: dz[row][3n+1] (d total / d logits, d values) and per-row loss terms.
__global__ void ppo_rows_kernel(const float* z, int ldz, int n, int64_t T, int64_t T_batch, const uint16_t* actions,
                                const double* old_logp, const double* adv, const double* ret, double clip,
                                double value_coef, double entropy_coef, float* dz, double* terms /* [T][3] */) {
    for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < T; r += int64_t(gridDim.x) * blockDim.x) {
        const float* zr = z + size_t(r) * ldz;
        const uint32_t act = actions[r];
        double lp[kMaxKnobs][3], pr[kMaxKnobs][3], H[kMaxKnobs];
        double newlp = 0.0, ent = 0.0;
        for (int k = 0; k < n; ++k) {
            const double z0 = zr[3 * k], z1 = zr[3 * k + 1], z2 = zr[3 * k + 2];
            const double m = fmax(z0, fmax(z1, z2));
            const double lse = log(exp(z0 - m) + exp(z1 - m) + exp(z2 - m));
            lp[k][0] = z0 - m - lse, lp[k][1] = z1 - m - lse, lp[k][2] = z2 - m - lse;
            H[k] = 0.0;
            for (int j = 0; j < 3; ++j) {
                pr[k][j] = exp(lp[k][j]);
                H[k] -= pr[k][j] * lp[k][j];
            }
            newlp += lp[k][(act >> (2 * k)) & 3];
            ent += H[k];
        }
        const double ratio = exp(newlp - old_logp[r]);
        const double A = adv[r];
        const double clipped = fmin(fmax(ratio, 1.0 - clip), 1.0 + clip);
        const double raw = ratio * A, cl = clipped * A;
        const double objective = fmin(raw, cl);
        const double v = zr[3 * n];
        const double err = v - ret[r];
        const double invB = 1.0 / double(T_batch);  // mean over the whole round's rows (all shards)
        const double coeff = raw <= cl ? A * ratio * invB : 0.0;
        float* d = dz + size_t(r) * ldz;
        for (int k = 0; k < n; ++k) {
            const int ak = (act >> (2 * k)) & 3;
            for (int j = 0; j < 3; ++j) {
                const double onehot = j == ak ? 1.0 : 0.0;
                const double g = -coeff * (onehot - pr[k][j]) + entropy_coef * invB * pr[k][j] * (lp[k][j] + H[k]);
                d[3 * k + j] = float(g);
            }
        }
        d[3 * n] = float(value_coef * 2.0 * err * invB);
        terms[r * 3 + 0] = objective;
        terms[r * 3 + 1] = err * err;
        terms[r * 3 + 2] = ent;
    }
}

// states (rows) -> X[T][n] fp32, encode_state (space.py:181-188)
__global__ void encode_kernel(const uint64_t* rows, int64_t T, int n, const RowFmt fmt, const int32_t* cards_dev,
                              float* X) {
    for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < T; r += int64_t(gridDim.x) * blockDim.x) {
        const uint64_t row = rows[r];
        for (int k = 0; k < n; ++k)
            X[size_t(r) * n + k] = float(double(fmt.get(row, k)) / double(max(1, cards_dev[k] - 1)));
    }
}

// Adam (nets.py:189-200), float64; grads come as the concatenation in PARAM_KEYS order.
__global__ void adam_kernel(double* p, double* m, double* v, const double* g, int count, double lr, double bias1,
                            double bias2) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
        // exact reference expression order, no FMA contraction
        const double gi = g[i];
        const double mi = __dadd_rn(__dmul_rn(0.9, m[i]), __dmul_rn(1.0 - 0.9, gi));
        const double vi = __dadd_rn(__dmul_rn(0.999, v[i]), __dmul_rn(1.0 - 0.999, __dmul_rn(gi, gi)));
        m[i] = mi;
        v[i] = vi;
        const double mh = __ddiv_rn(mi, bias1), vh = __ddiv_rn(vi, bias2);
        p[i] = __dsub_rn(p[i], __ddiv_rn(__dmul_rn(lr, mh), __dadd_rn(__dsqrt_rn(vh), 1e-8)));
    }
}

// Gather the dense-layout gradients back into PARAM_KEYS order.
__global__ void gather_grads_kernel(int n, int h, int g, const double* gw1, const double* gb1, const double* gw2,
                                    const double* gb2, const double* gw3, const double* gb3, double* out) {
    const ParamLayout L = param_layout(n, h, g);
    const int t = blockIdx.x * blockDim.x + threadIdx.x, T = gridDim.x * blockDim.x;
    const int n3 = 3 * n;
    for (int i = t; i < h * n; i += T) out[L.w1 + i] = gw1[i];
    for (int i = t; i < h; i += T) out[L.b1 + i] = gb1[i];
    for (int i = t; i < g * h; i += T) {
        out[L.w2p + i] = gw2[i];
        out[L.w2v + i] = gw2[g * h + i];
    }
    for (int i = t; i < g; i += T) {
        out[L.b2p + i] = gb2[i];
        out[L.b2v + i] = gb2[g + i];
        out[L.w3v + i] = gw3[n3 * 2 * g + g + i];
    }
    for (int i = t; i < n3 * g; i += T) out[L.w3p + i] = gw3[(i / g) * 2 * g + (i % g)];
    for (int i = t; i < n3; i += T) out[L.b3p + i] = gb3[i];
    if (t == 0) out[L.b3v] = gb3[n3];
}

}  // namespace kt

// ============================================================ orchestration
struct kt_agent {
    int n = 0, h = 0, g = 0, P = 0;
    double* p64 = nullptr;
    double* m64 = nullptr;
    double* v64 = nullptr;
    int64_t t = 0;
    kt::PaddedWeights64* w64 = nullptr;
    float* dense = nullptr;
    kt::DenseWeights dw{};
    std::vector<double> host_p;
    int device = 0;
};

namespace kt {

__global__ void lengths_kernel(const int32_t* len, int E, int64_t* steps, int64_t* visits) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
        steps[e] = len[e];
        visits[e] = int64_t(len[e]) + 1;
    }
}

__global__ void compact_round_kernel(int E, int S, const int32_t* len, const int64_t* step_off,
                                     const int64_t* visit_off, const uint64_t* visited, const uint64_t* states,
                                     const uint16_t* actions, const double* logp, const double* values,
                                     uint64_t* rows_out, int32_t* steps_out, uint64_t* st_c, uint16_t* ac_c,
                                     double* lp_c, double* v_c) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= E) return;
    const int L = len[warp];
    const int64_t vo = visit_off[warp], so = step_off[warp];
    for (int s = lane; s <= L; s += 32) {
        rows_out[vo + s] = visited[int64_t(warp) * (S + 1) + s];
        steps_out[vo + s] = s;
    }
    for (int s = lane; s < L; s += 32) {
        const int64_t src = int64_t(warp) * S + s;
        st_c[so + s] = states[src];
        ac_c[so + s] = actions[src];
        lp_c[so + s] = logp[src];
        v_c[so + s] = values[src];
    }
}

__global__ void loss_report_kernel(const double* sums, int64_t T, double value_coef, double entropy_coef,
                                   double* out) {
    const double pol = -__ddiv_rn(sums[0], double(T));
    const double vl = __ddiv_rn(sums[1], double(T));
    const double ent = __ddiv_rn(sums[2], double(T));
    out[0] = pol;
    out[1] = vl;
    out[2] = ent;
    out[3] = pol + value_coef * vl - entropy_coef * ent;
}

static void refresh_dense(kt_engine* e, kt_agent* ag) {
    e->pre_launch("dense_weights");
    dense_weights_kernel<<<32, 256, 0, e->stream>>>(ag->p64, ag->n, ag->h, ag->g, ag->dw);
    e->check_launch("dense_weights");
}

template <class Tv>
static void colsum(kt_engine* e, const Tv* X, int64_t rows, int cols, int ld, double* out) {
    const int blocks = int(std::max<int64_t>(1, ceil_div(rows, kColsumRows)));
    auto* part = static_cast<double*>(e->scratch("ppo.colsum", size_t(blocks) * cols * 8));
    e->pre_launch("colsum");
    colsum_partial_kernel<Tv><<<blocks, 256, 0, e->stream>>>(X, rows, cols, ld, part);
    e->check_launch("colsum");
    e->pre_launch("colsum_final");
    colsum_final_kernel<<<cols, 256, 0, e->stream>>>(part, blocks, cols, out);
    e->check_launch("colsum_final");
}

// out[c] = sum over the (row tile, warp) partials of column c (fixed order: colsum_final)
static void colsum_parts(kt_engine* e, const double* part, int parts, int cols, double* out) {
    e->pre_launch("colsum_final");
    colsum_final_kernel<<<cols, 256, 0, e->stream>>>(part, parts, cols, out);
    e->check_launch("colsum_final");
}

// weight gradient out[M][N] (float64) = A^T B over T rows, deterministic split-K
static void wgrad(kt_engine* e, int M, int N, int64_t T, const float* A, int lda, const float* B, int ldb,
                  double* out) {
    // split-K: one wave of the GEMM kernel's 3 resident CTAs per SM, each split >= 256 rows
    // (measured on B200 at T = 135K: 3/SM 3.0 ms, 2/SM 3.4, 6/SM 4.7 per 45 launches)
    const int tiles = int(ceil_div(M, 128) * ceil_div(N, 128));
    const int splits = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(T, 256), 3 * e->num_sms / tiles)));
    auto* part = static_cast<float*>(e->scratch("ppo.wgrad", size_t(splits) * M * N * 4));
    tc_gemm(e, true, false, M, N, int(T), A, lda, B, ldb, part, N, kEpiNone, nullptr, nullptr, 0, splits);
    const int64_t count = int64_t(M) * N;
    e->pre_launch("reduce_splits");
    reduce_splits_kernel<<<int(ceil_div(count, 32)), 256, 0, e->stream>>>(part, splits, count, out);
    e->check_launch("reduce_splits");
}

}  // namespace kt

extern "C" {

int kt_agent_create(kt_engine* e, int n, int h, int g, const double* params, const double* adam_m,
                    const double* adam_v, int64_t adam_t, kt_agent** out) {
    KT_API_BEGIN
    using namespace kt;
    if (n < 1 || n > kMaxKnobs) fail(KT_ERR_UNSUPPORTED, "engine agents support 1..8 knobs");
    if (h < 1 || h > kH || g < 1 || g > kG)
        fail(KT_ERR_UNSUPPORTED, "engine agents support shared_width <= 128 and head_width <= 64");
    auto* ag = new kt_agent();
    ag->n = n, ag->h = h, ag->g = g;
    ag->P = param_layout(n, h, g).total;
    ag->t = adam_t;
    ag->device = e->device;
    ag->host_p.assign(params, params + ag->P);
    const size_t pb = size_t(ag->P) * 8;
    KT_CUDA(cudaMalloc(&ag->p64, pb));
    KT_CUDA(cudaMalloc(&ag->m64, pb));
    KT_CUDA(cudaMalloc(&ag->v64, pb));
    KT_CUDA(cudaMemcpy(ag->p64, params, pb, cudaMemcpyHostToDevice));
    KT_CUDA(cudaMemcpy(ag->m64, adam_m, pb, cudaMemcpyHostToDevice));
    KT_CUDA(cudaMemcpy(ag->v64, adam_v, pb, cudaMemcpyHostToDevice));
    KT_CUDA(cudaMalloc(&ag->w64, sizeof(PaddedWeights64)));
    const int n3 = 3 * n + 1;
    const size_t dense = size_t(h) * n + h + size_t(2 * g) * h + 2 * g + size_t(n3) * 2 * g + n3;
    KT_CUDA(cudaMalloc(&ag->dense, dense * 4));
    float* d = ag->dense;
    ag->dw.w1 = d, d += size_t(h) * n;
    ag->dw.b1 = d, d += h;
    ag->dw.w2 = d, d += size_t(2 * g) * h;
    ag->dw.b2 = d, d += 2 * g;
    ag->dw.w3 = d, d += size_t(n3) * 2 * g;
    ag->dw.b3 = d;
    *out = ag;
    KT_API_END
}

int kt_agent_destroy(kt_agent* ag) {
    KT_API_BEGIN
    if (!ag) return KT_OK;
    cudaFree(ag->p64);
    cudaFree(ag->m64);
    cudaFree(ag->v64);
    cudaFree(ag->w64);
    cudaFree(ag->dense);
    delete ag;
    KT_API_END
}

int kt_agent_get_state(kt_engine* e, const kt_agent* ag, double* params, double* adam_m, double* adam_v,
                       int64_t* adam_t) {
    KT_API_BEGIN
    const size_t pb = size_t(ag->P) * 8;
    KT_CUDA(cudaMemcpyAsync(params, ag->p64, pb, cudaMemcpyDeviceToHost, e->stream));
    KT_CUDA(cudaMemcpyAsync(adam_m, ag->m64, pb, cudaMemcpyDeviceToHost, e->stream));
    KT_CUDA(cudaMemcpyAsync(adam_v, ag->v64, pb, cudaMemcpyDeviceToHost, e->stream));
    e->sync();
    *adam_t = ag->t;
    KT_API_END
}

int kt_search_round(kt_engine* e, kt_agent* ag, const kt_forest* f, const uint64_t* starts_dev, int32_t E,
                    const int32_t* cards, int n_knobs, const uint32_t* seed_words, int n_seed_words,
                    int64_t round_index, const kt_ppo_hyper* hp, uint64_t* rows_out_dev, double* scores_out_dev,
                    int32_t* steps_out_dev, int64_t* n_out, kt_round_info* info, double* logp_out_dev,
                    double* values_out_dev) {
    return kt_search_round_ex(e, ag, f, starts_dev, E, cards, n_knobs, seed_words, n_seed_words, round_index, hp,
                              rows_out_dev, scores_out_dev, steps_out_dev, n_out, info, logp_out_dev, values_out_dev,
                              nullptr);
}

int kt_search_round_ex(kt_engine* e, kt_agent* ag, const kt_forest* f, const uint64_t* starts_dev, int32_t E,
                       const int32_t* cards, int n_knobs, const uint32_t* seed_words, int n_seed_words,
                       int64_t round_index, const kt_ppo_hyper* hp, uint64_t* rows_out_dev, double* scores_out_dev,
                       int32_t* steps_out_dev, int64_t* n_out, kt_round_info* info, double* logp_out_dev,
                       double* values_out_dev, const kt_collective* coll) {
    KT_API_BEGIN
    using namespace kt;
    if (E < 1) fail(KT_ERR_VALUE, "run_search_round needs at least one start configuration");
    if (n_knobs != ag->n) fail(KT_ERR_DIMENSION, "agent and space disagree on the knob count");
    if (f->n_knobs != n_knobs) fail(KT_ERR_DIMENSION, "model and space disagree on the knob count");
    const int S = hp->max_steps;
    if (S < 1) fail(KT_ERR_VALUE, "max_steps_per_episode == 0 is handled by the host");
    if (n_seed_words < 1 || n_seed_words > 4) fail(KT_ERR_VALUE, "seed must fit in 128 bits");
    const int n = n_knobs;
    const ParamLayout L = param_layout(ag->n, ag->h, ag->g);
    launch_pad_weights64(e, ag->p64, ag->n, ag->h, ag->g, ag->w64);
    refresh_dense(e, ag);

    // ---- K1 rollout
    RolloutArgs ra{};
    ra.w64 = ag->w64;
    ra.n = n, ra.h = ag->h, ra.g = ag->g, ra.S = S, ra.E = E;
    for (int k = 0; k < n; ++k) ra.cards[k] = cards[k];
    ra.fmt = row_fmt(cards, n);
    if (ra.fmt.bytes != f->fmt.bytes) fail(KT_ERR_DIMENSION, "model and space disagree on the row layout");
    for (int i = 0; i < n_seed_words; ++i) ra.seed_words[i] = seed_words[i];
    ra.n_seed_words = n_seed_words;
    ra.n_round_words = u64_words(uint64_t(round_index), ra.round_words);
    ra.starts = starts_dev;
    ra.ep_offset = coll ? coll->episode_offset : 0;
    // in-place SUM over the ranks of a sharded round (agents split by episode), ordered on e->stream
    auto all_reduce = [&](double* buf, int64_t count) {
        if (!coll) return;
        const int rc = coll->all_reduce_sum_f64(coll->user, buf, count);
        if (rc != 0) fail(KT_ERR_INTERNAL, "collective all-reduce failed");
    };
    const size_t slots = size_t(E) * S;
    ra.visited = static_cast<uint64_t*>(e->scratch("rl.visited", size_t(E) * (S + 1) * 8));
    ra.states = static_cast<uint64_t*>(e->scratch("rl.states", slots * 8));
    ra.actions = static_cast<uint16_t*>(e->scratch("rl.actions", slots * 2));
    ra.logp = static_cast<double*>(e->scratch("rl.logp", slots * 8));
    ra.values = static_cast<double*>(e->scratch("rl.values", slots * 8));
    ra.lengths = static_cast<int32_t*>(e->scratch("rl.lengths", size_t(E) * 4));
    launch_rollout(e, ra);

    // ---- episode-major compaction (agent.py:331-363)
    auto* lens_s = static_cast<int64_t*>(e->scratch("rl.lens_s", size_t(E) * 8));
    auto* lens_v = static_cast<int64_t*>(e->scratch("rl.lens_v", size_t(E) * 8));
    auto* off_s = static_cast<int64_t*>(e->scratch("rl.off_s", size_t(E + 1) * 8));
    auto* off_v = static_cast<int64_t*>(e->scratch("rl.off_v", size_t(E + 1) * 8));
    e->pre_launch("round_lengths");
    lengths_kernel<<<int(std::min<int64_t>(1024, ceil_div(E, 256))), 256, 0, e->stream>>>(ra.lengths, E, lens_s,
                                                                                          lens_v);
    e->check_launch("round_lengths");
    exclusive_scan(e, lens_s, off_s, E);
    exclusive_scan(e, lens_v, off_v, E);
    int64_t totals[2];
    KT_CUDA(cudaMemcpyAsync(&totals[0], off_s + E, 8, cudaMemcpyDeviceToHost, e->stream));
    KT_CUDA(cudaMemcpyAsync(&totals[1], off_v + E, 8, cudaMemcpyDeviceToHost, e->stream));
    e->sync();
    const int64_t T = totals[0], N = totals[1];
    int64_t T_all = T;  // rows of the whole round (all shards): the PPO batch and statistics size
    if (coll) {
        auto* tb = static_cast<double*>(e->scratch("rl.tglobal", 8));
        const double tv = double(T);
        KT_CUDA(cudaMemcpyAsync(tb, &tv, 8, cudaMemcpyHostToDevice, e->stream));
        all_reduce(tb, 1);
        double th = 0.0;
        KT_CUDA(cudaMemcpyAsync(&th, tb, 8, cudaMemcpyDeviceToHost, e->stream));
        e->sync();
        T_all = int64_t(th);
    }
    auto* st_c = static_cast<uint64_t*>(e->scratch("rl.st_c", size_t(T) * 8));
    auto* ac_c = static_cast<uint16_t*>(e->scratch("rl.ac_c", size_t(T) * 2));
    auto* lp_c = static_cast<double*>(e->scratch("rl.lp_c", size_t(T) * 8));
    auto* v_c = static_cast<double*>(e->scratch("rl.v_c", size_t(T) * 8));
    e->pre_launch("compact_round");
    compact_round_kernel<<<int(ceil_div(int64_t(E) * 32, 256)), 256, 0, e->stream>>>(
        E, S, ra.lengths, off_s, off_v, ra.visited, ra.states, ra.actions, ra.logp, ra.values, rows_out_dev,
        steps_out_dev, st_c, ac_c, lp_c, v_c);
    e->check_launch("compact_round");
    if (logp_out_dev) KT_CUDA(cudaMemcpyAsync(logp_out_dev, lp_c, size_t(T) * 8, cudaMemcpyDeviceToDevice, e->stream));
    if (values_out_dev)
        KT_CUDA(cudaMemcpyAsync(values_out_dev, v_c, size_t(T) * 8, cudaMemcpyDeviceToDevice, e->stream));

    // ---- K2 scores of every visited configuration, rewards = landing scores
    score_trees(e, f, rows_out_dev, N, scores_out_dev);
    auto* rew = static_cast<double*>(e->scratch("rl.rewards", size_t(T) * 8));
    e->pre_launch("gather_rewards");
    gather_rewards_kernel<<<E, 64, 0, e->stream>>>(scores_out_dev, ra.lengths, off_s, off_v, E, rew);
    e->check_launch("gather_rewards");
    auto* sc = static_cast<double*>(e->scratch("rl.scalars", 16 * 8));  // sum, mean, sumsq per statistic
    const int nb = int(std::min<int64_t>(2048, ceil_div(T, 256)));
    pairwise_sum(e, rew, T, nullptr, sc + 0);
    all_reduce(sc + 0, 1);
    e->pre_launch("mean");
    mean_kernel<<<1, 1, 0, e->stream>>>(sc + 0, T_all, sc + 1);
    e->check_launch("mean");
    pairwise_sum(e, rew, T, sc + 1, sc + 2);
    all_reduce(sc + 2, 1);
    e->pre_launch("normalize");
    normalize_kernel<<<nb, 256, 0, e->stream>>>(rew, T, T_all, sc + 0, sc + 2, 1e-8, 0, nullptr, nullptr);
    e->check_launch("normalize");

    // ---- K4 GAE + advantage normalisation (agent.py:229-242)
    auto* adv = static_cast<double*>(e->scratch("rl.adv", size_t(T) * 8));
    auto* ret = static_cast<double*>(e->scratch("rl.ret", size_t(T) * 8));
    e->pre_launch("gae");
    gae_kernel<<<int(ceil_div(E, 128)), 128, 0, e->stream>>>(rew, v_c, ra.lengths, off_s, E, hp->discount,
                                                              hp->gae_parameter, adv);
    e->check_launch("gae");
    pairwise_sum(e, adv, T, nullptr, sc + 4);
    all_reduce(sc + 4, 1);
    e->pre_launch("mean");
    mean_kernel<<<1, 1, 0, e->stream>>>(sc + 4, T_all, sc + 5);
    e->check_launch("mean");
    pairwise_sum(e, adv, T, sc + 5, sc + 6);
    all_reduce(sc + 6, 1);
    e->pre_launch("normalize");
    normalize_kernel<<<nb, 256, 0, e->stream>>>(adv, T, T_all, sc + 4, sc + 6, 1e-8, 0, ret, v_c);
    e->check_launch("normalize");

    // ---- K5 PPO epochs (nets.py:94-200)
    const int h = ag->h, g2 = 2 * ag->g, n3 = 3 * n + 1;
    // Z / dZ rows padded to a multiple of 4 floats: the GEMMs that read them (wgrad, dgrad of
    // layer 3) take the 16-byte vector-load path instead of scalar loads (25 -> 28 columns)
    const int n3p = (n3 + 3) & ~3;
    auto* X = static_cast<float*>(e->scratch("ppo.X", size_t(T) * n * 4));
    auto* H1 = static_cast<float*>(e->scratch("ppo.H1", size_t(T) * h * 4));
    auto* H2 = static_cast<float*>(e->scratch("ppo.H2", size_t(T) * g2 * 4));
    auto* Z = static_cast<float*>(e->scratch("ppo.Z", size_t(T) * n3p * 4));
    auto* dZ = static_cast<float*>(e->scratch("ppo.dZ", size_t(T) * n3p * 4));
    auto* dP2 = static_cast<float*>(e->scratch("ppo.dP2", size_t(T) * g2 * 4));
    auto* dP1 = static_cast<float*>(e->scratch("ppo.dP1", size_t(T) * h * 4));
    auto* terms = static_cast<double*>(e->scratch("ppo.terms", size_t(T) * 3 * 8));
    auto* gbuf = static_cast<double*>(e->scratch("ppo.grads", size_t(h * n + h + g2 * h + g2 + n3 * g2 + n3) * 8));
    double* gw1 = gbuf;
    double* gb1 = gw1 + h * n;
    double* gw2 = gb1 + h;
    double* gb2 = gw2 + g2 * h;
    double* gw3 = gb2 + g2;
    double* gb3 = gw3 + n3 * g2;
    auto* gflat = static_cast<double*>(e->scratch("ppo.gflat", size_t(ag->P) * 8));
    const int tiles4 = int(ceil_div(T, 128)) * 4;  // dgrad epilogue partials: (row tile, warp)
    auto* colpart = static_cast<double*>(e->scratch("ppo.colpart", size_t(tiles4) * 128 * 8));
    auto* cards_dev = static_cast<int32_t*>(e->scratch("ppo.cards", 64));
    KT_CUDA(cudaMemcpyAsync(cards_dev, cards, size_t(n) * 4, cudaMemcpyHostToDevice, e->stream));
    e->pre_launch("encode_states");
    encode_kernel<<<nb, 256, 0, e->stream>>>(st_c, T, n, ra.fmt, cards_dev, X);
    e->check_launch("encode_states");
    auto* report = static_cast<double*>(e->scratch("ppo.report", 8 * 8));
    for (int ep = 0; ep < hp->epochs; ++ep) {
        if (ep > 0) refresh_dense(e, ag);
        const DenseWeights& w = ag->dw;
        tc_gemm(e, false, true, int(T), h, n, X, n, w.w1, n, H1, h, kEpiBiasTanh, w.b1, nullptr, 0, 1);
        tc_gemm(e, false, true, int(T), g2, h, H1, h, w.w2, h, H2, g2, kEpiBiasTanh, w.b2, nullptr, 0, 1);
        tc_gemm(e, false, true, int(T), n3, g2, H2, g2, w.w3, g2, Z, n3p, kEpiBias, w.b3, nullptr, 0, 1);
        e->pre_launch("ppo_rows");
        ppo_rows_kernel<<<nb, 256, 0, e->stream>>>(Z, n3p, n, T, T_all, ac_c, lp_c, adv, ret, hp->clip, hp->value_coef,
                                                    hp->entropy_coef, dZ, terms);
        e->check_launch("ppo_rows");
        wgrad(e, n3, g2, T, dZ, n3p, H2, g2, gw3);
        colsum(e, dZ, T, n3, n3p, gb3);
        // bias gradients of layers 2 and 1 = column sums of dP2 / dP1, accumulated by the dgrad
        // epilogues (float64 per row tile and warp) instead of re-reading T x 128 from HBM
        tc_gemm(e, false, false, int(T), g2, n3, dZ, n3p, w.w3, g2, dP2, g2, kEpiTanhDeriv, nullptr, H2, g2, 1,
                colpart);
        wgrad(e, g2, h, T, dP2, g2, H1, h, gw2);
        colsum_parts(e, colpart, tiles4, g2, gb2);
        tc_gemm(e, false, false, int(T), h, g2, dP2, g2, w.w2, h, dP1, h, kEpiTanhDeriv, nullptr, H1, h, 1, colpart);
        wgrad(e, h, n, T, dP1, h, X, n, gw1);
        colsum_parts(e, colpart, tiles4, h, gb1);
        e->pre_launch("gather_grads");
        gather_grads_kernel<<<32, 256, 0, e->stream>>>(n, ag->h, ag->g, gw1, gb1, gw2, gb2, gw3, gb3, gflat);
        e->check_launch("gather_grads");
        all_reduce(gflat, ag->P);  // PPO gradient all-reduce: every rank applies the same Adam step
        ag->t += 1;
        const double bias1 = 1.0 - std::pow(0.9, double(ag->t));
        const double bias2 = 1.0 - std::pow(0.999, double(ag->t));
        e->pre_launch("adam");
        adam_kernel<<<int(ceil_div(ag->P, 256)), 256, 0, e->stream>>>(ag->p64, ag->m64, ag->v64, gflat, ag->P,
                                                                      hp->adam_step_size, bias1, bias2);
        e->check_launch("adam");
        if (ep == hp->epochs - 1) {
            auto* tsum = static_cast<double*>(e->scratch("ppo.tsum", 3 * 8));
            colsum(e, terms, T, 3, 3, tsum);
            all_reduce(tsum, 3);
            e->pre_launch("loss_report");
            loss_report_kernel<<<1, 1, 0, e->stream>>>(tsum, T_all, hp->value_coef, hp->entropy_coef, report);
            e->check_launch("loss_report");
        }
    }
    // host mirror of the parameters (checkpoints)
    KT_CUDA(cudaMemcpyAsync(ag->host_p.data(), ag->p64, size_t(ag->P) * 8, cudaMemcpyDeviceToHost, e->stream));
    double rep[4];
    KT_CUDA(cudaMemcpyAsync(rep, report, 4 * 8, cudaMemcpyDeviceToHost, e->stream));
    e->sync();
    (void)L;
    *n_out = N;
    if (info) {
        info->steps = T;
        info->entries = N;
        info->guarded = 0;  // the float64 rollout needs no re-decided samples
        info->policy_loss = rep[0];
        info->value_loss = rep[1];
        info->entropy = rep[2];
        info->total = rep[3];
        info->guard_tau = 0.0;
    }
    KT_API_END
}


// compute_gae (agent.py:191-210) per episode on the device, terminal value 0: exposed for
// direct parity tests of gae_kernel.  rewards / values: [T] float64, episode-major; lengths: [E].
int kt_gae(kt_engine* e, const double* rewards_dev, const double* values_dev, const int32_t* lengths_dev, int32_t E,
           double discount, double gae_parameter, double* adv_out_dev) {
    KT_API_BEGIN
    using namespace kt;
    if (E < 1) fail(KT_ERR_VALUE, "compute_gae needs at least one episode");
    auto* lens = static_cast<int64_t*>(e->scratch("gae.lens", size_t(E) * 8));
    auto* lens2 = static_cast<int64_t*>(e->scratch("gae.lens2", size_t(E) * 8));
    auto* off = static_cast<int64_t*>(e->scratch("gae.off", size_t(E + 1) * 8));
    e->pre_launch("round_lengths");
    lengths_kernel<<<int(std::min<int64_t>(1024, ceil_div(E, 256))), 256, 0, e->stream>>>(lengths_dev, E, lens, lens2);
    e->check_launch("round_lengths");
    exclusive_scan(e, lens, off, E);
    e->pre_launch("gae");
    gae_kernel<<<int(ceil_div(E, 128)), 128, 0, e->stream>>>(rewards_dev, values_dev, lengths_dev, off, E, discount,
                                                              gae_parameter, adv_out_dev);
    e->check_launch("gae");
    KT_API_END
}
}  // extern "C"
