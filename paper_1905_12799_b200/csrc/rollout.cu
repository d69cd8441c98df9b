// rollout.cu — K1 policy_rollout: PPO search agents walking the knob lattice.
//
// Replaces the lockstep episode loop of run_search_round (agent.py:298-328) with
// nets.forward (nets.py:51-60), softmax / joint_log_prob (nets.py:63-80),
// _sample_actions (agent.py:261-264), encode_state and apply_action
// (space.py:167-188).  One CTA owns 128 episodes and runs all of their steps
// in-kernel: weights live in shared memory (77 KB), activations are kept
// transposed ([feature][agent]) so every lane reads its own agent's column
// while the weight operand is a broadcast float4.
//
// Determinism / parity.  Episode e draws its uniforms from
// PCG64(SeedSequence(seed, spawn_key=(round, e))) on the device, n per step
// (agent.py:292-296, :313).  The forward pass runs in fp32; an a-priori error
// bound tau (computed on the host from the weights' row norms, see
// rollout_guard_tau) brackets every |u - cdf| decision.  Any agent with a
// decision closer than tau is re-evaluated warp-cooperatively in float64 with
// the reference's formulas, so sampled actions equal the reference's except
// at measure-zero float64 boundaries (the north-star caveat).
#include <algorithm>
#include <cmath>
#include <vector>

#include "agent.cuh"
#include "rng.cuh"

namespace kt {



struct RolloutSmem {
    PaddedWeights w;
    float xt[kMaxKnobs][kAgentsPerCta];
    float h1t[kH][kAgentsPerCta];  // reused after GEMM2 for logits + float64 scratch
    float hpt[kG][kAgentsPerCta];
    float hvt[kG][kAgentsPerCta];
    double u[kAgentsPerCta][kMaxKnobs];
    uint64_t rows[kAgentsPerCta];
    double res_lp[kAgentsPerCta], res_v[kAgentsPerCta];
    uint32_t res_act[kAgentsPerCta];
    int overridden[kAgentsPerCta];
    int flagged[kAgentsPerCta];
    int n_flagged;
    int any_active;
};

// logits [agent][25] (24 logits + value) and per-warp float64 buffers live in h1t after GEMM2
constexpr int kLogitStride = kN3 + 1;

__device__ __forceinline__ double dtanh(double x) { return tanh(x); }

// float64 forward of one agent by one warp; returns logits in z[0..3n), value in *v (lane 0)
__device__ void forward64_warp(const RolloutArgs& a, const ParamLayout& L, const double x[kMaxKnobs], double* buf1,
                               double* buf2, double* z, double* v) {
    const int lane = threadIdx.x & 31;
    const double* p = a.p64;
    for (int o = lane; o < L.h; o += 32) {
        double s = p[L.b1 + o];
        for (int k = 0; k < L.n; ++k) s += x[k] * p[L.w1 + o * L.n + k];
        buf1[o] = dtanh(s);
    }
    __syncwarp();
    for (int o = lane; o < 2 * L.g; o += 32) {
        const bool pol = o < L.g;
        const int oo = pol ? o : o - L.g;
        const double* w = p + (pol ? L.w2p : L.w2v) + oo * L.h;
        double s = p[(pol ? L.b2p : L.b2v) + oo];
        for (int k = 0; k < L.h; ++k) s += buf1[k] * w[k];
        buf2[o] = dtanh(s);  // [0, g): hp, [g, 2g): hv
    }
    __syncwarp();
    for (int o = lane; o < 3 * L.n + 1; o += 32) {
        double s;
        if (o < 3 * L.n) {
            s = p[L.b3p + o];
            for (int k = 0; k < L.g; ++k) s += buf2[k] * p[L.w3p + o * L.g + k];
            z[o] = s;
        } else {
            s = p[L.b3v];
            for (int k = 0; k < L.g; ++k) s += buf2[L.g + k] * p[L.w3v + k];
            *v = s;
        }
    }
    __syncwarp();
}

__global__ void __launch_bounds__(kRolloutThreads, 1) rollout_kernel(RolloutArgs a) {
    extern __shared__ __align__(16) unsigned char s_raw[];
    RolloutSmem& sm = *reinterpret_cast<RolloutSmem*>(s_raw);
    const int tid = threadIdx.x;
    const int n = a.n;
    const ParamLayout L = param_layout(a.n, a.h, a.g);

    {  // weights -> smem
        const float4* src = reinterpret_cast<const float4*>(a.w32);
        float4* dst = reinterpret_cast<float4*>(&sm.w);
        for (int i = tid; i < int(sizeof(PaddedWeights) / 16); i += blockDim.x) dst[i] = src[i];
    }
    // per-agent state (threads 0..127 own one episode each)
    const int ag = tid;
    const int e = blockIdx.x * kAgentsPerCta + ag;
    const bool owner = ag < kAgentsPerCta && e < a.E;
    uint64_t row = 0;
    bool active = false;
    Pcg64 rng;
    if (owner) {
        row = a.starts[e];
        active = true;
        uint32_t spawn[4];
        int ns = 0;
        for (int i = 0; i < a.n_round_words; ++i) spawn[ns++] = a.round_words[i];
        int ew = ns;
        ns += u64_words(uint64_t(e), spawn + ew);
        rng = pcg64_from_seed_sequence(a.seed_words, a.n_seed_words, spawn, ns);
        a.visited[int64_t(e) * (a.S + 1)] = row;
    }
    float* logits = &sm.h1t[0][0];  // [agent][kLogitStride] after GEMM2
    double* scratch64 = reinterpret_cast<double*>(&sm.h1t[0][0] + kAgentsPerCta * kLogitStride + 64);
    int steps = 0;
    unsigned long long guarded = 0;

    for (int s = 0; s < a.S; ++s) {
        if (tid == 0) {
            sm.any_active = 0;
            sm.n_flagged = 0;
        }
        __syncthreads();
        if (owner && active) {
            atomicOr(&sm.any_active, 1);
            for (int k = 0; k < kMaxKnobs; ++k) {
                float x = 0.0f;
                if (k < n) {
                    const int den = max(1, a.cards[k] - 1);
                    x = float(double(row_byte(row, k)) / double(den));
                }
                sm.xt[k][ag] = x;
            }
            for (int k = 0; k < n; ++k) sm.u[ag][k] = rng.random();
            sm.rows[ag] = row;
            sm.overridden[ag] = 0;
        } else if (ag < kAgentsPerCta) {
            for (int k = 0; k < kMaxKnobs; ++k) sm.xt[k][ag] = 0.0f;
        }
        __syncthreads();
        if (!sm.any_active) break;

        const int col = tid & (kAgentsPerCta - 1);
        const int half = tid >> 7;
        // ---- h1 = tanh(x W1^T + b1): this thread's 64 outputs of its column
        {
            float acc[64];
#pragma unroll
            for (int o = 0; o < 64; ++o) acc[o] = sm.w.b1[half * 64 + o];
#pragma unroll
            for (int k = 0; k < kMaxKnobs; ++k) {
                const float xk = sm.xt[k][col];
                const float4* wr = reinterpret_cast<const float4*>(&sm.w.w1t[k][half * 64]);
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    const float4 w4 = wr[q];
                    acc[4 * q] = fmaf(xk, w4.x, acc[4 * q]);
                    acc[4 * q + 1] = fmaf(xk, w4.y, acc[4 * q + 1]);
                    acc[4 * q + 2] = fmaf(xk, w4.z, acc[4 * q + 2]);
                    acc[4 * q + 3] = fmaf(xk, w4.w, acc[4 * q + 3]);
                }
            }
#pragma unroll
            for (int o = 0; o < 64; ++o) sm.h1t[half * 64 + o][col] = tanhf(acc[o]);
        }
        __syncthreads();
        // ---- [hp | hv] = tanh(h1 [W2p | W2v]^T + b): half 0 -> hp, half 1 -> hv
        {
            float acc[64];
            const float* bias = half ? sm.w.b2v : sm.w.b2p;
#pragma unroll
            for (int o = 0; o < 64; ++o) acc[o] = bias[o];
            const float* wt = half ? &sm.w.w2vt[0][0] : &sm.w.w2pt[0][0];
#pragma unroll 2
            for (int k = 0; k < kH; ++k) {
                const float hk = sm.h1t[k][col];
                const float4* wr = reinterpret_cast<const float4*>(wt + k * kG);
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    const float4 w4 = wr[q];
                    acc[4 * q] = fmaf(hk, w4.x, acc[4 * q]);
                    acc[4 * q + 1] = fmaf(hk, w4.y, acc[4 * q + 1]);
                    acc[4 * q + 2] = fmaf(hk, w4.z, acc[4 * q + 2]);
                    acc[4 * q + 3] = fmaf(hk, w4.w, acc[4 * q + 3]);
                }
            }
            float* dst = half ? &sm.hvt[0][0] : &sm.hpt[0][0];
#pragma unroll
            for (int o = 0; o < 64; ++o) dst[o * kAgentsPerCta + col] = tanhf(acc[o]);
        }
        __syncthreads();
        // ---- logits (24) from hp, value from hv: half 0 -> logits 0..11, half 1 -> 12..23 + value
        {
            float acc[13];
#pragma unroll
            for (int o = 0; o < 12; ++o) acc[o] = sm.w.b3p[half * 12 + o];
            acc[12] = sm.w.b3v;
            for (int k = 0; k < kG; ++k) {
                const float hk = sm.hpt[k][col];
                const float* wr = &sm.w.w3pt[k][half * 12];
#pragma unroll
                for (int o = 0; o < 12; ++o) acc[o] = fmaf(hk, wr[o], acc[o]);
                if (half) acc[12] = fmaf(sm.hvt[k][col], sm.w.w3v[k], acc[12]);
            }
#pragma unroll
            for (int o = 0; o < 12; ++o) logits[col * kLogitStride + half * 12 + o] = acc[o];
            if (half) logits[col * kLogitStride + kN3] = acc[12];
        }
        __syncthreads();
        // ---- sample (agent threads)
        uint32_t act = 0;
        double lp_sum = 0.0;
        if (owner && active) {
            float lps[kMaxKnobs];
            float margin = INFINITY;
            for (int k = 0; k < n; ++k) {
                const float z0 = logits[ag * kLogitStride + 3 * k], z1 = logits[ag * kLogitStride + 3 * k + 1],
                            z2 = logits[ag * kLogitStride + 3 * k + 2];
                const float mz = fmaxf(z0, fmaxf(z1, z2));
                const float lse = logf(expf(z0 - mz) + expf(z1 - mz) + expf(z2 - mz));
                const float l0 = z0 - mz - lse, l1 = z1 - mz - lse, l2 = z2 - mz - lse;
                const float c0 = expf(l0), c1 = c0 + expf(l1);
                const double uk = sm.u[ag][k];
                const int ak = (uk > double(c0)) + (uk > double(c1));
                margin = fminf(margin, fminf(fabsf(float(uk - double(c0))), fabsf(float(uk - double(c1)))));
                act |= uint32_t(ak) << (2 * k);
                lps[k] = ak == 0 ? l0 : (ak == 1 ? l1 : l2);
            }
            float lsum = 0.0f;
            for (int k = 0; k < n; ++k) lsum += lps[k];
            lp_sum = double(lsum);
            if (!(margin > a.tau)) {
                const int slot = atomicAdd(&sm.n_flagged, 1);
                sm.flagged[slot] = ag;
            }
        }
        __syncthreads();
        // ---- float64 re-evaluation of agents whose decisions fall inside the guard band
        {
            const int warp = tid >> 5, lane = tid & 31;
            for (int f = warp; f < sm.n_flagged; f += kRolloutThreads / 32) {
                const int ga = sm.flagged[f];
                const uint64_t grow = sm.rows[ga];
                double x[kMaxKnobs];
                for (int k = 0; k < kMaxKnobs; ++k)
                    x[k] = k < n ? __ddiv_rn(double(row_byte(grow, k)), double(max(1, a.cards[k] - 1))) : 0.0;
                double* buf1 = scratch64 + warp * (kH + 2 * kG + kN3 + 8);
                double* buf2 = buf1 + kH;
                double* z = buf2 + 2 * kG;
                double* vv = z + kN3;
                forward64_warp(a, L, x, buf1, buf2, z, vv);
                if (lane == 0) {
                    uint32_t act = 0;
                    double picked[kMaxKnobs];
                    for (int k = 0; k < n; ++k) {
                        const double z0 = z[3 * k], z1 = z[3 * k + 1], z2 = z[3 * k + 2];
                        const double mz = fmax(z0, fmax(z1, z2));
                        const double y0 = z0 - mz, y1 = z1 - mz, y2 = z2 - mz;
                        const double lse = log(__dadd_rn(__dadd_rn(exp(y0), exp(y1)), exp(y2)));
                        const double l0 = y0 - lse, l1 = y1 - lse, l2 = y2 - lse;
                        const double c0 = exp(l0), c1 = __dadd_rn(c0, exp(l1));
                        const double uk = sm.u[ga][k];
                        const int ak = (uk > c0) + (uk > c1);
                        act |= uint32_t(ak) << (2 * k);
                        picked[k] = ak == 0 ? l0 : (ak == 1 ? l1 : l2);
                    }
                    sm.res_act[ga] = act;
                    sm.res_lp[ga] = np_sum_small(picked, n);
                    sm.res_v[ga] = *vv;
                    sm.overridden[ga] = 1;
                }
                __syncwarp();
            }
            if (tid == 0) guarded += sm.n_flagged;
        }
        __syncthreads();
        if (owner && active && sm.overridden[ag]) {
            act = sm.res_act[ag];
            lp_sum = sm.res_lp[ag];
        }
        if (owner && active) {
            const int64_t slot = int64_t(e) * a.S + s;
            a.states[slot] = row;
            a.actions[slot] = uint16_t(act);
            a.logp[slot] = lp_sum;
            a.values[slot] = sm.overridden[ag] ? sm.res_v[ag] : double(logits[ag * kLogitStride + kN3]);
            uint64_t nrow = row;
            bool stay = true;
            for (int k = 0; k < n; ++k) {
                const int ak = (act >> (2 * k)) & 3;
                stay &= ak == 1;
                int v = row_byte(row, k) + ak - 1;
                v = v < 0 ? 0 : (v > a.cards[k] - 1 ? a.cards[k] - 1 : v);
                nrow = (nrow & ~(0xffull << (8 * k))) | (uint64_t(v) << (8 * k));
            }
            row = nrow;
            a.visited[int64_t(e) * (a.S + 1) + s + 1] = row;
            ++steps;
            if (stay) active = false;
        }
        __syncthreads();
    }
    if (owner) a.lengths[e] = steps;
    if (tid == 0 && guarded && a.n_guarded) atomicAdd(a.n_guarded, guarded);
}

}  // namespace kt

namespace kt {

void launch_rollout(kt_engine* e, const RolloutArgs& a) {
    const size_t smem = sizeof(RolloutSmem);
    KT_CUDA(cudaFuncSetAttribute(rollout_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const int grid = int(ceil_div(a.E, kAgentsPerCta));
    e->pre_launch("policy_rollout");
    rollout_kernel<<<grid, kRolloutThreads, smem, e->stream>>>(a);
    e->check_launch("policy_rollout");
}

}  // namespace kt
