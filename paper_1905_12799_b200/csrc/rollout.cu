// rollout.cu — K1 policy_rollout: PPO search agents walking the knob lattice.
//
// Replaces the lockstep episode loop of run_search_round (agent.py:298-328) with
// nets.forward (nets.py:51-60), softmax / joint_log_prob (nets.py:63-80),
// _sample_actions (agent.py:261-264), encode_state and apply_action
// (space.py:167-188).  One CTA owns 32 episodes (one per lane) and runs all of
// their steps in-kernel.  The whole forward pass is float64 like the reference's
// numpy: B200 issues fp64 FMAs at half the fp32 rate, and the weights (151 KB of
// float64) fit in shared memory, where one TMA bulk copy stages them while the
// threads derive their PCG64 streams.  Activations live transposed
// ([feature][agent]); warp w computes outputs [16w, 16w+16) of a layer for its
// 32 agents — a lane two agents x 8 outputs, so each broadcast 16-byte weight load
// feeds four FMAs (the shared-load issue rate, not the FP64 pipe, bounded the
// one-agent-per-lane mapping: MIO throttle was its top stall).
//
// Determinism / parity.  Episode e draws its uniforms from
// PCG64(SeedSequence(seed, spawn_key=(round, e))) on the device, n per step
// (agent.py:292-296, :313).  Dot products accumulate sequentially in float64 and
// the softmax / cdf use the reference's formulas, so logits, values and log
// probabilities agree with numpy to a few ulps (BLAS summation order) and sampled
// actions are identical unless a uniform falls within ~1e-15 of a cdf boundary
// (the north-star caveat).
#include <algorithm>
#include <cmath>
#include <vector>

#include "agent.cuh"
#include "rng.cuh"
#include "umma.cuh"

namespace kt {

constexpr int kZStride = kN3 + 1;  // 24 logits + value per agent (odd stride: conflict-free columns)

struct RolloutSmem {
    PaddedWeights64 w;
    double xt[kMaxKnobs][kAgentsPerCta];
    double h[kH][kAgentsPerCta];  // h1, then [hp | hv] (rows 0..63 | 64..127)
    double z[kAgentsPerCta][kZStride];
    double u[kAgentsPerCta][kMaxKnobs];
    double lpk[kAgentsPerCta][kMaxKnobs];  // log p of the sampled action, per knob
    uint8_t ak[kAgentsPerCta][kMaxKnobs];
    unsigned long long mbar;
    int any_active;
};

__global__ void __launch_bounds__(kRolloutThreads, 1) rollout_kernel(RolloutArgs a) {
    extern __shared__ unsigned char s_raw[];
    RolloutSmem& sm = *reinterpret_cast<RolloutSmem*>(align_shared<128>(s_raw));
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int n = a.n;
    const uint32_t mbar = umma::smem_addr(&sm.mbar);
    if (tid == 0) {  // weights -> smem by TMA bulk copies, overlapped with the RNG set-up below
        umma::mbar_init(mbar, 1);
        umma::mbar_fence_init();
        constexpr uint32_t total = sizeof(PaddedWeights64), chunk = 32768;
        umma::mbar_arrive_expect_tx(mbar, total);
        const uint32_t dst = umma::smem_addr(&sm.w);
        const char* src = reinterpret_cast<const char*>(a.w64);
        for (uint32_t off = 0; off < total; off += chunk)
            umma::bulk_g2s(dst + off, src + off, min(chunk, total - off), mbar);
    }
    // agent state lives in warp 0: lane = episode of this CTA
    const int e = blockIdx.x * kAgentsPerCta + lane;
    const bool owner = warp == 0 && e < a.E;
    uint64_t row = 0;
    bool active = false;
    Pcg64 rng;
    if (owner) {
        row = a.starts[e];
        active = true;
        uint32_t spawn[4];
        int ns = 0;
        for (int i = 0; i < a.n_round_words; ++i) spawn[ns++] = a.round_words[i];
        ns += u64_words(uint64_t(e + a.ep_offset), spawn + ns);
        rng = pcg64_from_seed_sequence(a.seed_words, a.n_seed_words, spawn, ns);
        a.visited[int64_t(e) * (a.S + 1)] = row;
    }
    // no thread may poll the mbarrier before thread 0 has initialised it: shared memory still
    // holds whatever the SM's previous kernel left there (found as an intermittent launch
    // failure when several engines' kernels share the SMs)
    __syncthreads();
    umma::mbar_wait(mbar, 0);
    int steps = 0;
    const int o0 = warp * kRolloutOut;

    for (int s = 0; s < a.S; ++s) {
        if (warp == 0) {
            const bool act_now = owner && active;
            for (int k = 0; k < kMaxKnobs; ++k)
                sm.xt[k][lane] = (act_now && k < n) ? __ddiv_rn(double(a.fmt.get(row, k)), double(max(1, a.cards[k] - 1)))
                                                    : 0.0;
            if (act_now)
                for (int k = 0; k < n; ++k) sm.u[lane][k] = rng.random();
            const unsigned any = __any_sync(0xffffffffu, act_now);
            if (lane == 0) sm.any_active = int(any);
        }
        __syncthreads();
        if (!sm.any_active) break;

#if KT_ROLLOUT_PAIR
        // lane (half, p): agents 2p and 2p + 1, outputs [o1, o1 + 8) — every broadcast weight load
        // feeds both agents (half the shared loads per FMA of one agent per lane); per (output,
        // agent) the same sequential fma chain over k as the one-agent mapping
        const int half = lane >> 4, p2 = 2 * (lane & 15);
        const int o1 = o0 + 8 * half;
        // ---- h1 = tanh(x W1^T + b1)
        {
            double acc0[8], acc1[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) acc0[j] = acc1[j] = 0.0;
            for (int k = 0; k < n; ++k) {
                const double2 x2 = *reinterpret_cast<const double2*>(&sm.xt[k][p2]);
                const double2* wr = reinterpret_cast<const double2*>(&sm.w.w1t[k][o1]);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const double2 w2 = wr[q];
                    acc0[2 * q] = fma(x2.x, w2.x, acc0[2 * q]);
                    acc0[2 * q + 1] = fma(x2.x, w2.y, acc0[2 * q + 1]);
                    acc1[2 * q] = fma(x2.y, w2.x, acc1[2 * q]);
                    acc1[2 * q + 1] = fma(x2.y, w2.y, acc1[2 * q + 1]);
                }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const double b = sm.w.b1[o1 + j];
                *reinterpret_cast<double2*>(&sm.h[o1 + j][p2]) = make_double2(tanh(acc0[j] + b), tanh(acc1[j] + b));
            }
        }
        __syncthreads();
        // ---- [hp | hv] = tanh(h1 [W2p | W2v]^T + [b2p | b2v])
        {
            double acc0[8], acc1[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) acc0[j] = acc1[j] = 0.0;
            if ((o1 & (kG - 1)) < a.g) {  // outputs wholly inside the zero padding have nothing to add
#pragma unroll 4
                for (int k = 0; k < a.h; ++k) {
                    const double2 h2 = *reinterpret_cast<const double2*>(&sm.h[k][p2]);
                    const double2* wr = reinterpret_cast<const double2*>(&sm.w.w2t[k][o1]);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const double2 w2 = wr[q];
                        acc0[2 * q] = fma(h2.x, w2.x, acc0[2 * q]);
                        acc0[2 * q + 1] = fma(h2.x, w2.y, acc0[2 * q + 1]);
                        acc1[2 * q] = fma(h2.y, w2.x, acc1[2 * q]);
                        acc1[2 * q + 1] = fma(h2.y, w2.y, acc1[2 * q + 1]);
                    }
                }
            }
            __syncthreads();  // every warp has read h1
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const double b = sm.w.b2[o1 + j];
                *reinterpret_cast<double2*>(&sm.h[o1 + j][p2]) = make_double2(tanh(acc0[j] + b), tanh(acc1[j] + b));
            }
        }
        __syncthreads();
#else
        // ---- h1 = tanh(x W1^T + b1)
        {
            double acc[kRolloutOut];
#pragma unroll
            for (int j = 0; j < kRolloutOut; ++j) acc[j] = 0.0;
            for (int k = 0; k < n; ++k) {
                const double xk = sm.xt[k][lane];
                const double2* wr = reinterpret_cast<const double2*>(&sm.w.w1t[k][o0]);
#pragma unroll
                for (int q = 0; q < kRolloutOut / 2; ++q) {
                    const double2 w2 = wr[q];
                    acc[2 * q] = fma(xk, w2.x, acc[2 * q]);
                    acc[2 * q + 1] = fma(xk, w2.y, acc[2 * q + 1]);
                }
            }
#pragma unroll
            for (int j = 0; j < kRolloutOut; ++j) sm.h[o0 + j][lane] = tanh(acc[j] + sm.w.b1[o0 + j]);
        }
        __syncthreads();
        // ---- [hp | hv] = tanh(h1 [W2p | W2v]^T + [b2p | b2v])
        {
            double acc[kRolloutOut];
#pragma unroll
            for (int j = 0; j < kRolloutOut; ++j) acc[j] = 0.0;
            if ((o0 & (kG - 1)) < a.g) {  // warps wholly inside the zero padding have nothing to add
#pragma unroll 4
                for (int k = 0; k < a.h; ++k) {
                    const double hk = sm.h[k][lane];
                    const double2* wr = reinterpret_cast<const double2*>(&sm.w.w2t[k][o0]);
#pragma unroll
                    for (int q = 0; q < kRolloutOut / 2; ++q) {
                        const double2 w2 = wr[q];
                        acc[2 * q] = fma(hk, w2.x, acc[2 * q]);
                        acc[2 * q + 1] = fma(hk, w2.y, acc[2 * q + 1]);
                    }
                }
            }
            __syncthreads();  // every warp has read h1
#pragma unroll
            for (int j = 0; j < kRolloutOut; ++j) sm.h[o0 + j][lane] = tanh(acc[j] + sm.w.b2[o0 + j]);
        }
        __syncthreads();
#endif
        // ---- logits (warp w: knob w's three) and the value (warp n, or warp 7 when n == 8)
        {
            if (warp < n) {
                double z0 = 0.0, z1 = 0.0, z2 = 0.0;
                for (int k = 0; k < a.g; ++k) {
                    const double hk = sm.h[k][lane];
                    const double* wr = &sm.w.w3t[k][3 * warp];
                    z0 = fma(hk, wr[0], z0);
                    z1 = fma(hk, wr[1], z1);
                    z2 = fma(hk, wr[2], z2);
                }
                sm.z[lane][3 * warp] = z0 + sm.w.b3p[3 * warp];
                sm.z[lane][3 * warp + 1] = z1 + sm.w.b3p[3 * warp + 1];
                sm.z[lane][3 * warp + 2] = z2 + sm.w.b3p[3 * warp + 2];
            }
            if (warp == (kRolloutWarps > kMaxKnobs ? kMaxKnobs : (n < kMaxKnobs ? n : kMaxKnobs - 1))) {
                double v = 0.0;
                for (int k = 0; k < a.g; ++k) v = fma(sm.h[kG + k][lane], sm.w.w3v[k], v);
                sm.z[lane][kN3] = v + sm.w.b3v;
            }
        }
        __syncthreads();
        // ---- sample knob `warp` of agent `lane` (softmax / cdf as nets.py:63-80, agent.py:261-264)
        if (warp < n) {
            const double z0 = sm.z[lane][3 * warp], z1 = sm.z[lane][3 * warp + 1], z2 = sm.z[lane][3 * warp + 2];
            const double mz = fmax(z0, fmax(z1, z2));
            const double y0 = z0 - mz, y1 = z1 - mz, y2 = z2 - mz;
            const double lse = log(__dadd_rn(__dadd_rn(exp(y0), exp(y1)), exp(y2)));
            const double l0 = y0 - lse, l1 = y1 - lse, l2 = y2 - lse;
            const double c0 = exp(l0), c1 = __dadd_rn(c0, exp(l1));
            const double uk = sm.u[lane][warp];
            const int ak = (uk > c0) + (uk > c1);
            sm.ak[lane][warp] = uint8_t(ak);
            sm.lpk[lane][warp] = ak == 0 ? l0 : (ak == 1 ? l1 : l2);
        }
        __syncthreads();
        if (owner && active) {
            uint32_t act = 0;
            uint64_t nrow = row;
            bool stay = true;
            for (int k = 0; k < n; ++k) {
                const int ak = sm.ak[lane][k];
                act |= uint32_t(ak) << (2 * k);
                stay &= ak == 1;
                int v = a.fmt.get(row, k) + ak - 1;
                v = v < 0 ? 0 : (v > a.cards[k] - 1 ? a.cards[k] - 1 : v);
                nrow = a.fmt.set(nrow, k, v);
            }
            const int64_t slot = int64_t(e) * a.S + s;
            a.states[slot] = row;
            a.actions[slot] = uint16_t(act);
            a.logp[slot] = np_sum_small(sm.lpk[lane], n);
            a.values[slot] = sm.z[lane][kN3];
            row = nrow;
            a.visited[int64_t(e) * (a.S + 1) + s + 1] = row;
            ++steps;
            if (stay) active = false;
        }
        // the next step's first __syncthreads orders these reads before any overwrite
    }
    if (owner) a.lengths[e] = steps;
}

__global__ void pad_weights64_kernel(const double* p, int n, int h, int g, PaddedWeights64* w) {
    const ParamLayout L = param_layout(n, h, g);
    double* flat = reinterpret_cast<double*>(w);
    for (int i = threadIdx.x; i < int(sizeof(PaddedWeights64) / 8); i += blockDim.x) flat[i] = 0.0;
    __syncthreads();
    for (int i = threadIdx.x; i < h * n; i += blockDim.x) w->w1t[i % n][i / n] = p[L.w1 + i];
    for (int i = threadIdx.x; i < h; i += blockDim.x) w->b1[i] = p[L.b1 + i];
    for (int i = threadIdx.x; i < g * h; i += blockDim.x) {
        w->w2t[i % h][i / h] = p[L.w2p + i];
        w->w2t[i % h][kG + i / h] = p[L.w2v + i];
    }
    for (int i = threadIdx.x; i < g; i += blockDim.x) {
        w->b2[i] = p[L.b2p + i];
        w->b2[kG + i] = p[L.b2v + i];
        w->w3v[i] = p[L.w3v + i];
    }
    for (int i = threadIdx.x; i < 3 * n * g; i += blockDim.x) w->w3t[i % g][i / g] = p[L.w3p + i];
    for (int i = threadIdx.x; i < 3 * n; i += blockDim.x) w->b3p[i] = p[L.b3p + i];
    if (threadIdx.x == 0) w->b3v = p[L.b3v];
}

}  // namespace kt

namespace kt {

void launch_rollout(kt_engine* e, const RolloutArgs& a) {
    const size_t smem = sizeof(RolloutSmem) + 128;
    allow_dynamic_smem((const void*)rollout_kernel);
    const int grid = int(ceil_div(a.E, kAgentsPerCta));
    e->pre_launch("policy_rollout");
    rollout_kernel<<<grid, kRolloutThreads, smem, e->stream>>>(a);
    e->check_launch("policy_rollout");
}

}  // namespace kt

namespace kt {

void launch_pad_weights64(kt_engine* e, const double* p64, int n, int h, int g, PaddedWeights64* w) {
    e->pre_launch("pad_weights");
    pad_weights64_kernel<<<1, 1024, 0, e->stream>>>(p64, n, h, g, w);
    e->check_launch("pad_weights");
}

}  // namespace kt
