// agent.cuh — actor-critic parameter layout shared by the rollout (K1) and PPO (K4/K5) kernels.
//
// Parameters are kept in the reference's PARAM_KEYS order (nets.py:24), flattened:
//   w1 (h,n) b1 (h) w2p (g,h) b2p (g) w3p (3n,g) b3p (3n) w2v (g,h) b2v (g) w3v (1,g) b3v (1)
// Kernels use compile-time maxima (h <= 128, g <= 64, n <= 8) and zero padding,
// which leaves every output unchanged (tanh(0) = 0, zero weights add nothing).
#pragma once

#include "common.cuh"

namespace kt {

constexpr int kH = 128;      // max shared width
constexpr int kG = 64;       // max head width
constexpr int kN3 = 3 * kMaxKnobs;

struct ParamLayout {
    int n, h, g;
    int w1, b1, w2p, b2p, w3p, b3p, w2v, b2v, w3v, b3v, total;
};

__host__ __device__ inline ParamLayout param_layout(int n, int h, int g) {
    ParamLayout L;
    L.n = n, L.h = h, L.g = g;
    int o = 0;
    L.w1 = o, o += h * n;
    L.b1 = o, o += h;
    L.w2p = o, o += g * h;
    L.b2p = o, o += g;
    L.w3p = o, o += 3 * n * g;
    L.b3p = o, o += 3 * n;
    L.w2v = o, o += g * h;
    L.b2v = o, o += g;
    L.w3v = o, o += g;
    L.b3v = o, o += 1;
    L.total = o;
    return L;
}

// Padded float64 weights in the transposed (k-major) layouts the rollout reads from
// shared memory: every lane owns one agent and reads a broadcast weight row.
struct PaddedWeights64 {
    double w1t[kMaxKnobs][kH];  // w1t[k][o] = w1[o][k]
    double b1[kH];
    double w2t[kH][2 * kG];     // w2t[k][o] = w2p[o][k] (o < 64), w2v[o-64][k] (o >= 64)
    double b2[2 * kG];          // b2p | b2v
    double w3t[kG][kN3];        // w3t[k][o] = w3p[o][k]
    double b3p[kN3];
    double w3v[kG];
    double b3v;
    double pad;
};
static_assert(sizeof(PaddedWeights64) % 16 == 0, "bulk-copy granularity");

constexpr int kAgentsPerCta = 32;   // one agent per lane (state, sampling)
#ifndef KT_ROLLOUT_PAIR
#define KT_ROLLOUT_PAIR 1  // A/B per RL step (5 x 4,096 agents): rollout 3.24 -> 3.04 ms (the 16-warp mapping: 0)
#endif
#if KT_ROLLOUT_PAIR
// 8 warps; warp w: outputs [16w, 16w+16) of each layer, a lane two agents x 8 outputs
constexpr int kRolloutThreads = 256;
#else
// warp w: outputs [8w, 8w+8) of each layer (16 warps: 2x the latency hiding of 8 warps x 16
// outputs, half the accumulator registers), knob w when sampling, warp 8 the value head
constexpr int kRolloutThreads = 512;
#endif
constexpr int kRolloutWarps = kRolloutThreads / 32;
constexpr int kRolloutOut = kH / kRolloutWarps;

struct RolloutArgs {
    const PaddedWeights64* w64;
    int n, h, g;
    int S;              // max steps per episode
    int E;              // episodes
    int32_t cards[kMaxKnobs];
    RowFmt fmt;
    uint32_t seed_words[4];
    int n_seed_words;
    uint32_t round_words[2];
    int n_round_words;
    const uint64_t* starts;
    int64_t ep_offset;   // global index of episode 0 (sharded rounds: RNG spawn key = (round, ep_offset + e))
    // outputs (slots)
    uint64_t* visited;   // [E][S+1]
    uint64_t* states;    // [E][S]  config row before the move
    uint16_t* actions;   // [E][S]  2 bits per knob
    double* logp;        // [E][S]
    double* values;      // [E][S]
    int32_t* lengths;    // [E]
};

void launch_pad_weights64(kt_engine* e, const double* p64, int n, int h, int g, PaddedWeights64* w);
void launch_rollout(kt_engine* e, const RolloutArgs& a);

// fp32 GEMM on tcgen05 (gemm_tc.cu): C = epi(A(m,k) B(k,n)), TA: A MN-major, TB: B K-major.
void tc_gemm(kt_engine* e, bool TA, bool TB, int M, int N, int K, const float* A, int lda, const float* B, int ldb,
             float* C, int ldc, int epi, const float* bias, const float* aux, int ldaux, int splits,
             double* colpart = nullptr);

}  // namespace kt
