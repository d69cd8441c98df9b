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

// Padded fp32 weights in the transposed (k-major) layouts the tile kernels read.
struct PaddedWeights {
    float w1t[kMaxKnobs][kH];  // w1t[k][o] = w1[o][k]
    float b1[kH];
    float w2pt[kH][kG];        // w2pt[k][o] = w2p[o][k]
    float w2vt[kH][kG];
    float b2p[kG];
    float b2v[kG];
    float w3pt[kG][kN3];       // w3pt[k][o] = w3p[o][k]
    float b3p[kN3];
    float w3v[kG];
    float b3v;
    float pad[3];
};

constexpr int kAgentsPerCta = 128;
constexpr int kRolloutThreads = 256;

struct RolloutArgs {
    const PaddedWeights* w32;
    const double* p64;  // flat float64 parameters (PARAM_KEYS order)
    int n, h, g;
    int S;              // max steps per episode
    int E;              // episodes
    int32_t cards[kMaxKnobs];
    uint32_t seed_words[4];
    int n_seed_words;
    uint32_t round_words[2];
    int n_round_words;
    float tau;          // decision guard band
    const uint64_t* starts;
    // outputs (slots)
    uint64_t* visited;   // [E][S+1]
    uint64_t* states;    // [E][S]  config row before the move
    uint16_t* actions;   // [E][S]  2 bits per knob
    double* logp;        // [E][S]
    double* values;      // [E][S]
    int32_t* lengths;    // [E]
    unsigned long long* n_guarded;  // agent-steps re-evaluated in float64
};

void launch_rollout(kt_engine* e, const RolloutArgs& a);

// fp32 GEMM on tcgen05 (gemm_tc.cu): C = epi(A(m,k) B(k,n)), TA: A MN-major, TB: B K-major.
void tc_gemm(kt_engine* e, bool TA, bool TB, int M, int N, int K, const float* A, int lda, const float* B, int ldb,
             float* C, int ldc, int epi, const float* bias, const float* aux, int ldaux, int splits);

}  // namespace kt
