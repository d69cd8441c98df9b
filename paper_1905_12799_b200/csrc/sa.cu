// sa.cu — K10 sa_chains: simulated-annealing walkers on the surrogate.
//
// Replaces _propose_into + run_sa_round (sa.py:45-122).  One thread per chain
// runs all steps in-kernel: chains are independent Metropolis walkers, so the
// reference's lockstep batching (one predict per step) is only a CPU batching
// device — running each chain to completion is bit-identical because every
// chain owns its PCG64 stream (sa.py:4-9).
//
// Per chain c: stream = PCG64(SeedSequence(seed, spawn_key=(c,))) generated
// on the device; per step: integers(0, n) (knob), integers(0, 2) (sign), and
// random() only when the proposal lowers the score (the `delta >= 0 or ...`
// short circuit, sa.py:112).  The proposal is scored with the same packed
// forest walk as K2 (bit-exact), the temperature is T0 * cooling^s evaluated
// by repeated multiplication like the reference.
// T0 = np.std(start scores) (pairwise mean / pairwise sum of squares / sqrt),
// or 1.0 below 1e-12, or the explicit initial temperature.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "forest.cuh"
#include "pairwise.cuh"
#include "pwsum_warp.cuh"
#include "rng.cuh"

namespace kt {

__global__ void sa_temperature_kernel(const double* sum, const double* sumsq, int64_t count, int has_t0, double t0,
                                      double* mean_out, double* temp_out, int stage) {
    if (stage == 0) {
        *mean_out = __ddiv_rn(*sum, double(count));
    } else {
        if (has_t0) {
            *temp_out = t0;
        } else {
            const double sd = __dsqrt_rn(__ddiv_rn(*sumsq, double(count)));
            *temp_out = sd > 1e-12 ? sd : 1.0;
        }
    }
}

struct SAArgs {
    const uint64_t* forest;
    int words_per_tree, n_trees;
    double base;
    const uint64_t* starts;
    const double* start_scores;
    const double* temperature;
    int chains, steps, n;
    int32_t cards[kMaxKnobs];
    RowFmt fmt;
    uint32_t seed_words[4];
    int n_seed_words;
    double cooling;
    uint64_t* slot_rows;  // [chains][steps+1]
    double* slot_scores;
    int32_t* slot_steps;
    int64_t* counts;
    // fused start (warp kernel, few chains): every block scores all starts and derives the
    // temperature itself instead of the score_trees + pairwise-sum + temperature launches
    int fused, has_t0;
    double t0;
};

template <int D>
__device__ __forceinline__ double score_row(const uint64_t* forest, int words_per_tree, int n_trees, double base,
                                            uint64_t row, bool wide, const RowFmt& fmt) {
    double acc;
    if (wide) {
        const WideRow x = widen_row(row, fmt);
        acc = walk_tree_wide<D>(forest, x);
        for (int t = 1; t < n_trees; ++t) acc = __dadd_rn(acc, walk_tree_wide<D>(forest + t * words_per_tree, x));
    } else {
        const uint32_t lo = uint32_t(row), hi = uint32_t(row >> 32);
        acc = walk_tree<D>(forest, lo, hi);
        for (int t = 1; t < n_trees; ++t) acc = __dadd_rn(acc, walk_tree<D>(forest + t * words_per_tree, lo, hi));
    }
    return __dadd_rn(base, acc);
}

template <int D>
__global__ void __launch_bounds__(128) sa_chain_kernel(SAArgs a) {
    extern __shared__ uint64_t s_forest[];
    const int total = a.n_trees * a.words_per_tree;
    for (int i = threadIdx.x; i < total; i += blockDim.x) s_forest[i] = a.forest[i];
    __syncthreads();
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= a.chains) return;

    const uint32_t spawn = uint32_t(c);
    Pcg64 g = pcg64_from_seed_sequence(a.seed_words, a.n_seed_words, &spawn, 1);
    uint64_t row = a.starts[c];
    double score = a.start_scores[c];
    double temp = *a.temperature;
    const int64_t slot0 = int64_t(c) * (a.steps + 1);
    a.slot_rows[slot0] = row;
    a.slot_scores[slot0] = score;
    a.slot_steps[slot0] = 0;
    int64_t kept = 1;
    for (int s = 1; s <= a.steps; ++s) {
        const int knob = int(g.bounded32(uint32_t(a.n - 1)));
        const int sign = int(g.bounded32(1u)) * 2 - 1;
        int v = a.fmt.get(row, knob) + sign;
        v = v < 0 ? 0 : (v > a.cards[knob] - 1 ? a.cards[knob] - 1 : v);
        const uint64_t prop = a.fmt.set(row, knob, v);
        const double ps = score_row<D>(s_forest, a.words_per_tree, a.n_trees, a.base, prop, !a.fmt.bytes, a.fmt);
        const double delta = __dsub_rn(ps, score);
        bool accept = delta >= 0.0;
        if (!accept) accept = g.random() < exp(__ddiv_rn(delta, temp));
        if (accept) {
            row = prop;
            score = ps;
            a.slot_rows[slot0 + kept] = row;
            a.slot_scores[slot0 + kept] = score;
            a.slot_steps[slot0 + kept] = s;
            ++kept;
        }
        temp = __dmul_rn(temp, a.cooling);
    }
    a.counts[c] = kept;
}

// Warp-per-chain variant for few chains (a tuning round runs 64): the 32 lanes walk
// the trees of a proposal in parallel (lane l takes trees l, l + 32, ...), stage the leaf
// values in shared memory, then every lane accumulates them in tree order — the same
// sequential float64 sum as score_row, so the chain is bit-identical.  Every lane runs the chain's
// PCG64 stream redundantly (identical draws, no broadcast); lane 0 writes the slots.
template <int D>
__global__ void __launch_bounds__(128) sa_chain_warp_kernel(SAArgs a) {
    extern __shared__ uint64_t s_forest[];
    const int total = a.n_trees * a.words_per_tree;
    for (int i = threadIdx.x; i < total; i += blockDim.x) s_forest[i] = a.forest[i];
    __syncthreads();
    __shared__ double s_leaf[4][64];  // per warp: the proposal's leaf value of each tree
    __shared__ double s_temp;
    const double* start_scores = a.start_scores;
    if (a.fused) {
        // start scores (score_row = K2's float64 order) and T0 = np.std(start scores) (sa.py:93-97:
        // pairwise mean, pairwise sum of squared deviations, sqrt; 1.0 below 1e-12)
        double* s_sc = reinterpret_cast<double*>(s_forest + total);
        for (int i = threadIdx.x; i < a.chains; i += blockDim.x)
            s_sc[i] = score_row<D>(s_forest, a.words_per_tree, a.n_trees, a.base, a.starts[i], !a.fmt.bytes, a.fmt);
        __syncthreads();
        if (threadIdx.x < 32) {
            double t = a.t0;
            if (!a.has_t0) {
                const double mean = __ddiv_rn(pw_sum_warp([&](int i) { return s_sc[i]; }, a.chains), double(a.chains));
                const double ss = pw_sum_warp([&](int i) {
                    const double d = __dsub_rn(s_sc[i], mean);
                    return __dmul_rn(d, d);
                }, a.chains);
                const double sd = __dsqrt_rn(__ddiv_rn(ss, double(a.chains)));
                t = sd > 1e-12 ? sd : 1.0;
            }
            if (threadIdx.x == 0) s_temp = t;
        }
        __syncthreads();
        start_scores = s_sc;
    } else if (threadIdx.x == 0) {
        s_temp = *a.temperature;
    }
    __syncthreads();
    const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (c >= a.chains) return;  // whole warps
    double* my_leaf = s_leaf[threadIdx.x >> 5];
    const uint32_t spawn = uint32_t(c);
    Pcg64 g = pcg64_from_seed_sequence(a.seed_words, a.n_seed_words, &spawn, 1);
    uint64_t row = a.starts[c];
    double score = start_scores[c];
    double temp = s_temp;
    const int64_t slot0 = int64_t(c) * (a.steps + 1);
    if (lane == 0) {
        a.slot_rows[slot0] = row;
        a.slot_scores[slot0] = score;
        a.slot_steps[slot0] = 0;
    }
    const bool wide = !a.fmt.bytes;
    int64_t kept = 1;
    for (int s = 1; s <= a.steps; ++s) {
        const int knob = int(g.bounded32(uint32_t(a.n - 1)));
        const int sign = int(g.bounded32(1u)) * 2 - 1;
        int v = a.fmt.get(row, knob) + sign;
        v = v < 0 ? 0 : (v > a.cards[knob] - 1 ? a.cards[knob] - 1 : v);
        const uint64_t prop = a.fmt.set(row, knob, v);
        double leaf[2] = {0.0, 0.0};
        const uint32_t lo = uint32_t(prop), hi = uint32_t(prop >> 32);
        WideRow x{};
        if (wide) x = widen_row(prop, a.fmt);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int t = lane + 32 * q;
            if (t < a.n_trees) {
                const uint64_t* tr = s_forest + t * a.words_per_tree;
                leaf[q] = wide ? walk_tree_wide<D>(tr, x) : walk_tree<D>(tr, lo, hi);
            }
        }
        // tree-order sum from shared memory: the loads are independent of the running sum, so
        // only the dependent float64 adds remain on the step's critical path
        my_leaf[lane] = leaf[0];
        my_leaf[lane + 32] = leaf[1];
        __syncwarp();
        double acc = my_leaf[0];
#pragma unroll 8
        for (int t = 1; t < a.n_trees; ++t) acc = __dadd_rn(acc, my_leaf[t]);
        __syncwarp();  // every lane has read the leaves before the next step overwrites them
        const double ps = __dadd_rn(a.base, acc);
        const double delta = __dsub_rn(ps, score);
        bool accept = delta >= 0.0;
        if (!accept) accept = g.random() < exp(__ddiv_rn(delta, temp));
        if (accept) {
            row = prop;
            score = ps;
            if (lane == 0) {
                a.slot_rows[slot0 + kept] = row;
                a.slot_scores[slot0 + kept] = score;
                a.slot_steps[slot0 + kept] = s;
            }
            ++kept;
        }
        temp = __dmul_rn(temp, a.cooling);
    }
    if (lane == 0) a.counts[c] = kept;
}

__global__ void sa_compact_kernel(const uint64_t* slot_rows, const double* slot_scores, const int32_t* slot_steps,
                                  const int64_t* counts, const int64_t* offsets, int chains, int steps,
                                  uint64_t* rows_out, double* scores_out, int32_t* steps_out) {
    // one warp per chain: chain-major, coalesced within the chain's run
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= chains) return;
    const int64_t src = int64_t(warp) * (steps + 1), dst = offsets[warp], cnt = counts[warp];
    for (int64_t j = lane; j < cnt; j += 32) {
        rows_out[dst + j] = slot_rows[src + j];
        scores_out[dst + j] = slot_scores[src + j];
        steps_out[dst + j] = slot_steps[src + j];
    }
}

constexpr int kSaWarpChains = 8192;  // up to this many chains the warp-per-chain kernel is used
constexpr int kSaFusedChains = 1024;  // up to this many, the warp kernel also scores the starts

static bool sa_warp_path(const kt_forest* f, int chains) { return f->n_trees <= 64 && chains <= kSaWarpChains; }
static bool sa_fused_path(const kt_forest* f, int chains) {
    return sa_warp_path(f, chains) && chains <= kSaFusedChains &&
           (size_t(f->n_trees) * f->words_per_tree + chains) * 8 <= 200 * 1024;
}

template <int D>
static void launch_chains(kt_engine* e, const kt_forest* f, const SAArgs& a) {
    size_t smem = size_t(f->n_trees) * f->words_per_tree * 8;
    if (smem > 200 * 1024) fail(KT_ERR_UNSUPPORTED, "forest too large for the in-kernel SA walk");
    if (sa_warp_path(f, a.chains)) {  // few chains: a warp per chain
        if (a.fused) smem += size_t(a.chains) * 8;
        auto kern = sa_chain_warp_kernel<D>;
        allow_dynamic_smem((const void*)kern);
        e->pre_launch("sa_chains");
        kern<<<int(ceil_div(int64_t(a.chains) * 32, 128)), 128, smem, e->stream>>>(a);
        e->check_launch("sa_chains");
        return;
    }
    auto kern = sa_chain_kernel<D>;
    allow_dynamic_smem((const void*)kern);
    e->pre_launch("sa_chains");
    kern<<<int(ceil_div(a.chains, 128)), 128, smem, e->stream>>>(a);
    e->check_launch("sa_chains");
}

}  // namespace kt

extern "C" int kt_sa_chains(kt_engine* e, const kt_forest* f, const uint64_t* starts_dev, int32_t n_starts,
                            int32_t chains, int32_t steps, const int32_t* cards, int n_knobs,
                            const uint32_t* seed_words, int n_seed_words, int has_initial_temperature,
                            double initial_temperature, double cooling, uint64_t* rows_out_dev,
                            double* scores_out_dev, int32_t* steps_out_dev, int64_t* n_out) {
    KT_API_BEGIN
    using namespace kt;
    if (chains < 1) fail(KT_ERR_VALUE, "chains must be >= 1");
    if (steps < 1) fail(KT_ERR_VALUE, "steps_per_round must be >= 1");
    if (n_starts < 1) fail(KT_ERR_VALUE, "run_sa_round needs at least one start configuration");
    if (n_knobs != f->n_knobs) fail(KT_ERR_DIMENSION, "forest and space disagree on the knob count");
    if (n_seed_words < 1 || n_seed_words > 4) fail(KT_ERR_VALUE, "seed must fit in 128 bits");
    if (chains > 64 * 1024 * 1024) fail(KT_ERR_UNSUPPORTED, "at most 2^26 chains per call");
    const RowFmt fmt = row_fmt(cards, n_knobs);
    if (fmt.bytes != f->fmt.bytes) fail(KT_ERR_DIMENSION, "forest and space disagree on the row layout");
    // starts: the first min(n_starts, chains) given, the rest padded from the parent stream
    // (sa.py:79-85: pad_rng = default_rng(seed_seq); random_config draws integers(0, card) per knob)
    auto* starts = static_cast<uint64_t*>(e->scratch("sa.starts", size_t(chains) * 8));
    const int given = std::min(n_starts, chains);
    KT_CUDA(cudaMemcpyAsync(starts, starts_dev, size_t(given) * 8, cudaMemcpyDeviceToDevice, e->stream));
    if (given < chains) {
        Pcg64 pad = pcg64_from_seed_sequence(seed_words, n_seed_words, nullptr, 0);
        auto* h = static_cast<uint64_t*>(e->staging("sa.pad", size_t(chains - given) * 8));
        for (int c = 0; c < chains - given; ++c) {
            uint64_t row = 0;
            for (int q = 0; q < n_knobs; ++q) row = fmt.set(row, q, int(pad.bounded32(uint32_t(cards[q] - 1))));
            h[c] = row;
        }
        KT_CUDA(cudaMemcpyAsync(starts + given, h, size_t(chains - given) * 8, cudaMemcpyHostToDevice, e->stream));
    }
    if (f->n_trees == 0) fail(KT_ERR_UNSUPPORTED, "SA on a sentinel (tree-less) model is not supported by the engine");
    const bool fused = sa_fused_path(f, chains) && !std::getenv("KT_SA_UNFUSED");  // tests: the launch chain
    auto* start_scores = static_cast<double*>(e->scratch("sa.start_scores", size_t(chains) * 8));
    auto* scal = static_cast<double*>(e->scratch("sa.scalars", 4 * 8));  // sum, mean, sumsq, temperature
    if (!fused) {
        score_trees(e, f, starts, chains, start_scores);
        if (!has_initial_temperature) {
            pairwise_sum(e, start_scores, chains, nullptr, scal + 0);
            e->pre_launch("sa_mean");
            sa_temperature_kernel<<<1, 1, 0, e->stream>>>(scal + 0, nullptr, chains, 0, 0.0, scal + 1, nullptr, 0);
            e->check_launch("sa_mean");
            pairwise_sum(e, start_scores, chains, scal + 1, scal + 2);
        }
        e->pre_launch("sa_temperature");
        sa_temperature_kernel<<<1, 1, 0, e->stream>>>(nullptr, scal + 2, chains, has_initial_temperature,
                                                      initial_temperature, nullptr, scal + 3, 1);
        e->check_launch("sa_temperature");
    }

    SAArgs a{};
    a.fused = fused;
    a.has_t0 = has_initial_temperature;
    a.t0 = initial_temperature;
    a.forest = f->dev;
    a.words_per_tree = f->words_per_tree;
    a.n_trees = f->n_trees;
    a.base = f->base;
    a.starts = starts;
    a.start_scores = start_scores;
    a.temperature = scal + 3;
    a.chains = chains;
    a.steps = steps;
    a.n = n_knobs;
    for (int q = 0; q < n_knobs; ++q) a.cards[q] = cards[q];
    a.fmt = fmt;
    for (int q = 0; q < n_seed_words; ++q) a.seed_words[q] = seed_words[q];
    a.n_seed_words = n_seed_words;
    a.cooling = cooling;
    const size_t slots = size_t(chains) * (steps + 1);
    a.slot_rows = static_cast<uint64_t*>(e->scratch("sa.slot_rows", slots * 8));
    a.slot_scores = static_cast<double*>(e->scratch("sa.slot_scores", slots * 8));
    a.slot_steps = static_cast<int32_t*>(e->scratch("sa.slot_steps", slots * 4));
    a.counts = static_cast<int64_t*>(e->scratch("sa.counts", size_t(chains) * 8));
    switch (f->depth) {
        case 1: launch_chains<1>(e, f, a); break;
        case 2: launch_chains<2>(e, f, a); break;
        case 3: launch_chains<3>(e, f, a); break;
        case 4: launch_chains<4>(e, f, a); break;
        case 5: launch_chains<5>(e, f, a); break;
        case 6: launch_chains<6>(e, f, a); break;
        case 7: launch_chains<7>(e, f, a); break;
        case 8: launch_chains<8>(e, f, a); break;
        default: fail(KT_ERR_UNSUPPORTED, "tree depth > 8");
    }
    auto* offsets = static_cast<int64_t*>(e->scratch("sa.offsets", size_t(chains + 1) * 8));
    exclusive_scan(e, a.counts, offsets, chains);
    e->pre_launch("sa_compact");
    sa_compact_kernel<<<int(ceil_div(int64_t(chains) * 32, 256)), 256, 0, e->stream>>>(
        a.slot_rows, a.slot_scores, a.slot_steps, a.counts, offsets, chains, steps, rows_out_dev, scores_out_dev,
        steps_out_dev);
    e->check_launch("sa_compact");
    auto* h_total = static_cast<int64_t*>(e->staging("sa.total", 8));
    KT_CUDA(cudaMemcpyAsync(h_total, offsets + chains, 8, cudaMemcpyDeviceToHost, e->stream));
    e->sync();
    *n_out = *h_total;
    KT_API_END
}
