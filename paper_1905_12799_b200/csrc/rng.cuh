// rng.cuh — numpy-compatible SeedSequence + PCG64 (host and device).
//
// The reference derives every random stream as
//   default_rng(SeedSequence(entropy, spawn_key=...))   (sampler.py:89, sa.py:79-81,
//                                                        agent.py:292-296, driver.py:67-69)
// so the engine reproduces numpy's algorithms exactly:
//   * SeedSequence pool mixing and generate_state (numpy/random/bit_generator.pyx),
//   * PCG64 = pcg_setseq_128_xsl_rr_64 seeded with generate_state(4, uint64)
//     (numpy/random/_pcg64.pyx, src/pcg64/pcg64.h),
//   * random() = (next64 >> 11) * 2^-53, integers(0, n) = 32-bit Lemire on the
//     buffered next_uint32 (numpy/random/src/distributions/distributions.c).
#pragma once

#include <stdint.h>

namespace kt {

struct SeedPool {
    uint32_t w[4];
};

__host__ __device__ inline uint32_t ss_hashmix(uint32_t value, uint32_t& hash_const) {
    value ^= hash_const;
    hash_const *= 0x931e8875u;  // MULT_A
    value *= hash_const;
    value ^= value >> 16;
    return value;
}

__host__ __device__ inline uint32_t ss_mix(uint32_t x, uint32_t y) {
    uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;  // MIX_MULT_L, MIX_MULT_R
    r ^= r >> 16;
    return r;
}

// Assembled entropy = entropy words (padded with zeros to 4 when a spawn key is
// present) followed by the spawn-key words.
__host__ __device__ inline SeedPool seed_pool(const uint32_t* entropy, int ne, const uint32_t* spawn, int ns) {
    const int run_len = (ns > 0 && ne < 4) ? 4 : ne;
    const int total = run_len + ns;
    auto word = [&](int i) -> uint32_t {
        if (i < run_len) return i < ne ? entropy[i] : 0u;
        return spawn[i - run_len];
    };
    SeedPool p;
    uint32_t hc = 0x43b0d7e5u;  // INIT_A
    for (int i = 0; i < 4; ++i) p.w[i] = ss_hashmix(i < total ? word(i) : 0u, hc);
    for (int s = 0; s < 4; ++s)
        for (int d = 0; d < 4; ++d)
            if (s != d) p.w[d] = ss_mix(p.w[d], ss_hashmix(p.w[s], hc));
    for (int s = 4; s < total; ++s)
        for (int d = 0; d < 4; ++d) p.w[d] = ss_mix(p.w[d], ss_hashmix(word(s), hc));
    return p;
}

// generate_state(n_words, uint32)
__host__ __device__ inline void seed_generate(const SeedPool& p, uint32_t* out, int n_words) {
    uint32_t hc = 0x8b51f9ddu;  // INIT_B
    for (int i = 0; i < n_words; ++i) {
        uint32_t v = p.w[i & 3];
        v ^= hc;
        hc *= 0x58f38dedu;  // MULT_B
        v *= hc;
        v ^= v >> 16;
        out[i] = v;
    }
}

typedef unsigned __int128 u128;

struct Pcg64 {
    u128 state;
    u128 inc;
    uint32_t cached;
    int has_cached;

    __host__ __device__ static u128 mult() {
        return (u128(0x2360ED051FC65DA4ull) << 64) | u128(0x4385DF649FCCF645ull);
    }
    __host__ __device__ void step() { state = state * mult() + inc; }
    __host__ __device__ uint64_t next64() {
        step();
        uint64_t hi = uint64_t(state >> 64), lo = uint64_t(state);
        unsigned rot = unsigned(state >> 122);
        uint64_t x = hi ^ lo;
        return (x >> rot) | (x << ((64u - rot) & 63u));
    }
    __host__ __device__ uint32_t next32() {
        if (has_cached) {
            has_cached = 0;
            return cached;
        }
        uint64_t v = next64();
        has_cached = 1;
        cached = uint32_t(v >> 32);
        return uint32_t(v);
    }
    __host__ __device__ double random() { return double(next64() >> 11) * (1.0 / 9007199254740992.0); }
    // integers(0, rng + 1): rng == 0 consumes nothing.
    __host__ __device__ uint32_t bounded32(uint32_t rng) {
        if (rng == 0) return 0;
        if (rng == 0xffffffffu) return next32();
        const uint32_t excl = rng + 1;
        uint64_t m = uint64_t(next32()) * excl;
        uint32_t left = uint32_t(m);
        if (left < excl) {
            const uint32_t threshold = (0xffffffffu - rng) % excl;
            while (left < threshold) {
                m = uint64_t(next32()) * excl;
                left = uint32_t(m);
            }
        }
        return uint32_t(m >> 32);
    }
};

__host__ __device__ inline Pcg64 pcg64_from_pool(const SeedPool& pool) {
    uint32_t w[8];
    seed_generate(pool, w, 8);
    uint64_t v[4];
    for (int i = 0; i < 4; ++i) v[i] = uint64_t(w[2 * i]) | (uint64_t(w[2 * i + 1]) << 32);
    u128 initstate = (u128(v[0]) << 64) | v[1];
    u128 initseq = (u128(v[2]) << 64) | v[3];
    Pcg64 g;
    g.state = 0;
    g.inc = (initseq << 1) | 1;
    g.step();
    g.state += initstate;
    g.step();
    g.cached = 0;
    g.has_cached = 0;
    return g;
}

__host__ __device__ inline Pcg64 pcg64_from_seed_sequence(const uint32_t* entropy, int ne, const uint32_t* spawn,
                                                          int ns) {
    return pcg64_from_pool(seed_pool(entropy, ne, spawn, ns));
}

// Little-endian 32-bit words of a non-negative integer (numpy _int_to_uint32_array).
__host__ __device__ inline int u64_words(uint64_t x, uint32_t* out) {
    if (x == 0) {
        out[0] = 0;
        return 1;
    }
    int n = 0;
    while (x) {
        out[n++] = uint32_t(x);
        x >>= 32;
    }
    return n;
}

}  // namespace kt
