// forest.cuh — packed forest handle and the device tree walk (shared by K2 and K10).
#pragma once

#include <vector>

#include "common.cuh"

struct kt_forest {
    int n_knobs = 0;
    int depth = 1;
    int n_trees = 0;
    int words_per_tree = 0;  // 8-byte words: super nodes then leaves
    double base = 0.0;
    uint64_t* dev = nullptr;  // n_trees * words_per_tree words
    std::vector<uint64_t> host;
    int device = 0;
    kt::RowFmt fmt{};
    int wide = 0;  // rows use the bit-field layout: entries are knob | cut << 3
};

namespace kt {

// One tree of depth D: super nodes (two levels per 64-bit load), then leaves.
template <int D>
__device__ __forceinline__ double walk_tree(const uint64_t* __restrict__ t, uint32_t lo, uint32_t hi) {
    int pos = 0;     // index within the current level
    int base = 0;    // offset of the current super-node level
#pragma unroll
    for (int d = 0; d < D; d += 2) {
        // entry = knob << 12 | cut: PRMT reads only the selector's low 16 bits and puts
        // byte[knob] in the top byte (junk below), so byte >= cut <=> result >= cut << 24
        const uint64_t w = t[base + pos];
        const uint32_t wlo = uint32_t(w), whi = uint32_t(w >> 32);
        const int go = __byte_perm(lo, hi, wlo) >= (wlo << 24);
        pos = 2 * pos + go;
        if (d + 1 < D) {
            const uint32_t e1 = go ? whi : (wlo >> 16);
            pos = 2 * pos + int(__byte_perm(lo, hi, e1) >= (e1 << 24));
        }
        base += 1 << d;
    }
    return __longlong_as_double((long long)t[base + pos]);
}


// Wide rows: knob fields widened to 16 bits once per row (knobs 0-3 in w[0..1],
// 4-7 in w[2..3]); a node entry is knob | cut << 3 (cut <= 8191) and one PRMT
// selects the knob's two bytes, like the byte layout's single-byte select.
struct WideRow {
    uint32_t w[4];
};

__device__ __forceinline__ WideRow widen_row(uint64_t row, const RowFmt& f) {
    WideRow x{{0u, 0u, 0u, 0u}};
#pragma unroll
    for (int i = 0; i < kMaxKnobs; ++i) x.w[i >> 1] |= uint32_t(f.get(row, i)) << (16 * (i & 1));
    return x;
}

__device__ __forceinline__ uint32_t wide_field(const WideRow& x, uint32_t f) {
    const uint32_t j = f & 3u;
    const uint32_t sel = (2u * j) | ((2u * j + 1u) << 4);
    const bool up = (f & 4u) != 0u;
    return __byte_perm(up ? x.w[2] : x.w[0], up ? x.w[3] : x.w[1], sel) & 0xffffu;
}

template <int D>
__device__ __forceinline__ double walk_tree_wide(const uint64_t* __restrict__ t, const WideRow& x) {
    int pos = 0, base = 0;
#pragma unroll
    for (int d = 0; d < D; d += 2) {
        uint64_t w = t[base + pos];
        uint32_t e = uint32_t(w) & 0xffffu;
        int go = wide_field(x, e & 7u) >= (e >> 3);
        pos = 2 * pos + go;
        if (d + 1 < D) {
            uint32_t e1 = uint32_t(w >> (16 * (1 + go))) & 0xffffu;
            pos = 2 * pos + int(wide_field(x, e1 & 7u) >= (e1 >> 3));
        }
        base += 1 << d;
    }
    return __longlong_as_double((long long)t[base + pos]);
}

void score_trees(kt_engine* e, const kt_forest* f, const uint64_t* rows, int64_t count, double* out);

}  // namespace kt
