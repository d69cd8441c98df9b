// pwsum_warp.cuh — numpy's pairwise_sum order computed by one warp (device side).
//
// numpy/_core/src/umath/loops_utils.h.src pairwise_sum: <= 128 values with 8 strided
// accumulators, larger ranges split at n2 = n/2 - (n/2 % 8).  Used by the device fit
// (cost_model.py means / SSEs) and the SA chains' start temperature (sa.py:93-97).
#pragma once

#include "common.cuh"

namespace kt {

// Warp-cooperative numpy pairwise_sum of val(0..n-1) (all 32 lanes call it; every lane gets
// the result).  A <= 128-element leaf is loaded in one shot (4 values per lane) and its 8
// strided accumulators run on lanes 0..7 over shuffled values — the same additions in the
// same order as pw_leaf_dev; larger inputs walk numpy's split tree iteratively.
template <class Val>
__device__ double pw_leaf_warp(Val val, int base, int n) {
    const int lane = threadIdx.x & 31;
    double v[4];
#pragma unroll
    for (int s2 = 0; s2 < 4; ++s2) v[s2] = lane + 32 * s2 < n ? val(base + lane + 32 * s2) : 0.0;
    if (n < 8) {
        double res = 0.0;
        for (int i = 0; i < n; ++i) res = __dadd_rn(res, __shfl_sync(0xffffffffu, v[0], i));
        return res;
    }
    const int body = n - (n % 8);
    double r = 0.0;
#pragma unroll
    for (int t = 0; t < 16; ++t) {
        if (8 * t >= body) break;
        const double x = __shfl_sync(0xffffffffu, v[t / 4], (lane + 8 * (t % 4)) & 31);
        r = t ? __dadd_rn(r, x) : x;
    }
    double rr[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) rr[j] = __shfl_sync(0xffffffffu, r, j);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(rr[0], rr[1]), __dadd_rn(rr[2], rr[3])),
                           __dadd_rn(__dadd_rn(rr[4], rr[5]), __dadd_rn(rr[6], rr[7])));
    for (int i = body; i < n; ++i) {
        double x = 0.0;
#pragma unroll
        for (int s2 = 0; s2 < 4; ++s2) {
            const double y = __shfl_sync(0xffffffffu, v[s2], i & 31);
            if ((i >> 5) == s2) x = y;
        }
        res = __dadd_rn(res, x);
    }
    return res;
}
template <class Val>
__device__ double pw_sum_warp(Val val, int n) {
    if (n <= 128) return pw_leaf_warp(val, 0, n);
    constexpr int kMaxFrames = 32;
    int32_t off[kMaxFrames], len[kMaxFrames];
    double lsum[kMaxFrames];
    bool right[kMaxFrames];
    int sp = 0;
    off[0] = 0, len[0] = n, right[0] = false;
    for (;;) {
        while (len[sp] > 128) {
            int32_t n2 = len[sp] / 2;
            n2 -= n2 % 8;
            off[sp + 1] = off[sp];
            len[sp + 1] = n2;
            right[sp + 1] = false;
            ++sp;
        }
        double v = pw_leaf_warp(val, off[sp], len[sp]);
        for (;;) {
            if (sp == 0) return v;
            const int p = sp - 1;
            int32_t n2 = len[p] / 2;
            n2 -= n2 % 8;
            if (!right[sp]) {
                lsum[p] = v;
                off[sp] = off[p] + n2;
                len[sp] = len[p] - n2;
                right[sp] = true;
                break;
            }
            v = __dadd_rn(lsum[p], v);
            --sp;
        }
    }
}

}  // namespace kt
