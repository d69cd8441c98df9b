// landscape.cu — K3 score_landscape: the synthetic "fake hardware" oracle.
//
// Replaces synthetic_runtime / _hash_unit (backends.py:157-174):
//   runtime = base * (1 - sum_j depth_j * exp(-|x - c_j|^2 / r_j^2))
//   runtime *= 1 + noise * u,  u = 2 * (blake2b64("seed:i0,i1,...") / 2^64) - 1
//   runtime = max(runtime, 0.01 * base)
// |x - c_j|^2 is an integer (lattice points), so it is exact in any order; the
// remaining float64 ops follow the reference's evaluation order with explicit
// _rn intrinsics, and exp() is a bit-exact restatement of glibc's (the
// reference's math.exp; glibc_exp.cuh), so runtimes equal the reference's bit
// for bit.
//
// kt_landscape_best: the brute-force optimum of cli.py:77-90 (_enumerated_oracle)
// without the 10^6 enumeration cap (space.py:20): lexicographic ranks (last knob
// fastest, enumerate_space's order) are decoded into rows on the fly, scored, and
// reduced to (min runtime, lowest rank) — the first minimum, like the reference's
// strict `<` scan.
//
// blake2b (RFC 7693), unkeyed, 8-byte digest, one 128-byte block: the payload
// "seed:" + decimal indices joined by ',' is at most 21 + 1 + 8 * 4 bytes.
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "glibc_exp.cuh"

constexpr int kMaxCenters = 16;

struct kt_landscape {
    int n = 0;
    int n_centers = 0;
    double base = 1.0;
    double noise = 0.0;
    std::string prefix;  // str(seed) + ":"
    kt::RowFmt fmt{};
    int32_t centers[kMaxCenters][8] = {};
    double depths[kMaxCenters] = {};
    double radii[kMaxCenters] = {};
};

namespace kt {

struct LandscapeArgs {
    int n, n_centers, prefix_len;
    RowFmt fmt;
    double base, noise;
    int32_t centers[kMaxCenters][8];
    double depths[kMaxCenters];
    double r2[kMaxCenters];
    unsigned char prefix[64];
};

__device__ __constant__ uint64_t kBlakeIV[8] = {0x6a09e667f3bcc908ull, 0xbb67ae8584caa73bull, 0x3c6ef372fe94f82bull,
                                               0xa54ff53a5f1d36f1ull, 0x510e527fade682d1ull, 0x9b05688c2b3e6c1full,
                                               0x1f83d9abfb41bd6bull, 0x5be0cd19137e2179ull};

__device__ __forceinline__ uint64_t rotr64(uint64_t x, int r) { return (x >> r) | (x << (64 - r)); }

#define KT_G(a, b, c, d, x, y)      \
    a = a + b + x;                  \
    d = rotr64(d ^ a, 32);          \
    c = c + d;                      \
    b = rotr64(b ^ c, 24);          \
    a = a + b + y;                  \
    d = rotr64(d ^ a, 16);          \
    c = c + d;                      \
    b = rotr64(b ^ c, 63);

// blake2b-64 of a single final block m[16] holding `len` bytes.
__device__ uint64_t blake2b64_one_block(const uint64_t m[16], uint64_t len) {
    constexpr unsigned char sigma[12][16] = {
        {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
        {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4}, {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
        {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13}, {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
        {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11}, {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
        {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5}, {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
        {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};
    const uint64_t h0 = kBlakeIV[0] ^ 0x01010008ull;  // digest 8 bytes, no key
    uint64_t v0 = h0, v1 = kBlakeIV[1], v2 = kBlakeIV[2], v3 = kBlakeIV[3];
    uint64_t v4 = kBlakeIV[4], v5 = kBlakeIV[5], v6 = kBlakeIV[6], v7 = kBlakeIV[7];
    uint64_t v8 = kBlakeIV[0], v9 = kBlakeIV[1], v10 = kBlakeIV[2], v11 = kBlakeIV[3];
    uint64_t v12 = kBlakeIV[4] ^ len, v13 = kBlakeIV[5], v14 = ~kBlakeIV[6], v15 = kBlakeIV[7];
#pragma unroll
    for (int r = 0; r < 12; ++r) {
        const unsigned char* s = sigma[r];
        KT_G(v0, v4, v8, v12, m[s[0]], m[s[1]]);
        KT_G(v1, v5, v9, v13, m[s[2]], m[s[3]]);
        KT_G(v2, v6, v10, v14, m[s[4]], m[s[5]]);
        KT_G(v3, v7, v11, v15, m[s[6]], m[s[7]]);
        KT_G(v0, v5, v10, v15, m[s[8]], m[s[9]]);
        KT_G(v1, v6, v11, v12, m[s[10]], m[s[11]]);
        KT_G(v2, v7, v8, v13, m[s[12]], m[s[13]]);
        KT_G(v3, v4, v9, v14, m[s[14]], m[s[15]]);
    }
    return h0 ^ v0 ^ v8;
}

__device__ __forceinline__ void put_byte(uint64_t m[16], int pos, unsigned v) {
    m[pos >> 3] |= uint64_t(v & 0xffu) << (8 * (pos & 7));
}

// runtime of one configuration row (backends.py:164-174); `tab` = the exp table in shared memory
__device__ __forceinline__ double landscape_runtime(const LandscapeArgs& a, uint64_t row, const uint64_t* tab) {
    double depth_term = 0.0;
    for (int j = 0; j < a.n_centers; ++j) {
        int64_t d2 = 0;  // exact: numpy's ((x - c) ** 2).sum() of integer-valued float64
        for (int q = 0; q < a.n; ++q) {
            const int64_t d = a.fmt.get(row, q) - a.centers[j][q];
            d2 += d * d;
        }
        const double e = glibc_exp(__ddiv_rn(-double(d2), a.r2[j]), tab);
        depth_term = __dadd_rn(depth_term, __dmul_rn(a.depths[j], e));
    }
    double rt = __dmul_rn(a.base, __dsub_rn(1.0, depth_term));
    if (a.noise > 0.0) {
        uint64_t m[16];
#pragma unroll
        for (int w = 0; w < 16; ++w) m[w] = 0;
        int pos = 0;
        for (; pos < a.prefix_len; ++pos) put_byte(m, pos, a.prefix[pos]);
        for (int q = 0; q < a.n; ++q) {
            if (q) put_byte(m, pos++, ',');
            const int v = a.fmt.get(row, q);  // str(v): up to 5 digits
            if (v >= 10000) put_byte(m, pos++, '0' + v / 10000);
            if (v >= 1000) put_byte(m, pos++, '0' + (v / 1000) % 10);
            if (v >= 100) put_byte(m, pos++, '0' + (v / 100) % 10);
            if (v >= 10) put_byte(m, pos++, '0' + (v / 10) % 10);
            put_byte(m, pos++, '0' + v % 10);
        }
        const uint64_t h = blake2b64_one_block(m, uint64_t(pos));
        const uint64_t word = __byte_perm(uint32_t(h >> 32), 0, 0x0123) | (uint64_t(__byte_perm(uint32_t(h), 0, 0x0123)) << 32);
        const double unit = __dsub_rn(2.0 * (__ull2double_rn(word) * 5.421010862427522e-20), 1.0);  // 2^-64
        rt = __dmul_rn(rt, __dadd_rn(1.0, __dmul_rn(a.noise, unit)));
    }
    const double floor_rt = __dmul_rn(0.01, a.base);
    return floor_rt > rt ? floor_rt : rt;
}

__device__ __forceinline__ void load_exp_table(uint64_t* tab) {
    for (int i = threadIdx.x; i < 2 * kExpN; i += blockDim.x) tab[i] = kExpTableConst[i];
    __syncthreads();
}

__global__ void __launch_bounds__(256) landscape_kernel(const LandscapeArgs a, const uint64_t* __restrict__ rows,
                                                        int64_t count, double* __restrict__ out) {
    __shared__ uint64_t tab[2 * kExpN];
    load_exp_table(tab);
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x)
        out[i] = landscape_runtime(a, rows[i], tab);
}

struct EnumArgs {
    int64_t stride[kMaxKnobs];  // lexicographic rank strides, last knob fastest
    int32_t card[kMaxKnobs];
};

// (runtime, rank) order: smaller runtime first, then the lower rank (the first minimum)
__device__ __forceinline__ bool better(double v, int64_t r, double bv, int64_t br) {
    return v < bv || (v == bv && r < br);
}

constexpr int kBestThreads = 256;

// Grid-stride over ranks [lo, hi); each block writes its best (runtime, rank) pair.
__global__ void __launch_bounds__(kBestThreads) landscape_best_kernel(const LandscapeArgs a, const EnumArgs en,
                                                                     int64_t lo, int64_t hi, double* __restrict__ bv_out,
                                                                     int64_t* __restrict__ br_out) {
    __shared__ uint64_t tab[2 * kExpN];
    __shared__ double s_v[kBestThreads / 32];
    __shared__ int64_t s_r[kBestThreads / 32];
    load_exp_table(tab);
    double bv = __longlong_as_double(0x7ff0000000000000ll);  // +inf
    int64_t br = INT64_MAX;
    for (int64_t r = lo + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < hi; r += int64_t(gridDim.x) * blockDim.x) {
        uint64_t row = 0;
        for (int q = 0; q < a.n; ++q) row = a.fmt.set(row, q, int((r / en.stride[q]) % en.card[q]));
        const double v = landscape_runtime(a, row, tab);
        if (better(v, r, bv, br)) { bv = v; br = r; }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int64_t orr = __shfl_xor_sync(0xffffffffu, br, o);
        if (better(ov, orr, bv, br)) { bv = ov; br = orr; }
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) { s_v[w] = bv; s_r[w] = br; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < kBestThreads / 32; ++i)
            if (better(s_v[i], s_r[i], bv, br)) { bv = s_v[i]; br = s_r[i]; }
        bv_out[blockIdx.x] = bv;
        br_out[blockIdx.x] = br;
    }
}

}  // namespace kt

extern "C" {

int kt_landscape_create(kt_engine* e, int n_knobs, const int32_t* cards, int n_centers, const int32_t* centers,
                        const double* depths,
                        const double* radii, double base_runtime, double noise_rel, const char* seed_text,
                        kt_landscape** out) {
    KT_API_BEGIN
    using namespace kt;
    (void)e;
    if (n_knobs < 1 || n_knobs > kMaxKnobs) fail(KT_ERR_UNSUPPORTED, "1..8 knobs supported");
    if (n_centers < 1 || n_centers > kMaxCenters) fail(KT_ERR_UNSUPPORTED, "1..16 landscape centers supported");
    const RowFmt fmt = row_fmt(cards, n_knobs);
    auto* l = new kt_landscape();
    l->fmt = fmt;
    l->n = n_knobs;
    l->n_centers = n_centers;
    l->base = base_runtime;
    l->noise = noise_rel;
    l->prefix = std::string(seed_text ? seed_text : "") + ":";
    const size_t digits = fmt.cmax >= 10000 ? 5 : (fmt.cmax >= 1000 ? 4 : 3);
    if (l->prefix.size() + (digits + 1) * size_t(n_knobs) > 128 || l->prefix.size() > 64) {
        delete l;
        fail(KT_ERR_UNSUPPORTED, "landscape seed text too long for a one-block blake2b payload");
    }
    for (int j = 0; j < n_centers; ++j) {
        for (int q = 0; q < n_knobs; ++q) l->centers[j][q] = centers[j * n_knobs + q];
        l->depths[j] = depths[j];
        l->radii[j] = radii[j];
    }
    *out = l;
    KT_API_END
}

int kt_landscape_destroy(kt_landscape* l) {
    delete l;
    return KT_OK;
}

}  // extern "C"

namespace kt {
static LandscapeArgs landscape_args(const kt_landscape* l) {
    LandscapeArgs a{};
    a.n = l->n;
    a.fmt = l->fmt;
    a.n_centers = l->n_centers;
    a.base = l->base;
    a.noise = l->noise;
    a.prefix_len = int(l->prefix.size());
    std::memcpy(a.prefix, l->prefix.data(), l->prefix.size());
    for (int j = 0; j < l->n_centers; ++j) {
        for (int q = 0; q < 8; ++q) a.centers[j][q] = l->centers[j][q];
        a.depths[j] = l->depths[j];
        a.r2[j] = l->radii[j] * l->radii[j];
    }
    return a;
}
}  // namespace kt

extern "C" {

int kt_score_landscape(kt_engine* e, const kt_landscape* l, const uint64_t* rows_dev, int64_t count,
                       double* runtime_dev) {
    KT_API_BEGIN
    using namespace kt;
    if (count <= 0) return KT_OK;
    const LandscapeArgs a = landscape_args(l);
    const int grid = int(std::min<int64_t>(ceil_div(count, 256), int64_t(e->num_sms) * 8));
    e->pre_launch("score_landscape");
    landscape_kernel<<<grid, 256, 0, e->stream>>>(a, rows_dev, count, runtime_dev);
    e->check_launch("score_landscape");
    KT_API_END
}

int kt_landscape_best(kt_engine* e, const kt_landscape* l, const int32_t* cards, double* best_runtime,
                      int64_t* best_rank) {
    KT_API_BEGIN
    using namespace kt;
    const LandscapeArgs a = landscape_args(l);
    EnumArgs en{};
    int64_t total = 1;
    for (int q = a.n - 1; q >= 0; --q) {
        if (cards[q] < 1) fail(KT_ERR_VALUE, "cardinalities must be positive");
        en.stride[q] = total;
        en.card[q] = cards[q];
        if (total > INT64_MAX / cards[q]) fail(KT_ERR_UNSUPPORTED, "space too large to enumerate");
        total *= cards[q];
    }
    const int grid = e->num_sms * 8;
    auto* bv = static_cast<double*>(e->scratch("landscape.best", size_t(grid) * 16));
    auto* br = reinterpret_cast<int64_t*>(bv + grid);
    std::vector<double> hv(grid);
    std::vector<int64_t> hr(grid);
    double best_v = INFINITY;
    int64_t best_r = -1;
    constexpr int64_t kChunk = int64_t(1) << 30;  // bounded launches (watchdog-free, host can interleave)
    for (int64_t lo = 0; lo < total; lo += kChunk) {
        const int64_t hi = std::min(total, lo + kChunk);
        e->pre_launch("landscape_best");
        landscape_best_kernel<<<grid, kBestThreads, 0, e->stream>>>(a, en, lo, hi, bv, br);
        e->check_launch("landscape_best");
        KT_CUDA(cudaMemcpyAsync(hv.data(), bv, size_t(grid) * 8, cudaMemcpyDeviceToHost, e->stream));
        KT_CUDA(cudaMemcpyAsync(hr.data(), br, size_t(grid) * 8, cudaMemcpyDeviceToHost, e->stream));
        e->sync();
        for (int b = 0; b < grid; ++b)
            if (hr[b] >= 0 && hr[b] != INT64_MAX && (hv[b] < best_v || (hv[b] == best_v && hr[b] < best_r))) {
                best_v = hv[b];
                best_r = hr[b];
            }
    }
    *best_runtime = best_v;
    *best_rank = best_r;
    KT_API_END
}

}  // extern "C"
