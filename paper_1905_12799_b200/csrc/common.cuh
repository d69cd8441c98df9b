// common.cuh — shared types, error plumbing and numpy-order float helpers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <initializer_list>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/knobtuner_b200.h"

namespace kt {

// ---------------------------------------------------------------- errors
struct Error {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg);
void set_last_error(const std::string& msg);

#define KT_CUDA(call)                                                                   \
    do {                                                                                \
        cudaError_t _e = (call);                                                        \
        if (_e != cudaSuccess)                                                          \
            ::kt::fail(KT_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
    } while (0)

// Wrap an extern "C" body: converts exceptions into status codes.
#define KT_API_BEGIN try {
#define KT_API_END                                        \
    }                                                     \
    catch (const ::kt::Error& err) {                      \
        ::kt::set_last_error(err.msg);                    \
        return err.code;                                  \
    }                                                     \
    catch (const std::exception& ex) {                    \
        ::kt::set_last_error(ex.what());                  \
        return KT_ERR_INTERNAL;                           \
    }                                                     \
    return KT_OK;

// ---------------------------------------------------------------- layout
constexpr int kMaxKnobs = 8;      // a row is one uint64 (see RowFmt)
constexpr int kMaxCard = 255;     // index 255 never occurs -> usable as a sentinel
constexpr uint64_t kEmptyRow = ~0ull;

// Align a pointer into dynamic shared memory by pointer arithmetic on the shared
// array itself, so the compiler keeps the shared address space (LDS/STS).  Casting
// through uintptr_t would turn every access into a generic LD/ST.
template <unsigned ALIGN>
__device__ __forceinline__ unsigned char* align_shared(unsigned char* p) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
    return p + ((ALIGN - (a & (ALIGN - 1))) & (ALIGN - 1));
}


// Row layout of a space: knob i occupies bits [shift[i], shift[i] + width[i]) of
// the uint64 row.  Spaces whose cardinalities are all <= 255 use one byte per knob
// (shift 8i, width 8: `bytes` = 1, the fast paths); wider spaces (AlexNet's
// tile_f has 480 settings) pack minimal-width fields, sum of widths <= 64.
struct RowFmt {
    uint8_t shift[kMaxKnobs];
    uint8_t width[kMaxKnobs];
    int32_t cmax;   // largest index any knob can take (max cardinality - 1)
    int32_t bytes;  // 1: the byte-per-knob layout
    __host__ __device__ __forceinline__ int get(uint64_t row, int i) const {
        return int((row >> shift[i]) & ((1ull << width[i]) - 1ull));
    }
    __host__ __device__ __forceinline__ uint64_t set(uint64_t row, int i, int v) const {
        const uint64_t mask = ((1ull << width[i]) - 1ull) << shift[i];
        return (row & ~mask) | ((uint64_t(v) << shift[i]) & mask);
    }
};

// Same rule as paper_1905_12799_b200.space.row_layout (host side).
RowFmt row_fmt(const int32_t* cards, int n);

// ---------------------------------------------------------- numpy sums
// numpy's pairwise_sum for a contiguous run of n <= 8 float64 values
// (numpy/_core/src/umath/loops_utils.h.src): n < 8 sums sequentially from
// 0.0, n == 8 uses the 8-accumulator tree.  All ops are explicit _rn
// intrinsics so no FMA contraction can change the rounding.
__device__ __forceinline__ double np_sum_small(const double* t, int n) {
    if (n == 8) {
        double a = __dadd_rn(__dadd_rn(t[0], t[1]), __dadd_rn(t[2], t[3]));
        double b = __dadd_rn(__dadd_rn(t[4], t[5]), __dadd_rn(t[6], t[7]));
        return __dadd_rn(a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
        if (i < n) s = __dadd_rn(s, t[i]);
    return s;
}

// ((p - c)**2).sum(axis=-1) for a lattice point p (row) and float64 centroid c.
__device__ __forceinline__ double np_sq_dist(uint64_t row, const double* c, int n, const RowFmt& f) {
    double t[kMaxKnobs];
#pragma unroll
    for (int i = 0; i < kMaxKnobs; ++i) {
        if (i < n) {
            double d = __dsub_rn(double(f.get(row, i)), c[i]);
            t[i] = __dmul_rn(d, d);
        }
    }
    return np_sum_small(t, n);
}

__device__ __forceinline__ int64_t int_sq_dist(uint64_t a, uint64_t b, int n, const RowFmt& f) {
    int64_t s = 0;
#pragma unroll
    for (int i = 0; i < kMaxKnobs; ++i) {
        if (i < n) {
            const int64_t d = f.get(a, i) - f.get(b, i);
            s += d * d;
        }
    }
    return s;
}

// 64-bit mixer (murmur3 finaliser) for the dedup hash tables.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ull;
    k ^= k >> 33;
    return k;
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace kt

// ------------------------------------------------------------------ engine
struct kt_engine {
    int device = 0;
    int num_sms = 148;
    cudaStream_t own_stream = nullptr;
    cudaEvent_t order_event = nullptr;  // kt_engine_order
    cudaStream_t stream = nullptr;
    int64_t launches = 0;
    struct Buf {
        void* ptr = nullptr;
        size_t bytes = 0;
    };
    std::unordered_map<std::string, Buf> dev;
    std::unordered_map<std::string, Buf> pinned;

    // Optional per-kernel CUDA-event timing (kt_engine_set_timing).
    bool timing = false;
    cudaEvent_t open_start = nullptr;
    struct Pending {
        const char* name;
        cudaEvent_t start, stop;
    };
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> event_pool;
    struct Stat {
        int64_t count = 0;
        double ms = 0.0;
    };
    std::map<std::string, Stat> stats;

    // Named, growable device scratch (contents undefined after growth).
    void* scratch(const std::string& name, size_t bytes);
    // Named, growable pinned host staging buffer.
    void* staging(const std::string& name, size_t bytes);
    // Small device -> pinned-host read-back on the engine stream, written by a one-block kernel
    // through the pinned buffer's UVA mapping: it never queues behind a large D2H copy on the
    // copy engine (the e2e leg's 8 MB score copies).  host_dst must come from staging().
    void d2h(void* host_dst, const void* dev_src, size_t bytes);
    // up to 8 such read-backs in one launch
    struct D2H {
        void* dst;
        const void* src;
        size_t bytes;
    };
    void d2h(std::initializer_list<D2H> regions);
    void note_launch(int n = 1) { launches += n; }
    void pre_launch(const char* what);    // call right before a kernel launch
    void check_launch(const char* what);  // call right after it
    void flush_timing();
    cudaEvent_t take_event();
    void sync();
};

namespace kt {
// Launch helpers shared across translation units.
void allow_dynamic_smem(const void* kernel);
int occupancy_blocks(const void* kernel, int threads, size_t smem);  // cached per (device, kernel, shape)
int smem_optin(int device);             // cudaDevAttrMaxSharedMemoryPerBlockOptin, cached
size_t static_smem(const void* kernel);  // cudaFuncAttributes::sharedSizeBytes, cached
// out[i] = sum(in[0..i)), out[n] = total; n <= 16M (single-block scan).
void exclusive_scan(kt_engine* e, const int64_t* in, int64_t* out, int n);
// K6's first-occurrence hash table over rows[0, count): *first = per-slot lowest row index,
// *slot = each row's slot, so row i is a first occurrence iff first[slot[i]] == i (engine scratch).
void dedup_table(kt_engine* e, const uint64_t* rows, int64_t count, const uint32_t** first, const uint32_t** slot);
}  // namespace kt
