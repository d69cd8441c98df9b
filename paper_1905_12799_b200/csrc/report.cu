// report.cu — trajectory analysis on the device.
//
// Reference: knobtuner/report.py per_step_best (:53-69) — the round's best surrogate
// score after each search step — and pca_project (:227-253) — centred index vectors
// projected on the two leading principal axes.
//
//   * step_best: one float64 max per step index (scatter-max on an order-preserving
//     integer encoding of the doubles; exact), the running max is taken on the host.
//   * pca moments: exact int64 sums of the indices and of their pairwise products
//     (indices < 2^16, so every product and sum of up to 2^31 rows fits in int64); the
//     host forms mean and covariance in float64 from them.
//   * pca projection: per row, (x - mean) . v1 and . v2 in float64.
#include <cstring>
#include <vector>

#include "common.cuh"

namespace kt {
namespace {

__device__ __forceinline__ unsigned long long order_key(double x) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void step_best_kernel(const double* __restrict__ scores, const int32_t* __restrict__ steps, int64_t count,
                                 int cap, unsigned long long* best, int* horizon) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x) {
        const int s = steps[i];
        if (s < 0 || s >= cap) continue;  // reported by the horizon check on the host
        atomicMax(best + s, order_key(scores[i]));
        atomicMax(horizon, s);
    }
}

constexpr int kMomentThreads = 256;

// Per block: sums of x_i and x_i * x_j over its rows; then one int64 atomic per moment.
__global__ void __launch_bounds__(kMomentThreads) pca_moments_kernel(const uint64_t* __restrict__ rows, int64_t count,
                                                                      int n, const RowFmt fmt, long long* out) {
    __shared__ long long s_acc[kMaxKnobs + kMaxKnobs * kMaxKnobs];
    const int nm = n + n * n;
    for (int i = threadIdx.x; i < nm; i += blockDim.x) s_acc[i] = 0;
    __syncthreads();
    long long acc[kMaxKnobs + kMaxKnobs * kMaxKnobs];
#pragma unroll
    for (int i = 0; i < kMaxKnobs + kMaxKnobs * kMaxKnobs; ++i) acc[i] = 0;
    for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < count; r += int64_t(gridDim.x) * blockDim.x) {
        const uint64_t row = rows[r];
        long long x[kMaxKnobs];
#pragma unroll
        for (int i = 0; i < kMaxKnobs; ++i) x[i] = i < n ? fmt.get(row, i) : 0;
#pragma unroll
        for (int i = 0; i < kMaxKnobs; ++i) {
            acc[i] += x[i];
#pragma unroll
            for (int j = 0; j < kMaxKnobs; ++j) acc[kMaxKnobs + i * kMaxKnobs + j] += x[i] * x[j];
        }
    }
    // warp reduce, then shared, then global
#pragma unroll
    for (int i = 0; i < kMaxKnobs + kMaxKnobs * kMaxKnobs; ++i) {
        long long v = acc[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        acc[i] = v;
    }
    if ((threadIdx.x & 31) == 0) {
        for (int i = 0; i < n; ++i) atomicAdd(reinterpret_cast<unsigned long long*>(s_acc + i), (unsigned long long)acc[i]);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                atomicAdd(reinterpret_cast<unsigned long long*>(s_acc + n + i * n + j),
                          (unsigned long long)acc[kMaxKnobs + i * kMaxKnobs + j]);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nm; i += blockDim.x)
        atomicAdd(reinterpret_cast<unsigned long long*>(out + i), (unsigned long long)s_acc[i]);
}

struct Axes {
    double mean[kMaxKnobs], v1[kMaxKnobs], v2[kMaxKnobs];
};

__global__ void pca_project_kernel(const uint64_t* __restrict__ rows, int64_t count, int n, const RowFmt fmt, Axes ax,
                                   double* __restrict__ xs, double* __restrict__ ys) {
    for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < count; r += int64_t(gridDim.x) * blockDim.x) {
        const uint64_t row = rows[r];
        double a = 0.0, b = 0.0;
        for (int i = 0; i < n; ++i) {
            const double c = __dsub_rn(double(fmt.get(row, i)), ax.mean[i]);
            a = __fma_rn(c, ax.v1[i], a);
            b = __fma_rn(c, ax.v2[i], b);
        }
        xs[r] = a;
        ys[r] = b;
    }
}

}  // namespace
}  // namespace kt

extern "C" {

int kt_step_best(kt_engine* e, const double* scores_dev, const int32_t* steps_dev, int64_t count, int cap,
                 double* best_out, int32_t* horizon_out) {
    KT_API_BEGIN
    using namespace kt;
    if (count < 1) fail(KT_ERR_VALUE, "trajectory is empty");
    if (cap < 1) fail(KT_ERR_VALUE, "step capacity must be >= 1");
    auto* best = static_cast<unsigned long long*>(e->scratch("report.best", size_t(cap) * 8 + 8));
    int* hz = reinterpret_cast<int*>(best + cap);
    KT_CUDA(cudaMemsetAsync(best, 0, size_t(cap) * 8, e->stream));  // key 0 < every encoded double
    KT_CUDA(cudaMemsetAsync(hz, 0xff, 8, e->stream));  // the whole trailing word (read back)
    const int grid = int(std::min<int64_t>(ceil_div(count, 256), int64_t(e->num_sms) * 4));
    e->pre_launch("step_best");
    step_best_kernel<<<grid, 256, 0, e->stream>>>(scores_dev, steps_dev, count, cap, best, hz);
    e->check_launch("step_best");
    std::vector<unsigned long long> h(size_t(cap) + 1);
    KT_CUDA(cudaMemcpyAsync(h.data(), best, size_t(cap) * 8 + 8, cudaMemcpyDeviceToHost, e->stream));
    e->sync();
    int horizon;
    std::memcpy(&horizon, &h[cap], 4);
    for (int s = 0; s < cap; ++s) {
        const unsigned long long k = h[s];
        if (k == 0) {
            best_out[s] = -INFINITY;
            continue;
        }
        const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
        double x;
        std::memcpy(&x, &b, 8);
        best_out[s] = x;
    }
    *horizon_out = horizon;
    KT_API_END
}

int kt_pca_moments(kt_engine* e, const uint64_t* rows_dev, int64_t count, int n_knobs, const int32_t* cards,
                   int64_t* sums_out, int64_t* gram_out) {
    KT_API_BEGIN
    using namespace kt;
    if (n_knobs < 1 || n_knobs > kMaxKnobs) fail(KT_ERR_UNSUPPORTED, "1..8 knobs supported");
    if (count >= (int64_t(1) << 31)) fail(KT_ERR_UNSUPPORTED, "at most 2^31 rows");
    const RowFmt fmt = row_fmt(cards, n_knobs);
    const int nm = n_knobs + n_knobs * n_knobs;
    auto* acc = static_cast<long long*>(e->scratch("report.moments", size_t(nm) * 8));
    KT_CUDA(cudaMemsetAsync(acc, 0, size_t(nm) * 8, e->stream));
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(count, kMomentThreads), int64_t(e->num_sms) * 2)));
    e->pre_launch("pca_moments");
    pca_moments_kernel<<<grid, kMomentThreads, 0, e->stream>>>(rows_dev, count, n_knobs, fmt, acc);
    e->check_launch("pca_moments");
    std::vector<long long> h(static_cast<size_t>(nm));
    KT_CUDA(cudaMemcpyAsync(h.data(), acc, size_t(nm) * 8, cudaMemcpyDeviceToHost, e->stream));
    e->sync();
    for (int i = 0; i < n_knobs; ++i) sums_out[i] = h[size_t(i)];
    for (int i = 0; i < n_knobs * n_knobs; ++i) gram_out[i] = h[size_t(n_knobs + i)];
    KT_API_END
}

int kt_pca_project(kt_engine* e, const uint64_t* rows_dev, int64_t count, int n_knobs, const int32_t* cards,
                   const double* mean, const double* v1, const double* v2, double* xs_dev, double* ys_dev) {
    KT_API_BEGIN
    using namespace kt;
    if (n_knobs < 1 || n_knobs > kMaxKnobs) fail(KT_ERR_UNSUPPORTED, "1..8 knobs supported");
    Axes ax{};
    for (int i = 0; i < n_knobs; ++i) {
        ax.mean[i] = mean[i];
        ax.v1[i] = v1[i];
        ax.v2[i] = v2[i];
    }
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(count, 256), int64_t(e->num_sms) * 8)));
    e->pre_launch("pca_project");
    pca_project_kernel<<<grid, 256, 0, e->stream>>>(rows_dev, count, n_knobs, row_fmt(cards, n_knobs), ax, xs_dev,
                                                    ys_dev);
    e->check_launch("pca_project");
    KT_API_END
}

}  // extern "C"
