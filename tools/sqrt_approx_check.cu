// Exhaustive relative error of sqrt.approx.f32 against the correctly rounded sqrt over
// every float in [2^-30, 2^30] (the Lloyd kernels' bound square roots rely on it:
// sampler.cu kSqrtSlack).  nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/sq tools/sqrt_approx_check.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
__global__ void k(uint32_t lo, uint32_t hi, unsigned long long* worst) {
    double w = 0.0;
    for (uint32_t b = lo + blockIdx.x * blockDim.x + threadIdx.x; b < hi; b += gridDim.x * blockDim.x) {
        const float x = __uint_as_float(b);
        float r;
        asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
        const double e = sqrt((double)x);
        const double rel = fabs((double)r - e) / e;
        w = rel > w ? rel : w;
    }
    atomicMax(worst, (unsigned long long)__double_as_longlong(w));
}
int main() {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    cudaMemset(d, 0, 8);
    const uint32_t lo = (127u - 30u) << 23, hi = (127u + 30u) << 23;
    k<<<148 * 8, 256>>>(lo, hi, d);
    unsigned long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    double w;
    memcpy(&w, &h, 8);
    printf("sqrt.approx.f32 max relative error over [2^-30, 2^30]: %.3e (2^%.2f)\n", w, log2(w));
    return 0;
}
