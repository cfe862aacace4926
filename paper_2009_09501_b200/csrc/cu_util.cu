// Small device-query helpers shared by the kernel launchers.
#include "p3s_cu.h"

namespace p3s {
namespace cu {

int sm_count() {
    static int cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64 && cache[dev]) return cache[dev];
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n < 1) n = 1;
    if (dev >= 0 && dev < 64) cache[dev] = n;
    return n;
}

namespace {
// 8 independent chains per thread of x = x*a + b as separately rounded DMUL, DADD.
__global__ void __launch_bounds__(256) k_fp64_peak(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = 1.0 + 1e-9 * (threadIdx.x + k);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = __dadd_rn(__dmul_rn(x[k], a), b);
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}
}  // namespace

cudaError_t fp64_peak(double* ops_per_s) {
    const int blocks = sm_count() * 8, threads = 256, iters = 4096;
    double* dummy = nullptr;
    cudaError_t e = cudaMalloc(&dummy, sizeof(double));
    if (e != cudaSuccess) return e;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_fp64_peak<<<blocks, threads>>>(dummy, iters, 0.999999, 1e-7);  // warm-up
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(a);
        k_fp64_peak<<<blocks, threads>>>(dummy, iters, 0.999999, 1e-7);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    e = cudaGetLastError();
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(dummy);
    const double ops = 2.0 * 8.0 * iters * static_cast<double>(blocks) * threads;
    *ops_per_s = ops / (best * 1e-3);
    return e;
}

}  // namespace cu
}  // namespace p3s
