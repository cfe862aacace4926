// Latency probe: dependent chains of DADD / DMUL / FADD / LDS on one warp (clock64).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lat(double* out, long long* cyc, double a, float fa) {
    __shared__ double s[64];
    if (threadIdx.x < 64) s[threadIdx.x] = threadIdx.x * 0.5;
    __syncthreads();
    double x = a, y = a * 0.5;
    float f = fa;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) {
        x = __dadd_rn(x, 1.0000001);
        x = __dadd_rn(x, 0.9999999);
    }
    long long t1 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) {
        y = __dmul_rn(y, 1.0000001);
        y = __dmul_rn(y, 0.9999999);
    }
    long long t2 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) {
        f = __fadd_rn(f, 1.0000001f);
        f = __fadd_rn(f, 0.9999999f);
    }
    long long t3 = clock64();
    int idx = threadIdx.x & 1;
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) {
        idx = static_cast<int>(s[idx & 63]) & 1;
        idx = static_cast<int>(s[idx & 63]) & 1;
    }
    long long t4 = clock64();
    out[threadIdx.x] = x + y + f + idx;
    if (threadIdx.x == 0) {
        cyc[0] = t1 - t0;
        cyc[1] = t2 - t1;
        cyc[2] = t3 - t2;
        cyc[3] = t4 - t3;
    }
}

int main() {
    double* o;
    long long* c;
    cudaMalloc(&o, 64 * sizeof(double));
    cudaMallocManaged(&c, 4 * sizeof(long long));
    for (int rep = 0; rep < 3; ++rep) {
        k_lat<<<1, 32>>>(o, c, 1.0, 1.0f);
        cudaDeviceSynchronize();
    }
    printf("per-op latency (cycles): DADD %.1f  DMUL %.1f  FADD %.1f  LDS.64+cvt %.1f\n",
           c[0] / 2048.0, c[1] / 2048.0, c[2] / 2048.0, c[3] / 2048.0);
    return 0;
}
