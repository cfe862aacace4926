// Microbenchmark: data-dependent per-lane table gathers through the shared-memory pipe
// (LDS, 32-way replicated table: conflict-free), the texture pipe (tex1Dfetch) and a mix,
// all SMs; prints lookups per clock per SM. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>  // 0: LDS only, 1: TEX only, 2: 2 LDS : 1 TEX, 3: 1:1
__global__ void __launch_bounds__(512, 1) k(cudaTextureObject_t tex, const float* __restrict__ tbl_g,
                                           float* out, int iters) {
    extern __shared__ float tbl[];
    for (int i = threadIdx.x; i < 512 * 32; i += blockDim.x) tbl[i] = tbl_g[i / 32];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    unsigned s = threadIdx.x * 2654435761u + blockIdx.x;
    float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 12; ++j) {
            s = s * 1664525u + 1013904223u;
            const unsigned idx = (s >> 20) & 511u;
            float v;
            const bool use_tex = MODE == 1 || (MODE == 2 && j % 3 == 2) || (MODE == 3 && (j & 1));
            if (use_tex) v = tex1Dfetch<float>(tex, static_cast<int>(idx));
            else v = tbl[idx * 32 + lane];
            if ((j & 3) == 0) acc0 += v;
            else if ((j & 3) == 1) acc1 += v;
            else if ((j & 3) == 2) acc2 += v;
            else acc3 += v;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float *tbl, *out;
    cudaMalloc(&tbl, 512 * sizeof(float));
    cudaMalloc(&out, sms * 512 * sizeof(float));
    cudaMemset(tbl, 0, 512 * sizeof(float));
    cudaResourceDesc rd{};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = tbl;
    rd.res.linear.desc = cudaCreateChannelDesc<float>();
    rd.res.linear.sizeInBytes = 512 * sizeof(float);
    cudaTextureDesc td{};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t tex;
    cudaCreateTextureObject(&tex, &rd, &td, nullptr);
    const int iters = 4000;
    void (*ks[4])(cudaTextureObject_t, const float*, float*, int) = {k<0>, k<1>, k<2>, k<3>};
    const char* names[4] = {"LDS only", "TEX only", "LDS:TEX 2:1", "LDS:TEX 1:1"};
    for (int m = 0; m < 4; ++m) {
        cudaFuncSetAttribute(ks[m], cudaFuncAttributeMaxDynamicSharedMemorySize, 512 * 32 * 4);
        ks[m]<<<sms, 512, 512 * 32 * 4>>>(tex, tbl, out, 10);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        ks[m]<<<sms, 512, 512 * 32 * 4>>>(tex, tbl, out, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double lookups = double(sms) * 512 * iters * 12;
        const double clocks = ms * 1e-3 * clk * 1e3;
        printf("%-14s %.3f ms  %.1f lookups/clk/SM  (err %s)\n", names[m], ms, lookups / clocks / sms,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
