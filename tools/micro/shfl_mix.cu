// Microbenchmark: does SHFL take shared-memory wavefronts from a conflict-free LDS gather
// stream? Bilateral-shaped inner loop: per dx step one "row word" c (guide << 23), then 8
// table lookups at base_j + (c >> 16) (LEA.HI + LDS.32 + FADD). The row word comes from
//   MODE 0: an LDS.32 of a shared row (the kernel's current form: 9 wavefronts per 8 lookups)
//   MODE 1: a SHFL of a register the lane loaded once
//   MODE 2: register arithmetic (no load: the lookup-only floor)
// Prints lookups per clock per SM (all SMs, 16 warps each).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o shfl_mix shfl_mix.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float lds_f32(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(float* out, int iters) {
    extern __shared__ __align__(16) unsigned char sm[];
    float* tbl = reinterpret_cast<float*>(sm);                    // [512][32]
    uint32_t* row = reinterpret_cast<uint32_t*>(sm + 512 * 32 * 4);  // [16 warps][96]
    for (int i = threadIdx.x; i < 512 * 32; i += blockDim.x) tbl[i] = 1.0f / (1 + i / 32);
    for (int i = threadIdx.x; i < 16 * 96; i += blockDim.x) row[i] = ((i * 2654435761u) >> 24) << 23;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t tbl_s = static_cast<uint32_t>(__cvta_generic_to_shared(tbl));
    const uint32_t row_s = static_cast<uint32_t>(__cvta_generic_to_shared(row + warp * 96 + lane));
    uint32_t base[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) base[j] = tbl_s + (j * 30) * 128 + lane * 4;
    uint32_t my = row[warp * 96 + lane];
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int dx = 0; dx < 32; ++dx) {
            uint32_t c;
            if (MODE == 0) c = lds_u32(row_s + 4 * dx);
            else if (MODE == 1) c = __shfl_sync(0xFFFFFFFFu, my, (lane + dx) & 31);
            else c = my + (static_cast<uint32_t>(dx * 7) << 23);
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] += lds_f32(base[j] + (c >> 16));
        }
        my ^= static_cast<uint32_t>(it & 1) << 23;
    }
    float s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += acc[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float* out;
    cudaMalloc(&out, sms * 512 * sizeof(float));
    const int iters = 2000;
    const size_t smem = 512 * 32 * 4 + 16 * 96 * 4;
    void (*ks[3])(float*, int) = {k<0>, k<1>, k<2>};
    const char* names[3] = {"row via LDS", "row via SHFL", "row in regs"};
    for (int m = 0; m < 3; ++m) {
        cudaFuncSetAttribute(ks[m], cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        ks[m]<<<sms, 512, smem>>>(out, 10);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        float best = 1e30f;
        for (int r = 0; r < 3; ++r) {
            cudaEventRecord(a);
            ks[m]<<<sms, 512, smem>>>(out, iters);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        const double lookups = double(sms) * 512 * iters * 32 * 8;
        const double clocks = best * 1e-3 * clk * 1e3;
        printf("%-14s %.3f ms  %.2f lookups/clk/SM  (err %s)\n", names[m], best, lookups / clocks / sms,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
