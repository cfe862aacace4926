// Microbenchmark: the bilateral's inner loop shape (k_bilateral_sep bulk rows) in isolation,
// all SMs, 16 warps each, to find which part keeps the LDS pipe below its wavefront rate.
// Per dx step: two row-word LDS, the tap depths (I2F), SD2 = S2 * D2 (FMUL2), then for each of
// P outputs two LEA.HI + two table LDS + FFMA2 (weights) + FFMA2 (values).
//   MODE 0: the kernel's shape            MODE 1: no value FFMA2 (weights only)
//   MODE 2: depths from a shift (no I2F)   MODE 3: S2 from a register pair instead of a constant
//   MODE 4: + the kernel's per-row epilogue (halves added, FP64 sy * row sum into double
//           accumulators, sy by a runtime row index)
//   MODE 5: MODE 4 with the row sums folded by FFMA2 into float-pair accumulators instead
// Prints table lookups per clock per SM (LDS floor: 32 * 16 / 18 = 28.4 with the row words).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bil_inner bil_inner.cu
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
__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
    return (static_cast<unsigned long long>(__float_as_uint(hi)) << 32) | __float_as_uint(lo);
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ unsigned long long fmul2(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

struct Par {
    unsigned long long sx2[17];
    double sy[33];
};

constexpr int P = 8;

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(const __grid_constant__ Par sp, float* out, int iters) {
    extern __shared__ __align__(16) unsigned char sm[];
    float* tbl = reinterpret_cast<float*>(sm);                       // [767][32]
    uint32_t* row = reinterpret_cast<uint32_t*>(sm + 767 * 32 * 4);  // [16 warps][64]
    for (int i = threadIdx.x; i < 767 * 32; i += blockDim.x) tbl[i] = 1.0f / (1 + i / 32);
    for (int i = threadIdx.x; i < 16 * 64; i += blockDim.x)
        row[i] = (((i * 2654435761u) >> 24) << 23) | ((i * 40503u) & 0xFFu);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t tbl_s = static_cast<uint32_t>(__cvta_generic_to_shared(tbl));
    const uint32_t* rw = row + warp * 64 + lane + 16;
    uint32_t base[P];
#pragma unroll
    for (int i = 0; i < P; ++i) base[i] = tbl_s + static_cast<uint32_t>((255 - (i * 29) % 256) * 128 + lane * 4);
    unsigned long long SW[P], SV[P];
#pragma unroll
    for (int i = 0; i < P; ++i) SW[i] = SV[i] = 0ull;
    unsigned long long S2r = sp.sx2[lane & 15];
    double ws[P], vs[P];
    unsigned long long AW[P], AV[P];
#pragma unroll
    for (int i = 0; i < P; ++i) ws[i] = vs[i] = 0.0, AW[i] = AV[i] = 0ull;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int dx = 1; dx <= 16; ++dx) {
            const uint32_t a = lds_u32(static_cast<uint32_t>(__cvta_generic_to_shared(rw - dx)));
            const uint32_t b = lds_u32(static_cast<uint32_t>(__cvta_generic_to_shared(rw + dx)));
            const uint32_t ga = a >> 16, gb = b >> 16;
            unsigned long long D2;
            if (MODE == 2) D2 = pack2(__uint_as_float((a & 0xFFu) | 0x3F800000u), __uint_as_float((b & 0xFFu) | 0x3F800000u));
            else D2 = pack2(static_cast<float>(a & 0xFFu), static_cast<float>(b & 0xFFu));
            const unsigned long long S2 = MODE == 3 ? S2r : sp.sx2[dx];
            const unsigned long long SD2 = fmul2(S2, D2);
#pragma unroll
            for (int i = 0; i < P; ++i) {
                const unsigned long long R2 = pack2(lds_f32(base[i] + ga), lds_f32(base[i] + gb));
                SW[i] = ffma2(S2, R2, SW[i]);
                if (MODE != 1) SV[i] = ffma2(R2, SD2, SV[i]);
            }
        }
        if (MODE == 3) S2r ^= static_cast<unsigned long long>(it & 1);
        if (MODE == 4) {
            const int t = it % 26 + 7;
#pragma unroll
            for (int i = 0; i < P; ++i) {
                const double sy = sp.sy[t - i];
                const float a0 = __uint_as_float(static_cast<uint32_t>(SW[i])), a1 = __uint_as_float(static_cast<uint32_t>(SW[i] >> 32));
                const float b0 = __uint_as_float(static_cast<uint32_t>(SV[i])), b1 = __uint_as_float(static_cast<uint32_t>(SV[i] >> 32));
                ws[i] = __fma_rn(sy, static_cast<double>(__fadd_rn(a0, a1)), ws[i]);
                vs[i] = __fma_rn(sy, static_cast<double>(__fadd_rn(b0, b1)), vs[i]);
                SW[i] = SV[i] = 0ull;
            }
        }
        if (MODE == 5) {
            const int t = it % 26 + 7;
#pragma unroll
            for (int i = 0; i < P; ++i) {
                const float syf = static_cast<float>(sp.sy[t - i]);
                const unsigned long long SY2 = pack2(syf, syf);
                AW[i] = ffma2(SY2, SW[i], AW[i]);
                AV[i] = ffma2(SY2, SV[i], AV[i]);
                SW[i] = SV[i] = 0ull;
            }
        }
    }
#pragma unroll
    for (int i = 0; i < P; ++i) {
        SW[i] ^= AW[i];
        SV[i] ^= AV[i];
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < P; ++i) s += static_cast<float>(ws[i] + vs[i]);
#pragma unroll
    for (int i = 0; i < P; ++i) s += __uint_as_float(static_cast<uint32_t>(SW[i])) + __uint_as_float(static_cast<uint32_t>(SV[i] >> 32));
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float* out;
    cudaMalloc(&out, sms * 512 * sizeof(float));
    Par sp;
    for (int d = 0; d < 33; ++d) sp.sy[d] = 1.0 / (1 + d);
    for (int d = 0; d <= 16; ++d) {
        const float f = 1.0f / (1 + d);
        const unsigned long long u = __builtin_bit_cast(unsigned, f);
        sp.sx2[d] = (u << 32) | u;
    }
    const int iters = 1500;
    const size_t smem = 767 * 32 * 4 + 16 * 64 * 4;
    void (*ks[6])(Par, float*, int) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>};
    const char* names[6] = {"kernel shape", "no value FMA", "no I2F", "S2 in registers", "+ row epilogue", "+ f32 row fold"};
    for (int m = 0; m < 6; ++m) {
        cudaFuncSetAttribute(ks[m], cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        ks[m]<<<sms, 512, smem>>>(sp, out, 10);
        cudaError_t le = cudaDeviceSynchronize();
        if (le != cudaSuccess) printf("mode %d: %s\n", m, cudaGetErrorString(le));
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        float best = 1e30f;
        for (int r = 0; r < 3; ++r) {
            cudaEventRecord(a);
            ks[m]<<<sms, 512, smem>>>(sp, out, iters);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        const double lookups = double(sms) * 512 * iters * 16 * 2 * P;
        const double clocks = best * 1e-3 * clk * 1e3;
        printf("%-16s %.3f ms  %.2f lookups/clk/SM  (err %s)\n", names[m], best, lookups / clocks / sms,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
