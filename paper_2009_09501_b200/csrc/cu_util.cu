// Small device-query helpers shared by the kernel launchers.
#include <atomic>
#include <vector>

#include "p3s_cu.h"

namespace p3s {
namespace cu {

void record_event_any(cudaEvent_t e, cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if (cs == cudaStreamCaptureStatusActive)
        cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);
    else
        cudaEventRecord(e, st);
}

namespace {
// Zero up to kZeroRanges ranges of 4-byte words in one launch. cudaMemsetAsync nodes can be
// queued behind bulk copies on a copy engine (the banded convert keeps PCIe copies in flight
// while its kernels run); a kernel is not. The other way round, a kernel needs an SM slot,
// which other streams' persistent kernels may hold for milliseconds, so multi-stream paths
// keep the memsets.
__global__ void k_zero(ZeroRanges z) {
    const unsigned stride = gridDim.x * blockDim.x;
    for (int r = 0; r < z.n; ++r) {
        uint32_t* p = static_cast<uint32_t*>(z.p[r]);
        for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < z.words[r]; i += stride) p[i] = 0u;
    }
}
}  // namespace

namespace {
std::atomic<unsigned long long> g_launches{0};
}

void note_launch(cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) {
        cudaGetLastError();
        cs = cudaStreamCaptureStatusNone;
    }
    if (cs == cudaStreamCaptureStatusNone) g_launches.fetch_add(1, std::memory_order_relaxed);
}

void note_graph_launch(std::size_t kernels) { g_launches.fetch_add(kernels, std::memory_order_relaxed); }

std::size_t graph_kernel_nodes(cudaGraph_t g) {
    std::size_t n = 0;
    if (cudaGraphGetNodes(g, nullptr, &n) != cudaSuccess || n == 0) return 0;
    std::vector<cudaGraphNode_t> nodes(n);
    if (cudaGraphGetNodes(g, nodes.data(), &n) != cudaSuccess) return 0;
    std::size_t k = 0;
    for (auto nd : nodes) {
        cudaGraphNodeType t;
        if (cudaGraphNodeGetType(nd, &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++k;
    }
    return k;
}

unsigned long long launch_count() { return g_launches.load(std::memory_order_relaxed); }

cudaError_t zero(const ZeroRanges& z, cudaStream_t st, bool by_kernel) {
    if (!by_kernel) {
        for (int r = 0; r < z.n; ++r) {
            if (!z.words[r]) continue;
            const cudaError_t e = cudaMemsetAsync(z.p[r], 0, static_cast<size_t>(z.words[r]) * 4, st);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    }
    unsigned most = 1;
    for (int r = 0; r < z.n; ++r) most = z.words[r] > most ? z.words[r] : most;
    const unsigned blocks = (most + 255) / 256 < 256u ? (most + 255) / 256 : 256u;
    note_launch(st);
    k_zero<<<blocks, 256, 0, st>>>(z);
    return cudaGetLastError();
}

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

// Shared-memory lookup bandwidth: the access pattern of the bilateral's range table
// (lane l reads word k*32 + l of a 32-way replicated table: one LDS.32 per lane, every
// lane in its own bank). 16 independent loads per iteration off one base register, each
// consumed by one FADD, so the LDS pipe — not issue — is the limiter.
__global__ void __launch_bounds__(512) k_smem_peak(float* out, int iters) {
    __shared__ float tbl[256 * 32];
    for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) tbl[i] = 1e-6f * (i & 255);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    float acc[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = 0.f;
    int base = ((threadIdx.x >> 5) * 7) & 15;
    for (int i = 0; i < iters; ++i) {
        const float* t = tbl + base * 32 * 16 + lane;
#pragma unroll
        for (int k = 0; k < 16; ++k) acc[k] += t[k * 32];
        base = (base + 5) & 15;
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += acc[k];
    if (s == 12345.678f) out[0] = s;
}

// Same, but the bilateral's exact pattern: each lane gathers a data-dependent entry k of a
// 32-way replicated 512-entry table (word k*32 + lane: own bank, non-contiguous), with the
// address formed by one add from the previous value (16 independent chains per thread).
__global__ void __launch_bounds__(512) k_smem_gather(unsigned* out, int iters) {
    extern __shared__ unsigned gt[];  // [512][32]
    for (int i = threadIdx.x; i < 512 * 32; i += blockDim.x) {
        const int k = i >> 5;
        gt[i] = static_cast<unsigned>(((k * 37 + 11) & 511) * 128);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const unsigned base = static_cast<unsigned>(__cvta_generic_to_shared(gt)) + lane * 4u;
    unsigned v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = ((threadIdx.x * 7 + k * 29) & 511) * 128u;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            unsigned r;
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(base + v[k]));
            v[k] = r;
        }
    }
    unsigned s = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) s ^= v[k];
    if (s == 0x12345u) out[0] = s;
}
}  // namespace

cudaError_t smem_gather_peak(double* bytes_per_s) {
    const int blocks = sm_count() * 2, threads = 512, iters = 1024;
    const size_t smem = 512 * 32 * 4;
    unsigned* dummy = nullptr;
    cudaError_t e = cudaMalloc(&dummy, sizeof(unsigned));
    if (e != cudaSuccess) return e;
    cudaFuncSetAttribute(k_smem_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_smem_gather<<<blocks, threads, smem>>>(dummy, iters);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(a);
        k_smem_gather<<<blocks, threads, smem>>>(dummy, iters);
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
    *bytes_per_s = 4.0 * 16.0 * iters * static_cast<double>(blocks) * threads / (best * 1e-3);
    return e;
}

cudaError_t smem_peak(double* bytes_per_s) {
    const int blocks = sm_count() * 4, threads = 512, iters = 2048;
    float* dummy = nullptr;
    cudaError_t e = cudaMalloc(&dummy, sizeof(float));
    if (e != cudaSuccess) return e;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_smem_peak<<<blocks, threads>>>(dummy, iters);  // warm-up
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(a);
        k_smem_peak<<<blocks, threads>>>(dummy, iters);
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
    const double bytes = 4.0 * 16.0 * iters * static_cast<double>(blocks) * threads;
    *bytes_per_s = bytes / (best * 1e-3);
    return e;
}

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
