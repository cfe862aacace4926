// Interleaved RGB <-> planar on the device. The PPM payload is
// interleaved (reference pnm.cpp:115-120, 131-136) while the pipeline is planar
// (image.hpp:12-17); converting on the GPU lets decoded frames go to the device as raw
// payload bytes and come back ready to write, with no host (de)interleave pass.
// Both kernels are HBM-bound (3 bytes read + 3 written per pixel). Rows of a 16-pixel
// multiple start 16-byte aligned in both layouts, so a thread moves 16 pixels as three
// 16-byte words in and one 16-byte word per plane out (byte shuffles in registers); other
// widths take a per-pixel path.
#include "p3s_cu.h"

namespace p3s {
namespace cu {
namespace {

__device__ __forceinline__ uint8_t byte_of(const uint4 (&v)[3], int i) {
    const uint32_t w[12] = {v[0].x, v[0].y, v[0].z, v[0].w, v[1].x, v[1].y,
                            v[1].z, v[1].w, v[2].x, v[2].y, v[2].z, v[2].w};
    return static_cast<uint8_t>(w[i >> 2] >> (8 * (i & 3)));
}

// thread = 16 pixels of one row (vector path: w % 16 == 0, aligned buffers)
__global__ void k_deinterleave16(const uint8_t* __restrict__ src, int w, int h,
                                 uint8_t* __restrict__ r, uint8_t* __restrict__ g,
                                 uint8_t* __restrict__ b, int pitch) {
    const int chunks = w >> 4;
    const long long item = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (item >= static_cast<long long>(chunks) * h) return;
    const int y = static_cast<int>(item / chunks), c = static_cast<int>(item % chunks);
    const uint4* s = reinterpret_cast<const uint4*>(src + (static_cast<size_t>(y) * w + 16 * c) * 3);
    uint4 v[3] = {__ldcs(s), __ldcs(s + 1), __ldcs(s + 2)};
    uint32_t o[3][4];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t word = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) word |= static_cast<uint32_t>(byte_of(v, 3 * (4 * q + k) + ch)) << (8 * k);
            o[ch][q] = word;
        }
    const size_t off = static_cast<size_t>(y) * pitch + 16 * c;
    *reinterpret_cast<uint4*>(r + off) = make_uint4(o[0][0], o[0][1], o[0][2], o[0][3]);
    *reinterpret_cast<uint4*>(g + off) = make_uint4(o[1][0], o[1][1], o[1][2], o[1][3]);
    *reinterpret_cast<uint4*>(b + off) = make_uint4(o[2][0], o[2][1], o[2][2], o[2][3]);
}

__global__ void k_interleave16(const uint8_t* __restrict__ r, const uint8_t* __restrict__ g,
                               const uint8_t* __restrict__ b, int pitch, int w, int h,
                               uint8_t* __restrict__ dst) {
    const int chunks = w >> 4;
    const long long item = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (item >= static_cast<long long>(chunks) * h) return;
    const int y = static_cast<int>(item / chunks), c = static_cast<int>(item % chunks);
    const size_t off = static_cast<size_t>(y) * pitch + 16 * c;
    const uint4 pr = __ldg(reinterpret_cast<const uint4*>(r + off));
    const uint4 pg = __ldg(reinterpret_cast<const uint4*>(g + off));
    const uint4 pb = __ldg(reinterpret_cast<const uint4*>(b + off));
    const uint32_t cr[4] = {pr.x, pr.y, pr.z, pr.w}, cg[4] = {pg.x, pg.y, pg.z, pg.w},
                   cb[4] = {pb.x, pb.y, pb.z, pb.w};
    uint32_t o[12];
#pragma unroll
    for (int i = 0; i < 12; ++i) {
        uint32_t word = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int byte = 4 * i + k, px = byte / 3, ch = byte % 3;
            const uint32_t* pl = ch == 0 ? cr : (ch == 1 ? cg : cb);
            word |= ((pl[px >> 2] >> (8 * (px & 3))) & 0xFFu) << (8 * k);
        }
        o[i] = word;
    }
    uint4* d = reinterpret_cast<uint4*>(dst + (static_cast<size_t>(y) * w + 16 * c) * 3);
    __stcs(d, make_uint4(o[0], o[1], o[2], o[3]));
    __stcs(d + 1, make_uint4(o[4], o[5], o[6], o[7]));
    __stcs(d + 2, make_uint4(o[8], o[9], o[10], o[11]));
}

__global__ void k_deinterleave1(const uint8_t* __restrict__ src, int w, int h,
                                uint8_t* __restrict__ r, uint8_t* __restrict__ g,
                                uint8_t* __restrict__ b, int pitch) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<long long>(w) * h) return;
    const int y = static_cast<int>(i / w), x = static_cast<int>(i % w);
    const size_t off = static_cast<size_t>(y) * pitch + x;
    r[off] = src[3 * i];
    g[off] = src[3 * i + 1];
    b[off] = src[3 * i + 2];
}

__global__ void k_interleave1(const uint8_t* __restrict__ r, const uint8_t* __restrict__ g,
                              const uint8_t* __restrict__ b, int pitch, int w, int h,
                              uint8_t* __restrict__ dst) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<long long>(w) * h) return;
    const int y = static_cast<int>(i / w), x = static_cast<int>(i % w);
    const size_t off = static_cast<size_t>(y) * pitch + x;
    dst[3 * i] = r[off];
    dst[3 * i + 1] = g[off];
    dst[3 * i + 2] = b[off];
}

bool vec_ok(const void* a, const void* b, const void* c, const void* d, int w, int pitch) {
    const uintptr_t m = reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) |
                        reinterpret_cast<uintptr_t>(c) | reinterpret_cast<uintptr_t>(d) |
                        static_cast<uintptr_t>(pitch);
    return (w % 16) == 0 && (m & 15) == 0;
}

}  // namespace

cudaError_t deinterleave(const uint8_t* src, int w, int h, uint8_t* r, uint8_t* g, uint8_t* b,
                         int pitch, cudaStream_t st) {
    if (vec_ok(src, r, g, b, w, pitch)) {
        const long long items = static_cast<long long>(w / 16) * h;
        note_launch(st);
        k_deinterleave16<<<static_cast<unsigned>((items + 255) / 256), 256, 0, st>>>(src, w, h, r, g, b, pitch);
    } else {
        const long long items = static_cast<long long>(w) * h;
        note_launch(st);
        k_deinterleave1<<<static_cast<unsigned>((items + 255) / 256), 256, 0, st>>>(src, w, h, r, g, b, pitch);
    }
    return cudaGetLastError();
}

cudaError_t interleave(const uint8_t* r, const uint8_t* g, const uint8_t* b, int pitch, int w,
                       int h, uint8_t* dst, cudaStream_t st) {
    if (vec_ok(dst, r, g, b, w, pitch)) {
        const long long items = static_cast<long long>(w / 16) * h;
        note_launch(st);
        k_interleave16<<<static_cast<unsigned>((items + 255) / 256), 256, 0, st>>>(r, g, b, pitch, w, h, dst);
    } else {
        const long long items = static_cast<long long>(w) * h;
        note_launch(st);
        k_interleave1<<<static_cast<unsigned>((items + 255) / 256), 256, 0, st>>>(r, g, b, pitch, w, h, dst);
    }
    return cudaGetLastError();
}

namespace {
// One warp per (eye, row, group of 32 mask words): lane j tests word j; for every word with
// damage the warp copies its 32 bytes per plane (lane = pixel), one coalesced store each.
__global__ void __launch_bounds__(256) k_patch_host(PatchEye a, PatchEye b, int w, int h) {
    const int lane = threadIdx.x & 31;
    const int mwords = (w + 31) >> 5, groups = (mwords + 31) >> 5;
    const long long total = 2LL * h * groups;
    const long long nwarps = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
    for (long long it = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; it < total;
         it += nwarps) {
        const int e = static_cast<int>(it / (static_cast<long long>(h) * groups));
        const int rem = static_cast<int>(it - static_cast<long long>(e) * h * groups);
        const int y = rem / groups, g = rem - y * groups;
        const PatchEye& P = e ? b : a;
        const int j = g * 32 + lane;
        const uint32_t m = j < mwords ? __ldg(P.mask + static_cast<size_t>(y) * P.mpitch + j) : 0u;
        unsigned nz = __ballot_sync(0xFFFFFFFFu, m != 0u);
        while (nz) {
            const int k = __ffs(nz) - 1;
            nz &= nz - 1;
            const int x = (g * 32 + k) * 32 + lane;
            if (x < w) {
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    if (P.dev[c])
                        P.host[c][static_cast<size_t>(y) * P.hpitch + x] =
                            P.dev[c][static_cast<size_t>(y) * P.dpitch + x];
            }
        }
    }
}
}  // namespace

cudaError_t patch_host(PatchEye left, PatchEye right, Geom gm, cudaStream_t st) {
    const int mwords = (gm.w + 31) >> 5, groups = (mwords + 31) >> 5;
    const long long warps = 2LL * gm.h * groups;
    const int blocks = static_cast<int>(std::min<long long>((warps + 7) / 8, sm_count() * 8LL));
    note_launch(st);
    k_patch_host<<<blocks, 256, 0, st>>>(left, right, gm.w, gm.h);
    return cudaGetLastError();
}

}  // namespace cu
}  // namespace p3s
