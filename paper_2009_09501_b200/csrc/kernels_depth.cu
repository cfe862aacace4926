// Depth-map stage on sm_100a (reference proj/src/depth.cpp + image.cpp:13-21).
//
// K1 depth_front: one CTA per 128x16 pixel tile. R,G,B are read once with 8-byte vector
// loads (plus a 1-pixel clamped halo), luma is formed in shared memory and written out
// (it is also the bilateral guide), the 3x3 Sobel magnitude is evaluated from shared
// memory and reduced straight into per-block edge sums. The edge map itself never
// touches HBM. Algorithmic traffic: 3N read + N write.
//
// Integer arithmetic only in K1, so it is exact by construction. block_values/upsample
// reproduce the reference's double expressions with explicit round-to-nearest intrinsics
// (no FMA contraction regardless of compiler flags).
#include <cstdlib>

#include "p3s_cu.h"

namespace p3s {
namespace cu {
namespace {

constexpr int kTW = 128;  // tile width (pixels)
constexpr int kTH = 16;   // tile height
// smem row: left halo at kX0 - 1, pixel c at kX0 + c (8-byte aligned), right halo at kX0 + kTW
constexpr int kX0 = 8;
constexpr int kSW = kX0 + kTW + 8;
constexpr int kMaxBX = kTW / 4 + 2;  // local block columns a tile can touch (block >= 4)
constexpr int kMaxBY = kTH / 4 + 2;

__device__ __forceinline__ int clampi(int v, int hi) { return v < 0 ? 0 : (v > hi ? hi : v); }

// v / block for 0 <= v, v * block < 2^32, with magic = floor(2^32 / block) + 1 (host;
// magic = 0 when the frame is too large for that bound: plain division)
#define div_block(v, magic) \
    ((magic) ? static_cast<int>(__umulhi(static_cast<unsigned>(v), (magic))) : (v) / block)

__device__ __forceinline__ uint8_t luma_px(unsigned r, unsigned g, unsigned b) {
    return static_cast<uint8_t>((77u * r + 150u * g + 29u * b + 128u) >> 8);
}

// luma of 4 pixels (bytes of r4/g4/b4) -> 4 bytes. Two pixels per 32-bit word in 16-bit
// lanes: 77r + 150g + 29b + 128 <= 65408 never carries into the next lane.
__device__ __forceinline__ uint32_t luma4(uint32_t r4, uint32_t g4, uint32_t b4) {
    const uint32_t rl = __byte_perm(r4, 0, 0x4240), rh = __byte_perm(r4, 0, 0x4341);
    const uint32_t gl = __byte_perm(g4, 0, 0x4240), gh = __byte_perm(g4, 0, 0x4341);
    const uint32_t bl = __byte_perm(b4, 0, 0x4240), bh = __byte_perm(b4, 0, 0x4341);
    const uint32_t sl = 77u * rl + 150u * gl + 29u * bl + 0x00800080u;  // pixels 0, 2
    const uint32_t sh = 77u * rh + 150u * gh + 29u * bh + 0x00800080u;  // pixels 1, 3
    // luma bytes sit at bytes 1 and 3 of each word
    return __byte_perm(sl, sh, 0x7351);
}

__global__ void __launch_bounds__(256) k_depth_front(const uint8_t* __restrict__ R,
                                                     const uint8_t* __restrict__ G,
                                                     const uint8_t* __restrict__ B, int pitch,
                                                     int w, int h, uint8_t* __restrict__ luma,
                                                     unsigned long long* __restrict__ sums,
                                                     int block, int bx_total, int tile_row0,
                                                     unsigned magic) {
    __shared__ __align__(16) uint8_t s_y[kTH + 2][kSW];
    __shared__ unsigned s_sum[kMaxBY][kMaxBX];

    const int x0 = blockIdx.x * kTW;
    const int y0 = (tile_row0 + blockIdx.y) * kTH;
    const int tid = threadIdx.x;
    for (int i = tid; i < kMaxBY * kMaxBX; i += blockDim.x) (&s_sum[0][0])[i] = 0u;

    // ---- load R,G,B (tile + clamped 1-px halo) and form luma in smem ----
    const bool interior_x = x0 >= 1 && x0 + kTW + 1 <= w && (pitch % 8) == 0;
    if (interior_x) {
        // 18 rows x 16 chunks of 8 pixels, 8-byte vector loads
        for (int item = tid; item < (kTH + 2) * 16; item += blockDim.x) {
            const int sr = item >> 4, c8 = item & 15;
            const int gy = clampi(y0 - 1 + sr, h - 1);
            const size_t off = static_cast<size_t>(gy) * pitch + x0 + 8 * c8;
            const uint2 vr = __ldg(reinterpret_cast<const uint2*>(R + off));
            const uint2 vg = __ldg(reinterpret_cast<const uint2*>(G + off));
            const uint2 vb = __ldg(reinterpret_cast<const uint2*>(B + off));
            const uint2 yv = make_uint2(luma4(vr.x, vg.x, vb.x), luma4(vr.y, vg.y, vb.y));
            *reinterpret_cast<uint2*>(&s_y[sr][kX0 + 8 * c8]) = yv;
            const int oy = y0 - 1 + sr;
            if (sr >= 1 && sr <= kTH && oy < h)
                *reinterpret_cast<uint2*>(luma + static_cast<size_t>(oy) * pitch + x0 + 8 * c8) = yv;
        }
        for (int item = tid; item < (kTH + 2) * 2; item += blockDim.x) {
            const int sr = item >> 1, side = item & 1;
            const int gy = clampi(y0 - 1 + sr, h - 1);
            const int gx = side ? x0 + kTW : x0 - 1;
            const size_t off = static_cast<size_t>(gy) * pitch + gx;
            s_y[sr][side ? kX0 + kTW : kX0 - 1] = luma_px(R[off], G[off], B[off]);
        }
        __syncthreads();
    } else {
        for (int item = tid; item < (kTH + 2) * (kTW + 2); item += blockDim.x) {
            const int sr = item / (kTW + 2), sc = item % (kTW + 2);
            const int gy = clampi(y0 - 1 + sr, h - 1);
            const int gx = clampi(x0 - 1 + sc, w - 1);
            const size_t off = static_cast<size_t>(gy) * pitch + gx;
            s_y[sr][kX0 - 1 + sc] = luma_px(R[off], G[off], B[off]);
        }
        __syncthreads();
        for (int item = tid; item < kTH * kTW; item += blockDim.x) {
            const int r = item / kTW, c = item % kTW;
            const int oy = y0 + r, ox = x0 + c;
            if (oy < h && ox < w) luma[static_cast<size_t>(oy) * pitch + ox] = s_y[1 + r][kX0 + c];
        }
    }

    // ---- Sobel magnitude (depth.cpp:21-41) and block sums (depth.cpp:64-67) ----
    // thread -> row ty, 8 consecutive pixels starting at column 8*c8. Per window column j
    // (pixels x-1 .. x+8) the vertical [1 2 1] sum cs and the difference d = bottom - top are
    // formed once; then gx = cs[j+1] - cs[j-1] and gy = d[j-1] + 2 d[j] + d[j+1] (the
    // reference's expressions regrouped in exact integer arithmetic). The block column of a
    // pixel is tracked incrementally (one division per thread, not per pixel).
    {
        const int ty = tid >> 4, c8 = tid & 15;
        const int oy = y0 + ty;
        if (oy < h) {
            int cs[10], dd[10];
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                const uint8_t* row = &s_y[ty + r][kX0 + 8 * c8];
                const uint2 mid = *reinterpret_cast<const uint2*>(row);
                int p[10];
                p[0] = row[-1];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    p[1 + k] = (mid.x >> (8 * k)) & 0xFF;
                    p[5 + k] = (mid.y >> (8 * k)) & 0xFF;
                }
                p[9] = row[8];
#pragma unroll
                for (int j = 0; j < 10; ++j) {
                    if (r == 0) {
                        cs[j] = p[j];
                        dd[j] = -p[j];
                    } else if (r == 1) {
                        cs[j] += 2 * p[j];
                    } else {
                        cs[j] += p[j];
                        dd[j] += p[j];
                    }
                }
            }
            const int bx0 = div_block(x0, magic), by0 = div_block(y0, magic);
            const int lby = div_block(oy, magic) - by0;
            const int ox0 = x0 + 8 * c8;
            int lbx = div_block(ox0, magic) - bx0;
            int next = (bx0 + lbx + 1) * block;  // first column of the next block
            unsigned run = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int ox = ox0 + k;
                if (ox < w) {
                    const int gx = cs[k + 2] - cs[k];
                    const int gy = dd[k] + 2 * dd[k + 1] + dd[k + 2];
                    const unsigned mag = min((static_cast<unsigned>(abs(gx)) + static_cast<unsigned>(abs(gy))) >> 2, 255u);
                    if (ox == next) {
                        if (run) atomicAdd(&s_sum[lby][lbx], run);
                        ++lbx;
                        next += block;
                        run = 0;
                    }
                    run += mag;
                }
            }
            if (run) atomicAdd(&s_sum[lby][lbx], run);
        }
    }
    __syncthreads();
    {
        const int bx0 = div_block(x0, magic), by0 = div_block(y0, magic);
        const int nbx = div_block(min(x0 + kTW, w) - 1, magic) - bx0 + 1;
        const int nby = div_block(min(y0 + kTH, h) - 1, magic) - by0 + 1;
        for (int i = tid; i < nbx * nby; i += blockDim.x) {
            const int ly = i / nbx, lx = i % nbx;
            const unsigned v = s_sum[ly][lx];
            if (v)
                atomicAdd(&sums[static_cast<size_t>(by0 + ly) * bx_total + bx0 + lx],
                          static_cast<unsigned long long>(v));
        }
    }
}

// depth.cpp:55-71: value = (alpha*255.0) * (centre/row_denom) + beta * (sum / count).
__global__ void k_block_values(const unsigned long long* __restrict__ sums, int w, int h,
                               int block, int bx, int by, double alpha255, double beta,
                               double row_denom, double* __restrict__ values, int i0, int i1) {
    const int i = i0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= i1) return;
    const int iy = i / bx, ix = i % bx;
    const int y0 = iy * block, y1 = min(y0 + block, h);
    const int xa = ix * block, xb = min(xa + block, w);
    const double centre = __dadd_rn(static_cast<double>(y0),
                                    __ddiv_rn(static_cast<double>(y1 - 1 - y0), 2.0));
    const double ramp = __dmul_rn(alpha255, __ddiv_rn(centre, row_denom));
    const double mean = __ddiv_rn(static_cast<double>(sums[i]),
                                  static_cast<double>((y1 - y0) * (xb - xa)));
    values[i] = __dadd_rn(ramp, __dmul_rn(beta, mean));
}

__device__ __forceinline__ uint8_t round_half_up_u8(double v) {
    const double r = floor(__dadd_rn(v, 0.5));
    if (r <= 0.0) return 0;
    if (r >= 255.0) return 255;
    return static_cast<uint8_t>(static_cast<int>(r));
}

__device__ __forceinline__ double lerp_ref(double a, double b, double f) {
    // a * (1.0 - f) + b * f, each operation separately rounded (depth.cpp:115-117)
    return __dadd_rn(__dmul_rn(a, __dsub_rn(1.0, f)), __dmul_rn(b, f));
}

// depth.cpp:104-120. A CTA covers 1024 columns x 16 rows; a thread owns 4 adjacent columns
// (one 4-byte store per row). Within a band of rows sharing the same (iy, iy1) pair the
// horizontal lerps top(x) / bottom(x) are identical, so they are computed once per band and
// only the vertical lerp + rounding runs per pixel. Every double operation is the
// reference's, separately rounded, so the bytes are unchanged.
constexpr int kUpCols = 4, kUpThreads = 256, kUpRows = 16;

__global__ void __launch_bounds__(kUpThreads) k_upsample(const double* __restrict__ values, int bx,
                                                         const int* __restrict__ ci0,
                                                         const int* __restrict__ ci1,
                                                         const double* __restrict__ cf,
                                                         const int* __restrict__ ri0,
                                                         const int* __restrict__ ri1,
                                                         const double* __restrict__ rf, int w,
                                                         int h, int pitch,
                                                         uint8_t* __restrict__ depth, int ya, int yb) {
    const int x0 = (blockIdx.x * kUpThreads + threadIdx.x) * kUpCols;
    const int y0 = ya + blockIdx.y * kUpRows;
    if (x0 >= w) return;
    int a[kUpCols], b[kUpCols];
    double fx[kUpCols];
#pragma unroll
    for (int k = 0; k < kUpCols; ++k) {
        const int x = min(x0 + k, w - 1);
        a[k] = __ldg(ci0 + x);
        b[k] = __ldg(ci1 + x);
        fx[k] = __ldg(cf + x);
    }
    int cur0 = -1, cur1 = -1;
    double top[kUpCols], bot[kUpCols];
    const int y1 = min(y0 + kUpRows, yb);
    for (int y = y0; y < y1; ++y) {
        const int i0 = __ldg(ri0 + y), i1 = __ldg(ri1 + y);
        if (i0 != cur0 || i1 != cur1) {
            const double* vt = values + static_cast<size_t>(i0) * bx;
            const double* vb = values + static_cast<size_t>(i1) * bx;
#pragma unroll
            for (int k = 0; k < kUpCols; ++k) {
                top[k] = lerp_ref(__ldg(vt + a[k]), __ldg(vt + b[k]), fx[k]);
                bot[k] = lerp_ref(__ldg(vb + a[k]), __ldg(vb + b[k]), fx[k]);
            }
            cur0 = i0;
            cur1 = i1;
        }
        const double fy = __ldg(rf + y);
        uint32_t packed = 0;
#pragma unroll
        for (int k = 0; k < kUpCols; ++k)
            packed |= static_cast<uint32_t>(round_half_up_u8(lerp_ref(top[k], bot[k], fy))) << (8 * k);
        uint8_t* dst = depth + static_cast<size_t>(y) * pitch + x0;
        if (x0 + kUpCols <= pitch) {  // pitch % 16 == 0: 4-byte aligned, padding is scratch
            *reinterpret_cast<uint32_t*>(dst) = packed;
        } else {
            for (int k = 0; k < kUpCols && x0 + k < w; ++k) dst[k] = static_cast<uint8_t>(packed >> (8 * k));
        }
    }
}

// ---- fused depth front for 16-pixel blocks (the default depth_block) ----------------------
// K1 with the block values folded in: a CTA of 256 threads covers 1024 columns x one block
// row (16 image rows), i.e. 64 blocks of 16 x 16; four adjacent lanes own one block (four
// output rows each), reduce its Sobel sum with two shuffles and the first of them writes the
// block VALUE (depth.cpp:55-71) itself — no sums buffer, no atomics, no block_values launch.
//  phase 1  R, G, B rows y0-1 .. y0+16 (edge-clamped) with 16-byte loads (every thread issues
//           all of its rows' loads before converting), luma for 16 pixels at a time in 16-bit
//           lanes (luma4), into a shared 18-row luma tile (+ the two halo columns) and, for the
//           16 block rows, to the luma plane (16-byte stores);
//  phase 2  the 3x3 Sobel magnitude of 16 pixels per row in 16-bit lanes (2 pixels per 32-bit
//           word). With the window rows t (y-1), m (y), b (y+1):
//               gx + gy = 2 (A+ - A-),  A+ = m(x+1) + b(x+1) + b(x),  A- = t(x-1) + m(x-1) + t(x)
//               gx - gy = 2 (B+ - B-),  B+ = t(x+1) + m(x+1) + t(x),  B- = b(x-1) + m(x-1) + b(x)
//           and |gx| + |gy| = max(|gx + gy|, |gx - gy|), so the reference's
//           min(255, (|gx| + |gy|) / 4) = min(510, max(|A+ - A-|, |B+ - B-|)) >> 1 exactly
//           (integers, depth.cpp:34-37). |a - b| per lane = max - min (VIMNMX.U16x2).
// Requires block == 16, w % 16 == 0 and a 16-byte aligned pitch (depth_fused_ok).
constexpr int kFT = 256;           // threads per CTA
constexpr int kFW = 1024;          // columns per CTA (64 blocks)
constexpr int kFL = 16;            // smem column of image column x0 (halo at kFL - 1)
constexpr int kFS = kFL + kFW + 16;  // smem row stride

__device__ __forceinline__ uint32_t vmax2(uint32_t a, uint32_t b) { return __vmaxu2(a, b); }
__device__ __forceinline__ uint32_t vmin2(uint32_t a, uint32_t b) { return __vminu2(a, b); }
__device__ __forceinline__ uint32_t absdiff2(uint32_t a, uint32_t b) { return vmax2(a, b) - vmin2(a, b); }

// One smem luma row as 16-bit pairs: P[j] = (c2j, c2j+1), S[j] = (c2j-1, c2j) for j = 0..8
// (S[8] = (c15, c16)); row[-1] / row[16] are the neighbouring columns.
struct PairRow {
    uint32_t P[8], S[9];
};
__device__ __forceinline__ void load_pair_row(const uint8_t* row, PairRow& pr) {
    const uint4 v = *reinterpret_cast<const uint4*>(row);
    const uint32_t hl = static_cast<uint32_t>(row[-1]) << 16, hr = row[16];
    const uint32_t L[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 8; ++j) pr.P[j] = __byte_perm(L[j >> 1], 0u, (j & 1) ? 0x4342 : 0x4140);
    pr.S[0] = __byte_perm(hl, pr.P[0], 0x5432);
#pragma unroll
    for (int j = 1; j < 8; ++j) pr.S[j] = __byte_perm(pr.P[j - 1], pr.P[j], 0x5432);
    pr.S[8] = __byte_perm(pr.P[7], hr, 0x5432);
}

// R,G,B of 4 interleaved pixels (3 words r0 g0 b0 r1 | g1 b1 r2 g2 | b2 r3 g3 b3) as byte
// planes (4 pixels per word).
__device__ __forceinline__ void split_rgb4(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t& r,
                                           uint32_t& g, uint32_t& b) {
    r = __byte_perm(__byte_perm(w0, w1, 0x0630), w2, 0x5210);
    g = __byte_perm(__byte_perm(w0, w1, 0x0741), w2, 0x6210);
    b = __byte_perm(__byte_perm(w0, w1, 0x0052), w2, 0x7410);
}

// ILV: R is one RGB-interleaved image (row stride src_pitch; the PPM payload as uploaded),
// G and B are unused.
template <bool ILV>
__global__ void __launch_bounds__(kFT) k_depth_fused(const uint8_t* __restrict__ R,
                                                     const uint8_t* __restrict__ G,
                                                     const uint8_t* __restrict__ B, int pitch,
                                                     int w, int h, uint8_t* __restrict__ luma,
                                                     double* __restrict__ values, int bx_total,
                                                     double alpha255, double beta,
                                                     double row_denom, int tile_row0, int src_pitch) {
    __shared__ __align__(16) uint8_t s_l[kTH + 2][kFS];
    const int x0 = blockIdx.x * kFW;
    const int y0 = (tile_row0 + blockIdx.y) * kTH;
    const int t = threadIdx.x;
    const int ncols = min(kFW, w - x0);

    // ---- phase 1: luma tile (rows y0-1 .. y0+16, clamped); thread = chunk t & 63, rows
    // (t >> 6) + 4k ----
    {
        const int c0 = 16 * (t & 63), rq = t >> 6;
        if (c0 < ncols) {
            const size_t col = static_cast<size_t>(x0 + c0);
            uint4 vr[5], vg[5], vb[5];
#pragma unroll
            for (int k = 0; k < 5; ++k) {
                const int r = rq + 4 * k;
                if (r < kTH + 2) {
                    const int gy = clampi(y0 - 1 + r, h - 1);
                    if (ILV) {  // 48 interleaved bytes, planes recovered below
                        const uint4* src = reinterpret_cast<const uint4*>(R + static_cast<size_t>(gy) * src_pitch + 3 * col);
                        vr[k] = __ldg(src);
                        vg[k] = __ldg(src + 1);
                        vb[k] = __ldg(src + 2);
                    } else {
                        const size_t off = static_cast<size_t>(gy) * pitch + col;
                        vr[k] = __ldg(reinterpret_cast<const uint4*>(R + off));
                        vg[k] = __ldg(reinterpret_cast<const uint4*>(G + off));
                        vb[k] = __ldg(reinterpret_cast<const uint4*>(B + off));
                    }
                }
            }
            if (ILV) {
#pragma unroll
                for (int k = 0; k < 5; ++k) {
                    const uint32_t W[12] = {vr[k].x, vr[k].y, vr[k].z, vr[k].w, vg[k].x, vg[k].y,
                                            vg[k].z, vg[k].w, vb[k].x, vb[k].y, vb[k].z, vb[k].w};
                    uint32_t pr[4], pg[4], pb[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) split_rgb4(W[3 * i], W[3 * i + 1], W[3 * i + 2], pr[i], pg[i], pb[i]);
                    vr[k] = make_uint4(pr[0], pr[1], pr[2], pr[3]);
                    vg[k] = make_uint4(pg[0], pg[1], pg[2], pg[3]);
                    vb[k] = make_uint4(pb[0], pb[1], pb[2], pb[3]);
                }
            }
#pragma unroll
            for (int k = 0; k < 5; ++k) {
                const int r = rq + 4 * k;
                if (r < kTH + 2) {
                    const uint4 yv = make_uint4(luma4(vr[k].x, vg[k].x, vb[k].x), luma4(vr[k].y, vg[k].y, vb[k].y),
                                                luma4(vr[k].z, vg[k].z, vb[k].z), luma4(vr[k].w, vg[k].w, vb[k].w));
                    *reinterpret_cast<uint4*>(&s_l[r][kFL + c0]) = yv;
                    const int oy = y0 - 1 + r;
                    if (r >= 1 && r <= kTH && oy < h)
                        *reinterpret_cast<uint4*>(luma + static_cast<size_t>(oy) * pitch + col) = yv;
                }
            }
        }
        // halo columns x0-1 and x0+ncols (edge-clamped), 18 rows each
        if (t >= kFT - 2 * (kTH + 2)) {
            const int i = t - (kFT - 2 * (kTH + 2));
            const int r = i >> 1, side = i & 1;
            const int gy = clampi(y0 - 1 + r, h - 1);
            const int gx = side ? min(x0 + ncols, w - 1) : max(x0 - 1, 0);
            if (ILV) {
                const uint8_t* p = R + static_cast<size_t>(gy) * src_pitch + 3 * static_cast<size_t>(gx);
                s_l[r][side ? kFL + ncols : kFL - 1] = luma_px(p[0], p[1], p[2]);
            } else {
                const size_t off = static_cast<size_t>(gy) * pitch + gx;
                s_l[r][side ? kFL + ncols : kFL - 1] = luma_px(R[off], G[off], B[off]);
            }
        }
    }
    __syncthreads();

    // ---- phase 2: lanes 4b..4b+3 own block b; lane quarter q sums rows 4q..4q+3 ----
    const int blk = t >> 2, q = t & 3;
    const int c0 = 16 * blk;
    const int rows = min(kTH, h - y0);
    uint32_t acc = 0;
    if (c0 < ncols) {
        const int i0 = 4 * q, i1 = min(4 * q + 4, rows);
        PairRow top, mid, bot;
        load_pair_row(&s_l[i0][kFL + c0], top);
        load_pair_row(&s_l[i0 + 1][kFL + c0], mid);
        for (int i = i0; i < i1; ++i) {
            load_pair_row(&s_l[i + 2][kFL + c0], bot);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t ap = mid.S[j + 1] + bot.S[j + 1] + bot.P[j];
                const uint32_t an = top.S[j] + mid.S[j] + top.P[j];
                const uint32_t bp = top.S[j + 1] + mid.S[j + 1] + top.P[j];
                const uint32_t bn = bot.S[j] + mid.S[j] + bot.P[j];
                const uint32_t m = vmin2(vmax2(absdiff2(ap, an), absdiff2(bp, bn)), 0x01FE01FEu);
                acc += (m >> 1) & 0x00FF00FFu;  // <= 4 rows x 8 words x 255 per lane
            }
            top = mid;
            mid = bot;
        }
    }
    unsigned long long sum = (acc & 0xFFFFu) + (acc >> 16);
    sum += __shfl_xor_sync(0xFFFFFFFFu, sum, 1);
    sum += __shfl_xor_sync(0xFFFFFFFFu, sum, 2);
    if (q == 0 && c0 < ncols) {
        // depth.cpp:55-71 (same expression order as k_block_values)
        const int ya = y0, yb = y0 + rows;
        const double centre = __dadd_rn(static_cast<double>(ya), __ddiv_rn(static_cast<double>(yb - 1 - ya), 2.0));
        const double ramp = __dmul_rn(alpha255, __ddiv_rn(centre, row_denom));
        const double mean = __ddiv_rn(static_cast<double>(sum), static_cast<double>(rows * 16));
        values[static_cast<size_t>(tile_row0 + blockIdx.y) * bx_total + (x0 + c0) / 16] =
            __dadd_rn(ramp, __dmul_rn(beta, mean));
    }
}

// ---- upsample: a CTA = 1024 columns x 16 rows, a thread = 4 columns x 16 rows ------------
// Same arithmetic as k_upsample (depth.cpp:104-120, each double operation separately
// rounded); the CTA's 16 row-table entries are staged in shared memory first (no global
// load latency inside the row loop), and floor(v + 0.5) is taken on the FP64 pipe:
// t = v + 0.5 (the reference's add), then t + 2^52 rounded toward zero holds floor(t) in its
// low word (t in [0, 2^31)); v >= 0 since every block value and lerp weight is >= 0.
constexpr int kU2Cols = 4, kU2Rows = 16, kU2Threads = 256;

__global__ void __launch_bounds__(kU2Threads) k_upsample_rows(const double* __restrict__ values, int bx,
                                                              const int* __restrict__ ci0,
                                                              const int* __restrict__ ci1,
                                                              const double* __restrict__ cf,
                                                              const int* __restrict__ ri0,
                                                              const int* __restrict__ ri1,
                                                              const double* __restrict__ rf, int w,
                                                              int pitch, uint8_t* __restrict__ depth,
                                                              int ya, int yb) {
    __shared__ int s_i0[kU2Rows], s_i1[kU2Rows];
    __shared__ double s_f[kU2Rows];
    const int y0 = ya + blockIdx.y * kU2Rows;
    const int y1 = min(y0 + kU2Rows, yb);
    if (threadIdx.x < y1 - y0) {
        s_i0[threadIdx.x] = __ldg(ri0 + y0 + threadIdx.x);
        s_i1[threadIdx.x] = __ldg(ri1 + y0 + threadIdx.x);
        s_f[threadIdx.x] = __ldg(rf + y0 + threadIdx.x);
    }
    const int x0 = (blockIdx.x * kU2Threads + threadIdx.x) * kU2Cols;
    int a[kU2Cols], b[kU2Cols];
    double fx[kU2Cols];
#pragma unroll
    for (int k = 0; k < kU2Cols; ++k) {
        const int x = min(x0 + k, w - 1);
        a[k] = __ldg(ci0 + x);
        b[k] = __ldg(ci1 + x);
        fx[k] = __ldg(cf + x);
    }
    __syncthreads();
    if (x0 >= w) return;
    int cur0 = -1, cur1 = -1;
    double top[kU2Cols], bot[kU2Cols];
    const bool full = x0 + kU2Cols <= pitch;  // pitch % 16 == 0: 4-byte aligned, padding is scratch
    for (int y = y0; y < y1; ++y) {
        const int i0 = s_i0[y - y0], i1 = s_i1[y - y0];
        if (i0 != cur0 || i1 != cur1) {
            const double* vt = values + static_cast<size_t>(i0) * bx;
            const double* vb = values + static_cast<size_t>(i1) * bx;
#pragma unroll
            for (int k = 0; k < kU2Cols; ++k) {
                top[k] = lerp_ref(__ldg(vt + a[k]), __ldg(vt + b[k]), fx[k]);
                bot[k] = lerp_ref(__ldg(vb + a[k]), __ldg(vb + b[k]), fx[k]);
            }
            cur0 = i0;
            cur1 = i1;
        }
        const double fy = s_f[y - y0];
        const double omf = __dsub_rn(1.0, fy);
        uint32_t packed = 0;
#pragma unroll
        for (int k = 0; k < kU2Cols; ++k) {
            const double v = __dadd_rn(__dmul_rn(top[k], omf), __dmul_rn(bot[k], fy));
            const double f = __dadd_rz(__dadd_rn(v, 0.5), 4503599627370496.0);
            packed |= min(static_cast<uint32_t>(__double2loint(f)), 255u) << (8 * k);
        }
        uint8_t* dst = depth + static_cast<size_t>(y) * pitch + x0;
        if (full) {
            *reinterpret_cast<uint32_t*>(dst) = packed;
        } else {
            for (int k = 0; k < kU2Cols && x0 + k < w; ++k) dst[k] = static_cast<uint8_t>(packed >> (8 * k));
        }
    }
}

}  // namespace

cudaError_t depth_front(const uint8_t* r, const uint8_t* g, const uint8_t* b, Geom gm,
                        uint8_t* luma, unsigned long long* sums, int block, int bx,
                        cudaStream_t st, int tile_row0, int tile_row1) {
    const int rows = (gm.h + kTH - 1) / kTH;
    if (tile_row1 < 0 || tile_row1 > rows) tile_row1 = rows;
    if (tile_row1 <= tile_row0) return cudaSuccess;
    dim3 grid((gm.w + kTW - 1) / kTW, tile_row1 - tile_row0);
    const unsigned long long span = static_cast<unsigned long long>(std::max(gm.w, gm.h) + kTW);
    const unsigned magic = span * static_cast<unsigned>(block) < (1ull << 32)
                               ? static_cast<unsigned>((1ull << 32) / static_cast<unsigned>(block) + 1ull)
                               : 0u;
    note_launch(st);
    k_depth_front<<<grid, 256, 0, st>>>(r, g, b, gm.pitch, gm.w, gm.h, luma, sums, block, bx,
                                        tile_row0, magic);
    return cudaGetLastError();
}

cudaError_t block_values(const unsigned long long* sums, Geom gm, const DepthTables& t,
                         double* values, cudaStream_t st, int brow0, int brow1) {
    if (brow1 < 0 || brow1 > t.by) brow1 = t.by;
    const int i0 = brow0 * t.bx, i1 = brow1 * t.bx;
    if (i1 <= i0) return cudaSuccess;
    note_launch(st);
    k_block_values<<<(i1 - i0 + 255) / 256, 256, 0, st>>>(sums, gm.w, gm.h, t.block, t.bx, t.by,
                                                          t.alpha255, t.beta, t.row_denom, values,
                                                          i0, i1);
    return cudaGetLastError();
}

cudaError_t upsample(const double* values, Geom gm, const DepthTables& t, uint8_t* depth,
                     cudaStream_t st, int ya, int yb) {
    if (yb < 0 || yb > gm.h) yb = gm.h;
    if (yb <= ya) return cudaSuccess;
    if (gm.pitch % 16 == 0 && !std::getenv("P3S_UPSAMPLE4")) {
        dim3 grid((gm.w + kU2Threads * kU2Cols - 1) / (kU2Threads * kU2Cols),
                  (yb - ya + kU2Rows - 1) / kU2Rows);
        note_launch(st);
        k_upsample_rows<<<grid, kU2Threads, 0, st>>>(values, t.bx, t.col_i0, t.col_i1, t.col_f, t.row_i0,
                                                 t.row_i1, t.row_f, gm.w, gm.pitch, depth, ya, yb);
        return cudaGetLastError();
    }
    dim3 grid((gm.w + kUpThreads * kUpCols - 1) / (kUpThreads * kUpCols),
              (yb - ya + kUpRows - 1) / kUpRows);
    note_launch(st);
    k_upsample<<<grid, kUpThreads, 0, st>>>(values, t.bx, t.col_i0, t.col_i1, t.col_f, t.row_i0,
                                            t.row_i1, t.row_f, gm.w, gm.h, gm.pitch, depth, ya, yb);
    return cudaGetLastError();
}

int depth_tile_rows() { return kTH; }

bool depth_fused_ok(Geom gm, int block) {
    return block == kTH && gm.w % 16 == 0 && gm.pitch % 16 == 0 && gm.w >= 16;
}

cudaError_t depth_front_fused(const uint8_t* r, const uint8_t* g, const uint8_t* b, Geom gm,
                              uint8_t* luma, const DepthTables& t, double* values, cudaStream_t st,
                              int tile_row0, int tile_row1, int src_ipitch) {
    const int rows = (gm.h + kTH - 1) / kTH;
    if (tile_row1 < 0 || tile_row1 > rows) tile_row1 = rows;
    if (tile_row1 <= tile_row0) return cudaSuccess;
    dim3 grid((gm.w + kFW - 1) / kFW, tile_row1 - tile_row0);
    note_launch(st);
    if (src_ipitch > 0)
        k_depth_fused<true><<<grid, kFT, 0, st>>>(r, nullptr, nullptr, gm.pitch, gm.w, gm.h, luma, values,
                                                  t.bx, t.alpha255, t.beta, t.row_denom, tile_row0, src_ipitch);
    else
        k_depth_fused<false><<<grid, kFT, 0, st>>>(r, g, b, gm.pitch, gm.w, gm.h, luma, values, t.bx,
                                                   t.alpha255, t.beta, t.row_denom, tile_row0, 0);
    return cudaGetLastError();
}

}  // namespace cu
}  // namespace p3s
