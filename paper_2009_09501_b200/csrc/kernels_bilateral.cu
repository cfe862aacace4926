// K2: exact FP64 cross-bilateral filter on sm_100a (reference proj/src/bilateral.cpp:40-116).
//
// Bit-exactness contract (SURVEY.md §7 rule 3): for every output pixel the taps are
// accumulated in the reference's order — window rows dy ascending over the clipped
// window, in each row the centre tap, then dx = 1..r as a mirrored pair
// (ws += wl + wr; vs += wl*dL + wr*dR) or a single side at the image border — with every
// multiply and add separately rounded (__dmul_rn/__dadd_rn; no FMA). The spatial and
// range tables are computed on the host with the reference's libm exp (engine.cpp).
//
// Layout: a CTA is 8 warps; a warp owns 32 adjacent columns x P rows and each thread one
// column of P outputs (vertical register blocking). A (32+2r) x (8P+2r) tile of packed
// (depth<<8 | guide) u16 is staged in shared memory, so every loaded neighbour pair is
// reused by all P outputs of the thread (guide/depth loads amortised P-fold). The range
// table lives in shared memory replicated 16 ways ([d][lane & 15]) so the per-tap
// random-index LDS.64 is bank-conflict free. The spatial table is a __grid_constant__
// kernel parameter indexed with warp-uniform offsets (constant-bank operands), so each
// launch carries its own table and concurrent configs cannot race. Persistent CTAs walk
// the tile list so the range table is staged once per CTA.
//
// Image-border clipping in x uses a zero-weight sentinel: out-of-image taps read range
// entry 256 (= 0.0), and 0.0*x + y == y exactly, so a half-clipped pair reproduces the
// reference's single-sided update bit for bit. Clipping in y is done by the row loop
// bounds. Rows of a warp's window where only some outputs are inside their window are
// run with warp-uniform per-output predicates; the bulk rows run branch-free.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "p3s_cu.h"

#include <type_traits>

namespace p3s {
namespace cu {
namespace {

constexpr int kTX = 32;
constexpr int kNW = 8;
constexpr int kP = 8;  // outputs per thread (rows)
constexpr int kTY = kNW * kP;
constexpr int kRangeCopies = 16;
constexpr int kRangeEntries = 257;  // 256 + zero sentinel

template <int N>
struct __align__(8) SpatialParam {
    double s[N];
};

__device__ __forceinline__ uint8_t round_half_up_u8(double v) {
    const double r = floor(__dadd_rn(v, 0.5));
    if (r <= 0.0) return 0;
    if (r >= 255.0) return 255;
    return static_cast<uint8_t>(static_cast<int>(r));
}

// One window row (t = yq - yb + R) for the P outputs of this thread. Output i is inside
// its window iff 0 <= t - i <= 2R. ALL: every output is (the bulk rows), no predicates.
template <bool ALL, bool EDGE, int N>
__device__ __forceinline__ void bil_row(const SpatialParam<N>& sp, const uint16_t* __restrict__ row,
                                        const double* __restrict__ rng, int t, int R, int x,
                                        int w, const int (&gi)[kP], double (&ws)[kP],
                                        double (&vs)[kP]) {
    const int side = R + 1;
    {
        const unsigned c = row[0];
        const int gc = c & 0xFF;
        const double dc = static_cast<double>(c >> 8);
#pragma unroll
        for (int i = 0; i < kP; ++i) {
            if (!ALL && static_cast<unsigned>(t - i) > static_cast<unsigned>(2 * R)) continue;
            const double s = sp.s[(t - i) * side];
            const double wc = __dmul_rn(s, rng[__usad(gi[i], gc, 0) * kRangeCopies]);
            ws[i] = __dadd_rn(ws[i], wc);
            vs[i] = __dadd_rn(vs[i], __dmul_rn(wc, dc));
        }
    }
#pragma unroll 2
    for (int dx = 1; dx <= R; ++dx) {
        const unsigned a = row[-dx], b = row[dx];
        const int ga = a & 0xFF, gb = b & 0xFF;
        const double da = static_cast<double>(a >> 8), db = static_cast<double>(b >> 8);
        const bool oob_l = EDGE && (x - dx < 0);
        const bool oob_r = EDGE && (x + dx >= w);
#pragma unroll
        for (int i = 0; i < kP; ++i) {
            if (!ALL && static_cast<unsigned>(t - i) > static_cast<unsigned>(2 * R)) continue;
            const double s = sp.s[(t - i) * side + dx];
            const int il = oob_l ? 256 : static_cast<int>(__usad(gi[i], ga, 0));
            const int ir = oob_r ? 256 : static_cast<int>(__usad(gi[i], gb, 0));
            const double wl = __dmul_rn(s, rng[il * kRangeCopies]);
            const double wr = __dmul_rn(s, rng[ir * kRangeCopies]);
            ws[i] = __dadd_rn(ws[i], __dadd_rn(wl, wr));
            vs[i] = __dadd_rn(vs[i], __dadd_rn(__dmul_rn(wl, da), __dmul_rn(wr, db)));
        }
    }
}

template <bool EDGE, int N>
__device__ __forceinline__ void bil_rows(const SpatialParam<N>& sp, const uint16_t* tile_col,
                                         int SW, const double* rng, int R, int x, int w, int tlo,
                                         int thi, const int (&gi)[kP], double (&ws)[kP],
                                         double (&vs)[kP]) {
    // Rows t in [P-1, 2R] have every output inside its window; the ramps before and after
    // (and everything when 2R < P-1) run predicated. t ascends throughout, which is the
    // reference's dy-ascending order for every output.
    const int full_lo = kP - 1, full_hi = 2 * R;
    int t = tlo;
    for (; t <= min(full_lo - 1, thi); ++t)
        bil_row<false, EDGE>(sp, tile_col + t * SW, rng, t, R, x, w, gi, ws, vs);
    for (; t <= min(full_hi, thi); ++t)
        bil_row<true, EDGE>(sp, tile_col + t * SW, rng, t, R, x, w, gi, ws, vs);
    for (; t <= thi; ++t)
        bil_row<false, EDGE>(sp, tile_col + t * SW, rng, t, R, x, w, gi, ws, vs);
}

template <int N>
__global__ void __launch_bounds__(kNW * 32) k_bilateral_tiled(
    const __grid_constant__ SpatialParam<N> sp, const uint8_t* __restrict__ depth,
    const uint8_t* __restrict__ guide, int pitch, int w, int h, int R,
    const double* __restrict__ range_g, uint8_t* __restrict__ out, double* __restrict__ raw,
    int tiles_x, int ntiles) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* s_rng = reinterpret_cast<double*>(smem);
    uint16_t* s_tile = reinterpret_cast<uint16_t*>(smem + kRangeEntries * kRangeCopies * 8);
    const int SW = kTX + 2 * R;
    const int SH = kTY + 2 * R;

    for (int i = threadIdx.x; i < kRangeEntries * kRangeCopies; i += blockDim.x) {
        const int d = i / kRangeCopies;
        s_rng[i] = d < 256 ? range_g[d] : 0.0;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double* rng = s_rng + (lane & (kRangeCopies - 1));

    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int tx0 = (tile % tiles_x) * kTX;
        const int ty0 = (tile / tiles_x) * kTY;
        __syncthreads();
        for (int sy = warp; sy < SH; sy += kNW) {
            const int gy = ty0 - R + sy;
            const bool yin = gy >= 0 && gy < h;
            const uint8_t* grow = guide + static_cast<size_t>(yin ? gy : 0) * pitch;
            const uint8_t* drow = depth + static_cast<size_t>(yin ? gy : 0) * pitch;
            for (int sx = lane; sx < SW; sx += 32) {
                const int gx = tx0 - R + sx;
                unsigned v = 0;
                if (yin && gx >= 0 && gx < w) v = grow[gx] | (static_cast<unsigned>(drow[gx]) << 8);
                s_tile[sy * SW + sx] = static_cast<uint16_t>(v);
            }
        }
        __syncthreads();

        const int x = tx0 + lane;
        const int yb = ty0 + warp * kP;
        if (yb >= h) continue;
        const bool edge = (tx0 - R < 0) || (tx0 + kTX - 1 + R >= w);
        // tile column of this thread, at the smem row of t = 0 (yq = yb - R)
        const uint16_t* tile_col = s_tile + (warp * kP) * SW + lane + R;
        int gi[kP];
        double ws[kP], vs[kP];
#pragma unroll
        for (int i = 0; i < kP; ++i) {
            gi[i] = tile_col[(i + R) * SW] & 0xFF;
            ws[i] = 0.0;
            vs[i] = 0.0;
        }
        const int tlo = max(0, R - yb);
        const int thi = min(kP - 1 + 2 * R, h - 1 - yb + R);
        if (edge)
            bil_rows<true>(sp, tile_col, SW, rng, R, x, w, tlo, thi, gi, ws, vs);
        else
            bil_rows<false>(sp, tile_col, SW, rng, R, x, w, tlo, thi, gi, ws, vs);
        if (x < w) {
#pragma unroll
            for (int i = 0; i < kP; ++i) {
                const int y = yb + i;
                if (y < h) {
                    const double v = __ddiv_rn(vs[i], ws[i]);
                    out[static_cast<size_t>(y) * pitch + x] = round_half_up_u8(v);
                    if (raw) raw[static_cast<size_t>(y) * w + x] = v;
                }
            }
        }
    }
}

// ---- compile-time-radius variant (the default sigma_s = 8 -> R = 16) ----------------------
// Same schedule and accumulation order as k_bilateral_tiled, with the per-tap overhead cut:
//  * the radius is a compile-time constant (dx loop unrolled by 4: a full unroll overflows
//    the instruction cache — measured no_instruction stalls 1.7/issue);
//  * the range table is stored by SIGNED guide difference, k = gq - gi + 255, replicated
//    16 ways: the tile keeps gq*128 and each output keeps base_i = (255-gi)*128 + lane8,
//    so a lookup is one IADD + one conflict-free LDS.64 (no |.|, no scaling);
//  * the tile packs (depth << 16) | gq*128 in a u32.
// Edge tiles route out-of-image taps to the zero sentinel entry with a select.
constexpr int kSignedEntries = 512;  // k = 0..510, entry 511 = 0.0 sentinel

template <int R, int P, bool ALL, bool EDGE, int N>
__device__ __forceinline__ void bilr_row(const SpatialParam<N>& sp, const uint32_t* __restrict__ row,
                                         const char* __restrict__ tbl, int t, int x, int w,
                                         const int (&base)[P], double (&ws)[P],
                                         double (&vs)[P]) {
    constexpr int side = R + 1;
    constexpr int kZero = 511 * 128;
    {
        const uint32_t c = row[0];
        const int gc = static_cast<int>(c & 0xFFFFu);
        const double dc = static_cast<double>(c >> 16);
#pragma unroll
        for (int i = 0; i < P; ++i) {
            if (!ALL && static_cast<unsigned>(t - i) > static_cast<unsigned>(2 * R)) continue;
            const double s = sp.s[(t - i) * side];
            const double wc = __dmul_rn(s, *reinterpret_cast<const double*>(tbl + base[i] + gc));
            ws[i] = __dadd_rn(ws[i], wc);
            vs[i] = __dadd_rn(vs[i], __dmul_rn(wc, dc));
        }
    }
#pragma unroll 4
    for (int dx = 1; dx <= R; ++dx) {
        const uint32_t a = row[-dx], b = row[dx];
        const int ga = static_cast<int>(a & 0xFFFFu), gb = static_cast<int>(b & 0xFFFFu);
        const double da = static_cast<double>(a >> 16), db = static_cast<double>(b >> 16);
        const bool oob_l = EDGE && (x - dx < 0);
        const bool oob_r = EDGE && (x + dx >= w);
#pragma unroll
        for (int i = 0; i < P; ++i) {
            if (!ALL && static_cast<unsigned>(t - i) > static_cast<unsigned>(2 * R)) continue;
            const double s = sp.s[(t - i) * side + dx];
            const int ol = oob_l ? kZero + (base[i] & 127) : base[i] + ga;
            const int orr = oob_r ? kZero + (base[i] & 127) : base[i] + gb;
            const double wl = __dmul_rn(s, *reinterpret_cast<const double*>(tbl + ol));
            const double wr = __dmul_rn(s, *reinterpret_cast<const double*>(tbl + orr));
            ws[i] = __dadd_rn(ws[i], __dadd_rn(wl, wr));
            vs[i] = __dadd_rn(vs[i], __dadd_rn(__dmul_rn(wl, da), __dmul_rn(wr, db)));
        }
    }
}

template <int R, int P, bool EDGE, int N>
__device__ __forceinline__ void bilr_rows(const SpatialParam<N>& sp, const uint32_t* tile_col,
                                          const char* tbl, int x, int w, int tlo, int thi,
                                          const int (&base)[P], double (&ws)[P],
                                          double (&vs)[P]) {
    constexpr int SW = kTX + 2 * R;
    int t = tlo;
    for (; t <= min(P - 2, thi); ++t)
        bilr_row<R, P, false, EDGE>(sp, tile_col + t * SW, tbl, t, x, w, base, ws, vs);
    for (; t <= min(2 * R, thi); ++t)
        bilr_row<R, P, true, EDGE>(sp, tile_col + t * SW, tbl, t, x, w, base, ws, vs);
    for (; t <= thi; ++t)
        bilr_row<R, P, false, EDGE>(sp, tile_col + t * SW, tbl, t, x, w, base, ws, vs);
}

template <int R, int P, int NW, int MINB, int N>
__global__ void __launch_bounds__(NW * 32, MINB) k_bilateral_r(
    const __grid_constant__ SpatialParam<N> sp, const uint8_t* __restrict__ depth,
    const uint8_t* __restrict__ guide, int pitch, int w, int h,
    const double* __restrict__ range_g, uint8_t* __restrict__ out, double* __restrict__ raw,
    int tiles_x, int ntiles) {
    constexpr int TY = NW * P;
    constexpr int SW = kTX + 2 * R;
    constexpr int SH = TY + 2 * R;
    extern __shared__ __align__(16) unsigned char smem[];
    char* tbl = reinterpret_cast<char*>(smem);  // [512][16] doubles
    uint32_t* s_tile = reinterpret_cast<uint32_t*>(smem + kSignedEntries * kRangeCopies * 8);

    for (int i = threadIdx.x; i < kSignedEntries * kRangeCopies; i += blockDim.x) {
        const int k = i / kRangeCopies;
        const int d = k < 511 ? abs(k - 255) : 256;
        reinterpret_cast<double*>(tbl)[i] = d < 256 ? range_g[d] : 0.0;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int lane8 = (lane & (kRangeCopies - 1)) * 8;

    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int tx0 = (tile % tiles_x) * kTX;
        const int ty0 = (tile / tiles_x) * TY;
        __syncthreads();
        for (int sy = warp; sy < SH; sy += NW) {
            const int gy = ty0 - R + sy;
            const bool yin = gy >= 0 && gy < h;
            const uint8_t* grow = guide + static_cast<size_t>(yin ? gy : 0) * pitch;
            const uint8_t* drow = depth + static_cast<size_t>(yin ? gy : 0) * pitch;
            for (int sx = lane; sx < SW; sx += 32) {
                const int gx = tx0 - R + sx;
                uint32_t v = 0;
                if (yin && gx >= 0 && gx < w)
                    v = (static_cast<uint32_t>(grow[gx]) << 7) | (static_cast<uint32_t>(drow[gx]) << 16);
                s_tile[sy * SW + sx] = v;
            }
        }
        __syncthreads();

        const int x = tx0 + lane;
        const int yb = ty0 + warp * P;
        if (yb >= h) continue;
        const bool edge = (tx0 - R < 0) || (tx0 + kTX - 1 + R >= w);
        const uint32_t* tile_col = s_tile + (warp * P) * SW + lane + R;
        int base[P];
        double ws[P], vs[P];
#pragma unroll
        for (int i = 0; i < P; ++i) {
            const int gi = static_cast<int>((tile_col[(i + R) * SW] & 0xFFFFu) >> 7);
            base[i] = (255 - gi) * 128 + lane8;
            ws[i] = 0.0;
            vs[i] = 0.0;
        }
        const int tlo = max(0, R - yb);
        const int thi = min(P - 1 + 2 * R, h - 1 - yb + R);
        if (edge)
            bilr_rows<R, P, true>(sp, tile_col, tbl, x, w, tlo, thi, base, ws, vs);
        else
            bilr_rows<R, P, false>(sp, tile_col, tbl, x, w, tlo, thi, base, ws, vs);
        if (x < w) {
#pragma unroll
            for (int i = 0; i < P; ++i) {
                const int y = yb + i;
                if (y < h) {
                    const double v = __ddiv_rn(vs[i], ws[i]);
                    out[static_cast<size_t>(y) * pitch + x] = round_half_up_u8(v);
                    if (raw) raw[static_cast<size_t>(y) * w + x] = v;
                }
            }
        }
    }
}

// ---- certified FP32 fast path (radii 7..24) ----------------------------------------------
// Computes every output approximately and proves, per pixel, that the approximation rounds
// to the same byte as the reference's exact FP64 sequence; pixels it cannot prove are
// recomputed exactly (k_bilateral_fixup2, reference order). The output bytes are therefore
// identical to the reference's — only the arithmetic that decides them changes. The packed
// f32x2 helpers below carry two taps (the mirrored pair of a window row) per instruction;
// the error bound and certificate are documented at k_bilateral_sep.
__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void unpack2(unsigned long long v, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ unsigned long long fmul2(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ unsigned long long fadd2(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}

constexpr int kF32Copies = 32;  // LDS.32, one copy per lane: conflict-free

// ---- certified FP32, separable spatial factor (radius 16) ---------------------------------
// The spatial weight factors as
// s(dx,dy) = sx(dx) * sy(dy) (exp of a sum; host tables, each rounded to float), so inside a
// window row a tap contributes sx(dx)*R(|gi-gq|) to the weight sum and (sx(dx)*d_q)*R to the
// value sum: sx(dx) and sx(dx)*d_q depend only on the tap and are shared by the thread's P
// outputs (one FMUL2 per tap pair), leaving per tap pair and output 2 address adds
// (LEA.HI), 2 conflict-free LDS.32 range lookups and 2 FFMA2. The row's FP32 sums are
// scaled by sy(dy) when they are folded (below).
//  * tile element (u32): (goff << 16) | depth, goff = guide * 128 (byte offset of the range
//    row), or 511 * 128 for pixels outside the image: base_i + goff then lands in the zero
//    tail of the table for every centre guide, so image borders need no clipping code;
//  * table: entries k = gq - gi + 255 in [0, 510] hold R(|k - 255|) as float, 511..766 are
//    0; 32 copies, lane l reads copy l (bank l);
//  * depth u8 -> float: byte-select I2F.U8 on the XU pipe (otherwise idle in this loop).
// Rows fold into float-pair accumulators: (N_a, N_b) = sy * (SV_a, SV_b) + (N_a, N_b), one
// FFMA2 per row and output (and likewise D); the halves meet once, in FP64, for the quotient.
// (Folding each row in FP64 instead — add the halves, F2F, DFMA — stalled every warp at each
// row's end on the F2F -> DFMA latency: 9 % of the bulk rows' samples with no LDS issued.)
// Error bound (u = 2^-24, every term >= 0, d exact in float). Weight-sum terms: sx (1
// rounding), R (1), the product is exact inside the FFMA; value-sum terms: sx (1), R (1),
// sx*d (1). The row's FFMA chain adds <= R roundings, float(sy) 1, and the cross-row fold
// chain (the sy product is exact inside its FFMA) <= 2R + 1. So every term of N and D is
// within gamma_(3R+5) (+2^-46 for the FP64 half combine, table and division) of its exact
// value, |v~ - v| <= v * (6R + 10)u (1 + 1e-4), and the reference's own FP64 result is within
// v * 2200 * 2^-53 of v; underflowed float weights add < 1e-35 absolute against D >= 1 (the
// centre tap's weight is exactly 1). A byte is accepted only when v~ + 0.5 is farther than
// (6R + 12)u * v~ + 1e-9 from every integer (r = 16: 108u; ~0.12 % of 4K pixels go to the
// exact fix-up).
constexpr int kSepEntries = 767;  // 511 real + 256 zero
constexpr int kSepOob = 511 * 128;

__device__ __forceinline__ unsigned long long depth_pair(uint32_t a, uint32_t b) {
    // (2^23 + da, 2^23 + db) as f32x2 bit patterns
    const uint32_t lo = __byte_perm(a, 0x4B000000u, 0x7650);
    const uint32_t hi = __byte_perm(b, 0x4B000000u, 0x7650);
    return (static_cast<unsigned long long>(hi) << 32) | lo;
}

template <int R, int P>
struct SepParam {
    unsigned long long sx2[R + 1];  // (float(sx), float(sx)), dx = 0..R
    double sy[2 * R + 1];            // double(float(sy(dy))), dy + R
    unsigned long long sy2[2 * R + 1];  // (float(sy), float(sy)), dy + R (FOLD)
};

// One LDS.32 at a shared-window byte address (base already includes the table's address,
// so address = base + goff is a single LEA.HI).
__device__ __forceinline__ float lds_f32(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}

template <int R, int P, bool ALL, int U, typename Acc>
__device__ __forceinline__ void sep_row(const SepParam<R, P>& sp, const uint32_t* __restrict__ row,
                                        int t, const uint32_t (&base)[P], Acc (&ws)[P],
                                        Acc (&vs)[P]) {
    constexpr bool FOLD = sizeof(Acc) == 8 && !__is_same(Acc, double);
    unsigned long long SW[P], SV[P];
    {
        const uint32_t c = row[0];
        const uint32_t goff = c >> 16;
        const float dc = static_cast<float>(c & 0xFFu);  // I2F on the XU pipe (idle here)
#pragma unroll
        for (int i = 0; i < P; ++i) {
            SW[i] = 0ull;
            SV[i] = 0ull;
            if (!ALL && static_cast<unsigned>(t - i) > static_cast<unsigned>(2 * R)) continue;
            const float wc = lds_f32(base[i] + goff);
            SW[i] = pack2(wc, 0.0f);
            SV[i] = pack2(__fmul_rn(wc, dc), 0.0f);
        }
    }
#pragma unroll U
    for (int dx = 1; dx <= R; ++dx) {
        const uint32_t a = row[-dx], b = row[dx];
        const uint32_t ga = a >> 16, gb = b >> 16;
        const unsigned long long D2 = pack2(static_cast<float>(a & 0xFFu), static_cast<float>(b & 0xFFu));
        const unsigned long long S2 = sp.sx2[dx];
        const unsigned long long SD2 = fmul2(S2, D2);  // sx(dx) * d, shared by the P outputs
#pragma unroll
        for (int i = 0; i < P; ++i) {
            if (!ALL && static_cast<unsigned>(t - i) > static_cast<unsigned>(2 * R)) continue;
            const unsigned long long R2 = pack2(lds_f32(base[i] + ga), lds_f32(base[i] + gb));
            // the tap weights sit in the first operand slot of both FMAs, so the second takes
            // them from the operand reuse cache (register-file reads bound this loop's dispatch
            // as much as the LDS pipe does: 1.386 -> 1.376 ms at 4K)
            SW[i] = ffma2(S2, R2, SW[i]);
            SV[i] = ffma2(R2, SD2, SV[i]);
        }
    }
#pragma unroll
    for (int i = 0; i < P; ++i) {
        if (!ALL && static_cast<unsigned>(t - i) > static_cast<unsigned>(2 * R)) continue;
        if constexpr (FOLD) {
            // the row's pair sums folded into float-pair accumulators: sy * row + acc, one
            // FFMA2 each (the halves meet only in the final quotient, in FP64)
            const unsigned long long SY2 = sp.sy2[t - i];
            ws[i] = ffma2(SY2, SW[i], ws[i]);
            vs[i] = ffma2(SY2, SV[i], vs[i]);
        } else {
            float a0, a1, b0, b1;
            unpack2(SW[i], a0, a1);
            unpack2(SV[i], b0, b1);
            const double sy = sp.sy[t - i];
            ws[i] = __fma_rn(sy, static_cast<double>(__fadd_rn(a0, a1)), ws[i]);
            vs[i] = __fma_rn(sy, static_cast<double>(__fadd_rn(b0, b1)), vs[i]);
        }
    }
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <int R, int P, int NW, int U, bool FOLD = true>
__global__ void __launch_bounds__(NW * 32, 1) k_bilateral_sep(
    const __grid_constant__ SepParam<R, P> sp, const uint8_t* __restrict__ depth,
    const uint8_t* __restrict__ guide, int pitch, int w, int h,
    const double* __restrict__ range_g, uint8_t* __restrict__ out, uint32_t* __restrict__ list,
    uint32_t* __restrict__ count, int tiles_x, int tile_begin, int tile_end,
    uint32_t* __restrict__ tile_ctr, const float* __restrict__ table_g) {
    constexpr int TY = NW * P;
    constexpr int SW = kTX + 2 * R;
    constexpr int SH = TY + 2 * R;
    // raw rows are fetched as 16-byte chunks from the aligned column (tx0 - R) & ~15;
    // RO = (tx0 - R) mod 16 is the same for every tile (tx0 is a multiple of 32)
    constexpr int RO = ((kTX - R) % 16 + 16) % 16;
    constexpr int SWR = (RO + SW + 15) / 16 * 16;
    static_assert(R >= P - 1, "the ramp structure needs 2R + 1 >= P window rows per output");
    extern __shared__ __align__(16) unsigned char smem[];
    char* tbl = reinterpret_cast<char*>(smem);  // [767][32] floats
    uint32_t* s_tile = reinterpret_cast<uint32_t*>(smem + kSepEntries * kF32Copies * 4);
    // raw guide / depth bytes of the NEXT tile, fetched with cp.async while this one computes
    uint8_t* s_raw = smem + kSepEntries * kF32Copies * 4 + (SW * SH * 4 + 15) / 16 * 16;  // [2][SH][SWR]

    if (table_g) {
        // the plan's prebuilt replicated table: 16-byte async copies, landing with the
        // first tile's prefetch (same commit group)
        for (int i = threadIdx.x; i < kSepEntries * kF32Copies / 4; i += blockDim.x)
            cp_async16(tbl + 16 * i, table_g + 4 * i);
    } else {
        for (int i = threadIdx.x; i < kSepEntries * kF32Copies; i += blockDim.x) {
            const int k = i / kF32Copies;
            reinterpret_cast<float*>(tbl)[i] = k < 511 ? static_cast<float>(range_g[abs(k - 255)]) : 0.0f;
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // certificate (see the error bound above): (6R + 12)u v + 1e-9 with the FP32 row fold;
    // (2R + 12)u v + 1e-9 when rows fold in FP64 (R + 5 roundings per term)
    constexpr double kRel = (FOLD ? 6.0 * R + 12.0 : 2.0 * R + 12.0) / 16777216.0;
    // 16-byte chunks of the tile window rows that lie inside the image rows and the pitch;
    // the rest is never read (the packing step marks out-of-image pixels itself)
    auto prefetch = [&](int tile) {
        const int tx0 = (tile % tiles_x) * kTX, ty0 = (tile / tiles_x) * TY;
        const int gx0 = tx0 - R - RO;  // 16-byte aligned
        constexpr int kChunks = SWR / 16;
        for (int q = threadIdx.x; q < 2 * SH * kChunks; q += blockDim.x) {
            const int plane = q / (SH * kChunks), rem = q - plane * (SH * kChunks);
            const int sy = rem / kChunks, c = rem - sy * kChunks;
            const int gy = ty0 - R + sy, gx = gx0 + 16 * c;
            if (gy < 0 || gy >= h || gx < 0 || gx >= pitch) continue;
            const uint8_t* src = (plane ? depth : guide) + static_cast<size_t>(gy) * pitch + gx;
            cp_async16(s_raw + plane * SH * SWR + sy * SWR + 16 * c, src);
        }
        cp_async_commit();
    };
    // tiles [tile_begin, tile_end): the first one per CTA is blockIdx-based, the rest are
    // claimed from tile_ctr (dynamic: CTAs that start late, e.g. behind another launch's
    // tail, simply take fewer tiles)
    // the next tile index, double-buffered by iteration parity: slot it & 1 is written before
    // this iteration's first barrier and read after its second, and written again only two
    // iterations later, behind both barriers of the iteration in between
    __shared__ int s_next[2];
    int tile = tile_begin + static_cast<int>(blockIdx.x);
    if (tile < tile_end) prefetch(tile);
    else cp_async_commit();

    for (int it = 0; tile < tile_end; ++it) {
        const int tx0 = (tile % tiles_x) * kTX;
        const int ty0 = (tile / tiles_x) * TY;
        cp_async_wait_all();
        if (threadIdx.x == 0)
            s_next[it & 1] = tile_begin + static_cast<int>(gridDim.x) + static_cast<int>(atomicAdd(tile_ctr, 1u));
        __syncthreads();  // raw bytes of this tile landed; the previous tile's compute is done
        if constexpr (RO % 4 == 0 && SW % 4 == 0) {
            // 4 window columns per step: one 4-byte load per plane (the 4 bytes lie in one
            // 16-byte chunk, fetched whole or not at all) and one 16-byte store
            constexpr uint32_t kOobWord = static_cast<uint32_t>(kSepOob) << 16;
            for (int e4 = threadIdx.x; e4 < SH * SW / 4; e4 += blockDim.x) {
                const int e = 4 * e4;
                const int sy = e / SW, sx = e - sy * SW;
                const int gy = ty0 - R + sy, gx = tx0 - R + sx;
                uint4 o = make_uint4(kOobWord, kOobWord, kOobWord, kOobWord);
                if (gy >= 0 && gy < h && gx + 3 >= 0 && gx < w) {
                    const int ri = sy * SWR + sx + RO;
                    const uint32_t g4 = *reinterpret_cast<const uint32_t*>(s_raw + ri);
                    const uint32_t d4 = *reinterpret_cast<const uint32_t*>(s_raw + SH * SWR + ri);
                    auto px = [&](int k) {
                        return static_cast<unsigned>(gx + k) < static_cast<unsigned>(w)
                                   ? (((g4 >> (8 * k)) & 0xFFu) << 23) | ((d4 >> (8 * k)) & 0xFFu)
                                   : kOobWord;
                    };
                    o = make_uint4(px(0), px(1), px(2), px(3));
                }
                *reinterpret_cast<uint4*>(s_tile + e) = o;
            }
        } else {
            for (int e = threadIdx.x; e < SH * SW; e += blockDim.x) {
                const int sy = e / SW, sx = e - sy * SW;
                const int gy = ty0 - R + sy, gx = tx0 - R + sx;
                uint32_t v = static_cast<uint32_t>(kSepOob) << 16;
                if (gy >= 0 && gy < h && gx >= 0 && gx < w) {
                    const int ri = sy * SWR + sx + RO;
                    v = (static_cast<uint32_t>(s_raw[ri]) << 23) | s_raw[SH * SWR + ri];
                }
                s_tile[e] = v;
            }
        }
        __syncthreads();
        const int next = s_next[it & 1];
        if (next < tile_end) prefetch(next);
        tile = next;

        const int x = tx0 + lane;
        const int yb = ty0 + warp * P;
        if (yb >= h) continue;
        const uint32_t* tile_col = s_tile + (warp * P) * SW + lane + R;
        const uint32_t tbl_s = static_cast<uint32_t>(__cvta_generic_to_shared(tbl));
        uint32_t base[P];
        using Acc = typename std::conditional<FOLD, unsigned long long, double>::type;
        Acc ws[P], vs[P];
#pragma unroll
        for (int i = 0; i < P; ++i) {
            const int gi = static_cast<int>(tile_col[(i + R) * SW] >> 23) & 0xFF;
            base[i] = tbl_s + static_cast<uint32_t>((255 - gi) * 128 + lane * 4);
            ws[i] = 0;
            vs[i] = 0;
        }
        // Every window row of the band is processed: rows outside the image hold the OOB
        // guide offset (zero weight, exact zeros), so there is no clipping logic. The ramp
        // rows (only some outputs inside their window) are unrolled with compile-time t, so
        // their per-output predicates fold away; the bulk rows run all P outputs.
        // output i is final after window row 2R + i: its quotient, certificate, byte and list
        // entry are issued right there, so the tail-ramp outputs' FP64 epilogues overlap the
        // remaining rows' lookups instead of idling the LDS pipe at the end of the tile
        // (1.415 -> 1.386 ms at 4K)
        auto finalize = [&](int i) {
            const int y = yb + i;
            const bool valid = x < w && y < h;
            bool uncertain = false;
            if (valid) {
                double v;
                if constexpr (FOLD) {
                    float a0, a1, b0, b1;
                    unpack2(ws[i], a0, a1);
                    unpack2(vs[i], b0, b1);
                    v = __ddiv_rn(__dadd_rn(b0, b1), __dadd_rn(a0, a1));
                } else {
                    v = __ddiv_rn(vs[i], ws[i]);
                }
                const double f = __dadd_rn(v, 0.5);
                const double r = floor(f);
                const double dist = fmin(f - r, r + 1.0 - f);
                const double bound = v * kRel + 1e-9;
                uncertain = !(dist > bound);
                out[static_cast<size_t>(y) * pitch + x] =
                    uncertain ? 0 : static_cast<uint8_t>(min(max(static_cast<int>(r), 0), 255));
            }
            const unsigned m = __ballot_sync(0xFFFFFFFFu, uncertain);
            if (m) {
                uint32_t start = 0;
                if (lane == 0) start = atomicAdd(count, static_cast<uint32_t>(__popc(m)));
                start = __shfl_sync(0xFFFFFFFFu, start, 0);
                if (uncertain)
                    list[start + __popc(m & ((1u << lane) - 1u))] =
                        static_cast<uint32_t>(y) * static_cast<uint32_t>(w) + static_cast<uint32_t>(x);
            }
        };
#pragma unroll
        for (int t = 0; t < P - 1; ++t) sep_row<R, P, false, U>(sp, tile_col + t * SW, t, base, ws, vs);
        for (int t = P - 1; t <= 2 * R; ++t) sep_row<R, P, true, U>(sp, tile_col + t * SW, t, base, ws, vs);
        finalize(0);
#pragma unroll
        for (int t = 2 * R + 1; t < 2 * R + P; ++t) {
            sep_row<R, P, false, U>(sp, tile_col + t * SW, t, base, ws, vs);
            finalize(t - 2 * R);
        }
    }
}

// Exact recompute of the uncertified pixels (reference order): one warp per listed pixel,
// one resident wave of CTAs (4 warps each; their windows plus the FP64 range and spatial
// tables in shared memory, ~24 KB per CTA at r = 16), later pixels by grid stride.
// The window is staged with 16-byte loads. The terms of a batch of window rows — per row
// the centre (wc, wc*d), then per dx the mirrored pair (wl + wr, wl*dl + wr*dr) or the single
// in-image side, each separately rounded — are computed by all lanes in parallel; lane 0
// then adds them to the two running sums in the reference order (rows dy ascending; centre,
// dx = 1..R). Only that serial DADD chain remains on the critical path.
template <int R, int WPB>
__global__ void __launch_bounds__(WPB * 32) k_bilateral_fixup2(
    const uint8_t* __restrict__ depth, const uint8_t* __restrict__ guide, int pitch, int w,
    int h, const double* __restrict__ spatial, const double* __restrict__ range_g,
    uint8_t* __restrict__ out, const uint32_t* __restrict__ list,
    const uint32_t* __restrict__ count) {
    constexpr int S = 2 * R + 1, SP = (S + 15 + 15) / 16 * 16;  // window side, staged row length
    constexpr int kBatch = 4;                  // window rows per term batch (serial fallback)
    __shared__ __align__(16) uint8_t s_g[WPB][S][SP];
    __shared__ __align__(16) uint8_t s_d[WPB][S][SP];
    __shared__ double2 s_tu[WPB][kBatch][R + 1];
    // the FP64 range and spatial tables, staged once per CTA: the terms' table reads are
    // shared-memory gathers instead of L1 lookups (the fix-up was latency-bound on them)
    __shared__ double s_rng[256];
    __shared__ double s_sp[S * (R + 1)];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint32_t n = *count;
    const uint32_t nwarps = gridDim.x * WPB;
    if (blockIdx.x * WPB >= n) return;  // (uniform per CTA: no barrier below is skipped)
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s_rng[i] = __ldg(range_g + i);
    for (int i = threadIdx.x; i < S * (R + 1); i += blockDim.x) s_sp[i] = __ldg(spatial + i);
    __syncthreads();
    for (uint32_t k = blockIdx.x * WPB + wib; k < n; k += nwarps) {
        const uint32_t idx = list[k];
        const int x = static_cast<int>(idx % static_cast<uint32_t>(w));
        const int y = static_cast<int>(idx / static_cast<uint32_t>(w));
        // stage: 16-byte chunks from the aligned column c0 <= x - R; window column j of the
        // pixel sits at staged offset j + off
        const int c0 = (x - R) & ~15, off = (x - R) - c0;
        constexpr int kCh = (S + 15 + 15) / 16;
#pragma unroll
        for (int q0 = 0; q0 < (2 * S * kCh + 31) / 32; ++q0) {
            const int q = lane + 32 * q0;
            if (q >= 2 * S * kCh) break;
            const int plane = q / (S * kCh), rem = q - plane * (S * kCh);
            const int r = rem / kCh, ch = rem - r * kCh;
            const int gy = y - R + r, gx = c0 + 16 * ch;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (gy >= 0 && gy < h && gx >= 0 && gx < pitch)
                v = __ldg(reinterpret_cast<const uint4*>((plane ? depth : guide) +
                                                         static_cast<size_t>(gy) * pitch + gx));
            if (16 * ch + 16 <= SP)
                *reinterpret_cast<uint4*>(plane ? &s_d[wib][r][16 * ch] : &s_g[wib][r][16 * ch]) = v;
        }
        __syncwarp();
        const int gp = s_g[wib][R][R + off];
        const int dy0 = y - R < 0 ? -y : -R;
        const int dy1 = y + R >= h ? h - 1 - y : R;
        // Every term (per window row: the centre tap, then each mirrored pair as the
        // reference forms it, each separately rounded) is the reference's; only their
        // accumulation order decides the last bits. The lanes sum them in any order (<= kM
        // terms each, then a 5-level tree): the reference's sequential sum and this one are
        // both within gamma_(n-1) resp. gamma_(kM+4) of the exact sum of these non-negative
        // terms, so |v - v_ref| <= v (2 (n + kM + 3) + 2) u (u = 2^-53). When v + 0.5 is
        // farther than that (+1e-12) from every integer both round to the same byte;
        // otherwise (practically never) the serial reference-order chain below decides.
        {
            constexpr int kN = S * (R + 1);
            constexpr int kM = (kN + 31) / 32;
            double wsp = 0.0, vsp = 0.0;
            if (x >= R && x + R < w && y >= R && y + R < h) {
                // interior pixel (nearly all of them): every tap is in the image, so the terms
                // need no side tests; the centre is a pair with a zero right weight (t = wl + 0
                // and u = wl * d + 0 * d are the reference's wl and wl * d exactly). Two
                // accumulators per lane interleave the terms' FP64 chains (any order is covered
                // by the bound below: <= kM terms per lane chain).
                double w0 = 0.0, v0 = 0.0, w1 = 0.0, v1 = 0.0;
#pragma unroll
                for (int k = 0; k < kM; ++k) {
                    const int e = lane + 32 * k;
                    if (e >= kN) break;
                    const int r = e / (R + 1), j = e - r * (R + 1);
                    const uint8_t* gr = &s_g[wib][r][R + off];
                    const uint8_t* dr = &s_d[wib][r][R + off];
                    const double sj = s_sp[e];
                    const double wl = __dmul_rn(sj, s_rng[__usad(gp, gr[-j], 0)]);
                    const double wq = __dmul_rn(sj, s_rng[__usad(gp, gr[j], 0)]);
                    const double wr = j ? wq : 0.0;
                    const double t = __dadd_rn(wl, wr);
                    const double u = __dadd_rn(__dmul_rn(wl, static_cast<double>(dr[-j])),
                                               __dmul_rn(wr, static_cast<double>(dr[j])));
                    if (k & 1) {
                        w1 = __dadd_rn(w1, t);
                        v1 = __dadd_rn(v1, u);
                    } else {
                        w0 = __dadd_rn(w0, t);
                        v0 = __dadd_rn(v0, u);
                    }
                }
                wsp = __dadd_rn(w0, w1);
                vsp = __dadd_rn(v0, v1);
            } else
            for (int e = lane; e < kN; e += 32) {
                const int r = e / (R + 1), j = e - r * (R + 1), dy = r - R;
                if (dy < dy0 || dy > dy1) continue;
                const uint8_t* gr = &s_g[wib][r][R + off];
                const uint8_t* dr = &s_d[wib][r][R + off];
                const double sj = s_sp[r * (R + 1) + j];
                double t = 0.0, u = 0.0;
                if (j == 0) {
                    t = __dmul_rn(sj, s_rng[__usad(gp, gr[0], 0)]);
                    u = __dmul_rn(t, static_cast<double>(dr[0]));
                } else {
                    const bool lin = x - j >= 0, rin = x + j < w;
                    const double wl = lin ? __dmul_rn(sj, s_rng[__usad(gp, gr[-j], 0)]) : 0.0;
                    const double wr = rin ? __dmul_rn(sj, s_rng[__usad(gp, gr[j], 0)]) : 0.0;
                    if (lin && rin) {
                        t = __dadd_rn(wl, wr);
                        u = __dadd_rn(__dmul_rn(wl, static_cast<double>(dr[-j])),
                                      __dmul_rn(wr, static_cast<double>(dr[j])));
                    } else if (lin) {
                        t = wl;
                        u = __dmul_rn(wl, static_cast<double>(dr[-j]));
                    } else if (rin) {
                        t = wr;
                        u = __dmul_rn(wr, static_cast<double>(dr[j]));
                    }
                }
                wsp = __dadd_rn(wsp, t);
                vsp = __dadd_rn(vsp, u);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                wsp = __dadd_rn(wsp, __shfl_xor_sync(0xFFFFFFFFu, wsp, o));
                vsp = __dadd_rn(vsp, __shfl_xor_sync(0xFFFFFFFFu, vsp, o));
            }
            const double v = __ddiv_rn(vsp, wsp);
            const double f = __dadd_rn(v, 0.5);
            const double r = floor(f);
            const double dist = fmin(f - r, r + 1.0 - f);
            constexpr double kRel = (2.0 * (kN + kM + 3) + 2.0) * 1.1102230246251565e-16 * 1.01;
            if (dist > v * kRel + 1e-12) {  // every lane holds the same sums: uniform branch
                if (lane == 0)
                    out[static_cast<size_t>(y) * pitch + x] =
                        r <= 0.0 ? 0 : (r >= 255.0 ? 255 : static_cast<uint8_t>(static_cast<int>(r)));
                __syncwarp();
                continue;
            }
        }
        double ws = 0.0, vs = 0.0;
        for (int rb = 0; rb < S; rb += kBatch) {
            const int nr = min(kBatch, S - rb);
            for (int e = lane; e < nr * (R + 1); e += 32) {
                const int rr = e / (R + 1), j = e - rr * (R + 1);
                const int r = rb + rr, dy = r - R;
                double t = 0.0, u = 0.0;
                if (dy >= dy0 && dy <= dy1) {
                    const uint8_t* gr = &s_g[wib][r][R + off];
                    const uint8_t* dr = &s_d[wib][r][R + off];
                    const double sj = s_sp[r * (R + 1) + j];
                    if (j == 0) {
                        t = __dmul_rn(sj, s_rng[__usad(gp, gr[0], 0)]);
                        u = __dmul_rn(t, static_cast<double>(dr[0]));
                    } else {
                        const bool lin = x - j >= 0, rin = x + j < w;
                        const double wl = lin ? __dmul_rn(sj, s_rng[__usad(gp, gr[-j], 0)]) : 0.0;
                        const double wr = rin ? __dmul_rn(sj, s_rng[__usad(gp, gr[j], 0)]) : 0.0;
                        if (lin && rin) {
                            t = __dadd_rn(wl, wr);
                            u = __dadd_rn(__dmul_rn(wl, static_cast<double>(dr[-j])),
                                          __dmul_rn(wr, static_cast<double>(dr[j])));
                        } else if (lin) {
                            t = wl;
                            u = __dmul_rn(wl, static_cast<double>(dr[-j]));
                        } else if (rin) {
                            t = wr;
                            u = __dmul_rn(wr, static_cast<double>(dr[j]));
                        }
                        // both sides outside: +0 leaves the non-negative sums unchanged
                    }
                }
                s_tu[wib][rr][j] = make_double2(t, u);
            }
            __syncwarp();
            if (lane == 0) {
                for (int rr = 0; rr < nr; ++rr) {
                    const int dy = rb + rr - R;
                    if (dy < dy0 || dy > dy1) continue;
                    double2 v[R + 1];
#pragma unroll
                    for (int j = 0; j <= R; ++j) v[j] = s_tu[wib][rr][j];
#pragma unroll
                    for (int j = 0; j <= R; ++j) {
                        ws = __dadd_rn(ws, v[j].x);
                        vs = __dadd_rn(vs, v[j].y);
                    }
                }
            }
            __syncwarp();
        }
        if (lane == 0) out[static_cast<size_t>(y) * pitch + x] = round_half_up_u8(__ddiv_rn(vs, ws));
        __syncwarp();
    }
}

// Any radius: one thread per output, tables and pixels read through the L1 path.
__global__ void __launch_bounds__(256) k_bilateral_generic(
    const uint8_t* __restrict__ depth, const uint8_t* __restrict__ guide, int pitch, int w,
    int h, int R, const double* __restrict__ spatial, const double* __restrict__ range_g,
    uint8_t* __restrict__ out, double* __restrict__ raw) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    if (x >= w) return;
    const int side = R + 1;
    const int gp = guide[static_cast<size_t>(y) * pitch + x];
    double ws = 0.0, vs = 0.0;
    const int dy0 = y - R < 0 ? -y : -R;
    const int dy1 = y + R >= h ? h - 1 - y : R;
    for (int dy = dy0; dy <= dy1; ++dy) {
        const uint8_t* grow = guide + static_cast<size_t>(y + dy) * pitch;
        const uint8_t* drow = depth + static_cast<size_t>(y + dy) * pitch;
        const double* s = spatial + static_cast<size_t>(dy + R) * side;
        {
            const double wc = __dmul_rn(s[0], range_g[__usad(gp, grow[x], 0)]);
            ws = __dadd_rn(ws, wc);
            vs = __dadd_rn(vs, __dmul_rn(wc, static_cast<double>(drow[x])));
        }
        for (int dx = 1; dx <= R; ++dx) {
            const bool lin = x - dx >= 0, rin = x + dx < w;
            if (lin && rin) {
                const double wl = __dmul_rn(s[dx], range_g[__usad(gp, grow[x - dx], 0)]);
                const double wr = __dmul_rn(s[dx], range_g[__usad(gp, grow[x + dx], 0)]);
                ws = __dadd_rn(ws, __dadd_rn(wl, wr));
                vs = __dadd_rn(vs, __dadd_rn(__dmul_rn(wl, static_cast<double>(drow[x - dx])),
                                             __dmul_rn(wr, static_cast<double>(drow[x + dx]))));
            } else if (lin) {
                const double wl = __dmul_rn(s[dx], range_g[__usad(gp, grow[x - dx], 0)]);
                ws = __dadd_rn(ws, wl);
                vs = __dadd_rn(vs, __dmul_rn(wl, static_cast<double>(drow[x - dx])));
            } else if (rin) {
                const double wr = __dmul_rn(s[dx], range_g[__usad(gp, grow[x + dx], 0)]);
                ws = __dadd_rn(ws, wr);
                vs = __dadd_rn(vs, __dmul_rn(wr, static_cast<double>(drow[x + dx])));
            }
        }
    }
    const double v = __ddiv_rn(vs, ws);
    out[static_cast<size_t>(y) * pitch + x] = round_half_up_u8(v);
    if (raw) raw[static_cast<size_t>(y) * w + x] = v;
}

template <int N>
cudaError_t launch_tiled(const uint8_t* depth, const uint8_t* guide, Geom gm, int R,
                         const double* spatial_host_order, const double* range, uint8_t* out,
                         double* raw, cudaStream_t st) {
    SpatialParam<N> sp;
    const int n = (2 * R + 1) * (R + 1);
    for (int i = 0; i < n; ++i) sp.s[i] = spatial_host_order[i];
    for (int i = n; i < N; ++i) sp.s[i] = 0.0;
    const int SW = kTX + 2 * R, SH = kTY + 2 * R;
    const size_t smem = kRangeEntries * kRangeCopies * 8 + static_cast<size_t>(SW) * SH * 2;
    static std::atomic<unsigned long long> configured{0};
    once_per_device(configured, [] {
        cudaFuncSetAttribute(k_bilateral_tiled<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             200 * 1024);
    });
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bilateral_tiled<N>, kNW * 32, smem);
    if (per_sm < 1) per_sm = 1;
    const int tiles_x = (gm.w + kTX - 1) / kTX;
    const int tiles_y = (gm.h + kTY - 1) / kTY;
    const int ntiles = tiles_x * tiles_y;
    const int grid = min(ntiles, per_sm * sm_count());
    note_launch(st);
    k_bilateral_tiled<N><<<grid, kNW * 32, smem, st>>>(sp, depth, guide, gm.pitch, gm.w, gm.h, R,
                                                       range, out, raw, tiles_x, ntiles);
    return cudaGetLastError();
}

template <int R, int P, int NW, int MINB>
cudaError_t launch_r(const uint8_t* depth, const uint8_t* guide, Geom gm,
                     const double* spatial_host, const double* range, uint8_t* out, double* raw,
                     cudaStream_t st) {
    constexpr int N = (2 * R + 1) * (R + 1);
    SpatialParam<N> sp;
    for (int i = 0; i < N; ++i) sp.s[i] = spatial_host[i];
    constexpr int TY = NW * P;
    constexpr int SW = kTX + 2 * R, SH = TY + 2 * R;
    const size_t smem = kSignedEntries * kRangeCopies * 8 + static_cast<size_t>(SW) * SH * 4;
    static std::atomic<unsigned long long> configured{0};
    once_per_device(configured, [] {
        cudaFuncSetAttribute(k_bilateral_r<R, P, NW, MINB, N>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    });
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bilateral_r<R, P, NW, MINB, N>,
                                                  NW * 32, smem);
    if (per_sm < 1) per_sm = 1;
    const int tiles_x = (gm.w + kTX - 1) / kTX;
    const int tiles_y = (gm.h + TY - 1) / TY;
    const int ntiles = tiles_x * tiles_y;
    const int grid = min(ntiles, per_sm * sm_count());
    note_launch(st);
    k_bilateral_r<R, P, NW, MINB, N><<<grid, NW * 32, smem, st>>>(sp, depth, guide, gm.pitch, gm.w, gm.h,
                                                      range, out, raw, tiles_x, ntiles);
    return cudaGetLastError();
}

template <int R, int P, int NW, int U = 4, bool FOLD = true>
cudaError_t launch_sep_main(const uint8_t* depth, const uint8_t* guide, Geom gm,
                            const double* spatial_host, const double* range, uint8_t* out,
                            uint32_t* list, uint32_t* count, uint32_t* tile_ctr, int tr0, int tr1,
                            const float* table, cudaStream_t st) {
    SepParam<R, P> sp;
    // sx(d) = exp(-(d*d) * inv_s): the dy = 0 row of the host spatial table (same formula)
    const double* row0 = spatial_host + static_cast<size_t>(R) * (R + 1);
    for (int d = 0; d <= R; ++d) {
        const float f = static_cast<float>(row0[d]);
        unsigned u;
        memcpy(&u, &f, 4);
        sp.sx2[d] = (static_cast<unsigned long long>(u) << 32) | u;
    }
    for (int dy = -R; dy <= R; ++dy) {
        const float f = static_cast<float>(row0[dy < 0 ? -dy : dy]);
        sp.sy[dy + R] = static_cast<double>(f);
        unsigned u;
        memcpy(&u, &f, 4);
        sp.sy2[dy + R] = (static_cast<unsigned long long>(u) << 32) | u;
    }
    constexpr int TY = NW * P;
    constexpr int SW = kTX + 2 * R, SH = TY + 2 * R;
    constexpr int RO = ((kTX - R) % 16 + 16) % 16;
    constexpr int SWR = (RO + SW + 15) / 16 * 16;
    const size_t smem = kSepEntries * kF32Copies * 4 + (static_cast<size_t>(SW) * SH * 4 + 15) / 16 * 16 +
                        2 * static_cast<size_t>(SWR) * SH;
    static std::atomic<unsigned long long> configured{0};
    once_per_device(configured, [smem] {
        cudaFuncSetAttribute(k_bilateral_sep<R, P, NW, U, FOLD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
    });
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bilateral_sep<R, P, NW, U, FOLD>, NW * 32, smem);
    if (per_sm < 1) return cudaErrorLaunchOutOfResources;
    const int tiles_x = (gm.w + kTX - 1) / kTX;
    const int tiles_y = (gm.h + TY - 1) / TY;
    if (tr1 < 0 || tr1 > tiles_y) tr1 = tiles_y;
    if (tr1 <= tr0) return cudaSuccess;
    const int t0 = tr0 * tiles_x, t1 = tr1 * tiles_x;
    const int grid = min(t1 - t0, per_sm * sm_count());
    note_launch(st);
    k_bilateral_sep<R, P, NW, U, FOLD><<<grid, NW * 32, smem, st>>>(
        sp, depth, guide, gm.pitch, gm.w, gm.h, range, out, list, count, tiles_x, t0, t1, tile_ctr,
        table);
    return cudaGetLastError();
}

template <int R>
cudaError_t launch_sep_fixup(const uint8_t* depth, const uint8_t* guide, Geom gm,
                             const double* spatial_dev, const double* range, uint8_t* out,
                             const uint32_t* list, const uint32_t* count, cudaStream_t st,
                             int max_ctas) {
    // 4 warps per block up to R = 16 (static smem < 48 KB), 2 beyond; by default enough
    // warps for every listed pixel of a 4K frame in one wave
    constexpr int WPB = R <= 16 ? 4 : 2;
    // one resident wave (a second, partial one only adds its tail); the occupancy query is
    // made once per radius (same answer on every sm_100a device)
    static const int per_sm = [] {
        int n = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_bilateral_fixup2<R, WPB>, WPB * 32, 0);
        return std::max(1, std::min(n, 32 / WPB));
    }();
    int ctas = sm_count() * per_sm;
    if (max_ctas > 0 && max_ctas < ctas) ctas = max_ctas;
    note_launch(st);
    k_bilateral_fixup2<R, WPB><<<ctas, WPB * 32, 0, st>>>(
        depth, guide, gm.pitch, gm.w, gm.h, spatial_dev, range, out, list, count);
    return cudaGetLastError();
}

}  // namespace

cudaError_t bilateral_fast(const uint8_t* depth, const uint8_t* guide, Geom gm, int radius,
                           const double* spatial_host, const double* spatial_dev,
                           const double* range, uint8_t* out, uint32_t* list, uint32_t* count,
                           cudaStream_t st, cudaEvent_t after_main, const float* table) {
    if (!bilateral_fast_available(radius)) {
        const cudaError_t e = bilateral_tiled(depth, guide, gm, radius, spatial_host, range, out, nullptr, st);
        if (after_main) record_event_any(after_main, st);
        return e;
    }
    // count and the tile-claim counter (count[1]) start at zero
    ZeroRanges z{};
    z.p[0] = count;
    z.words[0] = 2;
    z.n = 1;
    cudaError_t e = zero(z, st);
    if (e != cudaSuccess) return e;
    e = bilateral_sep_main(depth, guide, gm, radius, spatial_host, range, out, list, count,
                           count + 1, 0, -1, table, st);
    if (e != cudaSuccess) return e;
    if (after_main) record_event_any(after_main, st);
    return bilateral_sep_fixup(depth, guide, gm, radius, spatial_dev, range, out, list, count, st);
}

// the certified kernel for radii 7..24 (sigma_s in (3, 12]); P = 8 outputs per thread,
// 16 warps, the dx loop fully unrolled
cudaError_t bilateral_sep_main(const uint8_t* depth, const uint8_t* guide, Geom gm, int radius,
                               const double* spatial_host, const double* range, uint8_t* out,
                               uint32_t* list, uint32_t* count, uint32_t* tile_ctr,
                               int tile_row0, int tile_row1, const float* table, cudaStream_t st) {
#define P3S_SEP(RR)                                                                          \
    case RR:                                                                                 \
        return launch_sep_main<RR, 8, 16, RR>(depth, guide, gm, spatial_host, range, out,    \
                                              list, count, tile_ctr, tile_row0, tile_row1,   \
                                              table, st);
    switch (radius) {
        P3S_SEP(7) P3S_SEP(8) P3S_SEP(9) P3S_SEP(10) P3S_SEP(11) P3S_SEP(12) P3S_SEP(13)
        P3S_SEP(14) P3S_SEP(15) P3S_SEP(16) P3S_SEP(17) P3S_SEP(18) P3S_SEP(19) P3S_SEP(20)
        P3S_SEP(21) P3S_SEP(22) P3S_SEP(23) P3S_SEP(24)
        default: break;
    }
#undef P3S_SEP
    return cudaErrorInvalidValue;
}

cudaError_t bilateral_sep_fixup(const uint8_t* depth, const uint8_t* guide, Geom gm, int radius,
                                const double* spatial_dev, const double* range, uint8_t* out,
                                const uint32_t* list, const uint32_t* count, cudaStream_t st,
                                int max_ctas) {
#define P3S_FIX(RR)                                                                          \
    case RR:                                                                                 \
        return launch_sep_fixup<RR>(depth, guide, gm, spatial_dev, range, out, list, count, st, \
                                    max_ctas);
    switch (radius) {
        P3S_FIX(7) P3S_FIX(8) P3S_FIX(9) P3S_FIX(10) P3S_FIX(11) P3S_FIX(12) P3S_FIX(13)
        P3S_FIX(14) P3S_FIX(15) P3S_FIX(16) P3S_FIX(17) P3S_FIX(18) P3S_FIX(19) P3S_FIX(20)
        P3S_FIX(21) P3S_FIX(22) P3S_FIX(23) P3S_FIX(24)
        default: break;
    }
#undef P3S_FIX
    return cudaErrorInvalidValue;
}

int bilateral_sep_tile_rows() { return 16 * 8; }

size_t bilateral_sep_table_bytes() { return static_cast<size_t>(kSepEntries) * kF32Copies * 4; }

namespace {
__global__ void k_build_sep_table(const double* __restrict__ range_g, float* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= kSepEntries * kF32Copies) return;
    const int k = i / kF32Copies;
    out[i] = k < 511 ? static_cast<float>(range_g[abs(k - 255)]) : 0.0f;
}
}  // namespace

cudaError_t build_sep_table(const double* range, float* table, cudaStream_t st) {
    const int n = kSepEntries * kF32Copies;
    note_launch(st);
    k_build_sep_table<<<(n + 255) / 256, 256, 0, st>>>(range, table);
    return cudaGetLastError();
}

bool bilateral_fast_available(int radius) {
    const char* v = getenv("P3S_BIL_FAST");
    return radius >= 7 && radius <= 24 && !(v && atoi(v) == 0);
}

// spatial: device table for the generic kernel, in the layout s[(dy+R)*(R+1)+dx] (dx>=0).
// The tiled kernels take the same table by value; engine.cpp passes the host copy via
// bilateral_tiled_host below.
cudaError_t bilateral(const uint8_t* depth, const uint8_t* guide, Geom gm, int radius,
                      const double* spatial, const double* range, uint8_t* out, double* raw,
                      cudaStream_t st) {
    dim3 grid((gm.w + 127) / 128, gm.h);
    note_launch(st);
    k_bilateral_generic<<<grid, 128, 0, st>>>(depth, guide, gm.pitch, gm.w, gm.h, radius,
                                              spatial, range, out, raw);
    return cudaGetLastError();
}

cudaError_t bilateral_tiled(const uint8_t* depth, const uint8_t* guide, Geom gm, int radius,
                            const double* spatial_host, const double* range, uint8_t* out,
                            double* raw, cudaStream_t st) {
    if (radius == 16)  // the reference tap order in FP64, P = 4 rows x 16 warps (3.2 ms at 4K)
        return launch_r<16, 4, 16, 2>(depth, guide, gm, spatial_host, range, out, raw, st);
    const int n = (2 * radius + 1) * (radius + 1);
    if (n <= 1024)
        return launch_tiled<1024>(depth, guide, gm, radius, spatial_host, range, out, raw, st);
    return launch_tiled<4000>(depth, guide, gm, radius, spatial_host, range, out, raw, st);
}

int bilateral_tiled_max_radius() { return 43; }  // (2r+1)(r+1) <= 4000

}  // namespace cu
}  // namespace p3s
