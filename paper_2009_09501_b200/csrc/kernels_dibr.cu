// K3a: DIBR left/right reconstruction on sm_100a (reference proj/src/dibr.cpp:33-111),
// optionally fused with the anaglyph composition (stereo_format.cpp:8-21).
//
// One CTA per image row. The source row (R, G, B) and its filtered depth are staged in
// shared memory with 16-byte vector loads. Forward mode splats every source pixel into a
// per-eye shared-memory z-buffer with atomicMax on a packed key
//     key = (d + 1) << 22 | (0x3FFFFF - x)
// whose maximum is "largest depth, then smallest source column" — exactly the winner of
// the reference's ascending-x scan with strict '>' (dibr.cpp:88-99) — and independent of
// the order atomics land in (plain stores first, atomicMax only for the few sources that
// lost a slot; see the splat phase). The resolve phase gathers each destination's winning colour
// from shared memory and writes 16 pixels per thread with 16-byte stores; a destination
// without a key is damaged. Output routing (EyeOut) writes only the planes a format
// needs: the fused anaglyph writes left.R and right.G/B straight into the output image,
// so the two eye frames never exist in HBM (4N read + 3N write + N/4 mask bits).
//
// Shift arithmetic is the reference's: sigma[d] = +s (d > T) or -s' (d <= T) is tabulated
// on the host; p.left = x - sigma, p.right = x + sigma are single IEEE adds (__dadd_rn /
// __dsub_rn, never contracted), truncated toward zero (__double2int_rz), so (-1, 0)
// maps to column 0 as in dibr.hpp:35.
#include <cstdlib>

#include "p3s_cu.h"

namespace p3s {
namespace cu {
namespace {

constexpr unsigned kXMask = 0x3FFFFFu;

__device__ __forceinline__ void store16(uint8_t* dst, const uint8_t (&v)[16], int x0, int w) {
    if (x0 + 16 <= w && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
        *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(v);
    } else {
        for (int k = 0; k < 16 && x0 + k < w; ++k) dst[k] = v[k];
    }
}

// Appends the set bits of `m` (pixel x0+k for bit k) to a damaged list, one global
// atomic per warp. Every lane of the warp must call it.
__device__ __forceinline__ void append_list(uint32_t* list, uint32_t* count, unsigned m,
                                            uint32_t base_index, int lane) {
    const int n = __popc(m);
    int incl = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
    uint32_t start = 0;
    if (lane == 31 && total) start = atomicAdd(count, static_cast<uint32_t>(total));
    start = __shfl_sync(0xFFFFFFFFu, start, 31);
    uint32_t pos = start + static_cast<uint32_t>(incl - n);
    while (m) {
        const int k = __ffs(m) - 1;
        m &= m - 1;
        list[pos++] = base_index + static_cast<uint32_t>(k);
    }
}

// Exact integer <-> double helpers on the FP64 pipe (no XU conversions):
//   xd(x)      = (2^52 + x) - 2^52, exact for 0 <= x < 2^31;
//   col(v)     = trunc(v) for v in (-1, w): (-1, 0) -> 0 as the reference's (int) cast,
//                else floor(v) = low word of (v + 2^52) rounded toward zero.
__device__ __forceinline__ double exact_xd(int x) {
    return __dsub_rn(__hiloint2double(0x43300000, x), 4503599627370496.0);
}
// Returns the truncated column if it lies in [0, w), else -1.
__device__ __forceinline__ int trunc_col(double v, int w) {
    if (!(v > -1.0) || !(v < static_cast<double>(w))) return -1;
    if (v < 0.0) return 0;
    return __double2loint(__dadd_rz(v, 4503599627370496.0));
}

// Integer column tables (engine.cpp dibr_col_table): for depth d and direction P (x + sigma)
// or M (x - sigma), the reference's trunc(fl(x +- sigma)) over x in [0, w) equals
//     col = x + off + (x >= X),  except col = 0 at x == z  (fl(x +- sigma) in (-1, 0)),
// valid iff 0 <= col < w. The host derives (off, X, z) from the exact double evaluation of
// every x and verifies the representation before a plan uses it (else the FP64 path runs).
// Packed per d as int4 {off & 0xFFFF | X << 16 (P), same (M), zP, zM}.
__device__ __forceinline__ int col_int(int packed, int z, int x) {
    const int off = static_cast<int>(static_cast<short>(packed & 0xFFFF));
    const int X = static_cast<int>(static_cast<unsigned>(packed) >> 16);
    const int c = x + off + (x >= X ? 1 : 0);
    return x == z ? 0 : c;
}

// ROUTE 0: anaglyph fused (left R, right G/B only, bit masks + lists).
// ROUTE 1: general (any planes of either eye, byte or bit masks, optional lists).
// INT: integer column tables (int4 per d) instead of FP64 shifts.
// Persistent CTAs walk the rows; the shift table is staged once per CTA. Shared memory per
// row: the source row (R, G, B, depth) and two key rows, 12 bytes per pixel. Phases use a
// lane-interleaved mapping (lane l handles pixel base + l): shared-memory accesses are
// consecutive across the warp, a warp's 32 output bytes per plane are one 32-byte sector
// store, and 32 pixels' damage flags are one __ballot_sync word.
// WIDE: rows wider than a CTA's shared memory (w > dibr_max_width()): the source row is
// read straight from global memory (L1-cached) and the two key rows live in a global
// per-CTA slot (wide_keys + blockIdx.x * 2 * wpad); the splat uses global atomicMax (same
// order-independent maximum). Same output bytes, masks and lists.
template <int ROUTE, bool INT, bool WIDE = false>
__global__ void __launch_bounds__(256) k_dibr(const uint8_t* __restrict__ R,
                                              const uint8_t* __restrict__ G,
                                              const uint8_t* __restrict__ B,
                                              const uint8_t* __restrict__ D, int pitch, int w, int h,
                                              const double* __restrict__ shift_g,
                                              const int4* __restrict__ cols_g, int backward,
                                              EyeOut L, EyeOut Rt, int ya, int yb,
                                              uint32_t* __restrict__ wide_keys = nullptr) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ double s_shift[INT ? 1 : 256];
    __shared__ int4 s_cols[INT ? 256 : 1];
    const int wpad = (w + 15) & ~15;
    const int nvec = wpad >> 4;
    uint8_t* s_src = smem;  // [4][wpad]: R, G, B, depth
    uint32_t* keyL = WIDE ? wide_keys + static_cast<size_t>(blockIdx.x) * 2 * wpad
                          : reinterpret_cast<uint32_t*>(smem + 4 * wpad);
    uint32_t* keyR = keyL + wpad;
    const int tid = threadIdx.x, lane = tid & 31;
    const uint8_t* s_r = s_src;
    const uint8_t* s_g = s_src + wpad;
    const uint8_t* s_b = s_src + 2 * wpad;
    const uint8_t* s_d = s_src + 3 * wpad;

    if (INT) {
        for (int i = tid; i < 256; i += blockDim.x) s_cols[i] = cols_g[i];
    } else {
        for (int i = tid; i < 256; i += blockDim.x) s_shift[i] = shift_g[i];
    }
    // destination columns of source x: a = trunc(x + sigma) (left eye / backward right),
    // b = trunc(x - sigma) (right eye / backward left); -1 when outside [0, w)
    auto cols = [&](int x, int& a, int& b) {
        const int d = s_d[x];
        if (INT) {
            const int4 t = s_cols[d];
            a = col_int(t.x, t.z, x);
            b = col_int(t.y, t.w, x);
            a = static_cast<unsigned>(a) < static_cast<unsigned>(w) ? a : -1;
            b = static_cast<unsigned>(b) < static_cast<unsigned>(w) ? b : -1;
        } else {
            const double sigma = s_shift[d];
            const double xd = exact_xd(x);
            a = trunc_col(__dadd_rn(xd, sigma), w);
            b = trunc_col(__dsub_rn(xd, sigma), w);
        }
    };

    for (int y = ya + static_cast<int>(blockIdx.x); y < yb; y += gridDim.x) {
        __syncthreads();  // previous row's readers are done with shared memory
        const size_t row = static_cast<size_t>(y) * pitch;
        if (WIDE) {
            s_r = R + row;
            s_g = G + row;
            s_b = B + row;
            s_d = D + row;
        } else {
            const uint8_t* planes_in[4] = {R + row, G + row, B + row, D + row};
#pragma unroll
            for (int pl = 0; pl < 4; ++pl)
                for (int v = tid; v < nvec; v += blockDim.x)
                    reinterpret_cast<uint4*>(s_src + pl * wpad)[v] =
                        __ldg(reinterpret_cast<const uint4*>(planes_in[pl]) + v);
        }
        if (!backward) {
            const uint4 z = make_uint4(0, 0, 0, 0);
            for (int c = tid; c < 2 * wpad / 4; c += blockDim.x) reinterpret_cast<uint4*>(keyL)[c] = z;
        }
        __syncthreads();

        if (!backward) {
            // Splat: shared atomicMax of (d+1) << 22 | (0x3FFFFF - x) into the destination
            // slot; the maximum (largest depth, then smallest column, dibr.cpp:88-99) does not
            // depend on the order the atomics land in. Left eye splats to trunc(p.right),
            // right eye to trunc(p.left).
            for (int x = tid; x < w; x += blockDim.x) {
                int a, b;
                cols(x, a, b);
                const unsigned key = (static_cast<unsigned>(s_d[x] + 1) << 22) | (kXMask - x);
                if (a >= 0) atomicMax(&keyL[a], key);
                if (b >= 0) atomicMax(&keyR[b], key);
            }
            __syncthreads();
        }

        const uint32_t row_base = static_cast<uint32_t>(y) * static_cast<uint32_t>(w);
        const size_t lrow = static_cast<size_t>(y) * L.pitch;
        const size_t rrow = static_cast<size_t>(y) * Rt.pitch;
        for (int xb = tid - lane; xb < w; xb += blockDim.x) {
            const int x = xb + lane;
            const bool act = x < w;
            int sl = -1, sr = -1;
            if (act) {
                if (backward) {
                    int a, b;
                    cols(x, a, b);
                    sl = b >= 0 ? b : x;  // trunc(p.left)
                    sr = a >= 0 ? a : x;  // trunc(p.right)
                } else {
                    // (WIDE: the keys were formed by L2 atomics; bypass L1, which may hold
                    // this slot's lines from the previous row)
                    const unsigned kl = WIDE ? __ldcg(keyL + x) : keyL[x];
                    const unsigned kr = WIDE ? __ldcg(keyR + x) : keyR[x];
                    sl = kl ? static_cast<int>(kXMask - (kl & kXMask)) : -1;
                    sr = kr ? static_cast<int>(kXMask - (kr & kXMask)) : -1;
                }
                if (ROUTE == 0) {
                    L.plane[0][lrow + x] = sl >= 0 ? s_r[sl] : 0;
                    Rt.plane[1][rrow + x] = sr >= 0 ? s_g[sr] : 0;
                    Rt.plane[2][rrow + x] = sr >= 0 ? s_b[sr] : 0;
                } else {
                    if (L.plane[0]) L.plane[0][lrow + x] = sl >= 0 ? s_r[sl] : 0;
                    if (L.plane[1]) L.plane[1][lrow + x] = sl >= 0 ? s_g[sl] : 0;
                    if (L.plane[2]) L.plane[2][lrow + x] = sl >= 0 ? s_b[sl] : 0;
                    if (Rt.plane[0]) Rt.plane[0][rrow + x] = sr >= 0 ? s_r[sr] : 0;
                    if (Rt.plane[1]) Rt.plane[1][rrow + x] = sr >= 0 ? s_g[sr] : 0;
                    if (Rt.plane[2]) Rt.plane[2][rrow + x] = sr >= 0 ? s_b[sr] : 0;
                    if (L.mask_bytes) L.mask_bytes[static_cast<size_t>(y) * L.mask_pitch + x] = sl < 0;
                    if (Rt.mask_bytes) Rt.mask_bytes[static_cast<size_t>(y) * Rt.mask_pitch + x] = sr < 0;
                }
            }
            if (backward) continue;  // uniform: no damage, no masks or lists to write
            const unsigned mL = __ballot_sync(0xFFFFFFFFu, act && sl < 0);
            const unsigned mR = __ballot_sync(0xFFFFFFFFu, act && sr < 0);
            if (lane == 0) {
                if (L.mask_bits) L.mask_bits[static_cast<size_t>(y) * L.mask_pitch + (xb >> 5)] = mL;
                if (Rt.mask_bits) Rt.mask_bits[static_cast<size_t>(y) * Rt.mask_pitch + (xb >> 5)] = mR;
            }
            if (L.list && mL) {
                uint32_t start = 0;
                if (lane == 0) start = atomicAdd(L.count, static_cast<uint32_t>(__popc(mL)));
                start = __shfl_sync(0xFFFFFFFFu, start, 0);
                if ((mL >> lane) & 1u) L.list[start + __popc(mL & ((1u << lane) - 1u))] = row_base + x;
            }
            if (Rt.list && mR) {
                uint32_t start = 0;
                if (lane == 0) start = atomicAdd(Rt.count, static_cast<uint32_t>(__popc(mR)));
                start = __shfl_sync(0xFFFFFFFFu, start, 0);
                if ((mR >> lane) & 1u) Rt.list[start + __popc(mR & ((1u << lane) - 1u))] = row_base + x;
            }
        }
    }
}

// Fused DIBR + anaglyph with integer column tables (the default route). Same semantics as
// k_dibr<0, true>, organised around shared memory so that every phase is conflict-free and
// HBM sees only 16-byte accesses:
//   stage    R, G, B, depth rows in with 16-byte loads; keys zeroed with 16-byte stores;
//   splat    lane-interleaved sources (lane l -> x = base + l): the destinations of a warp
//            are consecutive, so the shared atomicMax on the packed key hits distinct banks;
//            a single atomic pass (the maximum is order-independent);
//   resolve  lane-interleaved destinations: winner -> gathered bytes into output staging
//            rows, damage flags by ballot (one mask word and one list atomic per warp);
//   store    staging rows out with 16-byte stores.
// Requires 16-byte aligned output planes and pitches (the engine's arena guarantees it);
// bytes past w inside the pitch are written 0.
template <bool BACKWARD>
__global__ void __launch_bounds__(256) k_dibr_ana(const uint8_t* __restrict__ R,
                                                  const uint8_t* __restrict__ G,
                                                  const uint8_t* __restrict__ B,
                                                  const uint8_t* __restrict__ D, int pitch, int w,
                                                  int h, const int4* __restrict__ cols_g, EyeOut L,
                                                  EyeOut Rt, int ya, int yb) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ int4 s_cols[256];
    const int wpad = (w + 15) & ~15;
    const int nvec = wpad >> 4;
    uint8_t* s_r = smem;
    uint8_t* s_g = smem + wpad;
    uint8_t* s_b = smem + 2 * wpad;
    uint8_t* s_d = smem + 3 * wpad;
    uint8_t* o_r = smem + 4 * wpad;
    uint8_t* o_g = smem + 5 * wpad;
    uint8_t* o_b = smem + 6 * wpad;
    uint32_t* keyL = reinterpret_cast<uint32_t*>(smem + 7 * wpad + (16 - (7 * wpad) % 16) % 16);
    uint32_t* keyR = keyL + wpad;
    const int tid = threadIdx.x, lane = tid & 31;
    for (int i = tid; i < 256; i += blockDim.x) s_cols[i] = cols_g[i];

    for (int y = ya + static_cast<int>(blockIdx.x); y < yb; y += gridDim.x) {
        __syncthreads();
        const size_t row = static_cast<size_t>(y) * pitch;
        for (int v = tid; v < nvec; v += blockDim.x) {
            reinterpret_cast<uint4*>(s_r)[v] = __ldg(reinterpret_cast<const uint4*>(R + row) + v);
            reinterpret_cast<uint4*>(s_g)[v] = __ldg(reinterpret_cast<const uint4*>(G + row) + v);
            reinterpret_cast<uint4*>(s_b)[v] = __ldg(reinterpret_cast<const uint4*>(B + row) + v);
            reinterpret_cast<uint4*>(s_d)[v] = __ldg(reinterpret_cast<const uint4*>(D + row) + v);
        }
        if (!BACKWARD) {
            const uint4 z = make_uint4(0, 0, 0, 0);
            for (int v = tid; v < 2 * wpad / 4; v += blockDim.x) reinterpret_cast<uint4*>(keyL)[v] = z;
        }
        __syncthreads();
        if (!BACKWARD) {
            for (int x = tid; x < w; x += blockDim.x) {
                const int d = s_d[x];
                const int4 t = s_cols[d];
                const int a = col_int(t.x, t.z, x), b = col_int(t.y, t.w, x);
                const unsigned key = (static_cast<unsigned>(d + 1) << 22) | (kXMask - x);
                if (static_cast<unsigned>(a) < static_cast<unsigned>(w)) atomicMax(&keyL[a], key);
                if (static_cast<unsigned>(b) < static_cast<unsigned>(w)) atomicMax(&keyR[b], key);
            }
            __syncthreads();
        }
        const uint32_t row_base = static_cast<uint32_t>(y) * static_cast<uint32_t>(w);
        for (int xb = tid - lane; xb < wpad; xb += blockDim.x) {
            const int x = xb + lane;
            const bool act = x < w;
            int sl = -1, sr = -1;
            if (act) {
                if (BACKWARD) {
                    const int4 t = s_cols[s_d[x]];
                    const int a = col_int(t.x, t.z, x), b = col_int(t.y, t.w, x);
                    sl = static_cast<unsigned>(b) < static_cast<unsigned>(w) ? b : x;
                    sr = static_cast<unsigned>(a) < static_cast<unsigned>(w) ? a : x;
                } else {
                    const unsigned kl = keyL[x], kr = keyR[x];
                    sl = kl ? static_cast<int>(kXMask - (kl & kXMask)) : -1;
                    sr = kr ? static_cast<int>(kXMask - (kr & kXMask)) : -1;
                }
            }
            if (x < wpad) {  // (the last warp of a row may run past the padded width)
                o_r[x] = sl >= 0 ? s_r[sl] : 0;
                o_g[x] = sr >= 0 ? s_g[sr] : 0;
                o_b[x] = sr >= 0 ? s_b[sr] : 0;
            }
            if (BACKWARD || xb >= w) continue;  // (warp-uniform)
            const unsigned mL = __ballot_sync(0xFFFFFFFFu, act && sl < 0);
            const unsigned mR = __ballot_sync(0xFFFFFFFFu, act && sr < 0);
            if (lane == 0) {
                L.mask_bits[static_cast<size_t>(y) * L.mask_pitch + (xb >> 5)] = mL;
                Rt.mask_bits[static_cast<size_t>(y) * Rt.mask_pitch + (xb >> 5)] = mR;
            }
            if (mL) {
                uint32_t start = 0;
                if (lane == 0) start = atomicAdd(L.count, static_cast<uint32_t>(__popc(mL)));
                start = __shfl_sync(0xFFFFFFFFu, start, 0);
                if ((mL >> lane) & 1u) L.list[start + __popc(mL & ((1u << lane) - 1u))] = row_base + x;
            }
            if (mR) {
                uint32_t start = 0;
                if (lane == 0) start = atomicAdd(Rt.count, static_cast<uint32_t>(__popc(mR)));
                start = __shfl_sync(0xFFFFFFFFu, start, 0);
                if ((mR >> lane) & 1u) Rt.list[start + __popc(mR & ((1u << lane) - 1u))] = row_base + x;
            }
        }
        __syncthreads();
        for (int v = tid; v < nvec; v += blockDim.x) {
            const size_t o = static_cast<size_t>(16 * v);
            *reinterpret_cast<uint4*>(L.plane[0] + static_cast<size_t>(y) * L.pitch + o) =
                reinterpret_cast<const uint4*>(o_r)[v];
            *reinterpret_cast<uint4*>(Rt.plane[1] + static_cast<size_t>(y) * Rt.pitch + o) =
                reinterpret_cast<const uint4*>(o_g)[v];
            *reinterpret_cast<uint4*>(Rt.plane[2] + static_cast<size_t>(y) * Rt.pitch + o) =
                reinterpret_cast<const uint4*>(o_b)[v];
        }
    }
}

// Shared-window loads of arrays the splat only reads (not volatile: the compiler may hoist
// them across the reductions, which touch only the key rows; the barriers order everything
// else) and the z-buffer reduction itself (its result is read after a barrier).
__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) {
    uint32_t v;
    asm("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void red_max_shared(uint32_t addr, uint32_t v) {
    asm volatile("red.shared.max.u32 [%0], %1;" ::"r"(addr), "r"(v));
}

// Forward DIBR + anaglyph, quad version (the default route): the same z-buffer and output
// bytes as k_dibr_ana<false> with far fewer instructions per pixel.
//   stage    lane-contiguous 4-pixel words of R, G, B, depth (128-byte warp requests); the
//            source row is kept as one packed 0x00BBGGRR word per pixel, so a gather is one
//            LDS.32 for all channels; slot wpad is a zero word (unsplatted destinations);
//   splat    lane-interleaved sources (consecutive destinations across the warp:
//            conflict-free shared atomicMax on the packed key). Columns: the integer tables
//            give col = x + off + (x >= X), 0 at x == z; every X < w and z lies below
//            x_safe (the CTA's max over the 256 depths), so for x >= x_safe both eyes'
//            columns are x + off2[d] (off2 = off + (X < w)), formed by one add on a packed
//            pair of biased 16-bit offsets; x < x_safe (a few dozen pixels at the left edge)
//            takes the exact general form;
//   resolve  each thread owns 4 consecutive destinations: one 16-byte key load per eye, a
//            branch-free gather per pixel (index = ~key & 0x3FFFFF, clamped to the zero slot),
//            the output bytes assembled with byte permutes and written with one 4-byte store
//            per plane (128-byte warp stores); 4-bit damage nibbles are merged into 32-bit
//            mask words over 8-lane groups; one list atomic per warp and eye.
// MODE 0: anaglyph planes (left R, right G/B); MODE 1: all six eye planes (HSBS / FSBS
// routes), same z-buffer, masks and lists.
// ILV (MODE 0, w % 16 == 0): the source is one RGB-interleaved image (R = its base, row
// stride ipitch; the PPM payload as uploaded) and the anaglyph is written interleaved
// (L.plane[0] = its base, row stride L.pitch): the file / interleaved-video path with no
// separate (de)interleave pass.
template <int MODE, bool ILV = false>
__global__ void __launch_bounds__(256) k_dibr_quad(const uint8_t* __restrict__ R,
                                                   const uint8_t* __restrict__ G,
                                                   const uint8_t* __restrict__ B,
                                                   const uint8_t* __restrict__ D, int pitch,
                                                   int w, int h, const int4* __restrict__ cols_g,
                                                   EyeOut L, EyeOut Rt, int ya, int yb, int ipitch) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ int4 s_cols[256];
    __shared__ uint32_t s_off[256];
    __shared__ int s_xsafe;
    const int wpad = (w + 15) & ~15;
    const int nq = wpad >> 2;  // quads
    uint32_t* s_rgb = reinterpret_cast<uint32_t*>(smem);      // [wpad + 4]: slot wpad = 0
    uint32_t* keyL = s_rgb + wpad + 4;                         // [wpad + 4]: slot w = dump
    uint32_t* keyR = keyL + wpad + 4;                          // [wpad + 4]
    uint8_t* s_d = reinterpret_cast<uint8_t*>(keyR + wpad + 4);  // [wpad]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_xsafe = 0;
    if (tid < 4) s_rgb[wpad + tid] = 0u;
    __syncthreads();
    for (int i = tid; i < 256; i += blockDim.x) {
        const int4 c = cols_g[i];
        s_cols[i] = c;
        const int offP = static_cast<short>(c.x & 0xFFFF), XP = static_cast<int>(static_cast<unsigned>(c.x) >> 16);
        const int offM = static_cast<short>(c.y & 0xFFFF), XM = static_cast<int>(static_cast<unsigned>(c.y) >> 16);
        const int offP2 = offP + (XP < w ? 1 : 0), offM2 = offM + (XM < w ? 1 : 0);
        s_off[i] = (static_cast<uint32_t>(offP2 + 0x8000) & 0xFFFFu) | (static_cast<uint32_t>(offM2 + 0x8000) << 16);
        int xs = 0;
        if (XP < w) xs = max(xs, XP);
        if (XM < w) xs = max(xs, XM);
        if (c.z >= 0) xs = max(xs, c.z + 1);
        if (c.w >= 0) xs = max(xs, c.w + 1);
        // the packed add must not carry between the 16-bit lanes: x + off2 + 0x8000 < 2^16
        if (offP2 + w >= 0x8000 || offM2 + w >= 0x8000) xs = w;
        if (xs) atomicMax(&s_xsafe, xs);
    }
    const int nqr = (nq + 31) & ~31;
    const uint32_t wz = static_cast<uint32_t>(wpad);
    const uint32_t kinit = kXMask - wz;
    // 32-bit shared-window addresses, formed once (the splat's loads and atomics use them
    // directly: no generic-to-shared conversion inside the loop)
    const uint32_t sa_d = static_cast<uint32_t>(__cvta_generic_to_shared(s_d));
    const uint32_t sa_off = static_cast<uint32_t>(__cvta_generic_to_shared(s_off));
    const uint32_t sa_kl = static_cast<uint32_t>(__cvta_generic_to_shared(keyL));
    const uint32_t sa_kr = static_cast<uint32_t>(__cvta_generic_to_shared(keyR));
    const uint32_t uw = static_cast<uint32_t>(w);

    // The first kPre quads per thread of the NEXT row are loaded into registers while this row
    // is splatted and resolved (the row loads otherwise stall every row on HBM/L2 latency);
    // quads beyond kPre * blockDim.x (rows wider than 4096 px) load when staged.
    constexpr int kPre = 4;
    uint32_t pre[kPre][4];
    auto load_quad = [&](int yy, int q, uint32_t (&v)[4]) {
        v[3] = __ldg(reinterpret_cast<const uint32_t*>(D + static_cast<size_t>(yy) * pitch) + q);
        if (ILV) {
            const uint32_t* src = reinterpret_cast<const uint32_t*>(R + static_cast<size_t>(yy) * ipitch) + 3 * q;
            v[0] = __ldg(src);
            v[1] = __ldg(src + 1);
            v[2] = __ldg(src + 2);
        } else {
            const size_t rr = static_cast<size_t>(yy) * pitch;
            v[0] = __ldg(reinterpret_cast<const uint32_t*>(R + rr) + q);
            v[1] = __ldg(reinterpret_cast<const uint32_t*>(G + rr) + q);
            v[2] = __ldg(reinterpret_cast<const uint32_t*>(B + rr) + q);
        }
    };
    auto prefetch = [&](int yy) {
        if (yy >= yb) return;
#pragma unroll
        for (int k = 0; k < kPre; ++k) {
            const int q = tid + k * static_cast<int>(blockDim.x);
            if (q < nq) load_quad(yy, q, pre[k]);
        }
    };
    // packed 0x00BBGGRR words of 4 pixels (+ their depth bytes) into the row's shared arrays
    auto stage = [&](int q, const uint32_t (&v)[4]) {
        uint4 px;
        if (ILV) {  // 4 interleaved pixels = 3 words r0 g0 b0 r1 | g1 b1 r2 g2 | b2 r3 g3 b3
            px.x = v[0] & 0x00FFFFFFu;
            px.y = __byte_perm(v[0], v[1], 0x0543) & 0x00FFFFFFu;
            px.z = __byte_perm(v[1], v[2], 0x0432) & 0x00FFFFFFu;
            px.w = v[2] >> 8;
        } else {
            const uint32_t rg_lo = __byte_perm(v[0], v[1], 0x5140), rg_hi = __byte_perm(v[0], v[1], 0x7362);
            px.x = __byte_perm(rg_lo, v[2], 0x0410) & 0x00FFFFFFu;  // r0 g0 b0 0
            px.y = __byte_perm(rg_lo, v[2], 0x0532) & 0x00FFFFFFu;
            px.z = __byte_perm(rg_hi, v[2], 0x0610) & 0x00FFFFFFu;
            px.w = __byte_perm(rg_hi, v[2], 0x0732) & 0x00FFFFFFu;
        }
        reinterpret_cast<uint4*>(s_rgb)[q] = px;
        reinterpret_cast<uint32_t*>(s_d)[q] = v[3];
    };
    prefetch(ya + static_cast<int>(blockIdx.x));

    for (int y = ya + static_cast<int>(blockIdx.x); y < yb; y += gridDim.x) {
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kPre; ++k) {
            const int q = tid + k * static_cast<int>(blockDim.x);
            if (q < nq) stage(q, pre[k]);
        }
        for (int q = tid + kPre * static_cast<int>(blockDim.x); q < nq; q += blockDim.x) {
            uint32_t v[4];
            load_quad(y, q, v);
            stage(q, v);
        }
        // unsplatted destinations keep kinit: depth field 0 (damaged), and its gather index
        // ~kinit & kXMask is the zero slot wz, so the resolve needs no branch or clamp
        for (int q = tid; q < nq + 1; q += blockDim.x) {
            reinterpret_cast<uint4*>(keyL)[q] = make_uint4(kinit, kinit, kinit, kinit);
            reinterpret_cast<uint4*>(keyR)[q] = make_uint4(kinit, kinit, kinit, kinit);
        }
        prefetch(y + static_cast<int>(gridDim.x));
        __syncthreads();
        const int xsafe = s_xsafe;
        // destinations outside [0, w) go to the dump slot w (unsigned min), so every source
        // does both atomics unconditionally. Left edge (x < xsafe): the exact general form.
        int x = tid;
        for (; x < xsafe && x < w; x += blockDim.x) {
            const int d = s_d[x];
            const unsigned key = (static_cast<unsigned>(d + 1) << 22) | (kXMask - x);
            const int4 t = s_cols[d];
            const uint32_t a = min(static_cast<uint32_t>(col_int(t.x, t.z, x)), uw);
            const uint32_t b = min(static_cast<uint32_t>(col_int(t.y, t.w, x)), uw);
            red_max_shared(sa_kl + 4 * a, key);
            red_max_shared(sa_kr + 4 * b, key);
        }
        // the rest: both columns from one add on the packed biased offsets; two sources per
        // iteration, so their dependent loads (depth, then offsets) overlap
        const int step = static_cast<int>(blockDim.x);
        auto splat_fast = [&](int xx) {
            const uint32_t d = lds_u8(sa_d + xx);
            const uint32_t key = ((d + 1u) << 22) | (kXMask - static_cast<uint32_t>(xx));
            const uint32_t ab = lds_u32(sa_off + 4 * d) + static_cast<uint32_t>(xx) * 0x10001u;
            red_max_shared(sa_kl + 4 * min((ab & 0xFFFFu) - 0x8000u, uw), key);
            red_max_shared(sa_kr + 4 * min((ab >> 16) - 0x8000u, uw), key);
        };
        for (; x + step < w; x += 2 * step) {
            const uint32_t d0 = lds_u8(sa_d + x), d1 = lds_u8(sa_d + x + step);
            const uint32_t ab0 = lds_u32(sa_off + 4 * d0) + static_cast<uint32_t>(x) * 0x10001u;
            const uint32_t ab1 = lds_u32(sa_off + 4 * d1) + static_cast<uint32_t>(x + step) * 0x10001u;
            const uint32_t k0 = ((d0 + 1u) << 22) | (kXMask - static_cast<uint32_t>(x));
            const uint32_t k1 = ((d1 + 1u) << 22) | (kXMask - static_cast<uint32_t>(x + step));
            red_max_shared(sa_kl + 4 * min((ab0 & 0xFFFFu) - 0x8000u, uw), k0);
            red_max_shared(sa_kr + 4 * min((ab0 >> 16) - 0x8000u, uw), k0);
            red_max_shared(sa_kl + 4 * min((ab1 & 0xFFFFu) - 0x8000u, uw), k1);
            red_max_shared(sa_kr + 4 * min((ab1 >> 16) - 0x8000u, uw), k1);
        }
        if (x < w) splat_fast(x);
        __syncthreads();
        const uint32_t row_base = static_cast<uint32_t>(y) * static_cast<uint32_t>(w);
        for (int qb = warp * 32; qb < nqr; qb += blockDim.x) {
            const int q = qb + lane;
            const int x0 = 4 * q;
            unsigned mL = 0, mR = 0;
            if (q < nq) {
                const uint4 kl = reinterpret_cast<const uint4*>(keyL)[q];
                const uint4 kr = reinterpret_cast<const uint4*>(keyR)[q];
                const uint32_t kla[4] = {kl.x, kl.y, kl.z, kl.w}, kra[4] = {kr.x, kr.y, kr.z, kr.w};
                uint32_t vl[4], vr[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    // the winning source column, or the zero slot for an unsplatted destination
                    vl[k] = s_rgb[~kla[k] & kXMask];
                    vr[k] = s_rgb[~kra[k] & kXMask];
                    mL |= (kla[k] < 0x400000u ? 1u : 0u) << k;
                    mR |= (kra[k] < 0x400000u ? 1u : 0u) << k;
                }
                auto bytes = [](uint32_t v0, uint32_t v1, uint32_t v2, uint32_t v3, unsigned sel) {
                    return __byte_perm(__byte_perm(v0, v1, sel), __byte_perm(v2, v3, sel), 0x5410);
                };
                const uint32_t oR = bytes(vl[0], vl[1], vl[2], vl[3], 0x0040);
                const uint32_t oG = bytes(vr[0], vr[1], vr[2], vr[3], 0x0051);
                const uint32_t oB = bytes(vr[0], vr[1], vr[2], vr[3], 0x0062);
                // pixels x >= w (never a destination except the dump slot) have their mask
                // bits dropped below instead of testing x per pixel
                if (x0 + 4 > w) {
                    const unsigned valid = x0 >= w ? 0u : (1u << (w - x0)) - 1u;
                    mL &= valid;
                    mR &= valid;
                }
                // never write past w: in the direct-FSBS route the left eye's row continues
                // with the right eye's pixels
                const size_t lo = static_cast<size_t>(y) * L.pitch, ro = static_cast<size_t>(y) * Rt.pitch;
                auto put = [&](uint8_t* plane, size_t row, uint32_t v) {
                    if (x0 + 4 <= w) {
                        reinterpret_cast<uint32_t*>(plane + row)[q] = v;
                    } else {
                        for (int k = 0; x0 + k < w; ++k) plane[row + x0 + k] = static_cast<uint8_t>(v >> (8 * k));
                    }
                };
                if (ILV) {  // w % 16 == 0: whole quads; 12 interleaved bytes
                    const uint32_t rg0 = __byte_perm(oR, oG, 0x5140), rg1 = __byte_perm(oR, oG, 0x7362);
                    uint32_t* dst = reinterpret_cast<uint32_t*>(L.plane[0] + lo) + 3 * q;
                    dst[0] = __byte_perm(rg0, oB, 0x2410);                              // R0 G0 B0 R1
                    dst[1] = __byte_perm(__byte_perm(rg0, oB, 0x5353), rg1, 0x5410);   // G1 B1 R2 G2
                    dst[2] = __byte_perm(rg1, oB, 0x7326);                              // B2 R3 G3 B3
                } else if (x0 < w) {
                    put(L.plane[0], lo, oR);
                    put(Rt.plane[1], ro, oG);
                    put(Rt.plane[2], ro, oB);
                    if (MODE == 1) {
                        put(L.plane[1], lo, bytes(vl[0], vl[1], vl[2], vl[3], 0x0051));
                        put(L.plane[2], lo, bytes(vl[0], vl[1], vl[2], vl[3], 0x0062));
                        put(Rt.plane[0], ro, bytes(vr[0], vr[1], vr[2], vr[3], 0x0040));
                    }
                }
            }
            // mask words: 8 lanes x 4 pixels = 32 pixels; word index q >> 3
            unsigned wL = mL << (4 * (lane & 7)), wR = mR << (4 * (lane & 7));
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) {
                wL |= __shfl_xor_sync(0xFFFFFFFFu, wL, o);
                wR |= __shfl_xor_sync(0xFFFFFFFFu, wR, o);
            }
            const int mwords = (w + 31) >> 5;
            if ((lane & 7) == 0 && (q >> 3) < mwords) {
                L.mask_bits[static_cast<size_t>(y) * L.mask_pitch + (q >> 3)] = wL;
                Rt.mask_bits[static_cast<size_t>(y) * Rt.mask_pitch + (q >> 3)] = wR;
            }
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                unsigned m = e ? mR : mL;
                const EyeOut& eo = e ? Rt : L;
                const int n = __popc(m);
                if (!__any_sync(0xFFFFFFFFu, n)) continue;
                int incl = n;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                    if (lane >= o) incl += v;
                }
                const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
                uint32_t start = 0;
                if (lane == 31) start = atomicAdd(eo.count, static_cast<uint32_t>(total));
                start = __shfl_sync(0xFFFFFFFFu, start, 31);
                uint32_t pos = start + static_cast<uint32_t>(incl - n);
                while (m) {
                    const int k = __ffs(m) - 1;
                    m &= m - 1;
                    eo.list[pos++] = row_base + static_cast<uint32_t>(x0 + k);
                }
            }
        }
    }
}

// Byte mask -> damaged list (stage-level inpaint entry point).
__global__ void k_mask_to_list(const uint8_t* __restrict__ mask, int mpitch, int w, int h,
                               uint32_t* list, uint32_t* count, uint32_t* bits, int mwords) {
    const int lane = threadIdx.x & 31;
    const int y = blockIdx.y;
    const int x0 = (blockIdx.x * blockDim.x + threadIdx.x) * 16;
    unsigned m = 0;
    for (int k = 0; k < 16; ++k)
        if (x0 + k < w && mask[static_cast<size_t>(y) * mpitch + x0 + k]) m |= 1u << k;
    // the same damage as 32-pixel bit words (two threads per word), the inpaint's input
    const unsigned hi = __shfl_down_sync(0xFFFFFFFFu, m, 1);
    if (bits && !(lane & 1) && x0 < w) bits[static_cast<size_t>(y) * mwords + (x0 >> 5)] = m | (hi << 16);
    append_list(list, count, m, static_cast<uint32_t>(y) * w + x0, lane);
}

// HSBS squeeze (stereo_format.cpp:47-71): (a + b + 1) / 2 over column pairs; left eye to
// [0, w/2), right eye to [w/2, w). Thread = 16 output pixels of one half.
__global__ void k_hsbs(const uint8_t* __restrict__ l0, const uint8_t* __restrict__ l1,
                       const uint8_t* __restrict__ l2, const uint8_t* __restrict__ r0,
                       const uint8_t* __restrict__ r1, const uint8_t* __restrict__ r2,
                       int pitch, int w, uint8_t* o0, uint8_t* o1, uint8_t* o2, int opitch) {
    const int y = blockIdx.y;
    const int hw = w / 2;
    const int nchunk = (hw + 15) / 16;
    const int item = blockIdx.x * blockDim.x + threadIdx.x;
    if (item >= 2 * nchunk) return;
    const int eye = item / nchunk;
    const int x0 = (item % nchunk) * 16;
    const uint8_t* src[3] = {eye ? r0 : l0, eye ? r1 : l1, eye ? r2 : l2};
    uint8_t* dst[3] = {o0, o1, o2};
    for (int ch = 0; ch < 3; ++ch) {
        const uint8_t* s = src[ch] + static_cast<size_t>(y) * pitch;
        uint8_t v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const int x = min(x0 + k, hw - 1);
            v[k] = static_cast<uint8_t>((s[2 * x] + s[2 * x + 1] + 1u) / 2u);
        }
        store16(dst[ch] + static_cast<size_t>(y) * opitch + eye * hw + x0, v, x0, hw);
    }
}

// HSBS, 16 output pixels per thread from two 16-byte loads per plane: the column-pair
// rounded-up mean (a + b + 1) / 2 of 4 pairs at a time with SWAR byte arithmetic,
// (a | b) - ((a ^ b) >> 1) on the even/odd bytes gathered by PRMT (exact per byte).
__device__ __forceinline__ uint32_t pair_avg(uint32_t w0, uint32_t w1) {
    const uint32_t ev = __byte_perm(w0, w1, 0x6420), od = __byte_perm(w0, w1, 0x7531);
    return (ev | od) - (((ev ^ od) & 0xFEFEFEFEu) >> 1);
}

__global__ void k_hsbs16(const uint8_t* __restrict__ l0, const uint8_t* __restrict__ l1,
                         const uint8_t* __restrict__ l2, const uint8_t* __restrict__ r0,
                         const uint8_t* __restrict__ r1, const uint8_t* __restrict__ r2, int pitch,
                         int w, int h, uint8_t* o0, uint8_t* o1, uint8_t* o2, int opitch) {
    const int hw = w / 2;
    const int nchunk = hw / 16;  // full 16-pixel chunks per eye (hw % 16 == 0 here)
    const long long item = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long per_row = 2LL * 3 * nchunk;
    if (item >= per_row * h) return;
    const int y = static_cast<int>(item / per_row);
    int rem = static_cast<int>(item % per_row);
    const int eye = rem / (3 * nchunk);
    rem -= eye * 3 * nchunk;
    const int ch = rem / nchunk, c = rem - ch * nchunk;
    const uint8_t* src = (ch == 0 ? (eye ? r0 : l0) : ch == 1 ? (eye ? r1 : l1) : (eye ? r2 : l2)) +
                         static_cast<size_t>(y) * pitch + 32 * c;
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(src));
    const uint4 b = __ldg(reinterpret_cast<const uint4*>(src) + 1);
    uint8_t* dst = (ch == 0 ? o0 : ch == 1 ? o1 : o2) + static_cast<size_t>(y) * opitch + eye * hw + 16 * c;
    *reinterpret_cast<uint4*>(dst) =
        make_uint4(pair_avg(a.x, a.y), pair_avg(a.z, a.w), pair_avg(b.x, b.y), pair_avg(b.z, b.w));
}

}  // namespace

int dibr_wide_slots() { return 2 * sm_count(); }

size_t dibr_wide_key_words(int w) {
    if (w <= dibr_max_width()) return 0;
    return static_cast<size_t>(dibr_wide_slots()) * 2 * static_cast<size_t>((w + 15) & ~15);
}

cudaError_t dibr(const uint8_t* r, const uint8_t* g, const uint8_t* b, const uint8_t* depth,
                 Geom gm, const double* shift, const int4* cols, bool backward, EyeOut left,
                 EyeOut right, cudaStream_t st, int ya, int yb, uint32_t* wide_keys, int src_ipitch) {
    if (left.stride == 3) {
        // interleaved source + interleaved anaglyph: the quad kernel's ILV variant only
        const bool ok = cols && !backward && gm.w % 16 == 0 && left.plane[0] && right.plane[1] &&
                        right.plane[2] && left.mask_bits && right.mask_bits && left.list && right.list &&
                        static_cast<size_t>((gm.w + 15) & ~15) * 13 + 48 <= kDibrMaxSmem && src_ipitch > 0;
        if (!ok) return cudaErrorInvalidValue;
    }
    if (yb < 0 || yb > gm.h) yb = gm.h;
    if (yb <= ya) return cudaSuccess;
    const int rows = yb - ya;
    const int wpad = (gm.w + 15) & ~15;
    const size_t smem = static_cast<size_t>(wpad) * (backward ? 4 : 12);
    constexpr size_t kMax = kDibrMaxSmem;
    static std::atomic<unsigned long long> configured{0};
    once_per_device(configured, [] {
        cudaFuncSetAttribute(k_dibr<0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMax);
        cudaFuncSetAttribute(k_dibr<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMax);
        cudaFuncSetAttribute(k_dibr<0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMax);
        cudaFuncSetAttribute(k_dibr<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMax);
    });
    if (smem > kMax) {
        // rows wider than shared memory: global per-CTA key slots (dibr_wide_key_words)
        if (!wide_keys) return cudaErrorInvalidValue;
        void (*wk)(const uint8_t*, const uint8_t*, const uint8_t*, const uint8_t*, int, int, int,
                   const double*, const int4*, int, EyeOut, EyeOut, int, int, uint32_t*) =
            cols ? k_dibr<1, true, true> : k_dibr<1, false, true>;
        note_launch(st);
        wk<<<min(rows, dibr_wide_slots()), 256, 0, st>>>(r, g, b, depth, gm.pitch, gm.w, gm.h, shift, cols,
                                                          backward ? 1 : 0, left, right, ya, yb, wide_keys);
        return cudaGetLastError();
    }
    // the fused anaglyph route: left R and right G/B only, bit masks, lists
    const bool ana = left.plane[0] && !left.plane[1] && !left.plane[2] && !right.plane[0] &&
                     right.plane[1] && right.plane[2] && !left.mask_bytes && !right.mask_bytes;
    const bool aligned =
        ((reinterpret_cast<uintptr_t>(left.plane[0]) | reinterpret_cast<uintptr_t>(right.plane[1]) |
          reinterpret_cast<uintptr_t>(right.plane[2]) | static_cast<uintptr_t>(left.pitch) |
          static_cast<uintptr_t>(right.pitch)) & 15) == 0;
    const char* vec_env = getenv("P3S_DIBR_VEC");
    const int vec = vec_env ? atoi(vec_env) : 2;
    // all six eye planes, 4-byte aligned rows (the materialised-eyes and direct-FSBS routes)
    const bool six = left.plane[0] && left.plane[1] && left.plane[2] && right.plane[0] &&
                     right.plane[1] && right.plane[2] && !left.mask_bytes && !right.mask_bytes &&
                     ((reinterpret_cast<uintptr_t>(left.plane[0]) | reinterpret_cast<uintptr_t>(left.plane[1]) |
                       reinterpret_cast<uintptr_t>(left.plane[2]) | reinterpret_cast<uintptr_t>(right.plane[0]) |
                       reinterpret_cast<uintptr_t>(right.plane[1]) | reinterpret_cast<uintptr_t>(right.plane[2]) |
                       static_cast<uintptr_t>(left.pitch) | static_cast<uintptr_t>(right.pitch)) & 3) == 0;
    const bool ilv = left.stride == 3;  // checked above: the quad kernel's ILV variant
    if (ilv || (cols && !backward && left.mask_bits && right.mask_bits && left.list && right.list &&
                vec == 2 && ((ana && aligned) || six) && static_cast<size_t>(wpad) * 13 + 48 <= kMax)) {
        void (*qk)(const uint8_t*, const uint8_t*, const uint8_t*, const uint8_t*, int, int, int,
                   const int4*, EyeOut, EyeOut, int, int, int) =
            ilv ? k_dibr_quad<0, true> : ana ? k_dibr_quad<0> : k_dibr_quad<1>;
        static std::atomic<unsigned long long> qconf{0};
        once_per_device(qconf, [] {
            cudaFuncSetAttribute(k_dibr_quad<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMax);
            cudaFuncSetAttribute(k_dibr_quad<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMax);
            cudaFuncSetAttribute(k_dibr_quad<0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMax);
        });
        const size_t qsmem = static_cast<size_t>(wpad) * 13 + 48;
        int qper = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&qper, qk, 256, qsmem);
        if (qper < 1) qper = 1;
        note_launch(st);
        qk<<<min(rows, qper * sm_count()), 256, qsmem, st>>>(r, g, b, depth, gm.pitch, gm.w, gm.h,
                                                             cols, left, right, ya, yb, src_ipitch);
        return cudaGetLastError();
    }
    if (ana && cols && aligned && (backward || (left.mask_bits && right.mask_bits && left.list &&
                                                right.list)) &&
        vec != 0 && static_cast<size_t>(wpad) * (backward ? 7 : 15) + 16 <= kMax) {
        void (*vk)(const uint8_t*, const uint8_t*, const uint8_t*, const uint8_t*, int, int, int,
                   const int4*, EyeOut, EyeOut, int, int) = backward ? k_dibr_ana<true> : k_dibr_ana<false>;
        static std::atomic<unsigned long long> vconf{0};
        once_per_device(vconf, [] {
            cudaFuncSetAttribute(k_dibr_ana<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMax);
            cudaFuncSetAttribute(k_dibr_ana<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMax);
        });
        const size_t vsmem = static_cast<size_t>(wpad) * (backward ? 7 : 15) + 16;
        int vper = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&vper, vk, 256, vsmem);
        if (vper < 1) vper = 1;
        note_launch(st);
        vk<<<min(rows, vper * sm_count()), 256, vsmem, st>>>(r, g, b, depth, gm.pitch, gm.w, gm.h,
                                                             cols, left, right, ya, yb);
        return cudaGetLastError();
    }
    void (*kern)(const uint8_t*, const uint8_t*, const uint8_t*, const uint8_t*, int, int, int,
                 const double*, const int4*, int, EyeOut, EyeOut, int, int, uint32_t*) =
        ana ? (cols ? k_dibr<0, true> : k_dibr<0, false>) : (cols ? k_dibr<1, true> : k_dibr<1, false>);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem);
    if (per_sm < 1) per_sm = 1;
    const int grid = min(rows, per_sm * sm_count());
    note_launch(st);
    kern<<<grid, 256, smem, st>>>(r, g, b, depth, gm.pitch, gm.w, gm.h, shift, cols,
                                  backward ? 1 : 0, left, right, ya, yb, nullptr);
    return cudaGetLastError();
}

cudaError_t mask_to_list(const uint8_t* mask, int mpitch, Geom gm, uint32_t* list,
                         uint32_t* count, cudaStream_t st, uint32_t* bits, int mwords) {
    const int chunks = (gm.w + 15) / 16;
    dim3 grid((chunks + 127) / 128, gm.h);
    note_launch(st);
    k_mask_to_list<<<grid, 128, 0, st>>>(mask, mpitch, gm.w, gm.h, list, count, bits, mwords);
    return cudaGetLastError();
}

cudaError_t anaglyph(const uint8_t* const* left, const uint8_t* const* right, Geom gm,
                     uint8_t* const* out, int out_pitch, cudaStream_t st) {
    const uint8_t* src[3] = {left[0], right[1], right[2]};
    for (int ch = 0; ch < 3; ++ch) {
        cudaError_t e = cudaMemcpy2DAsync(out[ch], out_pitch, src[ch], gm.pitch, gm.w, gm.h,
                                          cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t side_by_side_half(const uint8_t* const* left, const uint8_t* const* right, Geom gm,
                              uint8_t* const* out, int out_pitch, cudaStream_t st) {
    const int hw = gm.w / 2;
    const uintptr_t al = reinterpret_cast<uintptr_t>(left[0]) | reinterpret_cast<uintptr_t>(left[1]) |
                         reinterpret_cast<uintptr_t>(left[2]) | reinterpret_cast<uintptr_t>(right[0]) |
                         reinterpret_cast<uintptr_t>(right[1]) | reinterpret_cast<uintptr_t>(right[2]) |
                         reinterpret_cast<uintptr_t>(out[0]) | reinterpret_cast<uintptr_t>(out[1]) |
                         reinterpret_cast<uintptr_t>(out[2]) | static_cast<uintptr_t>(gm.pitch) |
                         static_cast<uintptr_t>(out_pitch);
    if (hw % 16 == 0 && (al & 15) == 0) {
        const long long items = 2LL * 3 * (hw / 16) * gm.h;
        note_launch(st);
        k_hsbs16<<<static_cast<unsigned>((items + 255) / 256), 256, 0, st>>>(
            left[0], left[1], left[2], right[0], right[1], right[2], gm.pitch, gm.w, gm.h, out[0],
            out[1], out[2], out_pitch);
        return cudaGetLastError();
    }
    const int items = 2 * ((hw + 15) / 16);
    dim3 grid((items + 127) / 128, gm.h);
    note_launch(st);
    k_hsbs<<<grid, 128, 0, st>>>(left[0], left[1], left[2], right[0], right[1], right[2],
                                 gm.pitch, gm.w, out[0], out[1], out[2], out_pitch);
    return cudaGetLastError();
}

cudaError_t side_by_side_full(const uint8_t* const* left, const uint8_t* const* right, Geom gm,
                              uint8_t* const* out, int out_pitch, cudaStream_t st) {
    for (int ch = 0; ch < 3; ++ch) {
        cudaError_t e = cudaMemcpy2DAsync(out[ch], out_pitch, left[ch], gm.pitch, gm.w, gm.h,
                                          cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) return e;
        e = cudaMemcpy2DAsync(out[ch] + gm.w, out_pitch, right[ch], gm.pitch, gm.w, gm.h,
                              cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace cu
}  // namespace p3s
