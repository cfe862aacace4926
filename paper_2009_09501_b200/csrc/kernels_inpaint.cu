// K3b: Jacobi hole filling on sm_100a (reference proj/src/inpaint.cpp:29-130).
//
// Semantics kept exactly: every pass decides against the pass-start snapshot (a damaged
// pixel with >= 2 intact 8-neighbours takes the per-channel (2*sum + n) / (2n) mean),
// then applies all repairs; the first pass that repairs nothing while damage remains
// fills the rest with (128,128,128). Both eyes are independent instances
// (pipeline.cpp:56-65) and run in the same launch.
//
// Temporal blocking. The frame is cut into 32x32 tiles; a round runs kPasses Jacobi passes
// of one tile inside shared memory over the tile plus a kPasses-pixel halo (a 64x64 region,
// one warp per tile, lane l owning region rows l and l + 32). Information moves one pixel
// per pass, so after kPasses passes the tile interior equals the global Jacobi state;
// pixels outside the region are treated as not intact, which can only disturb the
// discarded halo. A pass that repairs nothing in the region is a fixed point of the
// simulation, so the remaining passes of the round are skipped.
//
// Bit-parallel passes. Damage and in-image flags are 64-bit row words, so the "at least two
// intact 8-neighbours" decision for a whole row is ~20 word operations; colours are only
// computed for the pixels a pass repairs (each damaged pixel exactly once), from the
// pass-start colours of its intact neighbours, staged in shared memory as one packed
// 0x00BBGGRR word per pixel (one shared load per neighbour; the three divisions by 2n are
// one multiply-high each with a per-n magic). A pass whose repairs are at most kDirect per
// lane (a vertical front: one or two per row) lets each lane repair its own rows; denser
// passes compact the repairs into one list first so the colour work spreads over the lanes.
//
// Cross-tile state is the damage of each 32-pixel row word of a tile interior as it stands
// at the end of a round: a 64-bit word (tag << 32 | damage bits), kept in two slots per
// word, tag = launch epoch << 12 | (round + 1). The init writes both slots of every word of
// a damaged tile with round tag 0 (the initial damage); round r writes slot r & 1 with tag
// r + 1. A tile starting round r takes, per word, the slot of this launch's epoch with the
// largest round tag <= r, i.e. the state at the end of round r - 1; a word with neither
// slot in this epoch belongs to an undamaged tile (damage 0). Slot (r - 1) & 1 is stable
// during round r and slot r & 1 only goes from an older tag to r + 1, so the racy reads are
// harmless and ONE grid barrier per round suffices. The words are stored column-major
// ([word][row]) so a warp reading 32 consecutive rows of one word is one coalesced 256-byte
// access; the epoch (persistent in the arena, advanced by each launch) means no per-frame
// clearing: only when it wraps (every 2^20 launches) does a launch zero the slots first.
// Per-pass global repair counts (interior pixels only) reproduce the reference's global
// stall rule and pass statistics exactly.
//
// Latency is what bounds this kernel (a wide disocclusion strip needs one pass per pixel of
// width, each round's tiles wait for the previous round), so every tile's global reads are
// issued together (mask + state words: one round trip; colour rows: one more), the first
// claim of a round is static (warp w takes list item w), and the grid barrier is one
// arrival atomic per CTA on a monotonic counter.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "p3s_cu.h"

namespace p3s {
namespace cu {
namespace {

constexpr int kT = 32;                 // tile side (interior)
constexpr int kPasses = 16;            // passes per round = halo width
constexpr int kE = kT + 2 * kPasses;   // region side (64: one u64 per row)
constexpr int kWarps = 8;              // one tile per warp
constexpr int kThreads = 32 * kWarps;
constexpr uint32_t kHeavy = 128;       // damaged pixels that make a tile "heavy" (run first)
#ifndef P3S_INPAINT_KDIRECT  // experiment builds: make VARIANT=x EXTRA=-DP3S_INPAINT_KDIRECT=n
#define P3S_INPAINT_KDIRECT 4
#endif
constexpr int kDirect = P3S_INPAINT_KDIRECT;  // per-lane repairs up to which a pass skips compaction
constexpr int kCtlWords = 128;         // ctl scratch: [eye][slot 0..2][kPasses + 1] + barrier
constexpr int kBarWord = 127;          // ctl word: the grid barrier's arrival counter
constexpr unsigned long long kInner = 0x0000FFFFFFFF0000ull;  // interior columns 16..47

struct Eye {
    InpaintEye io;
    unsigned long long* slot[2];  // [mwords][h] tagged damage words (column-major)
    int mwords;                   // (w + 31) / 32
};

constexpr unsigned kEpochBits = 20;  // launch epochs per slot clear

// Both eyes, passed as one __grid_constant__ parameter so the eye a tile belongs to is an
// indexed constant-bank read rather than a local-memory copy of the struct.
struct Eyes {
    Eye e[2];
};

struct Work {
    uint32_t* init_flags;  // [2][tiles] damaged-pixel count per tile (initial work list)
    uint32_t* heavy;       // [2 * tiles] tiles with >= kHeavy damaged pixels (round 0, first)
    uint32_t* lists;       // [3][2 * tiles] (eye * tiles + tile)
    uint32_t* counters;    // [0..5] = [3][2]: count, claim; [6] heavy count; [16] the launch
                           // epoch (persistent, not zeroed per launch)
    int cap;               // 2 * tiles
};

struct WarpSmem {
    // packed 0x00BBGGRR colours (intact pixels next to damage), column-major with an odd
    // stride: a vertical front (lanes on consecutive rows, one column) and a horizontal one
    // (one row, consecutive columns) both hit 32 distinct banks
    uint32_t col[kE][kE + 1];  // [column][row]
    unsigned long long itc[2][kE];      // intact (in-image, undamaged) bits per row; pass parity
    uint16_t rep[kE * kE];              // list-mode repairs of one pass (row << 6 | column)
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Predicated L2 loads (ld.global.cg under a predicate, 0 when off). __ldcg is a volatile asm
// statement, so `c ? __ldcg(p) : 0` compiles to a branch per load; these stay branch-free.
__device__ __forceinline__ unsigned long long ldcg_if(const unsigned long long* p, bool pred) {
    unsigned long long v = 0;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.global.cg.u64 %0, [%1];\n\t}"
                 : "+l"(v) : "l"(p), "r"(static_cast<unsigned>(pred)));
    return v;
}

__device__ __forceinline__ uint4 ldcg_if(const void* p, bool pred) {
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %5, 0;\n\t@q ld.global.cg.v4.u32 {%0, %1, %2, %3}, [%4];\n\t}"
                 : "+r"(v.x), "+r"(v.y), "+r"(v.z), "+r"(v.w) : "l"(p), "r"(static_cast<unsigned>(pred)));
    return v;
}

// Grid barrier of a co-resident (cooperative) launch: one arrival per CTA on a counter that
// only grows within a launch (zeroed before it), so the n-th barrier waits for n * gridDim.x.
__device__ __forceinline__ void grid_barrier(unsigned* ctr, unsigned& epoch) {
    __syncthreads();
    ++epoch;
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1u);
        const unsigned target = epoch * gridDim.x;
        while (ld_acquire(ctr) < target) {
        }
    }
    __syncthreads();
}

// Damage bits of one interior word as of the end of round r - 1 (this epoch's largest round
// tag <= r) from its two slot words; 0 when neither slot is of this epoch (undamaged tile).
__device__ __forceinline__ unsigned pick_slot(unsigned long long a, unsigned long long b, int r,
                                              unsigned epoch) {
    // tags of this epoch with round tag <= r, as (tag - epoch base) <= r
    const unsigned base = epoch << 12;
    const unsigned ra = static_cast<unsigned>(a >> 32) - base, rb = static_cast<unsigned>(b >> 32) - base;
    const bool va = ra <= static_cast<unsigned>(r), vb = rb <= static_cast<unsigned>(r);
    if (va && (!vb || ra >= rb)) return static_cast<unsigned>(a);
    if (vb) return static_cast<unsigned>(b);
    return 0u;
}

__device__ __forceinline__ unsigned word_state(const Eye& E, int gy, int wi, int h, int r, unsigned epoch) {
    if (wi < 0 || wi >= E.mwords) return 0u;
    const size_t o = static_cast<size_t>(wi) * h + gy;
    return pick_slot(__ldcg(E.slot[0] + o), __ldcg(E.slot[1] + o), r, epoch);
}

// Publishes the interior word of region row r (image row gy) at the end of round `round`.
__device__ __forceinline__ void publish_word(const Eye& E, int gy, int tx, int h, int round, unsigned epoch,
                                             unsigned long long dregion) {
    const unsigned long long v = (static_cast<unsigned long long>((epoch << 12) | (round + 1)) << 32) |
                                 ((dregion >> kPasses) & 0xFFFFFFFFull);
    __stcg(E.slot[round & 1] + static_cast<size_t>(tx) * h + gy, v);
}

// Cold paths are kept out of line (and not unrolled) so the hot tile code stays small and
// contiguous in the instruction cache.
// Bits of pixels with at least two set bits among their 8 neighbours in (up, mid, dn).
__device__ __forceinline__ unsigned long long two_plus(unsigned long long up, unsigned long long mid,
                                                       unsigned long long dn) {
    const unsigned long long v[8] = {up << 1, up, up >> 1, mid << 1, mid >> 1, dn << 1, dn, dn >> 1};
    unsigned long long one = 0, two = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        two |= one & v[k];
        one |= v[k];
    }
    return two;
}

// Packs 16 pixels of three planes (r, g, b: 16 bytes each) into 16 words 0x??BBGGRR.
__device__ __forceinline__ void pack16(const uint4& r, const uint4& g, const uint4& b, uint4 (&o)[4]) {
    const unsigned R[4] = {r.x, r.y, r.z, r.w}, G[4] = {g.x, g.y, g.z, g.w}, B[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const unsigned lo = __byte_perm(R[i], G[i], 0x5140);  // R0 G0 R1 G1
        const unsigned hi = __byte_perm(R[i], G[i], 0x7362);  // R2 G2 R3 G3
        o[i] = make_uint4(__byte_perm(lo, B[i], 0x4410), __byte_perm(lo, B[i], 0x5532),
                          __byte_perm(hi, B[i], 0x6610), __byte_perm(hi, B[i], 0x7732));
    }
}

// 16 interleaved pixels (48 bytes r0 g0 b0 r1 ...) into 16 words 0x??BBGGRR (the top byte
// is never read).
__device__ __forceinline__ void unpack_rgb16(const uint4& a, const uint4& b, const uint4& c, uint4 (&o)[4]) {
    const unsigned W[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {  // pixels 4i..4i+3: bytes 12i..12i+11 = words 3i..3i+2
        const unsigned w0 = W[3 * i], w1 = W[3 * i + 1], w2 = W[3 * i + 2];
        o[i] = make_uint4(w0, __byte_perm(w0, w1, 0x6543), __byte_perm(w1, w2, 0x5432), w2 >> 8);
    }
}

// 16 bytes of a plane row from column c, in-image columns only (0 elsewhere / no plane).
__device__ __noinline__ uint4 load16_bytes(const uint8_t* pl, int pitch, int gy, int c, int w, int stride) {
    unsigned b[4] = {0u, 0u, 0u, 0u};
    if (pl) {
#pragma unroll 1
        for (int k = 0; k < 16; ++k)
            if (c + k >= 0 && c + k < w)
                b[k >> 2] |= static_cast<unsigned>(__ldcg(pl + static_cast<size_t>(gy) * pitch +
                                                          static_cast<size_t>(c + k) * stride)) << (8 * (k & 3));
    }
    return make_uint4(b[0], b[1], b[2], b[3]);
}

// Stages the packed colours of the region pixels the round can read: those intact at its
// start and 8-adjacent to damage (need: [64] region-row masks), by 16-pixel quads. A warp
// instruction covers 8 rows x 4 quads (each row's 64 bytes contiguous: 8 rows are 8-16
// cache lines, not 32); all loads are issued before any is used.
template <int STRIDE>
__device__ __forceinline__ void load_colours(const InpaintEye& io, WarpSmem& S, const unsigned long long* need,
                                             int x0, int y0, int w, int h, bool vec, long long* sub = nullptr) {
#ifdef P3S_INPAINT_PHASES
    long long _s0 = clock64();
#endif
    const int lane = threadIdx.x & 31;
    uint4 v[8][3];
    bool ok[8], fast[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int r = 8 * i + (lane >> 2), c = x0 + 16 * (lane & 3), gy = y0 + r;
        ok[i] = ((need[r] >> (16 * (lane & 3))) & 0xFFFFull) != 0ull;  // in-image by construction
        fast[i] = ok[i] && vec && c >= 0 && STRIDE * (c + 16) <= io.pitch;
        if (STRIDE == 3) {
            // interleaved rows: the quad's 48 bytes (every channel; the ones this eye does
            // not produce are read but never used or written)
            const uint8_t* base = io.plane[0] ? io.plane[0] : io.plane[1] ? io.plane[1] - 1 : io.plane[2] - 2;
            const size_t o = static_cast<size_t>(gy) * io.pitch + 3 * static_cast<size_t>(c);
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) v[i][ch] = ldcg_if(base + o + 16 * ch, fast[i]);
        } else {
            const size_t o = static_cast<size_t>(gy) * io.pitch + c;
#pragma unroll
            for (int ch = 0; ch < 3; ++ch)
                v[i][ch] = ldcg_if(io.plane[ch] + o, fast[i] && io.plane[ch] != nullptr);
        }
    }
#ifdef P3S_INPAINT_PHASES
    long long _s1 = clock64();
    if (sub) sub[0] += _s1 - _s0;
#endif
#pragma unroll
    for (int i = 0; i < 8; ++i) {
#ifdef P3S_INPAINT_PHASES
        if (i == 1 && sub) {
            const long long _s2 = clock64();
            sub[1] += _s2 - _s1;
            _s1 = _s2;
        }
#endif
        if (!ok[i]) continue;
        const int r = 8 * i + (lane >> 2), q = lane & 3, c = x0 + 16 * q, gy = y0 + r;
        uint4 o[4];
        if (!fast[i]) {  // image edge or unaligned planes: bytes, in-image columns only
            v[i][0] = load16_bytes(io.plane[0], io.pitch, gy, c, w, STRIDE);
            v[i][1] = load16_bytes(io.plane[1], io.pitch, gy, c, w, STRIDE);
            v[i][2] = load16_bytes(io.plane[2], io.pitch, gy, c, w, STRIDE);
            pack16(v[i][0], v[i][1], v[i][2], o);
        } else if (STRIDE == 3) {
            unpack_rgb16(v[i][0], v[i][1], v[i][2], o);
        } else {
            pack16(v[i][0], v[i][1], v[i][2], o);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            S.col[16 * q + 4 * k + 0][r] = o[k].x;
            S.col[16 * q + 4 * k + 1][r] = o[k].y;
            S.col[16 * q + 4 * k + 2][r] = o[k].z;
            S.col[16 * q + 4 * k + 3][r] = o[k].w;
        }
    }
#ifdef P3S_INPAINT_PHASES
    if (sub) sub[2] += clock64() - _s1;
#endif
}

// The reference's repair of pixel (r, c): per-channel (2 * sum + n) / (2n) over its n intact
// 8-neighbours (inpaint.cpp:80-95), from the pass-start intact words of rows r-1, r, r+1.
__device__ __forceinline__ uint32_t repair_colour(const WarpSmem& S, const uint32_t* magic, int r, int c,
                                                  unsigned long long iu, unsigned long long im,
                                                  unsigned long long id) {
    uint32_t rb = 0, g = 0, n = 0;
    // unconditional loads (no branches): a neighbour that is not intact (possibly being
    // repaired by another lane in this pass, or outside the region) reads the pixel's own
    // cell instead, which only this lane writes, and the value is masked away
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy) {
        const unsigned long long wv = dy < 0 ? iu : (dy > 0 ? id : im);

        // bit 0 = column c - 1, bit 1 = c, bit 2 = c + 1 (outside the region: 0)
        unsigned tri = static_cast<unsigned>((c > 0 ? (wv >> (c - 1)) : (wv << 1)) & 7ull);
        if (dy == 0) tri &= 5u;
#pragma unroll
        for (int dx = -1; dx <= 1; ++dx) {
            if (dy == 0 && dx == 0) continue;
            const unsigned b = (tri >> (dx + 1)) & 1u;
            const uint32_t v = S.col[b ? c + dx : c][b ? r + dy : r] & (0u - b);
            rb += v & 0x00FF00FFu;
            g += (v >> 8) & 0xFFu;
            n += b;
        }
    }
    const uint32_t M = magic[n];  // ceil(2^32 / 2n): exact quotient for numerators < 2^12
    const uint32_t qr = __umulhi(2u * (rb & 0xFFFFu) + n, M);
    const uint32_t qg = __umulhi(2u * g + n, M);
    const uint32_t qb = __umulhi(2u * (rb >> 16) + n, M);
    return qr | (qg << 8) | (qb << 16);
}

__device__ __forceinline__ void repair(const InpaintEye& io, WarpSmem& S, const uint32_t* magic, int r, int c,
                                       unsigned long long iu, unsigned long long im, unsigned long long id,
                                       int x0, int y0) {
    // never an intact neighbour in its own pass: no other lane reads it. The interior's
    // repairs reach the planes once, at the end of the tile (publish_colours)
    S.col[c][r] = repair_colour(S, magic, r, c, iu, im, id);
}

// Writes the interior pixels this round repaired (rep: [64] region-row masks in shared
// memory) from S.col to the planes: lane = 4-pixel group of a row, 4 rows per instruction,
// so the byte stores of a row land in one 32-byte segment. Other tiles read only pixels that
// were intact at the round's start, so the deferred writes are invisible to them.
template <int STRIDE>
__device__ __forceinline__ void publish_colours(const InpaintEye& io, const WarpSmem& S,
                                                const unsigned long long* rep, int x0, int y0, bool vec) {
    const int lane = threadIdx.x & 31;
    const int g = lane & 7;  // interior columns 16 + 4g .. 16 + 4g + 3
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const int r = kPasses + 4 * b + (lane >> 3);
        const unsigned m = static_cast<unsigned>(rep[r] >> (kPasses + 4 * g)) & 0xFu;
        if (!m) continue;
        const size_t o = static_cast<size_t>(y0 + r) * io.pitch +
                         static_cast<size_t>(x0 + kPasses + 4 * g) * STRIDE;
        const int c = kPasses + 4 * g;
        const uint32_t q0 = S.col[c][r], q1 = S.col[c + 1][r], q2 = S.col[c + 2][r], q3 = S.col[c + 3][r];
        if (STRIDE == 3) {  // interleaved: byte stores of this eye's channels only
            const uint32_t q[4] = {q0, q1, q2, q3};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (!((m >> k) & 1u)) continue;
                if (io.plane[0]) io.plane[0][o + 3 * k] = static_cast<uint8_t>(q[k]);
                if (io.plane[1]) io.plane[1][o + 3 * k] = static_cast<uint8_t>(q[k] >> 8);
                if (io.plane[2]) io.plane[2][o + 3 * k] = static_cast<uint8_t>(q[k] >> 16);
            }
            continue;
        }
        if (m == 0xFu && vec) {  // the whole group: one 4-byte store per plane
            if (io.plane[0]) *reinterpret_cast<uint32_t*>(io.plane[0] + o) = __byte_perm(__byte_perm(q0, q1, 0x0040), __byte_perm(q2, q3, 0x0040), 0x5410);
            if (io.plane[1]) *reinterpret_cast<uint32_t*>(io.plane[1] + o) = __byte_perm(__byte_perm(q0, q1, 0x0051), __byte_perm(q2, q3, 0x0051), 0x5410);
            if (io.plane[2]) *reinterpret_cast<uint32_t*>(io.plane[2] + o) = __byte_perm(__byte_perm(q0, q1, 0x0062), __byte_perm(q2, q3, 0x0062), 0x5410);
            continue;
        }
        const uint32_t q[4] = {q0, q1, q2, q3};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (!((m >> k) & 1u)) continue;
            if (io.plane[0]) io.plane[0][o + k] = static_cast<uint8_t>(q[k]);
            if (io.plane[1]) io.plane[1][o + k] = static_cast<uint8_t>(q[k] >> 8);
            if (io.plane[2]) io.plane[2][o + k] = static_cast<uint8_t>(q[k] >> 16);
        }
    }
}

#ifdef P3S_INPAINT_PHASES
// experiment build only (make VARIANT=phases EXTRA=-DP3S_INPAINT_PHASES): per-phase SM
// cycles of the tiles of rounds >= 1, kept in registers and summed once per tile: [0] mask/
// state words, [1] colour rows, [2] decide, [3] colours (direct), [4] colours (list),
// [5] update, [6] tail; [7] tiles, [8] passes, [9] list-mode passes, [10] tile ns,
// [11] tile cycles
__device__ unsigned long long g_phase[20];
#define PH_MARK(i)                          \
    do {                                    \
        __syncwarp();                       \
        const long long _n = clock64();     \
        _ph[i] += _n - _pt;                 \
        _pt = _n;                           \
    } while (0)
#define PH_COUNT(i) ++_ph[i]
#else
#define PH_MARK(i) \
    do {           \
    } while (0)
#define PH_COUNT(i) \
    do {            \
    } while (0)
#endif

// One warp simulates up to kPasses Jacobi passes of one tile (+ halo) in shared memory.
template <int STRIDE>
__device__ void process_tile(const Eye& E, int tx, int ty, int w, int h, int round, unsigned epoch,
                             WarpSmem& S, const uint32_t* magic, bool vec, uint32_t* counts_slot,
                             bool& remains) {
    const InpaintEye& io = E.io;
    const int lane = threadIdx.x & 31;
    const unsigned full = 0xFFFFFFFFu;
    const int x0 = tx * kT - kPasses, y0 = ty * kT - kPasses;
    const int gy0 = y0 + lane, gy1 = y0 + lane + 32;
    const bool in0 = gy0 >= 0 && gy0 < h, in1 = gy1 >= 0 && gy1 < h;
    __syncwarp();  // the previous tile's shared-memory reads before this tile's writes
#ifdef P3S_INPAINT_PHASES
    long long _ph[15] = {};
    const long long _c0 = clock64();
    long long _pt = _c0;
    const unsigned long long _t0 = gtimer();
    PH_COUNT(7);
#endif
    // 1. damage words: the tagged state words of the three interior words the region spans
    //    (region columns 0..15 = bits 16..31 of word tx - 1, 16..47 = word tx, 48..63 = bits
    //    0..15 of word tx + 1), 12 coalesced loads issued before any is used
    const int lo = max(0, -x0), hi = min(64, w - x0);  // in-image region columns [lo, hi)
    const unsigned long long cols =
        hi <= lo ? 0ull : ((hi - lo == 64 ? ~0ull : ((1ull << (hi - lo)) - 1ull)) << lo);
    const unsigned long long img0 = in0 ? cols : 0ull, img1 = in1 ? cols : 0ull;
    unsigned long long sw[2][3][2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int gy = j ? gy1 : gy0;
        const bool in = j ? in1 : in0;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const int wi = tx - 1 + q;
            const bool ok = in && wi >= 0 && wi < E.mwords;
            const size_t o = static_cast<size_t>(wi) * h + gy;
            sw[j][q][0] = ldcg_if(E.slot[0] + o, ok);
            sw[j][q][1] = ldcg_if(E.slot[1] + o, ok);
        }
    }
    unsigned long long d0, d1;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const unsigned a = pick_slot(sw[j][0][0], sw[j][0][1], round, epoch);
        const unsigned b = pick_slot(sw[j][1][0], sw[j][1][1], round, epoch);
        const unsigned c = pick_slot(sw[j][2][0], sw[j][2][1], round, epoch);
        const unsigned long long m = static_cast<unsigned long long>(a >> 16) |
                                     (static_cast<unsigned long long>(b) << 16) |
                                     (static_cast<unsigned long long>(c & 0xFFFFu) << 48);
        (j ? d1 : d0) = m & (j ? img1 : img0);
    }
    S.itc[0][lane] = img0 & ~d0;
    S.itc[0][lane + 32] = img1 & ~d1;
    PH_MARK(0);
    // 2. colours of the intact pixels 8-adjacent to damage (the only ones the passes read;
    //    pixels repaired during the round get theirs in shared memory)
    unsigned long long* need = reinterpret_cast<unsigned long long*>(S.rep);  // free until the passes
    {
        const unsigned long long up0 = __shfl_up_sync(full, d0, 1), dn0 = __shfl_down_sync(full, d0, 1);
        const unsigned long long up1 = __shfl_up_sync(full, d1, 1), dn1 = __shfl_down_sync(full, d1, 1);
        const unsigned long long d0_31 = __shfl_sync(full, d0, 31), d1_0 = __shfl_sync(full, d1, 0);
        const unsigned long long a0 = (lane > 0 ? up0 : 0ull) | d0 | (lane < 31 ? dn0 : d1_0);
        const unsigned long long a1 = (lane > 0 ? up1 : d0_31) | d1 | (lane < 31 ? dn1 : 0ull);
        need[lane] = (a0 | (a0 << 1) | (a0 >> 1)) & img0 & ~d0;
        need[lane + 32] = (a1 | (a1 << 1) | (a1 >> 1)) & img1 & ~d1;
    }
    __syncwarp();
    const unsigned long long ds0 = d0, ds1 = d1;  // damage at the round's start
#ifdef P3S_INPAINT_PHASES
    load_colours<STRIDE>(io, S, need, x0, y0, w, h, vec, &_ph[10]);
#else
    load_colours<STRIDE>(io, S, need, x0, y0, w, h, vec);
#endif
    __syncwarp();
    PH_MARK(1);
    // 3. passes (S.itc[p] = the pass-start intact words; the pass writes S.itc[p ^ 1])
    uint32_t my_count = 0;  // lane k - 1: interior repairs of pass k
    int p = 0;
    for (int k = 1; k <= kPasses; ++k) {
        const unsigned long long* itc = S.itc[p];
        const unsigned long long u0 = lane > 0 ? itc[lane - 1] : 0ull, m0 = img0 & ~d0, n0 = itc[lane + 1];
        const unsigned long long u1 = itc[lane + 31], m1 = img1 & ~d1, n1 = lane < 31 ? itc[lane + 33] : 0ull;
        const unsigned long long rep0 = d0 & two_plus(u0, m0, n0);
        const unsigned long long rep1 = d1 & two_plus(u1, m1, n1);
        if (!__any_sync(full, (rep0 | rep1) != 0ull)) break;  // fixed point of the region
        PH_COUNT(8);
        // interior rows: 16..31 are lanes 16..31 of row set 0, 32..47 lanes 0..15 of set 1
        const int inner = __reduce_add_sync(full, lane >= 16 ? __popcll(rep0 & kInner) : __popcll(rep1 & kInner));
        if (lane == k - 1) my_count = static_cast<uint32_t>(inner);
        const unsigned cnt = __popcll(rep0) + __popcll(rep1);
        PH_MARK(2);
        if (__reduce_max_sync(full, cnt) <= static_cast<unsigned>(kDirect)) {
            // one repair of each of the lane's two rows per iteration (independent chains)
            unsigned long long b0 = rep0, b1 = rep1;
            while (b0 | b1) {
                const int c0 = __ffsll(static_cast<long long>(b0)) - 1, c1 = __ffsll(static_cast<long long>(b1)) - 1;
                const uint32_t v0 = repair_colour(S, magic, lane, max(c0, 0), u0, m0, n0);
                const uint32_t v1 = repair_colour(S, magic, lane + 32, max(c1, 0), u1, m1, n1);
                if (b0) S.col[c0][lane] = v0;
                if (b1) S.col[c1][lane + 32] = v1;
                b0 &= b0 - 1;
                b1 &= b1 - 1;
            }
            PH_MARK(3);
        } else {
            PH_COUNT(9);
            // compact the pass's repairs into one list so the colour work spreads over lanes
            unsigned incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned v = __shfl_up_sync(full, incl, o);
                if (lane >= o) incl += v;
            }
            const int total = static_cast<int>(__shfl_sync(full, incl, 31));
            int pos = static_cast<int>(incl - cnt);
            for (unsigned long long b = rep0; b; b &= b - 1)
                S.rep[pos++] = static_cast<uint16_t>((lane << 6) | (__ffsll(static_cast<long long>(b)) - 1));
            for (unsigned long long b = rep1; b; b &= b - 1)
                S.rep[pos++] = static_cast<uint16_t>(((lane + 32) << 6) | (__ffsll(static_cast<long long>(b)) - 1));
            __syncwarp();
            for (int i = lane; i < total; i += 32) {
                const int e = S.rep[i], r = e >> 6, c = e & 63;
                repair(io, S, magic, r, c, r > 0 ? itc[r - 1] : 0ull, itc[r], r + 1 < kE ? itc[r + 1] : 0ull,
                       x0, y0);
            }
            PH_MARK(4);
        }
        d0 &= ~rep0;
        d1 &= ~rep1;
        S.itc[p ^ 1][lane] = img0 & ~d0;
        S.itc[p ^ 1][lane + 32] = img1 & ~d1;
        p ^= 1;
        __syncwarp();  // the pass's colours and intact words before the next pass reads them
        // interior complete: its pixels never change again (repairs are final), so later
        // passes add no interior repairs; the halo's evolution is discarded anyway
        const bool left = lane >= 16 ? (d0 & kInner) != 0ull : (d1 & kInner) != 0ull;
        PH_MARK(5);
        if (!__any_sync(full, left)) break;
    }
    // 4. the round's interior repairs to the planes, pass counts, the interior's damage
    //    words; interior damage left -> runs again
    unsigned long long* repaired = reinterpret_cast<unsigned long long*>(S.rep);
    __syncwarp();
    repaired[lane] = ds0 & ~d0;
    repaired[lane + 32] = ds1 & ~d1;
    __syncwarp();
    publish_colours<STRIDE>(io, S, repaired, x0, y0, vec);
    if (my_count) atomicAdd(&counts_slot[lane + 1], my_count);
    const unsigned long long dint = lane >= 16 ? d0 : d1;
    const int gyi = lane >= 16 ? gy0 : gy1;
    if (gyi < h) publish_word(E, gyi, tx, h, round, epoch, dint);
    remains = __any_sync(full, (dint & kInner) != 0ull);
    PH_MARK(6);
#ifdef P3S_INPAINT_PHASES
    if (round > 0 && lane == 0) {
        for (int i = 0; i < 10; ++i) atomicAdd(&g_phase[i], static_cast<unsigned long long>(_ph[i]));
        atomicAdd(&g_phase[14], static_cast<unsigned long long>(_ph[10]));
        atomicAdd(&g_phase[15], static_cast<unsigned long long>(_ph[11]));
        atomicAdd(&g_phase[16], static_cast<unsigned long long>(_ph[12]));
        atomicAdd(&g_phase[10], gtimer() - _t0);
        atomicAdd(&g_phase[11], static_cast<unsigned long long>(clock64() - _c0));
    }
#endif
}

// Debug timeline (P3S_DEBUG_INPAINT): per round, [4] = round start (block 0, after the
// barrier), latest tile finish, max tile ns, tiles processed; nullptr in normal runs.
constexpr int kDbgRounds = 64;
__device__ unsigned long long* g_inp_rdbg = nullptr;

// STRIDE 3: the eyes' planes are channels of one RGB-interleaved image (InpaintEye.stride).
template <int STRIDE>
__global__ void __launch_bounds__(kThreads, 1) k_inpaint_tiles(const __grid_constant__ Eyes eyes, Work wk, int w, int h,
                                                               int tiles_x, int tiles_y, uint32_t* ctl,
                                                               long long* stats, int vec) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ uint32_t s_magic[9];
    WarpSmem& S = reinterpret_cast<WarpSmem*>(smem_raw)[threadIdx.x >> 5];
    const int ntiles = tiles_x * tiles_y;
    unsigned long long* rdbg = g_inp_rdbg;
    const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t gsize = gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    const uint32_t gw = gtid >> 5, nw = gsize >> 5;
    const Eye& L = eyes.e[0];
    const Eye& R = eyes.e[1];
    unsigned epoch_bar = 0;  // grid barriers passed
    if (threadIdx.x < 9) s_magic[threadIdx.x] = threadIdx.x >= 2 ? 0xFFFFFFFFu / (2u * threadIdx.x) + 1u : 0u;

    // launch epoch: 0 = fresh arena or wrapped -> zero every slot word first
    const unsigned epoch = __ldcg(wk.counters + 16);
    if (epoch == 0u) {
        for (int e = 0; e < 2; ++e) {
            const size_t nw = static_cast<size_t>(eyes.e[e].mwords) * h;
            for (size_t k = gtid; k < nw; k += gsize) {
                __stcg(eyes.e[e].slot[0] + k, 0ull);
                __stcg(eyes.e[e].slot[1] + k, 0ull);
            }
        }
        grid_barrier(ctl + kBarWord, epoch_bar);
    }
    // init: per-tile damage counts -> work lists (tiles with damage; heavy ones apart) and
    // both slots of every word of a damaged tile = its initial damage (round tag 0)
    uint32_t cnt[2];
    cnt[0] = __ldcg(L.io.count);
    cnt[1] = __ldcg(R.io.count);
    {
        // one warp per (eye, tile): lane = tile row, popcount of its interior mask word; a
        // warp's kInitBatch items' mask loads are issued together (one round trip, not one
        // per item: ~14 items per warp at 4K)
        constexpr int kInitBatch = 8;
        const uint32_t nitems = static_cast<uint32_t>(2 * ntiles);
        for (uint32_t item0 = gw; item0 < nitems; item0 += kInitBatch * nw) {
            unsigned mb[kInitBatch];
#pragma unroll
            for (int b = 0; b < kInitBatch; ++b) {
                const uint32_t item = item0 + b * nw;
                mb[b] = 0u;
                if (item >= nitems) continue;
                const int e = item >= static_cast<uint32_t>(ntiles);
                const int t = static_cast<int>(item) - e * ntiles, tx = t % tiles_x, ty = t / tiles_x;
                const int gy = ty * kT + lane;
                const InpaintEye& io = eyes.e[e].io;
                if (cnt[e] && gy < h) mb[b] = __ldg(io.mask_bits + static_cast<size_t>(gy) * io.mask_pitch + tx);
            }
#pragma unroll
            for (int b = 0; b < kInitBatch; ++b) {
            const uint32_t item = item0 + b * nw;
            if (item >= nitems) break;
            const int e = item >= static_cast<uint32_t>(ntiles);
            if (!cnt[e]) continue;
            const int t = static_cast<int>(item) - e * ntiles, tx = t % tiles_x, ty = t / tiles_x;
            const int gy = ty * kT + lane;
            const unsigned m = mb[b];
            const uint32_t c = __reduce_add_sync(0xFFFFFFFFu, static_cast<unsigned>(__popc(m)));
            if (c && gy < h) {
                const unsigned long long v = (static_cast<unsigned long long>(epoch << 12) << 32) | m;
                const size_t o = static_cast<size_t>(tx) * h + gy;
                __stcg(eyes.e[e].slot[0] + o, v);
                __stcg(eyes.e[e].slot[1] + o, v);
            }
            if (lane == 0 && c) {
                wk.init_flags[item] = c;
                const uint32_t pos = atomicAdd(&wk.counters[c >= kHeavy ? 6 : 0], 1u);
                (c >= kHeavy ? wk.heavy : wk.lists)[pos] = item;
            }
            }
        }
    }
    long long remaining[2] = {cnt[0], cnt[1]};
    bool done[2] = {cnt[0] == 0, cnt[1] == 0};
    long long passes[2] = {0, 0}, fallback[2] = {0, 0};
    unsigned long long busy[2] = {0, 0};  // this warp's tile ns per eye
    const unsigned long long t_start = gtimer();
    grid_barrier(ctl + kBarWord, epoch_bar);

    // ctl layout: [eye][slot 0..2][kPasses + 1] pass counts
    for (int round = 0; !(done[0] && done[1]); ++round) {
        const int slot = round % 3, nslot = (round + 1) % 3, rslot = (round + 2) % 3;
        if (rdbg && round < kDbgRounds && gtid == 0) rdbg[4 * round] = gtimer();
        if (gtid < 2 * (kPasses + 1)) {
            const int e = gtid / (kPasses + 1), k = gtid % (kPasses + 1);
            ctl[(e * 3 + nslot) * (kPasses + 1) + k] = 0;
        }
        if (gtid == 0) {  // list rslot was last read in round - 1; it is appended to in round + 1
            wk.counters[2 * rslot] = 0;
            wk.counters[2 * rslot + 1] = 0;
        }
        const uint32_t n = __ldcg(&wk.counters[2 * slot]);
        const uint32_t nheavy = round == 0 ? __ldcg(&wk.counters[6]) : 0u;
        const uint32_t total = n + nheavy;
        const uint32_t* list = wk.lists + static_cast<size_t>(slot) * wk.cap;
        uint32_t* next = wk.lists + static_cast<size_t>(nslot) * wk.cap;
        // claims: warp gw takes item gw, later items by atomic (heavy tiles first in round 0)
        for (uint32_t i = gw; i < total;) {
            const uint32_t item = __ldcg(i < nheavy ? wk.heavy + i : list + (i - nheavy));
            const int e = static_cast<int>(item) / ntiles, t = static_cast<int>(item) - e * ntiles;
            const bool skip = e ? done[1] : done[0];
            if (!skip) {
                bool remains = false;
                const unsigned long long tt0 = gtimer();
                process_tile<STRIDE>(eyes.e[e], t % tiles_x, t / tiles_x, w, h, round, epoch, S, s_magic, vec != 0,
                             ctl + (e * 3 + slot) * (kPasses + 1), remains);
                const unsigned long long tt1 = gtimer();
                (e ? busy[1] : busy[0]) += tt1 - tt0;  // selects keep both in registers
                if (rdbg && round < kDbgRounds && lane == 0) {
                    atomicMax(rdbg + 4 * round + 1, tt1);
                    atomicMax(rdbg + 4 * round + 2, tt1 - tt0);
                    atomicAdd(rdbg + 4 * round + 3, 1ull);
                }
                if (remains && lane == 0) {
                    const uint32_t pos = atomicAdd(&wk.counters[2 * nslot], 1u);
                    next[pos] = item;
                }
            }
            if (total <= nw) break;  // every item had its own warp
            uint32_t c = 0;
            if (lane == 0) c = atomicAdd(&wk.counters[2 * slot + 1], 1u);
            i = __shfl_sync(0xFFFFFFFFu, c, 0) + nw;
        }
        grid_barrier(ctl + kBarWord, epoch_bar);
        uint32_t cts[2][kPasses + 1];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
#pragma unroll
            for (int k = 1; k <= kPasses; ++k)
                cts[e][k] = done[e] ? 0u : __ldcg(ctl + (e * 3 + slot) * (kPasses + 1) + k);
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            if (done[e]) continue;
            bool stalled = false;
            for (int k = 1; k <= kPasses; ++k) {
                const long long rep = cts[e][k];
                if (rep == 0) {  // first pass with no repair while damage remains
                    passes[e] += k;
                    stalled = true;
                    break;
                }
                remaining[e] -= rep;
                if (remaining[e] == 0) {
                    passes[e] += k;
                    done[e] = true;
                    break;
                }
            }
            if (done[e]) continue;
            if (stalled) {
                // fixed point reached: fill what is left with mid-gray (inpaint.cpp:112-127)
                const InpaintEye& io = eyes.e[e].io;
                for (uint32_t k = gtid; k < cnt[e]; k += gsize) {
                    const uint32_t idx = io.list[k];
                    const int x = static_cast<int>(idx % static_cast<uint32_t>(w));
                    const int y = static_cast<int>(idx / static_cast<uint32_t>(w));
                    // damage as of the end of this round (tags <= round + 1)
                    if (!((word_state(eyes.e[e], y, x >> 5, h, round + 1, epoch) >> (x & 31)) & 1u)) continue;
                    const size_t o = static_cast<size_t>(y) * io.pitch + static_cast<size_t>(x) * io.stride;
                    for (int ch = 0; ch < 3; ++ch)
                        if (io.plane[ch]) io.plane[ch][o] = 128;
                }
                fallback[e] = remaining[e];
                done[e] = true;
            } else {
                passes[e] += kPasses;
            }
        }
    }
    // per-eye tile time (stats[6], stats[7]: zeroed before the launch), which splits the one
    // kernel's time into the reference's inpaint_left_ns / inpaint_right_ns
    if (stats && lane == 0 && (busy[0] | busy[1])) {
        unsigned long long* ns = reinterpret_cast<unsigned long long*>(stats + 6);
        if (busy[0]) atomicAdd(ns, busy[0]);
        if (busy[1]) atomicAdd(ns + 1, busy[1]);
    }
    if (gtid == 0) wk.counters[16] = (epoch + 1u) & ((1u << kEpochBits) - 1u);  // read by all at start
    if (rdbg && gtid == 0) {
        rdbg[4 * kDbgRounds] = gtimer();
        rdbg[4 * kDbgRounds + 1] = t_start;
    }
    if (gtid == 0 && stats) {
        for (int e = 0; e < 2; ++e) {
            stats[3 * e + 0] = passes[e];
            stats[3 * e + 1] = static_cast<long long>(cnt[e]) - fallback[e];
            stats[3 * e + 2] = fallback[e];
        }
    }
}

}  // namespace

// Damage words of one eye's two slots: 2 * mwords * h u64.
static size_t slot_bytes(int w, int h) {
    return 2 * static_cast<size_t>(h) * ((w + 31) / 32) * 8;
}

size_t inpaint_scratch_bytes(int w, int h) {
    const size_t tiles = static_cast<size_t>((w + kT - 1) / kT) * ((h + kT - 1) / kT);
    // damage slots [2 eyes] | tile counts [2][tiles] | lists [3][2 * tiles] | counters (128 B) |
    // heavy list [2 * tiles]
    return 2 * slot_bytes(w, h) + 2 * tiles * 4 + 3 * 2 * tiles * 4 + 128 + 2 * tiles * 4 + 256;
}

namespace {
// the work-counter words inside the inpaint arena (same layout as inpaint() builds)
uint32_t* work_counters(const InpaintEye& left, Geom gm) {
    const int tiles_x = (gm.w + kT - 1) / kT, tiles_y = (gm.h + kT - 1) / kT;
    const size_t tiles = static_cast<size_t>(tiles_x) * tiles_y;
    unsigned char* flags = reinterpret_cast<unsigned char*>(left.repair) + 2 * slot_bytes(gm.w, gm.h);
    return reinterpret_cast<uint32_t*>(flags + 2 * tiles * 4 + 3 * 2 * tiles * 4);
}
}  // namespace

cudaError_t inpaint_zero(InpaintEye left, Geom gm, uint32_t* scratch, long long* stats,
                         cudaStream_t st, bool by_kernel) {
    ZeroRanges z{};
    z.p[0] = scratch;
    z.words[0] = kCtlWords;
    z.p[1] = work_counters(left, gm);  // [0..15]; [16] (the launch epoch) persists
    z.words[1] = 16;
    z.p[2] = stats ? stats + 6 : nullptr;  // per-eye busy ns
    z.words[2] = stats ? 4u : 0u;
    z.n = 3;
    return zero(z, st, by_kernel);
}

cudaError_t inpaint(InpaintEye left, InpaintEye right, Geom gm, uint32_t capacity,
                    uint32_t* scratch, long long* stats, cudaStream_t st, int max_ctas,
                    int zero_mode) {
    (void)capacity;
    // scratch: ctl (kCtlWords u32, zeroed here: pass counts + the barrier counter); the damage
    // slots, tile flags and work lists live in the engine-provided inpaint arena
    // (InpaintEye.repair of the left eye points at it; see engine.cpp).
    const int tiles_x = (gm.w + kT - 1) / kT, tiles_y = (gm.h + kT - 1) / kT;
    const size_t tiles = static_cast<size_t>(tiles_x) * tiles_y;
    unsigned char* arena = reinterpret_cast<unsigned char*>(left.repair);
    const size_t sb = slot_bytes(gm.w, gm.h), half = sb / 2;
    const int mw = (gm.w + 31) / 32;
    Eyes E;
    E.e[0] = Eye{left, {reinterpret_cast<unsigned long long*>(arena), reinterpret_cast<unsigned long long*>(arena + half)}, mw};
    E.e[1] = Eye{right, {reinterpret_cast<unsigned long long*>(arena + sb), reinterpret_cast<unsigned long long*>(arena + sb + half)}, mw};
    unsigned char* flags = arena + 2 * sb;
    Work wk;
    wk.init_flags = reinterpret_cast<uint32_t*>(flags);
    wk.lists = reinterpret_cast<uint32_t*>(flags + 2 * tiles * 4);
    wk.counters = reinterpret_cast<uint32_t*>(flags + 2 * tiles * 4 + 3 * 2 * tiles * 4);
    wk.heavy = reinterpret_cast<uint32_t*>(flags + 2 * tiles * 4 + 3 * 2 * tiles * 4 + 128);
    wk.cap = static_cast<int>(2 * tiles);
    if (zero_mode != 2) {
        const cudaError_t e = inpaint_zero(left, gm, scratch, stats, st, zero_mode == 1);
        if (e != cudaSuccess) return e;
    }
    const size_t smem = kWarps * sizeof(WarpSmem);
    static std::atomic<unsigned long long> configured{0};
    once_per_device(configured, [smem] {
        cudaFuncSetAttribute(k_inpaint_tiles<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
        cudaFuncSetAttribute(k_inpaint_tiles<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
    });
    int per_sm = 0;
    if (left.stride != right.stride || (left.stride != 1 && left.stride != 3)) return cudaErrorInvalidValue;
    void* kern = left.stride == 3 ? reinterpret_cast<void*>(k_inpaint_tiles<3>)
                                  : reinterpret_cast<void*>(k_inpaint_tiles<1>);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
    if (per_sm < 1) return cudaErrorLaunchOutOfResources;
    int blocks = per_sm * sm_count();
    if (max_ctas > 0 && max_ctas < blocks) blocks = max_ctas;
    int w = gm.w, h = gm.h, tx = tiles_x, ty = tiles_y;
    // 16-byte colour loads need every produced plane and the pitch 16-byte aligned
    int vec = (left.pitch % 16 == 0 && right.pitch % 16 == 0) ? 1 : 0;
    for (int c = 0; c < 3; ++c)
        for (const InpaintEye* io : {&left, &right})
            if (io->plane[c] && (reinterpret_cast<uintptr_t>(io->plane[c] - (io->stride == 3 ? c : 0)) & 15)) vec = 0;
    void* args[] = {&E, &wk, &w, &h, &tx, &ty, &scratch, &stats, &vec};
    const bool want = getenv("P3S_DEBUG_INPAINT") != nullptr;
    static unsigned long long* rdbg = nullptr;
    if (want && !rdbg) {
        cudaMalloc(&rdbg, (4 * kDbgRounds + 4) * sizeof(unsigned long long));
        cudaMemcpyToSymbol(g_inp_rdbg, &rdbg, sizeof(rdbg));
    }
    if (want) cudaMemsetAsync(rdbg, 0, (4 * kDbgRounds + 4) * sizeof(unsigned long long), st);
    note_launch(st);
    cudaError_t e = cudaLaunchCooperativeKernel(kern, dim3(blocks),
                                    dim3(kThreads), args, smem, st);
#ifdef P3S_INPAINT_PHASES
    if (e == cudaSuccess) {
        unsigned long long ph[20];
        cudaStreamSynchronize(st);
        cudaMemcpyFromSymbol(ph, g_phase, sizeof(ph));
        const double tl = ph[7] ? static_cast<double>(ph[7]) : 1.0, ps = ph[8] ? static_cast<double>(ph[8]) : 1.0;
        const double ghz = ph[10] ? static_cast<double>(ph[11]) / ph[10] : 0.0;
        fprintf(stderr, "[p3s] inpaint phases (rounds >= 1, %llu warp tiles, %.2f passes/tile, %.1f%% list-mode, "
                        "SM %.3f GHz, %.1f us/tile): cycles per tile: words %.0f, colour rows %.0f, tail %.0f; "
                        "per pass: decide %.0f, colours %.0f, update %.0f\n",
                ph[7], ps / tl, 100.0 * ph[9] / ps, ghz, ph[10] / tl / 1e3, ph[0] / tl, ph[1] / tl, ph[6] / tl,
                ph[2] / ps, (ph[3] + ph[4]) / ps, ph[5] / ps);
        fprintf(stderr, "[p3s] inpaint probe: colour rows: issue %.0f, first unit %.0f, rest %.0f cycles\n",
                ph[14] / tl, ph[15] / tl, ph[16] / tl);
        const unsigned long long zz[20] = {};
        cudaMemcpyToSymbol(g_phase, zz, sizeof(zz));
    }
#endif
    if (want && e == cudaSuccess) {
        cudaStreamSynchronize(st);
        std::vector<unsigned long long> rb(4 * kDbgRounds + 4);
        cudaMemcpy(rb.data(), rdbg, rb.size() * 8, cudaMemcpyDeviceToHost);
        const unsigned long long tk = rb[4 * kDbgRounds + 1];
        fprintf(stderr, "[p3s] inpaint init: %.1f us\n", rb[0] > tk ? (rb[0] - tk) / 1e3 : 0.0);
        for (int r = 0; r < kDbgRounds && rb[4 * r]; ++r) {
            const unsigned long long t0 = rb[4 * r];
            const unsigned long long t1 = (r + 1 < kDbgRounds && rb[4 * (r + 1)]) ? rb[4 * (r + 1)] : rb[4 * kDbgRounds];
            fprintf(stderr, "[p3s] inpaint round %2d: %6.1f us (tiles done at %6.1f us, max tile %6.1f us, %llu tiles)\n",
                    r, (t1 - t0) / 1e3, rb[4 * r + 1] > t0 ? (rb[4 * r + 1] - t0) / 1e3 : 0.0, rb[4 * r + 2] / 1e3,
                    rb[4 * r + 3]);
        }
    }
    return e;
}

}  // namespace cu
}  // namespace p3s
