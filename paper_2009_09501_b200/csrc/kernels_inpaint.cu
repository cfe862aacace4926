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
// pass-start colours of its intact neighbours in shared memory.
//
// Cross-tile state is the damage of each 32-pixel row word of a tile interior as it stands
// at the end of a round: a 64-bit word (tag << 32 | damage bits), tag = round + 1, kept in
// two slots per word. Round r writes slot r & 1 (round 0 writes both, so no word of a
// damaged tile keeps another frame's content); a tile starting round r takes, per word, the
// slot with the largest tag <= r, i.e. the state at the end of round r - 1. Slot (r - 1) & 1
// is stable during round r, and slot r & 1 only ever goes from an older tag to r + 1, so the
// racy reads are harmless and ONE grid barrier per round suffices. A region row needs three
// of these words (6 independent loads), where per-pixel state words needed a serial chain
// of up to 64 L2 round trips per row in a dense strip. Per-pass global repair counts (interior pixels only)
// reproduce the reference's global stall rule and pass statistics exactly. Tiles are taken
// from a per-round work list with one atomic per claim (dynamic load balance).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "p3s_cu.h"

namespace cg = cooperative_groups;

namespace p3s {
namespace cu {
namespace {

constexpr int kT = 32;                 // tile side (interior)
constexpr int kPasses = 16;            // passes per round = halo width
constexpr int kE = kT + 2 * kPasses;   // region side (64: one u64 per row)
constexpr int kWarps = 8;              // one tile per warp
constexpr int kThreads = 32 * kWarps;
constexpr uint32_t kHeavy = 128;       // damaged pixels that make a tile "heavy"

struct Eye {
    InpaintEye io;
    unsigned long long* slot[2];  // [h][mwords] tagged damage words of tile interiors
    int mwords;                   // (w + 31) / 32
};

// Damage bits of word wi of row gy as of the end of round r - 1 (largest tag <= r); all ones
// when neither slot holds such a word (a word without initial damage: the caller ANDs it with
// the initial mask, which is 0 there).
__device__ __forceinline__ unsigned word_state(const Eye& E, int gy, int wi, int r) {
    if (wi < 0 || wi >= E.mwords) return 0u;
    const size_t o = static_cast<size_t>(gy) * E.mwords + wi;
    const unsigned long long a = __ldcg(E.slot[0] + o), b = __ldcg(E.slot[1] + o);
    const unsigned ta = static_cast<unsigned>(a >> 32), tb = static_cast<unsigned>(b >> 32);
    const bool va = ta - 1u < static_cast<unsigned>(r), vb = tb - 1u < static_cast<unsigned>(r);
    if (va && (!vb || ta >= tb)) return static_cast<unsigned>(a);
    if (vb) return static_cast<unsigned>(b);
    return 0xFFFFFFFFu;
}

// Publishes the interior word of region row r (image row gy) at the end of round `round`.
__device__ __forceinline__ void publish_word(const Eye& E, int gy, int tx, int round,
                                             unsigned long long dregion) {
    const unsigned long long v = (static_cast<unsigned long long>(round + 1) << 32) |
                                 ((dregion >> kPasses) & 0xFFFFFFFFull);
    const size_t o = static_cast<size_t>(gy) * E.mwords + tx;
    __stcg(E.slot[round & 1] + o, v);
    if (round == 0) __stcg(E.slot[1] + o, v);
}

struct Work {
    uint32_t* init_flags;  // [2][tiles] damaged-pixel count per tile (initial work list)
    uint32_t* heavy;       // [2 * tiles] tiles with >= kHeavy damaged pixels (run first)
    uint32_t* lists;       // [3][2 * tiles] (eye * tiles + tile)
    uint32_t* counters;    // [3][2]: count, claim
    int cap;               // 2 * tiles
};

struct WarpSmem {
    uint8_t col[3][kE][kE];      // colours (valid on intact pixels next to damage)
    unsigned long long dmg[kE];  // current damage bits per region row
    unsigned long long img[kE];  // in-image bits per region row
    uint16_t rep[kE * kE];       // the pass's repaired pixels (row << 6 | column)
};

// 64 damage bits of row gy starting at column gx0 (may be negative / past the width).
__device__ __forceinline__ unsigned long long row_bits(const InpaintEye& e, int gx0, int gy, int w,
                                                       unsigned long long& inimg) {
    unsigned long long inb = 0, m = 0;
    for (int j = 0; j < 64; j += 32) {
        unsigned lo = 0, in32 = 0;
        const int c0 = gx0 + j;
        if (e.mask_bits) {
            const int wi = c0 >> 5;  // floor division (c0 may be negative)
            const int sh = c0 & 31;
            const int words = (w + 31) >> 5;
            const uint32_t* rowp = e.mask_bits + static_cast<size_t>(gy) * e.mask_pitch;
            const unsigned a = (wi >= 0 && wi < words) ? __ldg(rowp + wi) : 0u;
            const unsigned b = (wi + 1 >= 0 && wi + 1 < words) ? __ldg(rowp + wi + 1) : 0u;
            lo = sh ? ((a >> sh) | (b << (32 - sh))) : a;
        } else {
            for (int k = 0; k < 32; ++k) {
                const int c = c0 + k;
                if (c >= 0 && c < w && __ldg(e.mask_bytes + static_cast<size_t>(gy) * e.mask_pitch + c))
                    lo |= 1u << k;
            }
        }
        const int lo_c = max(0, -c0), hi_c = min(32, w - c0);  // in-image columns [lo_c, hi_c)
        if (hi_c > lo_c)
            in32 = (hi_c - lo_c == 32 ? 0xFFFFFFFFu : ((1u << (hi_c - lo_c)) - 1u)) << lo_c;
        lo &= in32;
        m |= static_cast<unsigned long long>(lo) << j;
        inb |= static_cast<unsigned long long>(in32) << j;
    }
    inimg = inb;
    return m;
}

// Loads the 64 colour bytes of region row r (image row gy, columns x0 .. x0+63) of the
// channels the route needs. x0 is a multiple of 16; aligned planes use 16-byte loads.
__device__ __forceinline__ void load_row(const InpaintEye& io, WarpSmem& S, int r, int gy, int x0,
                                         int w) {
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        const uint8_t* pl = io.plane[ch];
        if (!pl) continue;
        const uint8_t* src = pl + static_cast<size_t>(gy) * io.pitch;
        const bool vec = ((reinterpret_cast<uintptr_t>(pl) | static_cast<uintptr_t>(io.pitch)) & 15) == 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int c = x0 + 16 * q;
            if (c + 16 <= 0 || c >= w) continue;
            if (vec && c >= 0 && c + 16 <= io.pitch) {
                *reinterpret_cast<uint4*>(&S.col[ch][r][16 * q]) = __ldcg(reinterpret_cast<const uint4*>(src + c));
            } else {
                for (int k = 0; k < 16; ++k)
                    if (c + k >= 0 && c + k < w) S.col[ch][r][16 * q + k] = src[c + k];
            }
        }
    }
}

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

#ifdef P3S_INPAINT_PHASES
// experiment build only (make VARIANT=phases EXTRA=-DP3S_INPAINT_PHASES): per-phase ns of
// the warp tiles of rounds >= 1, summed: [0] words, [1] colour rows, [2] pass decide,
// [3] compaction, [4] colours, [5] publish/update, [6] tail, [7] tiles, [8] passes
__device__ unsigned long long g_phase[16];
__device__ __forceinline__ unsigned long long ptimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define PH_MARK(i)                                                            \
    do {                                                                      \
        __syncwarp();                                                         \
        const unsigned long long _n = ptimer();                               \
        if (round > 0 && (threadIdx.x & 31) == 0) atomicAdd(&g_phase[i], _n - _pt); \
        _pt = _n;                                                             \
    } while (0)
#else
#define PH_MARK(i) \
    do {           \
    } while (0)
#endif

// One warp simulates up to kPasses Jacobi passes of one tile (+ halo) in shared memory.
__device__ void process_tile(const Eye& E, int tx, int ty, int w, int h, int round, WarpSmem& S,
                             uint32_t* counts_slot, bool& remains) {
    const InpaintEye& io = E.io;
    const int lane = threadIdx.x & 31;
    const int x0 = tx * kT - kPasses, y0 = ty * kT - kPasses;
    const unsigned long long kInner = 0x0000FFFFFFFF0000ull;  // interior columns 16..47
#ifdef P3S_INPAINT_PHASES
    unsigned long long _pt = ptimer();
    if (round > 0 && lane == 0) atomicAdd(&g_phase[7], 1ull);
#endif

    // 1. damage / in-image words; in later rounds, pixels repaired in earlier rounds (the
    //    tagged interior words of the end of round - 1) are intact
    unsigned long long d[2], img[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int r = lane + 32 * j, gy = y0 + r;
        unsigned long long in = 0, m = 0;
        if (gy >= 0 && gy < h) m = row_bits(io, x0, gy, w, in);
        if (round > 0 && m) {
            // region columns 0..15 = bits 16..31 of word tx - 1, 16..47 = word tx,
            // 48..63 = bits 0..15 of word tx + 1
            const unsigned a = word_state(E, gy, tx - 1, round), b = word_state(E, gy, tx, round),
                           c = word_state(E, gy, tx + 1, round);
            m &= static_cast<unsigned long long>(a >> 16) | (static_cast<unsigned long long>(b) << 16) |
                 (static_cast<unsigned long long>(c & 0xFFFFu) << 48);
        }
        d[j] = m;
        img[j] = in;
        S.dmg[r] = m;
        S.img[r] = in;
    }
    __syncwarp();
    PH_MARK(0);
    // 2. colours of every row next to damage (intact pixels there feed the means)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int r = lane + 32 * j, gy = y0 + r;
        const unsigned long long near = d[j] | (r > 0 ? S.dmg[r - 1] : 0) | (r + 1 < kE ? S.dmg[r + 1] : 0);
        if (near && gy >= 0 && gy < h) load_row(io, S, r, gy, x0, w);
    }
    __syncwarp();
    PH_MARK(1);
    // 3. passes
    for (int k = 1; k <= kPasses; ++k) {
        unsigned long long rep[2], iu[2], im[2], id[2];
        int inner = 0, any = 0;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int r = lane + 32 * j;
            iu[j] = r > 0 ? S.img[r - 1] & ~S.dmg[r - 1] : 0ull;
            im[j] = img[j] & ~d[j];
            id[j] = r + 1 < kE ? S.img[r + 1] & ~S.dmg[r + 1] : 0ull;
            rep[j] = d[j] & two_plus(iu[j], im[j], id[j]);
            any |= rep[j] != 0;
            if (r >= kPasses && r < kPasses + kT) inner += __popcll(rep[j] & kInner);
        }
        if (!__any_sync(0xFFFFFFFFu, any)) break;  // fixed point of the region
#ifdef P3S_INPAINT_PHASES
        if (round > 0 && lane == 0) atomicAdd(&g_phase[8], 1ull);
#endif
        PH_MARK(2);
        // compact the pass's repairs into one list so the colour work spreads over the lanes
        const int cnt = __popcll(rep[0]) + __popcll(rep[1]);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += v;
        }
        const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
        {
            int pos = incl - cnt;
#pragma unroll
            for (int j = 0; j < 2; ++j)
                for (unsigned long long b = rep[j]; b; b &= b - 1)
                    S.rep[pos++] = static_cast<uint16_t>(((lane + 32 * j) << 6) | (__ffsll(static_cast<long long>(b)) - 1));
        }
        __syncwarp();
        PH_MARK(3);
        // colours from the pass-start intact neighbours (S.dmg is still the pass-start
        // state; a repaired pixel is never an intact neighbour in its own pass, so the
        // in-place writes cannot be read by another lane in this pass)
        for (int i = lane; i < total; i += 32) {
            const int e = S.rep[i], r = e >> 6, c = e & 63;
            const unsigned long long iw[3] = {r > 0 ? S.img[r - 1] & ~S.dmg[r - 1] : 0ull,
                                              S.img[r] & ~S.dmg[r],
                                              r + 1 < kE ? S.img[r + 1] & ~S.dmg[r + 1] : 0ull};
            unsigned cntn = 0, a0 = 0, a1 = 0, a2 = 0;
#pragma unroll
            for (int dy = -1; dy <= 1; ++dy) {
#pragma unroll
                for (int dx = -1; dx <= 1; ++dx) {
                    if (!dx && !dy) continue;
                    const int cc = c + dx;
                    if (cc < 0 || cc >= kE || !((iw[dy + 1] >> cc) & 1ull)) continue;
                    ++cntn;
                    if (io.plane[0]) a0 += S.col[0][r + dy][cc];
                    if (io.plane[1]) a1 += S.col[1][r + dy][cc];
                    if (io.plane[2]) a2 += S.col[2][r + dy][cc];
                }
            }
            if (io.plane[0]) S.col[0][r][c] = static_cast<uint8_t>((2 * a0 + cntn) / (2 * cntn));
            if (io.plane[1]) S.col[1][r][c] = static_cast<uint8_t>((2 * a1 + cntn) / (2 * cntn));
            if (io.plane[2]) S.col[2][r][c] = static_cast<uint8_t>((2 * a2 + cntn) / (2 * cntn));
        }
        __syncwarp();
        PH_MARK(4);
        // interior repairs: publish colour + state word
        for (int i = lane; i < total; i += 32) {
            const int e = S.rep[i], r = e >> 6, c = e & 63;
            if (r < kPasses || r >= kPasses + kT || c < kPasses || c >= kPasses + kT) continue;
            const int gy = y0 + r, gx = x0 + c;
            const uint8_t c0 = S.col[0][r][c], c1 = S.col[1][r][c], c2 = S.col[2][r][c];
            const size_t o = static_cast<size_t>(gy) * io.pitch + gx;
            if (io.plane[0]) io.plane[0][o] = c0;
            if (io.plane[1]) io.plane[1][o] = c1;
            if (io.plane[2]) io.plane[2][o] = c2;
        }
        inner = __reduce_add_sync(0xFFFFFFFFu, inner);
        if (lane == 0 && inner) atomicAdd(&counts_slot[k], static_cast<uint32_t>(inner));
        __syncwarp();
        int inner_left = 0;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            d[j] &= ~rep[j];
            S.dmg[lane + 32 * j] = d[j];
            const int r = lane + 32 * j;
            if (r >= kPasses && r < kPasses + kT) inner_left |= (d[j] & kInner) != 0;
        }
        __syncwarp();
        PH_MARK(5);
        // interior complete: its pixels never change again (repairs are final), so later
        // passes add no interior repairs; the halo's evolution is discarded anyway
        if (!__any_sync(0xFFFFFFFFu, inner_left)) break;
    }
    PH_MARK(2);
    // 4. publish the interior's damage words; interior damage left -> the tile runs again
    int left = 0;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int r = lane + 32 * j, gy = y0 + r;
        if (r >= kPasses && r < kPasses + kT) {
            left |= (d[j] & kInner) != 0;
            if (gy < h) publish_word(E, gy, tx, round, d[j]);
        }
    }
    remains = __any_sync(0xFFFFFFFFu, left);
    __syncwarp();
    PH_MARK(6);
}

// Round-0 version of process_tile for heavy tiles: the whole CTA (kThreads threads) works
// on one region (warp 0's shared-memory slot), so the per-pass colour and publish work of a
// dense hole strip is spread over 8 warps instead of 1. Same simulation, same results; only
// the thread mapping differs (region rows on threads 0..63, the repair list on all threads).
__device__ void process_tile_cta(const Eye& E, int tx, int ty, int w, int h, WarpSmem& S,
                                 uint32_t* counts_slot, bool& remains) {
    const InpaintEye& io = E.io;
    const int tid = threadIdx.x;
    const int x0 = tx * kT - kPasses, y0 = ty * kT - kPasses;
    const unsigned long long kInner = 0x0000FFFFFFFF0000ull;  // interior columns 16..47
    // double-buffered pass counters: buffer k & 1 is reset during pass k - 1
    __shared__ int s_total[2], s_inner[2];
    const bool rowt = tid < kE;
    const bool inner_row = tid >= kPasses && tid < kPasses + kT;
    if (tid == 0) {
        s_total[1] = 0;
        s_inner[1] = 0;
    }
    unsigned long long d = 0, img = 0;
    if (rowt) {
        const int gy = y0 + tid;
        unsigned long long in = 0, m = 0;
        if (gy >= 0 && gy < h) m = row_bits(io, x0, gy, w, in);
        d = m;
        img = in;
        S.dmg[tid] = m;
        S.img[tid] = in;
    }
    __syncthreads();
    if (rowt) {
        const int r = tid, gy = y0 + r;
        const unsigned long long near = d | (r > 0 ? S.dmg[r - 1] : 0) | (r + 1 < kE ? S.dmg[r + 1] : 0);
        if (near && gy >= 0 && gy < h) load_row(io, S, r, gy, x0, w);
    }
    __syncthreads();
    for (int k = 1; k <= kPasses; ++k) {
        const int b = k & 1;
        unsigned long long rep = 0;
        if (rowt) {
            const int r = tid;
            const unsigned long long iu = r > 0 ? S.img[r - 1] & ~S.dmg[r - 1] : 0ull;
            const unsigned long long id = r + 1 < kE ? S.img[r + 1] & ~S.dmg[r + 1] : 0ull;
            rep = d & two_plus(iu, img & ~d, id);
            const int cnt = __popcll(rep);
            if (cnt) {
                int pos = atomicAdd(&s_total[b], cnt);  // list order is irrelevant (Jacobi pass)
                for (unsigned long long q = rep; q; q &= q - 1)
                    S.rep[pos++] = static_cast<uint16_t>((r << 6) | (__ffsll(static_cast<long long>(q)) - 1));
                if (inner_row && (rep & kInner)) atomicAdd(&s_inner[b], __popcll(rep & kInner));
            }
        }
        if (!__syncthreads_or(rep != 0)) break;  // fixed point of the region
        const int total = s_total[b];
        if (tid == 0) {
            s_total[b ^ 1] = 0;
            s_inner[b ^ 1] = 0;
        }
        for (int i = tid; i < total; i += blockDim.x) {
            const int e = S.rep[i], r = e >> 6, c = e & 63;
            const unsigned long long iw[3] = {r > 0 ? S.img[r - 1] & ~S.dmg[r - 1] : 0ull,
                                              S.img[r] & ~S.dmg[r],
                                              r + 1 < kE ? S.img[r + 1] & ~S.dmg[r + 1] : 0ull};
            unsigned cntn = 0, a0 = 0, a1 = 0, a2 = 0;
#pragma unroll
            for (int dy = -1; dy <= 1; ++dy) {
#pragma unroll
                for (int dx = -1; dx <= 1; ++dx) {
                    if (!dx && !dy) continue;
                    const int cc = c + dx;
                    if (cc < 0 || cc >= kE || !((iw[dy + 1] >> cc) & 1ull)) continue;
                    ++cntn;
                    if (io.plane[0]) a0 += S.col[0][r + dy][cc];
                    if (io.plane[1]) a1 += S.col[1][r + dy][cc];
                    if (io.plane[2]) a2 += S.col[2][r + dy][cc];
                }
            }
            if (io.plane[0]) S.col[0][r][c] = static_cast<uint8_t>((2 * a0 + cntn) / (2 * cntn));
            if (io.plane[1]) S.col[1][r][c] = static_cast<uint8_t>((2 * a1 + cntn) / (2 * cntn));
            if (io.plane[2]) S.col[2][r][c] = static_cast<uint8_t>((2 * a2 + cntn) / (2 * cntn));
        }
        __syncthreads();
        for (int i = tid; i < total; i += blockDim.x) {
            const int e = S.rep[i], r = e >> 6, c = e & 63;
            if (r < kPasses || r >= kPasses + kT || c < kPasses || c >= kPasses + kT) continue;
            const int gy = y0 + r, gx = x0 + c;
            const uint8_t c0 = S.col[0][r][c], c1 = S.col[1][r][c], c2 = S.col[2][r][c];
            const size_t o = static_cast<size_t>(gy) * io.pitch + gx;
            if (io.plane[0]) io.plane[0][o] = c0;
            if (io.plane[1]) io.plane[1][o] = c1;
            if (io.plane[2]) io.plane[2][o] = c2;
        }
        if (tid == 0 && s_inner[b]) atomicAdd(&counts_slot[k], static_cast<uint32_t>(s_inner[b]));
        if (rowt) {
            d &= ~rep;
            S.dmg[tid] = d;
        }
        // interior complete: later passes add no interior repairs (see process_tile)
        if (!__syncthreads_or(inner_row && (d & kInner))) break;
    }
    if (inner_row && y0 + tid < h) publish_word(E, y0 + tid, tx, 0, d);
    remains = __syncthreads_or(inner_row && (d & kInner)) != 0;
}

// Debug timeline (P3S_DEBUG_INPAINT): per warp, globaltimer ns at the phase boundaries of
// round 0 plus tile statistics. nullptr in normal runs.
__device__ unsigned long long* g_inp_dbg = nullptr;
// per-round debug (P3S_DEBUG_INPAINT): [kDbgRounds][4] = round start (block 0, after the
// barrier), latest warp finish of the round's tiles, max tile ns, tiles processed
constexpr int kDbgRounds = 64;
__device__ unsigned long long* g_inp_rdbg = nullptr;
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__global__ void __launch_bounds__(kThreads, 1) k_inpaint_tiles(Eye L, Eye R, Work wk, int w, int h,
                                                               int tiles_x, int tiles_y,
                                                               uint32_t* ctl, long long* stats) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WarpSmem& S = reinterpret_cast<WarpSmem*>(smem_raw)[threadIdx.x >> 5];
    const int ntiles = tiles_x * tiles_y;
    unsigned long long* dbg = g_inp_dbg;
    unsigned long long dt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (dbg) dt[0] = gtimer();
    const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t gsize = gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    Eye eyes[2] = {L, R};

    // init: state words of damaged pixels = 0; tiles holding damage -> work list 0
    uint32_t cnt[2];
    for (int e = 0; e < 2; ++e) {
        cnt[e] = __ldcg(eyes[e].io.count);
        for (uint32_t k = gtid; k < cnt[e]; k += gsize) {
            const uint32_t idx = eyes[e].io.list[k];
            const int x = static_cast<int>(idx % static_cast<uint32_t>(w));
            const int y = static_cast<int>(idx / static_cast<uint32_t>(w));
            const int t = (y / kT) * tiles_x + x / kT;
            const uint32_t old = atomicAdd(&wk.init_flags[e * ntiles + t], 1u);
            if (old + 1 == kHeavy) {  // round 0 starts with these (longest first)
                const uint32_t pos = atomicAdd(&wk.counters[6], 1u);
                wk.heavy[pos] = static_cast<uint32_t>(e * ntiles + t);
            }
            if (old == 0u) {
                const uint32_t pos = atomicAdd(&wk.counters[0], 1u);
                wk.lists[pos] = static_cast<uint32_t>(e * ntiles + t);
            }
        }
    }
    long long remaining[2] = {cnt[0], cnt[1]};
    bool done[2] = {cnt[0] == 0, cnt[1] == 0};
    long long passes[2] = {0, 0}, fallback[2] = {0, 0};
    if (dbg) dt[1] = gtimer();
    grid.sync();
    if (dbg) dt[2] = gtimer();

    // ctl layout: [eye][slot 0..2][kPasses + 1] pass counts
    unsigned long long* rdbg = g_inp_rdbg;
    for (int round = 0; !(done[0] && done[1]); ++round) {
        const int slot = round % 3, nslot = (round + 1) % 3, rslot = (round + 2) % 3;
        if (rdbg && round < kDbgRounds && blockIdx.x == 0 && threadIdx.x == 0) rdbg[4 * round] = gtimer();
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
        const uint32_t* list = wk.lists + static_cast<size_t>(slot) * wk.cap;
        uint32_t* next = wk.lists + static_cast<size_t>(nslot) * wk.cap;
        if (round == 0) {
            // heavy tiles first, one whole CTA per tile (counters[7] = CTA claim index)
            __shared__ uint32_t s_claim;
            WarpSmem& S0 = reinterpret_cast<WarpSmem*>(smem_raw)[0];
            for (;;) {
                if (threadIdx.x == 0) s_claim = atomicAdd(&wk.counters[7], 1u);
                __syncthreads();
                const uint32_t i = s_claim;
                __syncthreads();
                if (i >= nheavy) break;
                const uint32_t item = __ldcg(wk.heavy + i);
                const int e = static_cast<int>(item) / ntiles, t = static_cast<int>(item) - e * ntiles;
                if (done[e]) continue;
                bool remains = false;
                const unsigned long long tt0 = (dbg || rdbg) ? gtimer() : 0;
                process_tile_cta(e ? R : L, t % tiles_x, t / tiles_x, w, h, S0,
                                 ctl + (e * 3 + slot) * (kPasses + 1), remains);
                if (dbg && (threadIdx.x & 31) == 0) {
                    const unsigned long long dd = gtimer() - tt0;
                    dt[5] += 1;
                    dt[6] += dd;
                    dt[7] = dd > dt[7] ? dd : dt[7];
                }
                if (rdbg && threadIdx.x == 0) {
                    const unsigned long long now = gtimer();
                    atomicMax(rdbg + 1, now);
                    atomicMax(rdbg + 2, now - tt0);
                    atomicAdd(rdbg + 3, 1ull);
                }
                if (remains && threadIdx.x == 0) {
                    const uint32_t pos = atomicAdd(&wk.counters[2 * nslot], 1u);
                    next[pos] = item;
                }
            }
        }
        for (;;) {
            // round 0 takes the heavy tiles first (they bound the round), then the rest
            uint32_t i = 0;
            if (lane == 0) i = atomicAdd(&wk.counters[2 * slot + 1], 1u);
            i = __shfl_sync(0xFFFFFFFFu, i, 0);
            if (i >= n) break;
            const uint32_t item = __ldcg(list + i);
            if (round == 0 && __ldcg(wk.init_flags + item) >= kHeavy) continue;  // done by a CTA
            const int e = static_cast<int>(item) / ntiles, t = static_cast<int>(item) - e * ntiles;
            if (done[e]) continue;
            bool remains = false;
            const unsigned long long tt0 = (dbg || rdbg) ? gtimer() : 0;
            process_tile(e ? R : L, t % tiles_x, t / tiles_x, w, h, round, S,
                         ctl + (e * 3 + slot) * (kPasses + 1), remains);
            if (rdbg && round < kDbgRounds && lane == 0) {
                const unsigned long long now = gtimer();
                atomicMax(rdbg + 4 * round + 1, now);
                atomicMax(rdbg + 4 * round + 2, now - tt0);
                atomicAdd(rdbg + 4 * round + 3, 1ull);
            }
            if (dbg && round == 0) {
                const unsigned long long d = gtimer() - tt0;
                dt[5] += 1;
                dt[6] += d;
                dt[7] = d > dt[7] ? d : dt[7];
            }
            if (remains && lane == 0) {
                const uint32_t pos = atomicAdd(&wk.counters[2 * nslot], 1u);
                next[pos] = item;
            }
        }
        if (dbg && round == 0) dt[3] = gtimer();
        grid.sync();
        if (dbg && round == 0) {
            dt[4] = gtimer();
            if ((threadIdx.x & 31) == 0) {
                const int gw = blockIdx.x * kWarps + (threadIdx.x >> 5);
                for (int q = 0; q < 8; ++q) dbg[gw * 8 + q] = dt[q];
            }
        }
        for (int e = 0; e < 2; ++e) {
            if (done[e]) continue;
            const uint32_t* c = ctl + (e * 3 + slot) * (kPasses + 1);
            // all of the round's pass counts in one go (one L2 round trip, not one per pass)
            uint32_t cts[kPasses + 1];
#pragma unroll
            for (int k = 1; k <= kPasses; ++k) cts[k] = __ldcg(c + k);
            bool stalled = false;
            for (int k = 1; k <= kPasses; ++k) {
                const long long rep = cts[k];
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
                const InpaintEye& io = eyes[e].io;
                for (uint32_t k = gtid; k < cnt[e]; k += gsize) {
                    const uint32_t idx = io.list[k];
                    const int x = static_cast<int>(idx % static_cast<uint32_t>(w));
                    const int y = static_cast<int>(idx / static_cast<uint32_t>(w));
                    // damage as of the end of this round (tags <= round + 1)
                    if (!((word_state(eyes[e], y, x >> 5, round + 1) >> (x & 31)) & 1u)) continue;
                    const size_t o = static_cast<size_t>(y) * io.pitch + x;
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
    if (rdbg) {  // debug only (uniform across the grid): the end time of the last round
        grid.sync();
        if (gtid == 0) rdbg[4 * kDbgRounds] = gtimer();
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

// Damage words of one eye's two slots: 2 * h * mwords u64.
static size_t slot_bytes(int w, int h) {
    return 2 * static_cast<size_t>(h) * ((w + 31) / 32) * 8;
}

size_t inpaint_scratch_bytes(int w, int h) {
    const size_t tiles = static_cast<size_t>((w + kT - 1) / kT) * ((h + kT - 1) / kT);
    // damage slots [2 eyes] | tile counts [2][tiles] | lists [3][2 * tiles] | counters [4][2] |
    // heavy list [2 * tiles]
    return 2 * slot_bytes(w, h) + 2 * tiles * 4 + 3 * 2 * tiles * 4 + 64 + 2 * tiles * 4 + 256;
}

cudaError_t inpaint(InpaintEye left, InpaintEye right, Geom gm, uint32_t capacity,
                    uint32_t* scratch, long long* stats, cudaStream_t st, int max_ctas,
                    bool zero_by_kernel) {
    (void)capacity;
    // scratch: ctl (2*3*(kPasses+1) u32, zeroed here); the per-pixel state words, tile
    // flags and work lists live in the engine-provided inpaint arena (InpaintEye.repair of
    // the left eye points at it; see engine.cpp).
    const int tiles_x = (gm.w + kT - 1) / kT, tiles_y = (gm.h + kT - 1) / kT;
    const size_t tiles = static_cast<size_t>(tiles_x) * tiles_y;
    unsigned char* arena = reinterpret_cast<unsigned char*>(left.repair);
    const size_t sb = slot_bytes(gm.w, gm.h), half = sb / 2;
    const int mw = (gm.w + 31) / 32;
    Eye L{left, {reinterpret_cast<unsigned long long*>(arena), reinterpret_cast<unsigned long long*>(arena + half)}, mw};
    Eye R{right, {reinterpret_cast<unsigned long long*>(arena + sb), reinterpret_cast<unsigned long long*>(arena + sb + half)}, mw};
    unsigned char* flags = arena + 2 * sb;
    Work wk;
    wk.init_flags = reinterpret_cast<uint32_t*>(flags);
    wk.lists = reinterpret_cast<uint32_t*>(flags + 2 * tiles * 4);
    wk.counters = reinterpret_cast<uint32_t*>(flags + 2 * tiles * 4 + 3 * 2 * tiles * 4);
    wk.heavy = reinterpret_cast<uint32_t*>(flags + 2 * tiles * 4 + 3 * 2 * tiles * 4 + 64);
    wk.cap = static_cast<int>(2 * tiles);
    ZeroRanges z{};
    z.p[0] = scratch;
    z.words[0] = 2 * 3 * (kPasses + 1);
    z.p[1] = flags;
    z.words[1] = static_cast<unsigned>(2 * tiles);
    z.p[2] = wk.counters;
    z.words[2] = 8;
    z.n = 3;
    cudaError_t e = zero(z, st, zero_by_kernel);
    if (e != cudaSuccess) return e;
    const size_t smem = kWarps * sizeof(WarpSmem);
    static std::atomic<unsigned long long> configured{0};
    once_per_device(configured, [smem] {
        cudaFuncSetAttribute(k_inpaint_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
    });
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_inpaint_tiles, kThreads, smem);
    if (per_sm < 1) return cudaErrorLaunchOutOfResources;
    int blocks = per_sm * sm_count();
    if (max_ctas > 0 && max_ctas < blocks) blocks = max_ctas;
    int w = gm.w, h = gm.h, tx = tiles_x, ty = tiles_y;
    void* args[] = {&L, &R, &wk, &w, &h, &tx, &ty, &scratch, &stats};
    static unsigned long long* dbg = nullptr;
    const bool want = getenv("P3S_DEBUG_INPAINT") != nullptr;
    if (want && !dbg) {
        cudaMalloc(&dbg, static_cast<size_t>(blocks) * kWarps * 8 * sizeof(unsigned long long));
        cudaMemcpyToSymbol(g_inp_dbg, &dbg, sizeof(dbg));
    }
    static unsigned long long* rdbg = nullptr;
    if (want && !rdbg) {
        cudaMalloc(&rdbg, (4 * kDbgRounds + 4) * sizeof(unsigned long long));
        cudaMemcpyToSymbol(g_inp_rdbg, &rdbg, sizeof(rdbg));
    }
    if (want) cudaMemsetAsync(rdbg, 0, (4 * kDbgRounds + 4) * sizeof(unsigned long long), st);
    e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_inpaint_tiles), dim3(blocks),
                                    dim3(kThreads), args, smem, st);
#ifdef P3S_INPAINT_PHASES
    if (e == cudaSuccess) {
        unsigned long long ph[16];
        cudaStreamSynchronize(st);
        cudaMemcpyFromSymbol(ph, g_phase, sizeof(ph));
        const double tl = ph[7] ? static_cast<double>(ph[7]) : 1.0, ps = ph[8] ? static_cast<double>(ph[8]) : 1.0;
        fprintf(stderr, "[p3s] inpaint phases (rounds >= 1, %llu warp tiles, %.2f passes/tile): per tile words %.2f us, "
                        "colour rows %.2f us, tail %.2f us; per pass decide %.3f us, compact %.3f us, colours %.3f us, "
                        "publish %.3f us\n",
                ph[7], ps / tl, ph[0] / tl / 1e3, ph[1] / tl / 1e3, ph[6] / tl / 1e3, ph[2] / ps / 1e3, ph[3] / ps / 1e3,
                ph[4] / ps / 1e3, ph[5] / ps / 1e3);
        const unsigned long long z[16] = {};
        cudaMemcpyToSymbol(g_phase, z, sizeof(z));
    }
#endif
    if (want && e == cudaSuccess) {
        cudaStreamSynchronize(st);
        std::vector<unsigned long long> rb(4 * kDbgRounds + 4);
        cudaMemcpy(rb.data(), rdbg, rb.size() * 8, cudaMemcpyDeviceToHost);
        for (int r = 0; r < kDbgRounds && rb[4 * r]; ++r) {
            const unsigned long long t0 = rb[4 * r];
            const unsigned long long t1 = (r + 1 < kDbgRounds && rb[4 * (r + 1)]) ? rb[4 * (r + 1)] : rb[4 * kDbgRounds];
            fprintf(stderr, "[p3s] inpaint round %2d: %6.1f us (tiles done at %6.1f us, max tile %6.1f us, %llu tiles)\n",
                    r, (t1 - t0) / 1e3, rb[4 * r + 1] > t0 ? (rb[4 * r + 1] - t0) / 1e3 : 0.0, rb[4 * r + 2] / 1e3,
                    rb[4 * r + 3]);
        }
    }
    if (want && e == cudaSuccess) {
        cudaStreamSynchronize(st);
        const int nw = blocks * kWarps;
        std::vector<unsigned long long> hb(static_cast<size_t>(nw) * 8);
        cudaMemcpy(hb.data(), dbg, hb.size() * 8, cudaMemcpyDeviceToHost);
        unsigned long long t0 = ~0ull, init = 0, s1 = 0, rnd = 0, s2 = 0, maxtile = 0, tiles = 0, busy = 0;
        for (int i = 0; i < nw; ++i) t0 = std::min(t0, hb[8 * i]);
        for (int i = 0; i < nw; ++i) {
            const unsigned long long* d = &hb[8 * i];
            init = std::max(init, d[1] - t0);
            s1 = std::max(s1, d[2] - t0);
            rnd = std::max(rnd, d[3] - t0);
            s2 = std::max(s2, d[4] - t0);
            tiles += d[5];
            busy += d[6];
            maxtile = std::max(maxtile, d[7]);
        }
        fprintf(stderr, "[p3s] inpaint round0 (ns from first warp start): init done %llu, sync1 %llu, "
                        "tiles done %llu, sync2 %llu; tiles %llu, mean tile %llu ns, max tile %llu ns, "
                        "busy %.1f%%\n", init, s1, rnd, s2, tiles, tiles ? busy / tiles : 0ull, maxtile,
                100.0 * busy / (static_cast<double>(nw) * (rnd - s1 + 1)));
    }
    return e;
}

}  // namespace cu
}  // namespace p3s
