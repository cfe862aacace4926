// K3b: Jacobi hole filling on sm_100a (reference proj/src/inpaint.cpp:29-130).
//
// Semantics kept exactly: every pass decides against the pass-start snapshot (a damaged
// pixel with >= 2 intact 8-neighbours takes the per-channel (2*sum + n) / (2n) mean),
// then applies all repairs; the first pass that repairs nothing while damage remains
// fills the rest with (128,128,128). Both eyes are independent instances
// (pipeline.cpp:56-65) and run in the same launch.
//
// Temporal blocking. The frame is cut into 32x32 tiles; a round runs kPasses Jacobi passes
// of one tile inside shared memory (one warp per tile, 8 tiles per CTA) over the tile plus
// a kPasses-pixel halo. Only damage-mask words and the colours of intact pixels that touch
// damage are read from HBM; a pass with no local repair and no pending neighbour
// repair ends the simulation early (fixed point). Information
// moves one pixel per pass, so after kPasses passes the tile interior equals the global
// Jacobi state (pixels near the halo edge may be wrong, they are discarded). Only tiles
// whose interior still holds damage are processed.
//
// Cross-tile state is one 64-bit word per initially damaged pixel: 0 = damaged, else
// (1 << 63) | global pass of repair << 24 | colour bytes — the final truth, written once
// by the owning tile, read atomically by neighbours. A neighbour that reads a word written
// in the current round simply knows that pixel's future (it becomes intact after that
// pass), which is what its own simulation would have derived; a word still 0 is simulated.
// So one state buffer and ONE grid barrier per round suffice (the old kernel needed two
// barriers per pass). Per-pass global repair counts (interior pixels only) reproduce the
// reference's global stall rule and pass statistics exactly.
#include <cooperative_groups.h>

#include "p3s_cu.h"

namespace cg = cooperative_groups;

namespace p3s {
namespace cu {
namespace {

constexpr int kT = 32;                 // tile side (interior)
constexpr int kPasses = 16;            // passes per round = halo width
constexpr int kE = kT + 2 * kPasses;   // extended side (64: one u64 mask per row)
constexpr int kEN = kE * kE;
constexpr int kWarps = 8;              // one tile per warp
constexpr int kThreads = 32 * kWarps;
constexpr unsigned long long kRepaired = 1ull << 63;

struct Eye {
    InpaintEye io;
    unsigned long long* state;  // per pixel (only initially damaged entries used)
    uint8_t* flags;             // [2][tiles] round flags
};

struct WarpSmem {
    uint8_t st[kEN];            // 0 intact, 1 damaged, k+1 repaired at local pass k (valid only
                                // on damaged pixels and their in-image neighbours)
    uint8_t col[3][kEN];
    uint16_t lst[kEN];          // damaged pixels of the extended region
    unsigned long long dmg[kE]; // initial damage bits per extended row
    unsigned long long img[kE]; // in-image bits per extended row
    int rep[kPasses + 1];
};

// 64 damage bits of row gy starting at column gx0 (may be negative / past the width).
__device__ __forceinline__ unsigned long long row_bits(const InpaintEye& e, int gx0, int gy, int w,
                                                       unsigned long long& inimg) {
    unsigned long long inb = 0, m = 0;
    for (int j = 0; j < 64; j += 32) {
        // bits for columns gx0+j .. gx0+j+31
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
        for (int k = 0; k < 32; ++k) {
            const int c = c0 + k;
            if (c >= 0 && c < w) in32 |= 1u << k;
        }
        lo &= in32;
        m |= static_cast<unsigned long long>(lo) << j;
        inb |= static_cast<unsigned long long>(in32) << j;
    }
    inimg = inb;
    return m;
}

// One warp simulates kPasses Jacobi passes of one tile (+ halo) in its shared memory.
__device__ void process_tile(const Eye& E, int tx, int ty, int w, int h, int round, int tiles_x,
                             WarpSmem& S, uint32_t* counts_slot, uint8_t* next_flags) {
    const InpaintEye& io = E.io;
    const int lane = threadIdx.x & 31;
    const int x0 = tx * kT - kPasses, y0 = ty * kT - kPasses;
    const long long pass0 = static_cast<long long>(round) * kPasses;

    // 1. damage / in-image bits per extended row
    for (int r = lane; r < kE; r += 32) {
        const int gy = y0 + r;
        unsigned long long inimg = 0, m = 0;
        if (gy >= 0 && gy < h) m = row_bits(io, x0, gy, w, inimg);
        S.dmg[r] = m;
        S.img[r] = inimg;
    }
    if (lane <= kPasses) S.rep[lane] = 0;
    __syncwarp();
    // 2. Lists built from the bits alone (no memory round trip): lst[0, n) = the initially
    //    damaged pixels, lst[n, n + nn) = the in-image pixels of their 8-neighbourhood (a
    //    one-pixel dilation of the damage bits). Nothing else in the region is ever read.
    int n = 0, nn = 0;
    {
        // each lane owns rows lane and lane + 32
        unsigned long long md[2], mn[2];
        int cd = 0, cn = 0;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int r = lane + 32 * j;
            const unsigned long long m = S.dmg[r];
            const unsigned long long up = r > 0 ? S.dmg[r - 1] : 0, dn = r + 1 < kE ? S.dmg[r + 1] : 0;
            const unsigned long long near = m | up | dn;
            md[j] = m;
            mn[j] = (near | (near << 1) | (near >> 1)) & S.img[r] & ~m;
            cd += __popcll(md[j]);
            cn += __popcll(mn[j]);
        }
        int id = cd, in_ = cn;  // inclusive warp scans
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int a1 = __shfl_up_sync(0xFFFFFFFFu, id, o);
            const int a2 = __shfl_up_sync(0xFFFFFFFFu, in_, o);
            if (lane >= o) {
                id += a1;
                in_ += a2;
            }
        }
        n = __shfl_sync(0xFFFFFFFFu, id, 31);
        nn = __shfl_sync(0xFFFFFFFFu, in_, 31);
        int pd = id - cd, pn = n + in_ - cn;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int r = lane + 32 * j;
            for (unsigned long long m = md[j]; m; m &= m - 1) S.lst[pd++] = static_cast<uint16_t>(r * kE + __ffsll(m) - 1);
            for (unsigned long long m = mn[j]; m; m &= m - 1) S.lst[pn++] = static_cast<uint16_t>(r * kE + __ffsll(m) - 1);
        }
    }
    __syncwarp();
    // 3. loads, batched so each lane has several independent requests in flight
    int max_future = 0;
    constexpr int kB = 8;
    for (int base = 0; base < n + nn; base += 32 * kB) {
        unsigned long long v[kB];
        uint8_t c0[kB], c1[kB], c2[kB];
#pragma unroll
        for (int j = 0; j < kB; ++j) {
            const int i = base + lane + 32 * j;
            v[j] = 0;
            c0[j] = c1[j] = c2[j] = 0;
            if (i < n + nn) {
                const int e = S.lst[i];
                const int ly = e / kE, lx = e - ly * kE;
                const int gx = x0 + lx, gy = y0 + ly;
                if (i < n) {
                    v[j] = __ldcg(E.state + static_cast<size_t>(gy) * w + gx);
                } else {
                    const size_t o = static_cast<size_t>(gy) * io.pitch + gx;
                    if (io.plane[0]) c0[j] = io.plane[0][o];
                    if (io.plane[1]) c1[j] = io.plane[1][o];
                    if (io.plane[2]) c2[j] = io.plane[2][o];
                }
            }
        }
#pragma unroll
        for (int j = 0; j < kB; ++j) {
            const int i = base + lane + 32 * j;
            if (i >= n + nn) continue;
            const int e = S.lst[i];
            if (i < n) {
                if (v[j] & kRepaired) {
                    const long long g = static_cast<long long>((v[j] >> 24) & 0xFFFFFFFFull);
                    const int sv = g <= pass0 ? 0 : static_cast<int>(g - pass0 + 1);
                    if (sv > max_future) max_future = sv;
                    S.st[e] = static_cast<uint8_t>(sv);
                    S.col[0][e] = static_cast<uint8_t>(v[j]);
                    S.col[1][e] = static_cast<uint8_t>(v[j] >> 8);
                    S.col[2][e] = static_cast<uint8_t>(v[j] >> 16);
                } else {
                    S.st[e] = 1;
                }
            } else {
                S.st[e] = 0;
                S.col[0][e] = c0[j];
                S.col[1][e] = c1[j];
                S.col[2][e] = c2[j];
            }
        }
    }
    for (int o = 16; o; o >>= 1) max_future = max(max_future, __shfl_xor_sync(0xFFFFFFFFu, max_future, o));
    __syncwarp();
    // 3. passes
    for (int k = 1; k <= kPasses; ++k) {
        int local = 0;
        for (int i = lane; i < n; i += 32) {
            const int e = S.lst[i];
            if (S.st[e] != 1) continue;
            const int ly = e / kE, lx = e - ly * kE;
            unsigned cnt = 0, a0 = 0, a1 = 0, a2 = 0;
#pragma unroll
            for (int dy = -1; dy <= 1; ++dy) {
#pragma unroll
                for (int dx = -1; dx <= 1; ++dx) {
                    if (!dx && !dy) continue;
                    const int nx = lx + dx, ny = ly + dy;
                    if (nx < 0 || nx >= kE || ny < 0 || ny >= kE) continue;  // unknown: not intact
                    const int gx = x0 + nx, gy = y0 + ny;
                    if (gx < 0 || gx >= w || gy < 0 || gy >= h) continue;  // outside the image
                    const int ne = ny * kE + nx;
                    const int s = S.st[ne];
                    if (s == 0 || (s >= 2 && s <= k)) {
                        ++cnt;
                        a0 += S.col[0][ne];
                        a1 += S.col[1][ne];
                        a2 += S.col[2][ne];
                    }
                }
            }
            if (cnt >= 2) {
                S.col[0][e] = static_cast<uint8_t>((2 * a0 + cnt) / (2 * cnt));
                S.col[1][e] = static_cast<uint8_t>((2 * a1 + cnt) / (2 * cnt));
                S.col[2][e] = static_cast<uint8_t>((2 * a2 + cnt) / (2 * cnt));
                S.st[e] = static_cast<uint8_t>(k + 1);
                ++local;
                if (lx >= kPasses && lx < kPasses + kT && ly >= kPasses && ly < kPasses + kT)
                    atomicAdd(&S.rep[k], 1);
            }
        }
        __syncwarp();
        const int any = __reduce_add_sync(0xFFFFFFFFu, local);
        // no repair anywhere in the region and no neighbour-published repair still to come:
        // the simulated state is a fixed point, later passes cannot change it
        if (any == 0 && max_future <= k) break;
    }
    __syncwarp();
    // 4. publish the interior
    int left = 0;
    for (int i = lane; i < n; i += 32) {
        const int e = S.lst[i];
        const int ly = e / kE, lx = e - ly * kE;
        if (lx < kPasses || lx >= kPasses + kT || ly < kPasses || ly >= kPasses + kT) continue;
        const int s = S.st[e];
        if (s == 1) {
            ++left;
            continue;
        }
        const int gx = x0 + lx, gy = y0 + ly;
        const unsigned long long g = static_cast<unsigned long long>(pass0 + s - 1);
        const unsigned long long v = kRepaired | (g << 24) |
                                     (static_cast<unsigned long long>(S.col[2][e]) << 16) |
                                     (static_cast<unsigned long long>(S.col[1][e]) << 8) | S.col[0][e];
        E.state[static_cast<size_t>(gy) * w + gx] = v;
        const size_t o = static_cast<size_t>(gy) * io.pitch + gx;
        if (io.plane[0]) io.plane[0][o] = S.col[0][e];
        if (io.plane[1]) io.plane[1][o] = S.col[1][e];
        if (io.plane[2]) io.plane[2][o] = S.col[2][e];
    }
    left = __reduce_add_sync(0xFFFFFFFFu, left);
    if (lane >= 1 && lane <= kPasses && S.rep[lane]) atomicAdd(&counts_slot[lane], static_cast<uint32_t>(S.rep[lane]));
    if (lane == 0 && left) next_flags[ty * tiles_x + tx] = 1;
    __syncwarp();
}

__global__ void __launch_bounds__(kThreads, 1) k_inpaint_tiles(Eye L, Eye R, int w, int h,
                                                               int tiles_x, int tiles_y,
                                                               uint32_t* ctl, long long* stats) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WarpSmem& S = reinterpret_cast<WarpSmem*>(smem_raw)[threadIdx.x >> 5];
    const int ntiles = tiles_x * tiles_y;
    const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t gsize = gridDim.x * blockDim.x;
    const int gwarp = blockIdx.x * kWarps + (threadIdx.x >> 5);
    const int nwarps = gridDim.x * kWarps;
    Eye eyes[2] = {L, R};

    // init: state words of damaged pixels = 0, round-0 flags of tiles holding damage
    uint32_t cnt[2];
    for (int e = 0; e < 2; ++e) {
        cnt[e] = __ldcg(eyes[e].io.count);
        for (uint32_t k = gtid; k < cnt[e]; k += gsize) {
            const uint32_t idx = eyes[e].io.list[k];
            eyes[e].state[idx] = 0ull;
            const int x = static_cast<int>(idx % static_cast<uint32_t>(w));
            const int y = static_cast<int>(idx / static_cast<uint32_t>(w));
            eyes[e].flags[(y / kT) * tiles_x + x / kT] = 1;
        }
    }
    long long remaining[2] = {cnt[0], cnt[1]};
    bool done[2] = {cnt[0] == 0, cnt[1] == 0};
    long long passes[2] = {0, 0}, fallback[2] = {0, 0};
    grid.sync();

    // ctl layout: [eye][slot 0..2][kPasses + 1] pass counts
    for (int round = 0; !(done[0] && done[1]); ++round) {
        const int slot = round % 3, nslot = (round + 1) % 3;
        if (gtid < 2 * (kPasses + 1)) {
            const int e = gtid / (kPasses + 1), k = gtid % (kPasses + 1);
            ctl[(e * 3 + nslot) * (kPasses + 1) + k] = 0;
        }
        for (int item = gwarp; item < 2 * ntiles; item += nwarps) {
            const int e = item / ntiles, t = item - e * ntiles;
            if (done[e]) continue;
            uint8_t* cur = eyes[e].flags + (round & 1) * ntiles;
            uint8_t* nxt = eyes[e].flags + ((round + 1) & 1) * ntiles;
            if (!cur[t]) continue;
            process_tile(eyes[e], t % tiles_x, t / tiles_x, w, h, round, tiles_x, S,
                         ctl + (e * 3 + slot) * (kPasses + 1), nxt);
            if ((threadIdx.x & 31) == 0) cur[t] = 0;
        }
        grid.sync();
        for (int e = 0; e < 2; ++e) {
            if (done[e]) continue;
            const uint32_t* c = ctl + (e * 3 + slot) * (kPasses + 1);
            bool stalled = false;
            for (int k = 1; k <= kPasses; ++k) {
                const long long rep = __ldcg(c + k);
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
                    if (__ldcg(eyes[e].state + idx) & kRepaired) continue;
                    const int x = static_cast<int>(idx % static_cast<uint32_t>(w));
                    const int y = static_cast<int>(idx / static_cast<uint32_t>(w));
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
    if (gtid == 0 && stats) {
        for (int e = 0; e < 2; ++e) {
            stats[3 * e + 0] = passes[e];
            stats[3 * e + 1] = static_cast<long long>(cnt[e]) - fallback[e];
            stats[3 * e + 2] = fallback[e];
        }
    }
}

}  // namespace

size_t inpaint_scratch_bytes(int w, int h) {
    const size_t n = static_cast<size_t>(w) * h;
    const size_t tiles = static_cast<size_t>((w + kT - 1) / kT) * ((h + kT - 1) / kT);
    return 2 * (n * sizeof(unsigned long long) + 2 * tiles) + 256;
}

cudaError_t inpaint(InpaintEye left, InpaintEye right, Geom gm, uint32_t capacity,
                    uint32_t* scratch, long long* stats, cudaStream_t st) {
    (void)capacity;
    // scratch layout: ctl (2*3*(kPasses+1) u32, zeroed) lives in `scratch` (64+ words);
    // state words and tile flags in the engine-provided inpaint arena (InpaintEye.repair
    // of the left eye points at it; see engine.cpp).
    const int tiles_x = (gm.w + kT - 1) / kT, tiles_y = (gm.h + kT - 1) / kT;
    const size_t n = static_cast<size_t>(gm.w) * gm.h;
    const size_t tiles = static_cast<size_t>(tiles_x) * tiles_y;
    unsigned char* arena = reinterpret_cast<unsigned char*>(left.repair);
    Eye L{left, reinterpret_cast<unsigned long long*>(arena), arena + 2 * n * 8};
    Eye R{right, reinterpret_cast<unsigned long long*>(arena + n * 8), arena + 2 * n * 8 + 2 * tiles};
    cudaError_t e = cudaMemsetAsync(scratch, 0, 2 * 3 * (kPasses + 1) * sizeof(uint32_t), st);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(arena + 2 * n * 8, 0, 4 * tiles, st);
    if (e != cudaSuccess) return e;
    const size_t smem = kWarps * sizeof(WarpSmem);
    static bool configured[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !configured[dev]) {
        cudaFuncSetAttribute(k_inpaint_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
        configured[dev] = true;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_inpaint_tiles, kThreads, smem);
    if (per_sm < 1) return cudaErrorLaunchOutOfResources;
    const int blocks = per_sm * sm_count();
    int w = gm.w, h = gm.h, tx = tiles_x, ty = tiles_y;
    void* args[] = {&L, &R, &w, &h, &tx, &ty, &scratch, &stats};
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_inpaint_tiles), dim3(blocks),
                                       dim3(kThreads), args, smem, st);
}

}  // namespace cu
}  // namespace p3s
