// K3b: Jacobi hole filling on sm_100a (reference proj/src/inpaint.cpp:29-130).
//
// Semantics kept exactly: every pass decides against the pass-start snapshot (a damaged
// pixel with >= 2 intact 8-neighbours takes the per-channel (2*sum + n) / (2n) mean),
// then applies all repairs; the first pass that repairs nothing while damage remains
// fills the rest with (128,128,128). Both eyes are independent instances
// (pipeline.cpp:56-65) and run in the same launch.
//
// Temporal blocking. The frame is cut into 32x32 tiles; a round runs kPasses Jacobi passes
// of one tile inside shared memory over the tile plus a kPasses-pixel halo. Information
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
constexpr int kE = kT + 2 * kPasses;   // extended side
constexpr int kEN = kE * kE;
constexpr int kThreads = 256;
constexpr unsigned long long kRepaired = 1ull << 63;

struct Eye {
    InpaintEye io;
    unsigned long long* state;  // per pixel (only initially damaged entries used)
    uint8_t* flags;             // [2][tiles] round flags
};

__device__ __forceinline__ bool damaged0(const InpaintEye& e, int x, int y) {
    if (e.mask_bits) return (__ldg(e.mask_bits + static_cast<size_t>(y) * e.mask_pitch + (x >> 5)) >> (x & 31)) & 1u;
    return __ldg(e.mask_bytes + static_cast<size_t>(y) * e.mask_pitch + x) != 0;
}

// st: 0 intact, 1 damaged, k+1 repaired at local pass k (intact for passes > k), 255 outside image
__device__ void process_tile(const Eye& E, int tx, int ty, int w, int h, int round, int tiles_x,
                             uint8_t* st, uint8_t* col, uint16_t* lst, int* s_n, int* s_rep,
                             int* s_left, uint32_t* counts_slot, uint8_t* next_flags) {
    const InpaintEye& io = E.io;
    const int x0 = tx * kT - kPasses, y0 = ty * kT - kPasses;
    const long long pass0 = static_cast<long long>(round) * kPasses;  // passes before this round
    const int tid = threadIdx.x;
    if (tid == 0) {
        *s_n = 0;
        *s_left = 0;
    }
    if (tid < kPasses + 1) s_rep[tid] = 0;
    __syncthreads();
    // load the extended region
    for (int e = tid; e < kEN; e += kThreads) {
        const int ly = e / kE, lx = e - ly * kE;
        const int gx = x0 + lx, gy = y0 + ly;
        uint8_t s = 255;
        uint8_t c0 = 0, c1 = 0, c2 = 0;
        if (gx >= 0 && gx < w && gy >= 0 && gy < h) {
            const size_t o = static_cast<size_t>(gy) * io.pitch + gx;
            if (!damaged0(io, gx, gy)) {
                s = 0;
                if (io.plane[0]) c0 = io.plane[0][o];
                if (io.plane[1]) c1 = io.plane[1][o];
                if (io.plane[2]) c2 = io.plane[2][o];
            } else {
                const unsigned long long v =
                    __ldcg(E.state + static_cast<size_t>(gy) * w + gx);
                if (v & kRepaired) {
                    const long long g = static_cast<long long>((v >> 24) & 0xFFFFFFFFull);
                    s = g <= pass0 ? 0 : static_cast<uint8_t>(g - pass0 + 1);
                    c0 = static_cast<uint8_t>(v);
                    c1 = static_cast<uint8_t>(v >> 8);
                    c2 = static_cast<uint8_t>(v >> 16);
                } else {
                    s = 1;
                    const int at = atomicAdd(s_n, 1);
                    lst[at] = static_cast<uint16_t>(e);
                }
            }
        }
        st[e] = s;
        col[e] = c0;
        col[kEN + e] = c1;
        col[2 * kEN + e] = c2;
    }
    __syncthreads();
    const int n = *s_n;
    for (int k = 1; k <= kPasses; ++k) {
        for (int i = tid; i < n; i += kThreads) {
            const int e = lst[i];
            if (st[e] != 1) continue;
            const int ly = e / kE, lx = e - ly * kE;
            unsigned cnt = 0, a0 = 0, a1 = 0, a2 = 0;
#pragma unroll
            for (int dy = -1; dy <= 1; ++dy) {
#pragma unroll
                for (int dx = -1; dx <= 1; ++dx) {
                    if (!dx && !dy) continue;
                    const int nx = lx + dx, ny = ly + dy;
                    if (nx < 0 || nx >= kE || ny < 0 || ny >= kE) continue;  // unknown: not intact
                    const int ne = ny * kE + nx;
                    const int s = st[ne];
                    if (s == 0 || (s >= 2 && s != 255 && s <= k)) {  // intact at pass start
                        ++cnt;
                        a0 += col[ne];
                        a1 += col[kEN + ne];
                        a2 += col[2 * kEN + ne];
                    }
                }
            }
            if (cnt >= 2) {
                col[e] = static_cast<uint8_t>((2 * a0 + cnt) / (2 * cnt));
                col[kEN + e] = static_cast<uint8_t>((2 * a1 + cnt) / (2 * cnt));
                col[2 * kEN + e] = static_cast<uint8_t>((2 * a2 + cnt) / (2 * cnt));
                st[e] = static_cast<uint8_t>(k + 1);
                if (lx >= kPasses && lx < kPasses + kT && ly >= kPasses && ly < kPasses + kT)
                    atomicAdd(&s_rep[k], 1);
            }
        }
        __syncthreads();
    }
    // publish the interior
    for (int i = tid; i < n; i += kThreads) {
        const int e = lst[i];
        const int ly = e / kE, lx = e - ly * kE;
        if (lx < kPasses || lx >= kPasses + kT || ly < kPasses || ly >= kPasses + kT) continue;
        const int gx = x0 + lx, gy = y0 + ly;
        const int s = st[e];
        if (s == 1) {
            atomicAdd(s_left, 1);
            continue;
        }
        const unsigned long long g = static_cast<unsigned long long>(pass0 + s - 1);
        const unsigned long long v = kRepaired | (g << 24) |
                                     (static_cast<unsigned long long>(col[2 * kEN + e]) << 16) |
                                     (static_cast<unsigned long long>(col[kEN + e]) << 8) | col[e];
        E.state[static_cast<size_t>(gy) * w + gx] = v;
        const size_t o = static_cast<size_t>(gy) * io.pitch + gx;
        if (io.plane[0]) io.plane[0][o] = col[e];
        if (io.plane[1]) io.plane[1][o] = col[kEN + e];
        if (io.plane[2]) io.plane[2][o] = col[2 * kEN + e];
    }
    __syncthreads();
    if (tid >= 1 && tid <= kPasses && s_rep[tid]) atomicAdd(&counts_slot[tid], static_cast<uint32_t>(s_rep[tid]));
    if (tid == 0 && *s_left) next_flags[ty * tiles_x + tx] = 1;
    __syncthreads();
}

__global__ void __launch_bounds__(kThreads) k_inpaint_tiles(Eye L, Eye R, int w, int h,
                                                            int tiles_x, int tiles_y,
                                                            uint32_t* ctl, long long* stats) {
    cg::grid_group grid = cg::this_grid();
    __shared__ uint8_t st[kEN];
    __shared__ uint8_t col[3 * kEN];
    __shared__ uint16_t lst[kEN];
    __shared__ int s_n, s_left, s_rep[kPasses + 1];
    const int ntiles = tiles_x * tiles_y;
    const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t gsize = gridDim.x * blockDim.x;
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
        for (int item = blockIdx.x; item < 2 * ntiles; item += gridDim.x) {
            const int e = item / ntiles, t = item - e * ntiles;
            if (done[e]) continue;
            uint8_t* cur = eyes[e].flags + (round & 1) * ntiles;
            uint8_t* nxt = eyes[e].flags + ((round + 1) & 1) * ntiles;
            if (!cur[t]) continue;
            process_tile(eyes[e], t % tiles_x, t / tiles_x, w, h, round, tiles_x, st, col, lst,
                         &s_n, s_rep, &s_left, ctl + (e * 3 + slot) * (kPasses + 1), nxt);
            if (threadIdx.x == 0) cur[t] = 0;
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
    static int per_sm_cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    int per_sm = dev < 64 ? per_sm_cache[dev] : 0;
    if (per_sm == 0) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_inpaint_tiles, kThreads, 0);
        if (per_sm < 1) per_sm = 1;
        if (per_sm > 4) per_sm = 4;
        if (dev < 64) per_sm_cache[dev] = per_sm;
    }
    const int blocks = per_sm * sm_count();
    int w = gm.w, h = gm.h, tx = tiles_x, ty = tiles_y;
    void* args[] = {&L, &R, &w, &h, &tx, &ty, &scratch, &stats};
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_inpaint_tiles), dim3(blocks),
                                       dim3(kThreads), args, 0, st);
}

}  // namespace cu
}  // namespace p3s
