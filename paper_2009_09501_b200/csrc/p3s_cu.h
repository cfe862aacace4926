// p3s_cu.h — the thin internal layer between the host orchestrator (engine.cpp) and the
// sm_100a kernels (*.cu). Plain functions over device pointers, sizes, POD parameters
// and a cudaStream_t; each enqueues work and returns a cudaError_t. No torch, no STL.
//
// Device image layout: planar u8, row-major, `pitch` bytes per row (pitch % 16 == 0 so
// every kernel can use 16-byte vector accesses), plane stride = pitch * h.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <stdint.h>

namespace p3s {
namespace cu {

// Reference pseudo3d.h:43-47 format bits.
enum : unsigned { kAnaglyph = 1u, kHsbs = 2u, kFsbs = 4u };

struct Geom {
    int w, h, pitch;
};

// Per-(size, config) constant tables, computed on the host with the reference's exact
// double expressions (engine.cpp) and uploaded once per plan.
struct DepthTables {
    const int* col_i0;     // [w]  left block-centre index  (depth.cpp:96-102 locate)
    const int* col_i1;     // [w]  min(i0+1, bx-1)
    const double* col_f;   // [w]  interpolation fraction
    const int* row_i0;     // [h]
    const int* row_i1;     // [h]
    const double* row_f;   // [h]
    int bx, by, block;
    double alpha255;       // alpha * 255.0 (left-to-right as depth.cpp:60)
    double beta;
    double row_denom;      // h > 1 ? h - 1 : 1
};

// K1: luma plane + per-block Sobel-magnitude sums (image.cpp:13-21, depth.cpp:21-74).
// sums must be zeroed (bx*by u64) before the call. Optional row band: tiles of
// depth_tile_rows() image rows [tile_row0, tile_row1) (-1: to the end); the block sums of
// a block row are complete once every tile row covering it has run.
cudaError_t depth_front(const uint8_t* r, const uint8_t* g, const uint8_t* b, Geom gm,
                        uint8_t* luma, unsigned long long* sums, int block, int bx,
                        cudaStream_t st, int tile_row0 = 0, int tile_row1 = -1);
int depth_tile_rows();
// K1 with the block values folded in, for depth_block == depth_tile_rows() (16), w % 16 == 0
// and a 16-byte aligned pitch (depth_fused_ok): luma plane + block values of block rows
// [tile_row0, tile_row1) in one launch, no sums buffer (block_values is not called).
bool depth_fused_ok(Geom gm, int block);
// src_ipitch > 0: r is one RGB-interleaved image with that row stride (g, b unused; needs
// src_ipitch % 16 == 0).
cudaError_t depth_front_fused(const uint8_t* r, const uint8_t* g, const uint8_t* b, Geom gm,
                              uint8_t* luma, const DepthTables& t, double* values, cudaStream_t st,
                              int tile_row0 = 0, int tile_row1 = -1, int src_ipitch = 0);
// Block values (depth.cpp:55-71) from the sums, block rows [brow0, brow1).
cudaError_t block_values(const unsigned long long* sums, Geom gm, const DepthTables& t,
                         double* values, cudaStream_t st, int brow0 = 0, int brow1 = -1);
// Bilinear upsample to the u8 depth map (depth.cpp:104-120), image rows [ya, yb).
cudaError_t upsample(const double* values, Geom gm, const DepthTables& t, uint8_t* depth,
                     cudaStream_t st, int ya = 0, int yb = -1);

// K2: exact FP64 cross-bilateral (bilateral.cpp:40-116). spatial: (2r+1) x (r+1) doubles,
// s[(dy+r)*(r+1) + dx] for dx >= 0; range: 256 doubles. raw (optional, w-strided)
// receives the unrounded means (cross_bilateral_raw), out the rounded u8 map.
// bilateral_tiled takes the spatial table from HOST memory (it travels as a kernel
// parameter) and handles radius <= bilateral_tiled_max_radius(); bilateral (generic,
// any radius) reads a DEVICE copy.
cudaError_t bilateral_tiled(const uint8_t* depth, const uint8_t* guide, Geom gm, int radius,
                            const double* spatial_host, const double* range, uint8_t* out,
                            double* raw, cudaStream_t st);
int bilateral_tiled_max_radius();
// Certified FP32 fast path (same output bytes): approximate every pixel, prove the byte,
// recompute the unprovable ones exactly. `list`/`count`: device scratch for the fallback
// pixel list (capacity w*h). Falls back to bilateral_tiled for radii it does not cover.
cudaError_t bilateral_fast(const uint8_t* depth, const uint8_t* guide, Geom gm, int radius,
                           const double* spatial_host, const double* spatial_dev,
                           const double* range, uint8_t* out, uint32_t* list, uint32_t* count,
                           cudaStream_t st, cudaEvent_t after_main = nullptr,
                           const float* table = nullptr);
// The certified path in parts, for row-banded schedules: bilateral_sep_main runs the FP32
// kernel over tile rows [tile_row0, tile_row1) of bilateral_sep_tile_rows() image rows
// (appending to list/count, which the caller zeroes once per frame; tile_ctr: one zeroed
// u32 per launch for dynamic tile claims); bilateral_sep_fixup then recomputes every listed
// pixel. Only for radii where bilateral_fast_available().
cudaError_t bilateral_sep_main(const uint8_t* depth, const uint8_t* guide, Geom gm, int radius,
                               const double* spatial_host, const double* range, uint8_t* out,
                               uint32_t* list, uint32_t* count, uint32_t* tile_ctr,
                               int tile_row0, int tile_row1, const float* table, cudaStream_t st);
cudaError_t bilateral_sep_fixup(const uint8_t* depth, const uint8_t* guide, Geom gm, int radius,
                                const double* spatial_dev, const double* range, uint8_t* out,
                                const uint32_t* list, const uint32_t* count, cudaStream_t st,
                                int max_ctas = 0 /* 0: one warp per listed pixel of a 4K frame */);
int bilateral_sep_tile_rows();
// The certified kernel's replicated FP32 range table (bilateral_sep_table_bytes(), built once
// per plan from the FP64 range table); table = nullptr builds it in every CTA instead.
size_t bilateral_sep_table_bytes();
cudaError_t build_sep_table(const double* range, float* table, cudaStream_t st);
// cudaEventRecord, or an event-record graph node while `st` is being captured.
void record_event_any(cudaEvent_t e, cudaStream_t st);
// Per-device one-time launch setup (cudaFuncSetAttribute): runs `setup` until it has
// completed once on the current device. Host threads may race into it; the setup is
// idempotent and the device is marked only after it ran, so no launch can see it missing.
template <class F>
inline void once_per_device(std::atomic<unsigned long long>& done, F&& setup) {
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = dev >= 0 && dev < 64 ? 1ull << dev : 0ull;
    if (bit && (done.load(std::memory_order_acquire) & bit)) return;
    setup();
    if (bit) done.fetch_or(bit, std::memory_order_release);
}
// Zero several ranges of whole 4-byte words (4-byte aligned): one kernel launch when
// by_kernel (copy engines busy with PCIe traffic), else one memset per range (SMs busy
// with other streams' kernels).
// Kernel-launch accounting (the bench's gpu_launches): every launch site calls note_launch
// (not counted while its stream is being captured into a graph); a graph replay adds the
// kernel nodes of its graph.
void note_launch(cudaStream_t st);
void note_graph_launch(std::size_t kernels);
std::size_t graph_kernel_nodes(cudaGraph_t g);
unsigned long long launch_count();

constexpr int kZeroRanges = 4;
struct ZeroRanges {
    void* p[kZeroRanges];
    unsigned words[kZeroRanges];
    int n;
};
cudaError_t zero(const ZeroRanges& z, cudaStream_t st, bool by_kernel = false);
bool bilateral_fast_available(int radius);
cudaError_t bilateral(const uint8_t* depth, const uint8_t* guide, Geom gm, int radius,
                      const double* spatial, const double* range, uint8_t* out, double* raw,
                      cudaStream_t st);

// DIBR output routing. Each eye writes up to three planes (nullptr = channel not needed,
// e.g. anaglyph needs only left.R and right.G/B). Planes of one eye share a pitch.
struct EyeOut {
    uint8_t* plane[3];     // stride 3: one RGB-interleaved image, plane[c] = base + c
    int pitch;
    int stride = 1;        // 1: planar; 3: interleaved (the fused-anaglyph quad kernel only)
    uint8_t* mask_bytes;   // byte mask (reference DamageMask layout), pitch = mask_pitch
    uint32_t* mask_bits;   // or bit mask: ceil(w/32) words per row, bit x%32, 1 = damaged
    int mask_pitch;        // bytes per row (bytes) or words per row (bits)
    uint32_t* list;        // damaged pixel indices (y*w + x), appended
    uint32_t* count;       // list length (device counter, zeroed before the call)
};

// DIBR (dibr.cpp:43-104). shift: 256 doubles sigma[d] (p.left = x - sigma, p.right =
// x + sigma; see engine.cpp). cols (optional, 256 int4): the host-verified integer column
// tables (engine.cpp dibr_col_table); when given, no FP64 runs on the device.
// backward = cfg.dibr_mode == kBackwardFallback.
// A DIBR row lives in one CTA's shared memory (12 bytes per pixel for the general kernel)
// up to dibr_max_width(); wider rows keep their z-buffer keys in global per-CTA slots of
// dibr_wide_key_words(w) u32 (0 when not needed), passed to dibr() as wide_keys.
constexpr size_t kDibrMaxSmem = 220 * 1024;  // + the kernels' static tables <= 227 KB
inline int dibr_max_width() { return static_cast<int>(kDibrMaxSmem / 12) & ~15; }
int dibr_wide_slots();
size_t dibr_wide_key_words(int w);
// Host patch after a banded early download: every 32-pixel word whose mask bit is set
// (damage the inpaint repaired after the rows left) is copied from the device planes to the
// host planes (pinned, so device-visible under UVA) with coalesced 32-byte stores.
struct PatchEye {
    const uint8_t* dev[3];  // nullptr: plane not produced by this eye
    uint8_t* host[3];
    int dpitch, hpitch;
    const uint32_t* mask;
    int mpitch;
};
cudaError_t patch_host(PatchEye left, PatchEye right, Geom gm, cudaStream_t st);
cudaError_t dibr(const uint8_t* r, const uint8_t* g, const uint8_t* b, const uint8_t* depth,
                 Geom gm, const double* shift, const int4* cols, bool backward, EyeOut left,
                 EyeOut right, cudaStream_t st, int ya = 0, int yb = -1,  // rows [ya, yb)
                 uint32_t* wide_keys = nullptr,
                 int src_ipitch = 0 /* left.stride == 3: r = interleaved source, row stride */);

// Byte mask -> damaged list and (bits != nullptr) 32-pixel damage words of mwords per row
// (stage-level inpaint entry point).
cudaError_t mask_to_list(const uint8_t* mask, int mpitch, Geom gm, uint32_t* list,
                         uint32_t* count, cudaStream_t st, uint32_t* bits = nullptr, int mwords = 0);

// Inpaint (inpaint.cpp:29-130) on both eyes at once, in place on the EyeOut planes.
// Work lists come from dibr(). stats (device, 8 x i64): passes/repaired/fallback per eye,
// then the per-eye tile-processing ns (the split of the kernel's time between the eyes).
// The damage is read from mask_bits (the INITIAL damage, 32-pixel words, read-only; the
// byte mask is not read). `repair` of the left eye points at a device arena of
// inpaint_scratch_bytes(w, h) (tagged damage words, tile counts, work lists; persistent).
struct InpaintEye {
    uint8_t* plane[3];     // channel c of pixel (x, y) at plane[c] + y * pitch + x * stride
    int pitch;
    int stride = 1;        // 1: planar; 3: RGB-interleaved rows (plane[c] = base + c)
    uint8_t* mask_bytes;
    uint32_t* mask_bits;
    int mask_pitch;
    uint32_t* list;        // in: damaged indices (length *count)
    uint32_t* count;
    uint32_t* list2;       // unused (kept for layout compatibility)
    uint32_t* repair;      // left eye: inpaint arena
};
size_t inpaint_scratch_bytes(int w, int h);
// zero: 0 = the call zeroes its control words with memsets, 1 = with a kernel, 2 = not at
// all (the caller ran inpaint_zero earlier in stream order, off the critical path)
cudaError_t inpaint(InpaintEye left, InpaintEye right, Geom gm, uint32_t capacity,
                    uint32_t* scratch /* >= 128 words, zeroed by the call */, long long* stats,
                    cudaStream_t st, int max_ctas = 0 /* 0: one CTA per SM */,
                    int zero = 0);
// The control-word zeroing inpaint() would do (pass counts, barrier, work counters, busy ns)
cudaError_t inpaint_zero(InpaintEye left, Geom gm, uint32_t* scratch, long long* stats,
                         cudaStream_t st, bool by_kernel);

// Formats from materialised eyes (stereo_format.cpp:8-73).
cudaError_t anaglyph(const uint8_t* const* left, const uint8_t* const* right, Geom gm,
                     uint8_t* const* out, int out_pitch, cudaStream_t st);
cudaError_t side_by_side_half(const uint8_t* const* left, const uint8_t* const* right, Geom gm,
                              uint8_t* const* out, int out_pitch, cudaStream_t st);
cudaError_t side_by_side_full(const uint8_t* const* left, const uint8_t* const* right, Geom gm,
                              uint8_t* const* out, int out_pitch, cudaStream_t st);

// Interleaved RGB (PPM payload order, w*h*3 bytes) <-> planes of `pitch` (kernels_io.cu).
cudaError_t deinterleave(const uint8_t* src, int w, int h, uint8_t* r, uint8_t* g, uint8_t* b,
                         int pitch, cudaStream_t st);
cudaError_t interleave(const uint8_t* r, const uint8_t* g, const uint8_t* b, int pitch, int w,
                       int h, uint8_t* dst, cudaStream_t st);

int sm_count();
// Non-FMA FP64 issue-rate microbenchmark (independent DMUL/DADD chains), ops per second.
cudaError_t fp64_peak(double* ops_per_s);
// Measured conflict-free shared-memory lookup bandwidth (LDS.32 gathers, all SMs), bytes/s.
cudaError_t smem_peak(double* bytes_per_s);
// Same for data-dependent per-lane gathers from a 32-way replicated table (the bilateral's pattern).
cudaError_t smem_gather_peak(double* bytes_per_s);

}  // namespace cu
}  // namespace p3s
