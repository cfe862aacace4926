/* p3s_gpu.h — B200 extensions to the pseudo3d C ABI (libpseudo3d_b200.so).
 *
 * pseudo3d.h is the drop-in surface (the reference's 49 functions). This header adds
 * what a GPU build needs on top, all plain C over host/device pointers:
 *   - stage entry points over host planes — the reference C++ stage API of
 *     proj/include/pseudo3d/{depth,bilateral,dibr,inpaint,stereo_format}.hpp as C, used
 *     by the parity tests to diff every intermediate against the oracle;
 *   - a device-resident pipeline (frames already in HBM; kernel-only throughput);
 *   - a multi-stream video converter (pinned host frames in, H2D/compute/D2H overlapped);
 *   - small device/event/pinned-memory helpers for harnesses.
 * All functions return p3s_status and set p3s_last_error() like pseudo3d.h.
 */
#ifndef P3S_GPU_H
#define P3S_GPU_H

#include "pseudo3d.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Flat view of p3s_config (reference config.hpp:25-43). base < 0 means auto. */
typedef struct p3s_params {
    int base;
    int pop_threshold;
    double sigma_spatial;
    double sigma_range;
    int depth_block;
    int inpaint_block;
    double alpha;
    double beta;
    int mode;         /* p3s_dibr_mode */
    unsigned formats; /* p3s_format bits */
} p3s_params;

P3S_API p3s_status p3s_config_get_params(const p3s_config* cfg, p3s_params* out);
/* Validates the whole candidate; on failure the config is unchanged. */
P3S_API p3s_status p3s_config_set_params(p3s_config* cfg, const p3s_params* params);

P3S_API int p3s_gpu_device_count(void);
/* Binds the calling thread to a CUDA device (all later calls on this thread use it). */
P3S_API p3s_status p3s_gpu_set_device(int ordinal);
P3S_API p3s_status p3s_gpu_device_name(char* buf, size_t cap);
/* Row-band plan of the synchronous p3s_convert schedule (host arithmetic, no device
 * needed): writes up to cap bands as 5 ints each (upload rows, depth-front tile rows,
 * block rows, depth rows, filter tile rows: where the band ENDS) and returns the band count
 * (0: the frame is converted in one piece), or -1 with p3s_last_error set. */
P3S_API int p3s_gpu_band_plan(int w, int h, const p3s_config* cfg, int* out, int cap);
/* 1 if conversions of width w with cfg use the host-verified integer DIBR column tables,
 * 0 if they keep the FP64 device path, -1 on invalid arguments (host only). */
P3S_API int p3s_gpu_dibr_integer_columns(int w, const p3s_config* cfg);
/* Streaming multiprocessors of the calling thread's device. */
P3S_API p3s_status p3s_gpu_sm_count(int* out);

/* ---- stage entry points (host planes in/out, row-major w*h, no pitch) ---- */
/* image.cpp:13-21 */
P3S_API p3s_status p3s_gpu_luma(const uint8_t* r, const uint8_t* g, const uint8_t* b, int w,
                                int h, uint8_t* out);
/* depth.cpp:21-74: luma -> Sobel -> block values; values: ceil(w/B)*ceil(h/B) doubles */
P3S_API p3s_status p3s_gpu_block_depth(const uint8_t* r, const uint8_t* g, const uint8_t* b,
                                       int w, int h, const p3s_config* cfg, double* values);
/* depth.cpp:76-121 */
P3S_API p3s_status p3s_gpu_upsample(const double* values, int w, int h, int block, uint8_t* out);
/* depth.cpp:127-129 */
P3S_API p3s_status p3s_gpu_generate_depth(const uint8_t* r, const uint8_t* g, const uint8_t* b,
                                          int w, int h, const p3s_config* cfg, uint8_t* depth);
/* bilateral.cpp:103-116 (rounded) and :88-101 (raw means, w*h doubles) */
P3S_API p3s_status p3s_gpu_cross_bilateral(const uint8_t* depth, const uint8_t* guide, int w,
                                           int h, const p3s_config* cfg, uint8_t* out);
P3S_API p3s_status p3s_gpu_cross_bilateral_raw(const uint8_t* depth, const uint8_t* guide, int w,
                                               int h, const p3s_config* cfg, double* out);
/* dibr.cpp:106-111 (mode from cfg); masks 1 = damaged */
P3S_API p3s_status p3s_gpu_reconstruct(const uint8_t* r, const uint8_t* g, const uint8_t* b,
                                       const uint8_t* depth, int w, int h, const p3s_config* cfg,
                                       uint8_t* lr, uint8_t* lg, uint8_t* lb, uint8_t* rr,
                                       uint8_t* rg, uint8_t* rb, uint8_t* lmask, uint8_t* rmask);
/* inpaint.cpp:29-130; stats: passes, repaired, fallback_filled */
P3S_API p3s_status p3s_gpu_inpaint(const uint8_t* r, const uint8_t* g, const uint8_t* b,
                                   const uint8_t* mask, int w, int h, const p3s_config* cfg,
                                   uint8_t* outr, uint8_t* outg, uint8_t* outb, int64_t* stats);
/* stereo_format.cpp:8-73; half: out w x h, full: out 2w x h */
P3S_API p3s_status p3s_gpu_anaglyph(const uint8_t* lr, const uint8_t* lg, const uint8_t* lb,
                                    const uint8_t* rr, const uint8_t* rg, const uint8_t* rb,
                                    int w, int h, uint8_t* outr, uint8_t* outg, uint8_t* outb);
P3S_API p3s_status p3s_gpu_side_by_side(const uint8_t* lr, const uint8_t* lg, const uint8_t* lb,
                                        const uint8_t* rr, const uint8_t* rg, const uint8_t* rb,
                                        int w, int h, int half, uint8_t* outr, uint8_t* outg,
                                        uint8_t* outb);

/* ---- device-resident pipeline ----
 * A plan for one (size, config) on the calling thread's device, with its own stream.
 * Input frames live in device memory as 3 planes of pitch*h bytes (plane stride pitch*h).
 * run() only enqueues (returns before the GPU finishes). */
typedef struct p3s_pipeline p3s_pipeline;
P3S_API p3s_status p3s_pipeline_create(int w, int h, const p3s_config* cfg, p3s_pipeline** out);
P3S_API void p3s_pipeline_free(p3s_pipeline* p);
P3S_API int p3s_pipeline_pitch(const p3s_pipeline* p);
P3S_API size_t p3s_pipeline_frame_bytes(const p3s_pipeline* p);
P3S_API void* p3s_pipeline_stream(const p3s_pipeline* p);
/* timed != 0 records CUDA events between stages (p3s_pipeline_timings). stream may be
 * NULL (the pipeline's own stream). */
P3S_API p3s_status p3s_pipeline_run(p3s_pipeline* p, const uint8_t* d_src, int timed, void* stream);
P3S_API p3s_status p3s_pipeline_timings(p3s_pipeline* p, p3s_timings* out);
/* Sums the stage times of every timed run since the last reset (each run keeps its own
 * events, so a timed loop needs no per-step synchronisation); count = runs summed. */
P3S_API p3s_status p3s_pipeline_timing_sum(p3s_pipeline* p, p3s_timings* sum, int64_t* count,
                                           int reset);
/* Same accumulation for the main bilateral kernel alone (without the exact fix-up). */
P3S_API p3s_status p3s_pipeline_bilateral_kernel_sum(p3s_pipeline* p, int64_t* sum_ns,
                                                     int64_t* count, int reset);
/* CTAs of the cooperative inpaint kernel (0 = one per SM, the default). With several
 * pipelines running concurrently, fewer CTAs leave SMs to the other frames' kernels (more
 * aggregate frames/s); one stream wants every SM (lowest latency). */
P3S_API p3s_status p3s_pipeline_set_inpaint_ctas(p3s_pipeline* p, int ctas);
/* Copies results of the last run to host planes (any pointer may be NULL), then syncs. */
P3S_API p3s_status p3s_pipeline_download(p3s_pipeline* p, uint8_t* depth, uint8_t* filtered,
                                         p3s_format format, uint8_t* outr, uint8_t* outg,
                                         uint8_t* outb);
/* stats[6]: left passes, repaired, fallback; right passes, repaired, fallback */
P3S_API p3s_status p3s_pipeline_inpaint_stats(p3s_pipeline* p, int64_t* stats);
/* H2D of host planes (w*h each) into a device frame with the pipeline's pitch; async on
 * `stream` (NULL = pipeline stream). Host planes should be pinned for a true async copy. */
P3S_API p3s_status p3s_pipeline_upload(p3s_pipeline* p, const uint8_t* r, const uint8_t* g,
                                       const uint8_t* b, uint8_t* d_dst, void* stream);

/* ---- video: frames pipelined through `streams` plans on the calling thread's device.
 * frames[i] / outs[i] point at 3 consecutive planes (w*h bytes each; outs of FSBS are
 * 2w*h each) in host memory, ideally pinned (p3s_host_alloc). Output = the lowest
 * requested format bit. Frame i runs on stream i % streams: its H2D, kernels and D2H
 * overlap the neighbouring frames'. Blocks until all n frames are back on the host. */
typedef struct p3s_video p3s_video;
P3S_API p3s_status p3s_video_create(int w, int h, const p3s_config* cfg, int streams,
                                    p3s_video** out);
/* Frame-sharded over several GPUs of one box: one host thread per device (`streams` plans
 * each) takes the next frame index from a shared counter, so frames of uneven cost balance
 * themselves; outputs land at their index. Frames are independent, so nothing crosses
 * NVLink and no collective runs. If a device fails, it is retired and every frame it took
 * is re-run on the others (the call still succeeds while one device is healthy). A device
 * may be listed more than once. */
P3S_API p3s_status p3s_video_create_devices(int w, int h, const p3s_config* cfg,
                                            const int* devices, int ndev, int streams,
                                            p3s_video** out);
P3S_API int p3s_video_shards(const p3s_video* v);
P3S_API p3s_status p3s_video_convert(p3s_video* v, const uint8_t* const* frames, int n,
                                     uint8_t* const* outs);
/* Same with RGB-interleaved frames (the PPM payload: w*h*3 bytes, R,G,B per pixel) in and
 * the output format interleaved out (ow*h*3 bytes): the (de)interleave runs on the GPU. */
P3S_API p3s_status p3s_video_convert_interleaved(p3s_video* v, const uint8_t* const* frames,
                                                 int n, uint8_t* const* outs);
P3S_API void p3s_video_free(p3s_video* v);
/* Frames re-run on healthy devices after a device failed (summed over calls), and the
 * devices still in service. A failed device is retired for the video's lifetime. */
P3S_API long long p3s_video_requeued(const p3s_video* v);
P3S_API int p3s_video_healthy_shards(const p3s_video* v);
/* NUMA node of a CUDA device (-1 unknown) and a pinned block whose pages sit on it (for
 * per-GPU frame rings on multi-socket hosts; release with p3s_host_free). */
P3S_API int p3s_gpu_numa_node(int device);
/* Kernels this library has launched in this process (direct launches plus the kernel nodes
 * of every graph replay): the bench's gpu_launches is a difference of two readings. */
P3S_API unsigned long long p3s_gpu_launch_count(void);
P3S_API void* p3s_host_alloc_near(int device, size_t bytes);

/* ---- helpers ---- */
P3S_API p3s_status p3s_gpu_malloc(size_t bytes, void** out); /* zero-filled */
P3S_API void p3s_gpu_free(void* p);
P3S_API p3s_status p3s_gpu_memset(void* p, int value, size_t bytes);
P3S_API p3s_status p3s_gpu_stream_sync(void* stream);
P3S_API p3s_status p3s_gpu_device_sync(void);
P3S_API p3s_status p3s_gpu_event_create(void** out);
P3S_API p3s_status p3s_gpu_event_record(void* ev, void* stream);
/* Makes `stream` wait for the work recorded in `ev` (cudaStreamWaitEvent). */
P3S_API p3s_status p3s_gpu_stream_wait_event(void* stream, void* ev);
P3S_API p3s_status p3s_gpu_event_elapsed_ms(void* start, void* stop, float* ms);
P3S_API void p3s_gpu_event_destroy(void* ev);
P3S_API void* p3s_host_alloc(size_t bytes); /* pinned pool */
/* Measured non-FMA FP64 issue rate of the current device (DADD/DMUL ops per second), the
 * roofline denominator of the exact bilateral kernel. */
P3S_API p3s_status p3s_gpu_fp64_peak(double* ops_per_s);
/* Measured conflict-free shared-memory load bandwidth (bytes/s, all SMs): gather = 0 for
 * lane-contiguous LDS.32, 1 for data-dependent per-lane gathers from a 32-way replicated
 * table (the certified FP32 bilateral's range lookups, its limiting stream). */
P3S_API p3s_status p3s_gpu_smem_peak(double* bytes_per_s, int gather);
/* Which bilateral kernel p3s_convert uses for this config (no GPU needed): 1 = certified
 * FP32 + exact FP64 fix-up (radius 16), 0 = exact FP64 kernels. */
P3S_API p3s_status p3s_gpu_bilateral_path(const p3s_config* cfg, int* certified_fp32);
P3S_API void p3s_host_free(void* p);
/* The reference's seeded synthetic frame (bench.cpp:23-46: mt19937_64 seeded with
 * seed ^ (w << 32) ^ h, one draw per pixel in raster order) written into three caller
 * planes of w*h bytes. Host code, no GPU needed; the bench's and the tests' input source. */
P3S_API p3s_status p3s_synthetic_frame(int w, int h, uint64_t seed, uint8_t* r, uint8_t* g,
                                       uint8_t* b);

#ifdef __cplusplus
}
#endif

#endif /* P3S_GPU_H */
