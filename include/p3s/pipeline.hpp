// p3s/pipeline.hpp — the C++ stage API of the B200 pseudo-stereo pipeline.
//
// Same stage names, parameters and results as the reference's C++ API
// (reference include/pseudo3d/{depth,bilateral,dibr,inpaint,stereo_format,pipeline}.hpp);
// where the reference takes an `Executor&` thread pool, these take a `Device&`, the
// per-thread CUDA context (stream, cached plans, device buffers) of one GPU. Every
// function runs on the GPU through the hand-written sm_100a kernels; there is no CPU
// compute path. Inputs and outputs are host images (pinned), so each call is
// H2D -> kernels -> D2H; the device-resident path for throughput work is
// p3s::Pipeline (below) and the C entry points in p3s_gpu.h.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "p3s/core.hpp"

namespace p3s {

class Device;

// Reference pipeline.hpp:16-27. GPU: CUDA-event time of each stage's kernels.
struct StageTimings {
    std::int64_t depth_gen_ns = 0;
    std::int64_t filter_ns = 0;
    std::int64_t dibr_ns = 0;
    std::int64_t inpaint_left_ns = 0;
    std::int64_t inpaint_right_ns = 0;
    std::int64_t format_ns = 0;
    std::int64_t pure_ns() const {
        return filter_ns + dibr_ns + inpaint_left_ns + inpaint_right_ns + format_ns;
    }
};

// Row-band plan of the synchronous convert: where
// each band ends, in the units of every stage. Host-only arithmetic (no device needed);
// empty when the frame is too short for two bands.
struct BandEnd {
    int in_rows;  // upload rows [0, in_rows) are needed
    int dtile;    // depth-front tile rows (16 image rows each) [0, dtile)
    int brow;     // block rows [0, brow)
    int urow;     // depth rows [0, urow)
    int btile;    // filter tile rows (128 image rows each) [0, btile)
};
std::vector<BandEnd> band_plan(int width, int height, int radius, int depth_block,
                               const char* ends_override = nullptr);
// Whether plans of this width/config use the host-verified integer DIBR column tables
// (dibr.cpp:33-41 as x + off + (x >= X)); false keeps the FP64 device path. Host only.
bool dibr_integer_columns(int width, const ConversionConfig& cfg);

// Reference pipeline.hpp:29-35.
struct ConversionResult {
    std::map<StereoFormat, ImageRGB8> outputs;  // exactly the requested formats
    GrayMap depth;
    GrayMap filtered_depth;
    StageTimings timings;
};

// Reference dibr.hpp:14-20.
struct StereoFrames {
    ImageRGB8 left, right;
    DamageMask left_mask, right_mask;
};

// Reference inpaint.hpp:10-14.
struct InpaintStats {
    int passes = 0;
    std::size_t repaired = 0;
    std::size_t fallback_filled = 0;
};

// Reference depth.hpp:13-27.
struct BlockGrid {
    int blocks_x = 0, blocks_y = 0, block = 0, width = 0, height = 0;
    std::vector<double> values;
};

// The CUDA context of the calling thread on one GPU. Device::current() binds lazily to
// the thread's current CUDA device; throws DeviceError if there is none.
class Device {
public:
    static Device& current();
    explicit Device(int ordinal);
    ~Device();
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;

    int ordinal() const;
    void* stream() const;  // cudaStream_t
    struct Impl;
    Impl& impl() { return *impl_; }

private:
    std::unique_ptr<Impl> impl_;
};

// ---- stages (reference depth.hpp, bilateral.hpp, dibr.hpp, inpaint.hpp,
//      stereo_format.hpp, pipeline.hpp) --------------------------------------------------
GrayMap luma(const ImageRGB8& img, Device& dev);
BlockGrid block_depth(const ImageRGB8& img, const ConversionConfig& cfg, Device& dev);
GrayMap upsample_block_grid(const BlockGrid& grid, Device& dev);
GrayMap generate_depth(const ImageRGB8& img, const ConversionConfig& cfg, Device& dev);
GrayMap cross_bilateral(const GrayMap& depth, const GrayMap& guide, const ConversionConfig& cfg,
                        Device& dev);
std::vector<double> cross_bilateral_raw(const GrayMap& depth, const GrayMap& guide,
                                        const ConversionConfig& cfg, Device& dev);
StereoFrames reconstruct(const ImageRGB8& src, const GrayMap& depth, const ConversionConfig& cfg,
                         Device& dev);
ImageRGB8 inpaint(const ImageRGB8& frame, const DamageMask& mask, const ConversionConfig& cfg,
                  Device& dev, InpaintStats* stats = nullptr);
ImageRGB8 anaglyph(const ImageRGB8& left, const ImageRGB8& right, Device& dev);
ImageRGB8 side_by_side(const ImageRGB8& left, const ImageRGB8& right, bool half, Device& dev);

// Full pipeline (reference pipeline.cpp:29-78): one H2D, all stages on the device, one
// D2H of the requested outputs plus depth and filtered depth.
ConversionResult convert_image(const ImageRGB8& src, const ConversionConfig& cfg, Device& dev);

// The depth and filtered-depth maps of a conversion (the C ABI's p3s_result_depth /
// _filtered_depth): a device copy made right after the frame's filter, downloaded into
// pinned host maps in the background on a per-device copy stream (it does not hold up the
// call that produced it; only the D2H direction of the link is shared with the outputs).
// depth() / filtered() wait for that download; the device copy returns to a pool as soon as
// it is done.
class DeferredMaps {
public:
    DeferredMaps(int device, int w, int h, void* dev_buf);
    ~DeferredMaps();
    DeferredMaps(const DeferredMaps&) = delete;
    DeferredMaps& operator=(const DeferredMaps&) = delete;
    // Queues the D2H after `ready_event` (a cudaEvent_t recorded after the device copy) on
    // the device's copy stream.
    void start_download(void* ready_event);
    // Waits for both maps once (thread-safe); later calls return the cached host maps.
    const GrayMap& depth();
    const GrayMap& filtered();

private:
    void materialize();
    int device_, w_, h_;
    void* buf_;  // 2 * w * h bytes: depth then filtered depth (unpitched)
    GrayMap depth_, filtered_;
    void* done_ = nullptr;  // cudaEvent_t: the background download's completion
    bool ready_ = false;
    std::mutex mu_;
};

// convert_image without the depth / filtered-depth downloads: outputs and timings come back
// to the host, the two maps stay on the device in `maps`.
ConversionResult convert_image_deferred(const ImageRGB8& src, const ConversionConfig& cfg,
                                        Device& dev, std::shared_ptr<DeferredMaps>& maps);

// ---- device-resident pipeline ------------------------------------------------------------
// A plan for one (size, config) on one device: tables, device buffers, a stream. run()
// enqueues the whole pipeline for a frame already in device memory (planar, pitch()
// bytes per row, plane stride pitch()*h) and returns immediately.
class Pipeline {
public:
    Pipeline(int width, int height, const ConversionConfig& cfg, Device& dev);
    ~Pipeline();
    int pitch() const;
    int width() const;
    int height() const;
    void* stream() const;
    // Device frame layout for inputs: 3 planes of pitch()*height() bytes.
    std::size_t frame_bytes() const;
    void run(const std::uint8_t* d_src, void* stream = nullptr);
    // Same, with CUDA events between stages (read back with last_timings()).
    void run_timed(const std::uint8_t* d_src, void* stream = nullptr);
    StageTimings last_timings();
    // Sum of the stage times of every timed run since the last reset (synchronises).
    StageTimings accumulated_timings(long long* count, bool reset = true);
    // Sum of the main bilateral kernel's time (without the exact fix-up) over the same timed
    // runs, for the roofline of the dominant kernel.
    long long bilateral_kernel_ns(long long* count, bool reset = true);
    // CTAs of the cooperative inpaint kernel (0 = one per SM, the default). With several
    // pipelines running concurrently, fewer CTAs leave SMs to the other frames (more
    // aggregate frames/s); a single stream wants every SM (lowest latency). Recaptures the
    // plan's graphs.
    void set_inpaint_ctas(int ctas);
    // Device pointers of the results of the last run (pitch(), or fsbs_pitch() for FSBS).
    const std::uint8_t* d_depth() const;
    const std::uint8_t* d_filtered() const;
    const std::uint8_t* d_output(StereoFormat f) const;
    int output_pitch(StereoFormat f) const;
    // Copies the last results to host images (async on `stream`, then synchronised).
    void download(ConversionResult& out, void* stream = nullptr);
    // Host-side per-eye inpaint stats of the last run (synchronises).
    void inpaint_stats(InpaintStats& left, InpaintStats& right);
    // The pipeline's own device input frame (3 * pitch() * height() bytes).
    std::uint8_t* d_input();
    // Async H2D of host planes (width*height each) into a device frame with pitch().
    void upload(const std::uint8_t* r, const std::uint8_t* g, const std::uint8_t* b,
                std::uint8_t* d_dst, void* stream = nullptr);
    // Async D2H of the last results into host planes (nullptr = skip); sync if asked.
    void download_to(std::uint8_t* depth, std::uint8_t* filtered, StereoFormat f,
                     std::uint8_t* const* out, void* stream = nullptr, bool sync = true);
    // Interleaved RGB (the PPM payload, width*height*3 bytes) in and out: the payload is
    // copied to a device staging buffer and split into planes on the GPU; outputs are
    // interleaved on the GPU and copied back as ready-to-write payload
    // (output width * height * 3 bytes). Async on `stream`.
    void upload_interleaved(const std::uint8_t* rgb, std::uint8_t* d_dst, void* stream = nullptr);
    void download_interleaved(StereoFormat f, std::uint8_t* rgb_out, void* stream = nullptr,
                              bool sync = true);
    // One interleaved frame (host payload, width*height*3 bytes) through the pipeline: H2D into
    // the staging buffer, then the fused kernels read the payload directly and write the
    // anaglyph interleaved (anaglyph-only forward configs with 16-pixel blocks and w % 16 == 0),
    // or the payload is split into planes on the GPU first (every other config). Read the
    // outputs back with download_interleaved. Async on `stream`; timed = run_timed's events.
    void run_interleaved(const std::uint8_t* rgb, bool timed = false, void* stream = nullptr);
    struct Impl;

private:
    std::shared_ptr<Impl> impl_;
};

}  // namespace p3s
