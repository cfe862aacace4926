// The drop-in C ABI (include/pseudo3d.h: the reference's 49 functions, replacing
// /root/reference/proj/src/capi.cpp:20-385) plus the B200 extensions of include/p3s_gpu.h.
//
// Behaviour kept from the reference: opaque caller-owned handles, borrowed result views,
// thread-local last error cleared on success, the exception -> status taxonomy
// (capi.cpp:60-79), config setters that validate the whole candidate and roll back
// (capi.cpp:95-104), and its error strings. New: CUDA failures (no device, OOM, launch
// errors) map to P3S_ERR_INTERNAL with the CUDA message; there is no CPU fallback.
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <exception>
#include <map>
#include <mutex>
#include <memory>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "p3s/pipeline.hpp"
#include "p3s_gpu.h"
#include "p3s_cu.h"
#include "p3s_host.hpp"
#include "p3s_nvtx.hpp"
#include "pseudo3d.h"

struct p3s_image {
    p3s::ImageRGB8 img;
};
struct p3s_graymap {
    p3s::GrayMap map;
};
struct p3s_buffer {
    std::vector<std::uint8_t> bytes;
};
struct p3s_config {
    p3s::ConversionConfig cfg;
    int threads = 0;
};
struct p3s_result {
    std::map<unsigned, p3s_image> outputs;
    // depth / filtered depth stay on the GPU until first asked for (deferred); the host
    // graymaps below are filled from it on first access
    std::shared_ptr<p3s::DeferredMaps> deferred;
    mutable std::mutex mu;
    mutable p3s_graymap depth;
    mutable p3s_graymap filtered_depth;
    mutable bool maps_ready = false;
    p3s_timings timings{};
};
struct p3s_bench_report {
    p3s::BenchReport report;
};
struct p3s_pipeline {
    std::unique_ptr<p3s::Pipeline> p;
};
struct p3s_video {
    // One shard per GPU, one host thread each. Frames are independent (reference
    // sequence.cpp:59-77), so shards take the next frame index from a shared counter (a
    // dynamic queue: frames of uneven cost, e.g. parallax-dependent inpaint, balance
    // themselves) and pipeline it over their streams; outputs land at their frame index.
    // A shard whose device fails is retired and every frame it took is re-queued to the
    // healthy shards.
    struct Shard {
        int device = 0;
        bool failed = false;
        std::vector<std::unique_ptr<p3s::Pipeline>> pipes;
    };
    std::vector<Shard> shards;
    int w = 0, h = 0;
    unsigned format = 1;
    long long requeued = 0;     // frames re-run after a shard failed (all calls)
    int fail_shard = -1;        // test hook (P3S_VIDEO_FAIL="shard:frames"): that shard
    int fail_after = 0;         // throws a DeviceError after taking `fail_after` frames
};

namespace {

thread_local std::string g_last_error;

p3s_status fail(p3s_status st, const std::string& msg) {
    g_last_error = msg;
    return st;
}

template <class F>
p3s_status guarded(F&& body) noexcept {
    try {
        body();
        g_last_error.clear();
        return P3S_OK;
    } catch (const p3s::PnmError& e) {
        return fail(P3S_ERR_DECODE, e.what());
    } catch (const p3s::SequenceError& e) {
        return fail(P3S_ERR_DECODE, e.what());
    } catch (const p3s::IoError& e) {
        return fail(P3S_ERR_IO, e.what());
    } catch (const p3s::DeviceError& e) {
        return fail(P3S_ERR_INTERNAL, e.what());
    } catch (const std::invalid_argument& e) {
        return fail(P3S_ERR_INVALID, e.what());
    } catch (const std::bad_alloc&) {
        return fail(P3S_ERR_INTERNAL, "out of memory");
    } catch (const std::exception& e) {
        return fail(P3S_ERR_INTERNAL, e.what());
    }
}

p3s_timings to_c(const p3s::StageTimings& t) {
    p3s_timings o;
    o.depth_gen_ns = t.depth_gen_ns;
    o.filter_ns = t.filter_ns;
    o.dibr_ns = t.dibr_ns;
    o.inpaint_left_ns = t.inpaint_left_ns;
    o.inpaint_right_ns = t.inpaint_right_ns;
    o.format_ns = t.format_ns;
    o.pure_ns = t.pure_ns();
    return o;
}

template <class F>
p3s_status update_config(p3s_config* cfg, F&& mutate) {
    if (!cfg) return fail(P3S_ERR_INVALID, "null config");
    p3s::ConversionConfig cand = cfg->cfg;
    mutate(cand);
    return guarded([&] {
        cand.validate();
        cfg->cfg = cand;
    });
}

p3s::ImageRGB8 image_from(const uint8_t* r, const uint8_t* g, const uint8_t* b, int w, int h) {
    p3s::ImageRGB8 img(w, h, false);
    const std::size_t n = img.size();
    std::memcpy(img.r.data(), r, n);
    std::memcpy(img.g.data(), g, n);
    std::memcpy(img.b.data(), b, n);
    return img;
}

void image_to(const p3s::ImageRGB8& img, uint8_t* r, uint8_t* g, uint8_t* b) {
    const std::size_t n = img.size();
    std::memcpy(r, img.r.data(), n);
    std::memcpy(g, img.g.data(), n);
    std::memcpy(b, img.b.data(), n);
}

p3s::GrayMap gray_from(const uint8_t* p, int w, int h) {
    p3s::GrayMap m(w, h, false);
    std::memcpy(m.data.data(), p, m.size());
    return m;
}

}  // namespace

extern "C" {

const char* p3s_version(void) { return "1.0.0"; }

const char* p3s_status_name(p3s_status s) {
    switch (s) {
        case P3S_OK: return "ok";
        case P3S_ERR_INVALID: return "invalid argument";
        case P3S_ERR_IO: return "io error";
        case P3S_ERR_DECODE: return "decode error";
        case P3S_ERR_INTERNAL: return "internal error";
    }
    return "unknown";
}

const char* p3s_last_error(void) { return g_last_error.c_str(); }

// ---- buffers ----
const uint8_t* p3s_buffer_data(const p3s_buffer* b) { return b ? b->bytes.data() : nullptr; }
size_t p3s_buffer_size(const p3s_buffer* b) { return b ? b->bytes.size() : 0; }
void p3s_buffer_free(p3s_buffer* b) { delete b; }

// ---- images ----
p3s_status p3s_image_create(int width, int height, p3s_image** out) {
    if (!out) return fail(P3S_ERR_INVALID, "null output pointer");
    return guarded([&] { *out = new p3s_image{p3s::ImageRGB8(width, height)}; });
}
void p3s_image_free(p3s_image* img) { delete img; }
int p3s_image_width(const p3s_image* img) { return img ? img->img.width : 0; }
int p3s_image_height(const p3s_image* img) { return img ? img->img.height : 0; }
const uint8_t* p3s_image_plane(const p3s_image* img, int channel) {
    if (!img || channel < 0 || channel > 2) return nullptr;
    return img->img.plane(channel).data();
}
uint8_t* p3s_image_plane_mut(p3s_image* img, int channel) {
    return const_cast<uint8_t*>(p3s_image_plane(img, channel));
}
p3s_status p3s_image_decode_ppm(const uint8_t* data, size_t size, p3s_image** out) {
    if (!data || !out) return fail(P3S_ERR_INVALID, "null argument");
    return guarded([&] { *out = new p3s_image{p3s::decode_ppm(data, size)}; });
}
p3s_status p3s_image_encode_ppm(const p3s_image* img, p3s_buffer** out) {
    if (!img || !out) return fail(P3S_ERR_INVALID, "null argument");
    return guarded([&] { *out = new p3s_buffer{p3s::encode_ppm(img->img)}; });
}
p3s_status p3s_image_load_ppm(const char* path, p3s_image** out) {
    if (!path || !out) return fail(P3S_ERR_INVALID, "null argument");
    return guarded([&] {
        const auto bytes = p3s::read_file(path);
        *out = new p3s_image{p3s::decode_ppm(bytes.data(), bytes.size())};
    });
}
p3s_status p3s_image_save_ppm(const char* path, const p3s_image* img) {
    if (!path || !img) return fail(P3S_ERR_INVALID, "null argument");
    return guarded([&] {
        const auto bytes = p3s::encode_ppm(img->img);
        p3s::write_file(path, bytes.data(), bytes.size());
    });
}

// ---- gray maps ----
void p3s_graymap_free(p3s_graymap* m) { delete m; }
int p3s_graymap_width(const p3s_graymap* m) { return m ? m->map.width : 0; }
int p3s_graymap_height(const p3s_graymap* m) { return m ? m->map.height : 0; }
const uint8_t* p3s_graymap_data(const p3s_graymap* m) { return m ? m->map.data.data() : nullptr; }
p3s_status p3s_graymap_decode_pgm(const uint8_t* data, size_t size, p3s_graymap** out) {
    if (!data || !out) return fail(P3S_ERR_INVALID, "null argument");
    return guarded([&] { *out = new p3s_graymap{p3s::decode_pgm(data, size)}; });
}
p3s_status p3s_graymap_encode_pgm(const p3s_graymap* m, p3s_buffer** out) {
    if (!m || !out) return fail(P3S_ERR_INVALID, "null argument");
    return guarded([&] { *out = new p3s_buffer{p3s::encode_pgm(m->map)}; });
}
p3s_status p3s_graymap_load_pgm(const char* path, p3s_graymap** out) {
    if (!path || !out) return fail(P3S_ERR_INVALID, "null argument");
    return guarded([&] {
        const auto bytes = p3s::read_file(path);
        *out = new p3s_graymap{p3s::decode_pgm(bytes.data(), bytes.size())};
    });
}
p3s_status p3s_graymap_save_pgm(const char* path, const p3s_graymap* m) {
    if (!path || !m) return fail(P3S_ERR_INVALID, "null argument");
    return guarded([&] {
        const auto bytes = p3s::encode_pgm(m->map);
        p3s::write_file(path, bytes.data(), bytes.size());
    });
}

// ---- configuration ----
p3s_config* p3s_config_create(void) { return new (std::nothrow) p3s_config; }
void p3s_config_free(p3s_config* cfg) { delete cfg; }
p3s_status p3s_config_set_base(p3s_config* cfg, int base) {
    return update_config(cfg, [&](p3s::ConversionConfig& c) { c.base = base; });
}
p3s_status p3s_config_set_auto_base(p3s_config* cfg) {
    return update_config(cfg, [&](p3s::ConversionConfig& c) {
        c.base = p3s::ConversionConfig::kAutoBase;
    });
}
p3s_status p3s_config_set_pop_threshold(p3s_config* cfg, int t) {
    return update_config(cfg, [&](p3s::ConversionConfig& c) { c.pop_threshold = t; });
}
p3s_status p3s_config_set_sigma_spatial(p3s_config* cfg, double s) {
    return update_config(cfg, [&](p3s::ConversionConfig& c) { c.sigma_spatial = s; });
}
p3s_status p3s_config_set_sigma_range(p3s_config* cfg, double s) {
    return update_config(cfg, [&](p3s::ConversionConfig& c) { c.sigma_range = s; });
}
p3s_status p3s_config_set_depth_block(p3s_config* cfg, int b) {
    return update_config(cfg, [&](p3s::ConversionConfig& c) { c.depth_block = b; });
}
p3s_status p3s_config_set_inpaint_block(p3s_config* cfg, int b) {
    return update_config(cfg, [&](p3s::ConversionConfig& c) { c.inpaint_block = b; });
}
p3s_status p3s_config_set_depth_weights(p3s_config* cfg, double alpha, double beta) {
    return update_config(cfg, [&](p3s::ConversionConfig& c) {
        c.alpha = alpha;
        c.beta = beta;
    });
}
p3s_status p3s_config_set_mode(p3s_config* cfg, p3s_dibr_mode mode) {
    if (mode != P3S_MODE_FORWARD_ZBUFFER && mode != P3S_MODE_BACKWARD_FALLBACK)
        return fail(P3S_ERR_INVALID, "unknown dibr mode");
    return update_config(cfg, [&](p3s::ConversionConfig& c) {
        c.dibr_mode = mode == P3S_MODE_FORWARD_ZBUFFER ? p3s::DibrMode::kForwardZBuffer
                                                       : p3s::DibrMode::kBackwardFallback;
    });
}
p3s_status p3s_config_set_formats(p3s_config* cfg, unsigned mask) {
    return update_config(cfg, [&](p3s::ConversionConfig& c) { c.formats = mask; });
}
p3s_status p3s_config_set_threads(p3s_config* cfg, int threads) {
    if (!cfg) return fail(P3S_ERR_INVALID, "null config");
    cfg->threads = threads;
    return P3S_OK;
}

// ---- conversion ----
p3s_status p3s_convert(const p3s_image* src, const p3s_config* cfg, p3s_result** out) {
    if (!src || !cfg || !out) return fail(P3S_ERR_INVALID, "null argument");
    return guarded([&] {
        auto res = std::make_unique<p3s_result>();
        p3s::ConversionResult core = p3s::convert_image_deferred(
            src->img, cfg->cfg, p3s::Device::current(), res->deferred);
        for (auto& [fmt, img] : core.outputs)
            res->outputs.emplace(static_cast<unsigned>(fmt), p3s_image{std::move(img)});
        res->timings = to_c(core.timings);
        *out = res.release();
    });
}
p3s_status p3s_result_output(const p3s_result* r, p3s_format format, const p3s_image** out) {
    if (!r || !out) return fail(P3S_ERR_INVALID, "null argument");
    const auto it = r->outputs.find(static_cast<unsigned>(format));
    if (it == r->outputs.end())
        return fail(P3S_ERR_INVALID, "format was not requested in the configuration");
    *out = &it->second;
    return P3S_OK;
}
namespace {
// Downloads the deferred maps on first access. Returns false (last error set) on failure.
bool result_maps(const p3s_result* r) {
    std::lock_guard<std::mutex> lk(r->mu);
    if (r->maps_ready) return true;
    try {
        if (r->deferred) {
            r->depth.map = r->deferred->depth();
            r->filtered_depth.map = r->deferred->filtered();
        }
        r->maps_ready = true;
        return true;
    } catch (const std::exception& e) {
        g_last_error = std::string("downloading the depth maps failed: ") + e.what();
        return false;
    }
}
}  // namespace

const p3s_graymap* p3s_result_depth(const p3s_result* r) {
    return r && result_maps(r) ? &r->depth : nullptr;
}
const p3s_graymap* p3s_result_filtered_depth(const p3s_result* r) {
    return r && result_maps(r) ? &r->filtered_depth : nullptr;
}
p3s_status p3s_result_timings(const p3s_result* r, p3s_timings* out) {
    if (!r || !out) return fail(P3S_ERR_INVALID, "null argument");
    *out = r->timings;
    return P3S_OK;
}
void p3s_result_free(p3s_result* r) { delete r; }

p3s_status p3s_depth_map(const p3s_image* src, const p3s_config* cfg, p3s_graymap** out) {
    if (!src || !cfg || !out) return fail(P3S_ERR_INVALID, "null argument");
    return guarded([&] {
        cfg->cfg.validate();
        *out = new p3s_graymap{p3s::generate_depth(src->img, cfg->cfg, p3s::Device::current())};
    });
}

// ---- sequences ----
p3s_status p3s_convert_sequence(const char* in_dir, const char* pattern, const char* out_dir,
                                const p3s_config* cfg, p3s_sequence_summary* summary,
                                p3s_buffer** timing_csv) {
    if (!in_dir || !pattern || !out_dir || !cfg) return fail(P3S_ERR_INVALID, "null argument");
    return guarded([&] {
        const p3s::SequenceReport rep =
            p3s::convert_sequence_dir(in_dir, pattern, out_dir, cfg->cfg, cfg->threads);
        if (summary) {
            summary->frames = static_cast<int64_t>(rep.frames.size());
            summary->pure_sum_ns = rep.pure_sum_ns();
            summary->pure_min_ns = rep.pure_min_ns();
            summary->pure_max_ns = rep.pure_max_ns();
            summary->pure_mean_ns = rep.pure_mean_ns();
            summary->wall_ns = rep.wall_ns;
        }
        if (timing_csv) {
            const std::string csv = rep.to_csv(p3s::resolve_threads(cfg->threads));
            *timing_csv = new p3s_buffer{{csv.begin(), csv.end()}};
        }
    });
}

// ---- bench ----
p3s_status p3s_bench(const int* widths, const int* heights, size_t nsizes,
                     const int* thread_counts, size_t nthreads, int reps, uint64_t seed,
                     const p3s_config* cfg, p3s_bench_report** out) {
    if (!widths || !heights || !thread_counts || !cfg || !out)
        return fail(P3S_ERR_INVALID, "null argument");
    return guarded([&] {
        std::vector<std::pair<int, int>> sizes;
        for (size_t i = 0; i < nsizes; ++i) sizes.emplace_back(widths[i], heights[i]);
        std::vector<int> threads(thread_counts, thread_counts + nthreads);
        *out = new p3s_bench_report{p3s::run_bench(sizes, threads, reps, seed, cfg->cfg)};
    });
}
p3s_status p3s_bench_report_csv(const p3s_bench_report* r, p3s_buffer** out) {
    if (!r || !out) return fail(P3S_ERR_INVALID, "null argument");
    return guarded([&] {
        const std::string csv = r->report.to_csv();
        *out = new p3s_buffer{{csv.begin(), csv.end()}};
    });
}
double p3s_bench_report_speedup(const p3s_bench_report* r, int width, int height, int threads) {
    return r ? r->report.speedup(width, height, threads) : 0.0;
}
void p3s_bench_report_free(p3s_bench_report* r) { delete r; }

// ============================ p3s_gpu.h extensions ========================================

p3s_status p3s_config_get_params(const p3s_config* cfg, p3s_params* o) {
    if (!cfg || !o) return fail(P3S_ERR_INVALID, "null argument");
    const p3s::ConversionConfig& c = cfg->cfg;
    o->base = c.base;
    o->pop_threshold = c.pop_threshold;
    o->sigma_spatial = c.sigma_spatial;
    o->sigma_range = c.sigma_range;
    o->depth_block = c.depth_block;
    o->inpaint_block = c.inpaint_block;
    o->alpha = c.alpha;
    o->beta = c.beta;
    o->mode = c.dibr_mode == p3s::DibrMode::kBackwardFallback ? 1 : 0;
    o->formats = c.formats;
    return P3S_OK;
}

p3s_status p3s_config_set_params(p3s_config* cfg, const p3s_params* p) {
    if (!p) return fail(P3S_ERR_INVALID, "null argument");
    if (p->mode != 0 && p->mode != 1) return fail(P3S_ERR_INVALID, "unknown dibr mode");
    return update_config(cfg, [&](p3s::ConversionConfig& c) {
        c.base = p->base < 0 ? p3s::ConversionConfig::kAutoBase : p->base;
        c.pop_threshold = p->pop_threshold;
        c.sigma_spatial = p->sigma_spatial;
        c.sigma_range = p->sigma_range;
        c.depth_block = p->depth_block;
        c.inpaint_block = p->inpaint_block;
        c.alpha = p->alpha;
        c.beta = p->beta;
        c.dibr_mode = p->mode ? p3s::DibrMode::kBackwardFallback : p3s::DibrMode::kForwardZBuffer;
        c.formats = p->formats;
    });
}

int p3s_gpu_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

p3s_status p3s_gpu_set_device(int ordinal) {
    return guarded([&] {
        const cudaError_t e = cudaSetDevice(ordinal);
        if (e != cudaSuccess) {
            cudaGetLastError();
            throw p3s::DeviceError(std::string("cudaSetDevice: ") + cudaGetErrorString(e));
        }
        p3s::Device::current();
    });
}

p3s_status p3s_gpu_device_name(char* buf, size_t cap) {
    if (!buf || !cap) return fail(P3S_ERR_INVALID, "null argument");
    return guarded([&] {
        p3s::Device& d = p3s::Device::current();
        cudaDeviceProp prop;
        if (cudaGetDeviceProperties(&prop, d.ordinal()) != cudaSuccess)
            throw p3s::DeviceError("cudaGetDeviceProperties failed");
        std::strncpy(buf, prop.name, cap - 1);
        buf[cap - 1] = 0;
    });
}

int p3s_gpu_band_plan(int w, int h, const p3s_config* cfg, int* out, int cap) {
    if (!cfg || (cap > 0 && !out) || w <= 0 || h <= 0) {
        fail(P3S_ERR_INVALID, "invalid argument");
        return -1;
    }
    int n = -1;
    const p3s_status st = guarded([&] {
        cfg->cfg.validate();
        const int radius = static_cast<int>(std::ceil(2.0 * cfg->cfg.sigma_spatial));
        const std::vector<p3s::BandEnd> b = p3s::band_plan(w, h, radius, cfg->cfg.depth_block);
        for (std::size_t i = 0; i < b.size() && static_cast<int>(i) < cap; ++i) {
            const int v[5] = {b[i].in_rows, b[i].dtile, b[i].brow, b[i].urow, b[i].btile};
            for (int j = 0; j < 5; ++j) out[5 * i + j] = v[j];
        }
        n = static_cast<int>(b.size());
    });
    return st == P3S_OK ? n : -1;
}

int p3s_gpu_dibr_integer_columns(int w, const p3s_config* cfg) {
    if (!cfg || w <= 0) {
        fail(P3S_ERR_INVALID, "invalid argument");
        return -1;
    }
    int r = -1;
    const p3s_status st = guarded([&] {
        cfg->cfg.validate();
        r = p3s::dibr_integer_columns(w, cfg->cfg) ? 1 : 0;
    });
    return st == P3S_OK ? r : -1;
}

p3s_status p3s_gpu_sm_count(int* out) {
    if (!out) return fail(P3S_ERR_INVALID, "null argument");
    return guarded([&] {
        p3s::Device& d = p3s::Device::current();
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d.ordinal()) != cudaSuccess)
            throw p3s::DeviceError("cudaDeviceGetAttribute failed");
        *out = n;
    });
}

#define NEED(...)                                                          \
    do {                                                                   \
        const void* ptrs_[] = {__VA_ARGS__};                               \
        for (const void* q_ : ptrs_)                                       \
            if (!q_) return fail(P3S_ERR_INVALID, "null argument");        \
    } while (0)

p3s_status p3s_gpu_luma(const uint8_t* r, const uint8_t* g, const uint8_t* b, int w, int h,
                        uint8_t* out) {
    NEED(r, g, b, out);
    return guarded([&] {
        const p3s::GrayMap m = p3s::luma(image_from(r, g, b, w, h), p3s::Device::current());
        std::memcpy(out, m.data.data(), m.size());
    });
}

p3s_status p3s_gpu_block_depth(const uint8_t* r, const uint8_t* g, const uint8_t* b, int w, int h,
                               const p3s_config* cfg, double* values) {
    NEED(r, g, b, cfg, values);
    return guarded([&] {
        const p3s::BlockGrid gr =
            p3s::block_depth(image_from(r, g, b, w, h), cfg->cfg, p3s::Device::current());
        std::memcpy(values, gr.values.data(), gr.values.size() * sizeof(double));
    });
}

p3s_status p3s_gpu_upsample(const double* values, int w, int h, int block, uint8_t* out) {
    NEED(values, out);
    return guarded([&] {
        if (block < 4) throw std::invalid_argument("depth_block must be >= 4");
        p3s::BlockGrid g;
        g.block = block;
        g.width = w;
        g.height = h;
        p3s::pixel_count(w, h);
        g.blocks_x = (w + block - 1) / block;
        g.blocks_y = (h + block - 1) / block;
        g.values.assign(values, values + static_cast<size_t>(g.blocks_x) * g.blocks_y);
        const p3s::GrayMap m = p3s::upsample_block_grid(g, p3s::Device::current());
        std::memcpy(out, m.data.data(), m.size());
    });
}

p3s_status p3s_gpu_generate_depth(const uint8_t* r, const uint8_t* g, const uint8_t* b, int w,
                                  int h, const p3s_config* cfg, uint8_t* depth) {
    NEED(r, g, b, cfg, depth);
    return guarded([&] {
        const p3s::GrayMap m =
            p3s::generate_depth(image_from(r, g, b, w, h), cfg->cfg, p3s::Device::current());
        std::memcpy(depth, m.data.data(), m.size());
    });
}

p3s_status p3s_gpu_cross_bilateral(const uint8_t* depth, const uint8_t* guide, int w, int h,
                                   const p3s_config* cfg, uint8_t* out) {
    NEED(depth, guide, cfg, out);
    return guarded([&] {
        cfg->cfg.validate();
        const p3s::GrayMap m = p3s::cross_bilateral(gray_from(depth, w, h), gray_from(guide, w, h),
                                                    cfg->cfg, p3s::Device::current());
        std::memcpy(out, m.data.data(), m.size());
    });
}

p3s_status p3s_gpu_cross_bilateral_raw(const uint8_t* depth, const uint8_t* guide, int w, int h,
                                       const p3s_config* cfg, double* out) {
    NEED(depth, guide, cfg, out);
    return guarded([&] {
        cfg->cfg.validate();
        const std::vector<double> v = p3s::cross_bilateral_raw(
            gray_from(depth, w, h), gray_from(guide, w, h), cfg->cfg, p3s::Device::current());
        std::memcpy(out, v.data(), v.size() * sizeof(double));
    });
}

p3s_status p3s_gpu_reconstruct(const uint8_t* r, const uint8_t* g, const uint8_t* b,
                               const uint8_t* depth, int w, int h, const p3s_config* cfg,
                               uint8_t* lr, uint8_t* lg, uint8_t* lb, uint8_t* rr, uint8_t* rg,
                               uint8_t* rb, uint8_t* lmask, uint8_t* rmask) {
    NEED(r, g, b, depth, cfg, lr, lg, lb, rr, rg, rb, lmask, rmask);
    return guarded([&] {
        cfg->cfg.validate();
        const p3s::StereoFrames f = p3s::reconstruct(image_from(r, g, b, w, h),
                                                     gray_from(depth, w, h), cfg->cfg,
                                                     p3s::Device::current());
        image_to(f.left, lr, lg, lb);
        image_to(f.right, rr, rg, rb);
        std::memcpy(lmask, f.left_mask.damaged.data(), f.left_mask.size());
        std::memcpy(rmask, f.right_mask.damaged.data(), f.right_mask.size());
    });
}

p3s_status p3s_gpu_inpaint(const uint8_t* r, const uint8_t* g, const uint8_t* b,
                           const uint8_t* mask, int w, int h, const p3s_config* cfg, uint8_t* outr,
                           uint8_t* outg, uint8_t* outb, int64_t* stats) {
    NEED(r, g, b, mask, cfg, outr, outg, outb);
    return guarded([&] {
        cfg->cfg.validate();
        p3s::DamageMask m(w, h);
        std::memcpy(m.damaged.data(), mask, m.size());
        p3s::InpaintStats st;
        const p3s::ImageRGB8 o =
            p3s::inpaint(image_from(r, g, b, w, h), m, cfg->cfg, p3s::Device::current(), &st);
        image_to(o, outr, outg, outb);
        if (stats) {
            stats[0] = st.passes;
            stats[1] = static_cast<int64_t>(st.repaired);
            stats[2] = static_cast<int64_t>(st.fallback_filled);
        }
    });
}

p3s_status p3s_gpu_anaglyph(const uint8_t* lr, const uint8_t* lg, const uint8_t* lb,
                            const uint8_t* rr, const uint8_t* rg, const uint8_t* rb, int w, int h,
                            uint8_t* outr, uint8_t* outg, uint8_t* outb) {
    NEED(lr, lg, lb, rr, rg, rb, outr, outg, outb);
    return guarded([&] {
        const p3s::ImageRGB8 o = p3s::anaglyph(image_from(lr, lg, lb, w, h),
                                               image_from(rr, rg, rb, w, h), p3s::Device::current());
        image_to(o, outr, outg, outb);
    });
}

p3s_status p3s_gpu_side_by_side(const uint8_t* lr, const uint8_t* lg, const uint8_t* lb,
                                const uint8_t* rr, const uint8_t* rg, const uint8_t* rb, int w,
                                int h, int half, uint8_t* outr, uint8_t* outg, uint8_t* outb) {
    NEED(lr, lg, lb, rr, rg, rb, outr, outg, outb);
    return guarded([&] {
        const p3s::ImageRGB8 o =
            p3s::side_by_side(image_from(lr, lg, lb, w, h), image_from(rr, rg, rb, w, h),
                              half != 0, p3s::Device::current());
        image_to(o, outr, outg, outb);
    });
}

// ---- device-resident pipeline ----
p3s_status p3s_pipeline_create(int w, int h, const p3s_config* cfg, p3s_pipeline** out) {
    NEED(cfg, out);
    return guarded([&] {
        auto p = std::make_unique<p3s_pipeline>();
        p->p = std::make_unique<p3s::Pipeline>(w, h, cfg->cfg, p3s::Device::current());
        *out = p.release();
    });
}
void p3s_pipeline_free(p3s_pipeline* p) { delete p; }
int p3s_pipeline_pitch(const p3s_pipeline* p) { return p ? p->p->pitch() : 0; }
size_t p3s_pipeline_frame_bytes(const p3s_pipeline* p) { return p ? p->p->frame_bytes() : 0; }
void* p3s_pipeline_stream(const p3s_pipeline* p) { return p ? p->p->stream() : nullptr; }

p3s_status p3s_pipeline_run(p3s_pipeline* p, const uint8_t* d_src, int timed, void* stream) {
    NEED(p, d_src);
    return guarded([&] {
        if (timed)
            p->p->run_timed(d_src, stream);
        else
            p->p->run(d_src, stream);
    });
}

p3s_status p3s_pipeline_timings(p3s_pipeline* p, p3s_timings* out) {
    NEED(p, out);
    return guarded([&] { *out = to_c(p->p->last_timings()); });
}

p3s_status p3s_pipeline_timing_sum(p3s_pipeline* p, p3s_timings* sum, int64_t* count,
                                   int reset) {
    NEED(p, sum);
    return guarded([&] {
        long long n = 0;
        *sum = to_c(p->p->accumulated_timings(&n, reset != 0));
        if (count) *count = n;
    });
}

p3s_status p3s_pipeline_bilateral_kernel_sum(p3s_pipeline* p, int64_t* sum_ns, int64_t* count,
                                             int reset) {
    NEED(p, sum_ns);
    return guarded([&] {
        long long n = 0;
        *sum_ns = p->p->bilateral_kernel_ns(&n, reset != 0);
        if (count) *count = n;
    });
}

p3s_status p3s_pipeline_set_inpaint_ctas(p3s_pipeline* p, int ctas) {
    NEED(p);
    if (ctas < 0) return fail(P3S_ERR_INVALID, "inpaint CTAs must be >= 0");
    return guarded([&] { p->p->set_inpaint_ctas(ctas); });
}

p3s_status p3s_pipeline_download(p3s_pipeline* p, uint8_t* depth, uint8_t* filtered,
                                 p3s_format format, uint8_t* outr, uint8_t* outg, uint8_t* outb) {
    NEED(p);
    return guarded([&] {
        uint8_t* o[3] = {outr, outg, outb};
        p->p->download_to(depth, filtered, static_cast<p3s::StereoFormat>(format),
                          (outr || outg || outb) ? o : nullptr, nullptr, true);
    });
}

p3s_status p3s_pipeline_inpaint_stats(p3s_pipeline* p, int64_t* stats) {
    NEED(p, stats);
    return guarded([&] {
        p3s::InpaintStats l, r;
        p->p->inpaint_stats(l, r);
        stats[0] = l.passes;
        stats[1] = static_cast<int64_t>(l.repaired);
        stats[2] = static_cast<int64_t>(l.fallback_filled);
        stats[3] = r.passes;
        stats[4] = static_cast<int64_t>(r.repaired);
        stats[5] = static_cast<int64_t>(r.fallback_filled);
    });
}

p3s_status p3s_pipeline_upload(p3s_pipeline* p, const uint8_t* r, const uint8_t* g,
                               const uint8_t* b, uint8_t* d_dst, void* stream) {
    NEED(p, r, g, b, d_dst);
    return guarded([&] { p->p->upload(r, g, b, d_dst, stream); });
}

// ---- video ----
namespace {

p3s_status video_create(int w, int h, const p3s_config* cfg, const int* devices, int ndev,
                        int streams, p3s_video** out) {
    NEED(cfg, out);
    return guarded([&] {
        if (streams < 1) throw std::invalid_argument("video needs at least one stream");
        if (ndev < 1) throw std::invalid_argument("video needs at least one device");
        cfg->cfg.validate();
        auto v = std::make_unique<p3s_video>();
        v->w = w;
        v->h = h;
        const unsigned f = cfg->cfg.formats;
        v->format = (f & 1u) ? 1u : (f & 2u) ? 2u : 4u;
        int caller = 0;
        cudaGetDevice(&caller);
        try {
            for (int k = 0; k < ndev; ++k) {
                const int d = devices ? devices[k] : caller;
                if (cudaSetDevice(d) != cudaSuccess) {
                    cudaGetLastError();
                    throw p3s::DeviceError("cannot select CUDA device " + std::to_string(d));
                }
                p3s::Device& dev = p3s::Device::current();
                p3s_video::Shard shard;
                shard.device = d;
                // several frames in flight: each cooperative inpaint takes a quarter of the
                // SMs, leaving the rest to the other streams' filters (Pipeline::set_inpaint_ctas)
                int sms = 0;
                cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
                const char* env = std::getenv("P3S_VIDEO_INPAINT_CTAS");
                const int ctas = env ? std::atoi(env) : (streams > 1 ? sms / 4 : 0);
                for (int i = 0; i < streams; ++i) {
                    shard.pipes.push_back(std::make_unique<p3s::Pipeline>(w, h, cfg->cfg, dev));
                    shard.pipes.back()->set_inpaint_ctas(ctas);
                }
                v->shards.push_back(std::move(shard));
            }
        } catch (...) {
            cudaSetDevice(caller);
            throw;
        }
        cudaSetDevice(caller);
        if (const char* f = std::getenv("P3S_VIDEO_FAIL")) {
            v->fail_shard = std::atoi(f);
            const char* c = std::strchr(f, ':');
            v->fail_after = c ? std::atoi(c + 1) : 0;
        }
        *out = v.release();
    });
}

// One convert call's shared state: the frame counter, the re-queue of failed shards' frames
// and the first failure.
struct VideoRun {
    const uint8_t* const* frames;
    uint8_t* const* outs;
    int n;
    bool interleaved;
    std::atomic<int> next{0};
    std::mutex mu;
    std::deque<int> retry;
    std::exception_ptr first_error;

    int take() {
        {
            std::lock_guard<std::mutex> lk(mu);
            if (!retry.empty()) {
                const int i = retry.front();
                retry.pop_front();
                return i;
            }
        }
        const int i = next.fetch_add(1);
        return i < n ? i : -1;
    }
};

void video_frame(p3s::Pipeline& p, const p3s_video& v, const VideoRun& run, int i, std::size_t N,
                 std::size_t on);

// Shard k's host thread: takes frames until the run is drained, pipelined over its streams.
// interleaved: frames/outs are RGB-interleaved payloads (converted on the device).
void video_shard(p3s_video& v, std::size_t k, VideoRun& run) {
    p3s_video::Shard& sh = v.shards[k];
    std::vector<int> taken;
    try {
        if (cudaSetDevice(sh.device) != cudaSuccess) {
            cudaGetLastError();
            throw p3s::DeviceError("cannot select CUDA device " + std::to_string(sh.device));
        }
        const std::size_t N = static_cast<std::size_t>(v.w) * v.h;
        const std::size_t on = v.format == 4u ? 2 * N : N;
        const std::size_t S = sh.pipes.size();
        std::size_t j = 0;
        for (int i; (i = run.take()) >= 0; ++j) {
            taken.push_back(i);
            if (static_cast<int>(k) == v.fail_shard && static_cast<int>(taken.size()) > v.fail_after)
                throw p3s::DeviceError("injected device failure (P3S_VIDEO_FAIL) on shard " + std::to_string(k));
            p3s::Pipeline& p = *sh.pipes[j % S];
            video_frame(p, v, run, i, N, on);
        }
        for (auto& p : sh.pipes) {
            const cudaError_t e = cudaStreamSynchronize(static_cast<cudaStream_t>(p->stream()));
            if (e != cudaSuccess) throw p3s::DeviceError(cudaGetErrorString(e));
        }
    } catch (...) {
        // the device is retired; its frames (done or not: outputs are simply rewritten) go
        // back to the healthy shards once its queued work has drained (or failed)
        for (auto& p : sh.pipes) cudaStreamSynchronize(static_cast<cudaStream_t>(p->stream()));
        cudaGetLastError();
        std::lock_guard<std::mutex> lk(run.mu);
        sh.failed = true;
        if (!run.first_error) run.first_error = std::current_exception();
        for (int i : taken) run.retry.push_back(i);
        v.requeued += static_cast<long long>(taken.size());
    }
}
}  // namespace

namespace {
void video_frame(p3s::Pipeline& p, const p3s_video& v, const VideoRun& run, int i, std::size_t N,
                 std::size_t on) {
    const bool interleaved = run.interleaved;
    const uint8_t* const* frames = run.frames;
    uint8_t* const* outs = run.outs;
    p3s::NvtxRange nv(interleaved ? "p3s_video frame (interleaved)" : "p3s_video frame");
    {
        const uint8_t* f = frames[i];
        if (interleaved) {
            p.run_interleaved(f);
            p.download_interleaved(static_cast<p3s::StereoFormat>(v.format), outs[i], nullptr, false);
            return;
        }
        p.upload(f, f + N, f + 2 * N, p.d_input());
        p.run(p.d_input());
        uint8_t* o[3] = {outs[i], outs[i] + on, outs[i] + 2 * on};
        p.download_to(nullptr, nullptr, static_cast<p3s::StereoFormat>(v.format), o, nullptr,
                      false);
    }
}

}  // namespace

p3s_status p3s_video_create(int w, int h, const p3s_config* cfg, int streams, p3s_video** out) {
    return video_create(w, h, cfg, nullptr, 1, streams, out);
}

p3s_status p3s_video_create_devices(int w, int h, const p3s_config* cfg, const int* devices,
                                    int ndev, int streams, p3s_video** out) {
    NEED(devices);
    return video_create(w, h, cfg, devices, ndev, streams, out);
}

int p3s_video_shards(const p3s_video* v) { return v ? static_cast<int>(v->shards.size()) : 0; }

long long p3s_video_requeued(const p3s_video* v) { return v ? v->requeued : 0; }

int p3s_video_healthy_shards(const p3s_video* v) {
    if (!v) return 0;
    int n = 0;
    for (const auto& s : v->shards) n += !s.failed;
    return n;
}

void* p3s_host_alloc_near(int device, size_t bytes) {
    try {
        return p3s::pinned_alloc_near(device, bytes);
    } catch (...) {
        return nullptr;
    }
}

int p3s_gpu_numa_node(int device) { return p3s::device_numa_node(device); }

unsigned long long p3s_gpu_launch_count(void) { return p3s::cu::launch_count(); }

namespace {
p3s_status video_convert(p3s_video* v, const uint8_t* const* frames, int n, uint8_t* const* outs,
                         bool interleaved) {
    NEED(v, frames, outs);
    return guarded([&] {
        int caller = 0;
        cudaGetDevice(&caller);
        struct Restore {
            int d;
            ~Restore() { cudaSetDevice(d); }
        } restore{caller};
        if (n < 0) throw std::invalid_argument("frame count must be >= 0");
        VideoRun run;
        run.frames = frames;
        run.outs = outs;
        run.n = n;
        run.interleaved = interleaved;
        // one host thread per healthy GPU, no data crossing between GPUs; repeated while
        // frames of a failed shard wait in the re-queue and a healthy shard is left
        for (;;) {
            std::vector<std::size_t> live;
            for (std::size_t k = 0; k < v->shards.size(); ++k)
                if (!v->shards[k].failed) live.push_back(k);
            if (live.empty()) {
                if (run.first_error) std::rethrow_exception(run.first_error);
                throw p3s::DeviceError("video: every device of this video has failed");
            }
            if (live.size() == 1) {
                video_shard(*v, live[0], run);
            } else {
                std::vector<std::thread> threads;
                for (std::size_t k : live) threads.emplace_back([&, k] { video_shard(*v, k, run); });
                for (auto& t : threads) t.join();
            }
            std::lock_guard<std::mutex> lk(run.mu);
            if (run.retry.empty() && run.next.load() >= n) break;
        }
    });
}
}  // namespace

p3s_status p3s_video_convert(p3s_video* v, const uint8_t* const* frames, int n,
                             uint8_t* const* outs) {
    return video_convert(v, frames, n, outs, false);
}

p3s_status p3s_video_convert_interleaved(p3s_video* v, const uint8_t* const* frames, int n,
                                         uint8_t* const* outs) {
    return video_convert(v, frames, n, outs, true);
}

void p3s_video_free(p3s_video* v) { delete v; }

// ---- helpers ----
p3s_status p3s_gpu_malloc(size_t bytes, void** out) {
    NEED(out);
    return guarded([&] {
        p3s::Device::current();
        if (cudaMalloc(out, bytes) != cudaSuccess) {
            cudaGetLastError();
            throw std::bad_alloc();
        }
        // zero-filled, so row padding of frames built in it is defined
        if (cudaMemset(*out, 0, bytes) != cudaSuccess) {
            cudaGetLastError();
            cudaFree(*out);
            throw p3s::DeviceError("cudaMemset failed");
        }
    });
}
void p3s_gpu_free(void* p) {
    if (p) cudaFree(p);
}
p3s_status p3s_gpu_memset(void* p, int value, size_t bytes) {
    NEED(p);
    return guarded([&] {
        const cudaError_t e = cudaMemset(p, value, bytes);
        if (e != cudaSuccess) throw p3s::DeviceError(cudaGetErrorString(e));
    });
}
p3s_status p3s_gpu_stream_sync(void* stream) {
    return guarded([&] {
        const cudaError_t e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
        if (e != cudaSuccess) throw p3s::DeviceError(cudaGetErrorString(e));
    });
}
p3s_status p3s_gpu_device_sync(void) {
    return guarded([&] {
        const cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) throw p3s::DeviceError(cudaGetErrorString(e));
    });
}
p3s_status p3s_gpu_event_create(void** out) {
    NEED(out);
    return guarded([&] {
        cudaEvent_t ev;
        if (cudaEventCreate(&ev) != cudaSuccess) throw p3s::DeviceError("cudaEventCreate failed");
        *out = ev;
    });
}
p3s_status p3s_gpu_event_record(void* ev, void* stream) {
    NEED(ev);
    return guarded([&] {
        if (cudaEventRecord(static_cast<cudaEvent_t>(ev), static_cast<cudaStream_t>(stream)) !=
            cudaSuccess)
            throw p3s::DeviceError("cudaEventRecord failed");
    });
}
p3s_status p3s_gpu_stream_wait_event(void* stream, void* ev) {
    NEED(ev);
    return guarded([&] {
        if (cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), static_cast<cudaEvent_t>(ev), 0) !=
            cudaSuccess)
            throw p3s::DeviceError("cudaStreamWaitEvent failed");
    });
}
p3s_status p3s_gpu_event_elapsed_ms(void* a, void* b, float* ms) {
    NEED(a, b, ms);
    return guarded([&] {
        if (cudaEventSynchronize(static_cast<cudaEvent_t>(b)) != cudaSuccess ||
            cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(a), static_cast<cudaEvent_t>(b)) !=
                cudaSuccess)
            throw p3s::DeviceError("cudaEventElapsedTime failed");
    });
}
void p3s_gpu_event_destroy(void* ev) {
    if (ev) cudaEventDestroy(static_cast<cudaEvent_t>(ev));
}
void* p3s_host_alloc(size_t bytes) {
    try {
        return p3s::pinned_alloc(bytes);
    } catch (...) {
        return nullptr;
    }
}
void p3s_host_free(void* p) { p3s::pinned_free(p); }

p3s_status p3s_gpu_fp64_peak(double* ops_per_s) {
    NEED(ops_per_s);
    return guarded([&] {
        p3s::Device::current();
        const cudaError_t e = p3s::cu::fp64_peak(ops_per_s);
        if (e != cudaSuccess) throw p3s::DeviceError(cudaGetErrorString(e));
    });
}

p3s_status p3s_gpu_bilateral_path(const p3s_config* cfg, int* certified_fp32) {
    NEED(cfg, certified_fp32);
    return guarded([&] {
        const int r = static_cast<int>(std::ceil(2.0 * cfg->cfg.sigma_spatial));
        *certified_fp32 = p3s::cu::bilateral_fast_available(r) ? 1 : 0;
    });
}

p3s_status p3s_synthetic_frame(int w, int h, uint64_t seed, uint8_t* r, uint8_t* g, uint8_t* b) {
    NEED(r, g, b);
    return guarded([&] {
        if (w <= 0 || h <= 0) throw std::invalid_argument("synthetic_frame: dimensions must be positive");
        const p3s::ImageRGB8 img = p3s::synthetic_frame(w, h, seed);
        const std::size_t n = static_cast<std::size_t>(w) * h;
        std::memcpy(r, img.r.data(), n);
        std::memcpy(g, img.g.data(), n);
        std::memcpy(b, img.b.data(), n);
    });
}

p3s_status p3s_gpu_smem_peak(double* bytes_per_s, int gather) {
    NEED(bytes_per_s);
    return guarded([&] {
        p3s::Device::current();
        const cudaError_t e =
            gather ? p3s::cu::smem_gather_peak(bytes_per_s) : p3s::cu::smem_peak(bytes_per_s);
        if (e != cudaSuccess) throw p3s::DeviceError(cudaGetErrorString(e));
    });
}

}  // extern "C"
