// TEST INFRASTRUCTURE ONLY — exposes the compiled reference's C++ stage API under the
// oracle.h entry points, so tests can diff every intermediate of the CUDA path against
// the reference itself. Linked only with the reference's own sources
// (/root/reference/proj/src/*.cpp, built by oracle/Makefile into oracle/_ref/); no
// reference source is copied into this repository.
#include <chrono>
#include <cstring>
#include <stdexcept>
#include <string>

#include "oracle.h"
#include "pseudo3d/bench.hpp"
#include "pseudo3d/bilateral.hpp"
#include "pseudo3d/config.hpp"
#include "pseudo3d/depth.hpp"
#include "pseudo3d/dibr.hpp"
#include "pseudo3d/executor.hpp"
#include "pseudo3d/image.hpp"
#include "pseudo3d/inpaint.hpp"
#include "pseudo3d/pipeline.hpp"
#include "pseudo3d/stereo_format.hpp"

namespace {

p3s::ConversionConfig to_ref(const oracle_cfg* c) {
    p3s::ConversionConfig r;
    r.base = c->base;
    r.pop_threshold = c->pop_threshold;
    r.sigma_spatial = c->sigma_spatial;
    r.sigma_range = c->sigma_range;
    r.depth_block = c->depth_block;
    r.inpaint_block = c->inpaint_block;
    r.alpha = c->alpha;
    r.beta = c->beta;
    r.dibr_mode = c->mode == 1 ? p3s::DibrMode::kBackwardFallback : p3s::DibrMode::kForwardZBuffer;
    r.formats = c->formats;
    return r;
}

p3s::ImageRGB8 image_in(const uint8_t* r, const uint8_t* g, const uint8_t* b, int w, int h) {
    p3s::ImageRGB8 img(w, h);
    const size_t n = img.size();
    std::memcpy(img.r.data(), r, n);
    std::memcpy(img.g.data(), g, n);
    std::memcpy(img.b.data(), b, n);
    return img;
}

void image_out(const p3s::ImageRGB8& img, uint8_t* r, uint8_t* g, uint8_t* b) {
    const size_t n = img.size();
    std::memcpy(r, img.r.data(), n);
    std::memcpy(g, img.g.data(), n);
    std::memcpy(b, img.b.data(), n);
}

p3s::GrayMap gray_in(const uint8_t* p, int w, int h) {
    p3s::GrayMap m(w, h);
    std::memcpy(m.data.data(), p, m.size());
    return m;
}

int fail(char* msg, size_t cap, const char* what) {
    if (msg && cap) {
        std::strncpy(msg, what, cap - 1);
        msg[cap - 1] = 0;
    }
    return 1;
}

}  // namespace

extern "C" {

const char* oracle_kind(void) { return "reference"; }

void oracle_default_cfg(oracle_cfg* c) {
    p3s::ConversionConfig d;
    c->base = d.base;
    c->pop_threshold = d.pop_threshold;
    c->sigma_spatial = d.sigma_spatial;
    c->sigma_range = d.sigma_range;
    c->depth_block = d.depth_block;
    c->inpaint_block = d.inpaint_block;
    c->alpha = d.alpha;
    c->beta = d.beta;
    c->mode = d.dibr_mode == p3s::DibrMode::kBackwardFallback ? 1 : 0;
    c->formats = d.formats;
}

int oracle_validate(const oracle_cfg* c, char* msg, size_t cap) {
    try {
        to_ref(c).validate();
        return 0;
    } catch (const std::exception& e) {
        return fail(msg, cap, e.what());
    }
}

int oracle_effective_base(const oracle_cfg* c, int width) { return to_ref(c).effective_base(width); }

void oracle_synthetic_frame(int w, int h, uint64_t seed, uint8_t* r, uint8_t* g, uint8_t* b) {
    image_out(p3s::synthetic_frame(w, h, seed), r, g, b);
}

void oracle_luma(const uint8_t* r, const uint8_t* g, const uint8_t* b, size_t n, uint8_t* y) {
    const p3s::GrayMap m = p3s::luma(image_in(r, g, b, static_cast<int>(n), 1));
    std::memcpy(y, m.data.data(), n);
}

void oracle_sobel(const uint8_t* gray, int w, int h, uint8_t* out) {
    const p3s::GrayMap m = p3s::sobel_magnitude(gray_in(gray, w, h));
    std::memcpy(out, m.data.data(), m.size());
}

void oracle_block_depth(const uint8_t* edges, int w, int h, const oracle_cfg* c, double* values) {
    const p3s::BlockGrid g = p3s::block_depth(gray_in(edges, w, h), to_ref(c));
    std::memcpy(values, g.values.data(), g.values.size() * sizeof(double));
}

void oracle_upsample(const double* values, int w, int h, int block, uint8_t* out) {
    p3s::BlockGrid g;
    g.block = block;
    g.width = w;
    g.height = h;
    g.blocks_x = (w + block - 1) / block;
    g.blocks_y = (h + block - 1) / block;
    g.values.assign(values, values + static_cast<size_t>(g.blocks_x) * g.blocks_y);
    const p3s::GrayMap m = p3s::upsample_block_grid(g);
    std::memcpy(out, m.data.data(), m.size());
}

void oracle_generate_depth(const uint8_t* r, const uint8_t* g, const uint8_t* b, int w, int h,
                           const oracle_cfg* c, uint8_t* depth) {
    const p3s::GrayMap m = p3s::generate_depth(image_in(r, g, b, w, h), to_ref(c));
    std::memcpy(depth, m.data.data(), m.size());
}

void oracle_cross_bilateral_raw(const uint8_t* depth, const uint8_t* guide, int w, int h,
                                const oracle_cfg* c, int threads, double* out) {
    p3s::Executor ex(threads);
    const std::vector<double> v =
        p3s::cross_bilateral_raw(gray_in(depth, w, h), gray_in(guide, w, h), to_ref(c), ex);
    std::memcpy(out, v.data(), v.size() * sizeof(double));
}

void oracle_cross_bilateral(const uint8_t* depth, const uint8_t* guide, int w, int h,
                            const oracle_cfg* c, int threads, uint8_t* out) {
    p3s::Executor ex(threads);
    const p3s::GrayMap m =
        p3s::cross_bilateral(gray_in(depth, w, h), gray_in(guide, w, h), to_ref(c), ex);
    std::memcpy(out, m.data.data(), m.size());
}

void oracle_shift_pair(int x, int depth, int base, int pop_threshold, double* left,
                       double* right) {
    const p3s::ShiftPair p =
        p3s::shift_pair(x, static_cast<std::uint8_t>(depth), base, pop_threshold);
    *left = p.left;
    *right = p.right;
}

void oracle_reconstruct(const uint8_t* r, const uint8_t* g, const uint8_t* b,
                        const uint8_t* depth, int w, int h, const oracle_cfg* c, int threads,
                        uint8_t* lr, uint8_t* lg, uint8_t* lb, uint8_t* rr, uint8_t* rg,
                        uint8_t* rb, uint8_t* lmask, uint8_t* rmask) {
    p3s::Executor ex(threads);
    const p3s::StereoFrames f =
        p3s::reconstruct(image_in(r, g, b, w, h), gray_in(depth, w, h), to_ref(c), ex);
    image_out(f.left, lr, lg, lb);
    image_out(f.right, rr, rg, rb);
    std::memcpy(lmask, f.left_mask.damaged.data(), f.left_mask.size());
    std::memcpy(rmask, f.right_mask.damaged.data(), f.right_mask.size());
}

void oracle_inpaint(const uint8_t* r, const uint8_t* g, const uint8_t* b, const uint8_t* mask,
                    int w, int h, const oracle_cfg* c, int threads, uint8_t* outr,
                    uint8_t* outg, uint8_t* outb, int64_t* stats) {
    p3s::Executor ex(threads);
    p3s::DamageMask m(w, h);
    std::memcpy(m.damaged.data(), mask, m.size());
    p3s::InpaintStats st;
    const p3s::ImageRGB8 out = p3s::inpaint(image_in(r, g, b, w, h), m, to_ref(c), ex, &st);
    image_out(out, outr, outg, outb);
    stats[0] = st.passes;
    stats[1] = static_cast<int64_t>(st.repaired);
    stats[2] = static_cast<int64_t>(st.fallback_filled);
}

void oracle_anaglyph(const uint8_t* lr, const uint8_t* lg, const uint8_t* lb, const uint8_t* rr,
                     const uint8_t* rg, const uint8_t* rb, int w, int h, uint8_t* outr,
                     uint8_t* outg, uint8_t* outb) {
    p3s::Executor ex(1);
    image_out(p3s::anaglyph(image_in(lr, lg, lb, w, h), image_in(rr, rg, rb, w, h), ex), outr,
              outg, outb);
}

int oracle_side_by_side(const uint8_t* lr, const uint8_t* lg, const uint8_t* lb,
                        const uint8_t* rr, const uint8_t* rg, const uint8_t* rb, int w, int h,
                        int half, uint8_t* outr, uint8_t* outg, uint8_t* outb) {
    p3s::Executor ex(1);
    try {
        image_out(p3s::side_by_side(image_in(lr, lg, lb, w, h), image_in(rr, rg, rb, w, h),
                                    half != 0, ex),
                  outr, outg, outb);
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    }
}

int oracle_convert(const uint8_t* r, const uint8_t* g, const uint8_t* b, int w, int h,
                   const oracle_cfg* c, int threads, uint8_t* depth, uint8_t* filtered,
                   uint8_t* ana_r, uint8_t* ana_g, uint8_t* ana_b, uint8_t* hsbs_r,
                   uint8_t* hsbs_g, uint8_t* hsbs_b, uint8_t* fsbs_r, uint8_t* fsbs_g,
                   uint8_t* fsbs_b, int64_t* t, char* msg, size_t cap) {
    try {
        p3s::Executor ex(threads);
        const p3s::ConversionResult res =
            p3s::convert_image(image_in(r, g, b, w, h), to_ref(c), ex);
        std::memcpy(depth, res.depth.data.data(), res.depth.size());
        std::memcpy(filtered, res.filtered_depth.data.data(), res.filtered_depth.size());
        for (const auto& [fmt, img] : res.outputs) {
            if (fmt == p3s::kFormatAnaglyph) image_out(img, ana_r, ana_g, ana_b);
            if (fmt == p3s::kFormatHsbs) image_out(img, hsbs_r, hsbs_g, hsbs_b);
            if (fmt == p3s::kFormatFsbs) image_out(img, fsbs_r, fsbs_g, fsbs_b);
        }
        const p3s::StageTimings& s = res.timings;
        t[0] = s.depth_gen_ns;
        t[1] = s.filter_ns;
        t[2] = s.dibr_ns;
        t[3] = s.inpaint_left_ns;
        t[4] = s.inpaint_right_ns;
        t[5] = s.format_ns;
        t[6] = s.pure_ns();
        return 0;
    } catch (const std::exception& e) {
        return fail(msg, cap, e.what());
    }
}

}  // extern "C"
