/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the pseudo-stereo hot path.
 *
 * Two libraries export this exact symbol set so tests can swap them:
 *   oracle/_build/libp3s_oracle.so — p3s_oracle.c, a plain-C restatement of the
 *                                    reference algorithm (file:line cited per function);
 *   oracle/_ref/libp3s_ref.so      — the reference itself, compiled from
 *                                    /root/reference/proj/src/ (all .cpp) by oracle/Makefile,
 *                                    plus ref_shim.cpp (these same entry points over the
 *                                    reference's C++ stage API).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load either library. The product (paper_2009_09501_b200) never links it.
 *
 * All images are planar u8, row-major, no pitch (reference image.hpp:12-17).
 */
#ifndef P3S_ORACLE_H
#define P3S_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirror of p3s::ConversionConfig (reference config.hpp:25-43). */
typedef struct oracle_cfg {
    int base; /* -1 = auto: 2*floor(w/256+0.5) */
    int pop_threshold;
    double sigma_spatial;
    double sigma_range;
    int depth_block;
    int inpaint_block;
    double alpha;
    double beta;
    int mode; /* 0 forward z-buffer, 1 backward fallback */
    unsigned formats;
} oracle_cfg;

void oracle_default_cfg(oracle_cfg* cfg);
/* 0 when valid, else 1 and the reference's message copied into msg. */
int oracle_validate(const oracle_cfg* cfg, char* msg, size_t cap);
int oracle_effective_base(const oracle_cfg* cfg, int width);

void oracle_synthetic_frame(int w, int h, uint64_t seed, uint8_t* r, uint8_t* g, uint8_t* b);
void oracle_luma(const uint8_t* r, const uint8_t* g, const uint8_t* b, size_t n, uint8_t* y);
void oracle_sobel(const uint8_t* gray, int w, int h, uint8_t* out);
/* values: ceil(w/block) * ceil(h/block) doubles, row-major. */
void oracle_block_depth(const uint8_t* edges, int w, int h, const oracle_cfg* cfg, double* values);
void oracle_upsample(const double* values, int w, int h, int block, uint8_t* out);
void oracle_generate_depth(const uint8_t* r, const uint8_t* g, const uint8_t* b, int w, int h,
                           const oracle_cfg* cfg, uint8_t* depth);
void oracle_cross_bilateral_raw(const uint8_t* depth, const uint8_t* guide, int w, int h,
                                const oracle_cfg* cfg, int threads, double* out);
void oracle_cross_bilateral(const uint8_t* depth, const uint8_t* guide, int w, int h,
                            const oracle_cfg* cfg, int threads, uint8_t* out);
void oracle_shift_pair(int x, int depth, int base, int pop_threshold, double* left, double* right);
void oracle_reconstruct(const uint8_t* r, const uint8_t* g, const uint8_t* b,
                        const uint8_t* depth, int w, int h, const oracle_cfg* cfg, int threads,
                        uint8_t* lr, uint8_t* lg, uint8_t* lb, uint8_t* rr, uint8_t* rg,
                        uint8_t* rb, uint8_t* lmask, uint8_t* rmask);
/* stats[0]=passes, stats[1]=repaired, stats[2]=fallback_filled. */
void oracle_inpaint(const uint8_t* r, const uint8_t* g, const uint8_t* b, const uint8_t* mask,
                    int w, int h, const oracle_cfg* cfg, int threads, uint8_t* outr,
                    uint8_t* outg, uint8_t* outb, int64_t* stats);
void oracle_anaglyph(const uint8_t* lr, const uint8_t* lg, const uint8_t* lb, const uint8_t* rr,
                     const uint8_t* rg, const uint8_t* rb, int w, int h, uint8_t* outr,
                     uint8_t* outg, uint8_t* outb);
/* half: out is w x h (w even, else returns 1); full: out is 2w x h. */
int oracle_side_by_side(const uint8_t* lr, const uint8_t* lg, const uint8_t* lb,
                        const uint8_t* rr, const uint8_t* rg, const uint8_t* rb, int w, int h,
                        int half, uint8_t* outr, uint8_t* outg, uint8_t* outb);
/* Full convert_image (reference pipeline.cpp:29-78). Any output pointer may be NULL when
 * the format is not requested. Returns 0, or 1 with msg on a validation/format error.
 * timings: 7 int64 (depth, filter, dibr, inpaint L, inpaint R, format, pure) ns. */
int oracle_convert(const uint8_t* r, const uint8_t* g, const uint8_t* b, int w, int h,
                   const oracle_cfg* cfg, int threads, uint8_t* depth, uint8_t* filtered,
                   uint8_t* ana_r, uint8_t* ana_g, uint8_t* ana_b, uint8_t* hsbs_r,
                   uint8_t* hsbs_g, uint8_t* hsbs_b, uint8_t* fsbs_r, uint8_t* fsbs_g,
                   uint8_t* fsbs_b, int64_t* timings, char* msg, size_t cap);

/* Which implementation this library is: "port" or "reference". */
const char* oracle_kind(void);

#ifdef __cplusplus
}
#endif

#endif
