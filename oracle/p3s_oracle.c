/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference pseudo-stereo path.
 *
 * This is the checker, never the product: only tests/, __graft_entry__.smoke() and
 * bench.py's CPU-baseline legs load it. Every function cites the reference file:line
 * (under /root/reference/proj) whose behaviour it restates. Parity of this port with the
 * reference is pinned by tests/test_oracle.py against tests/golden/ (fixtures produced
 * by the compiled reference, tests/golden/make_golden.py) and, where oracle/_ref exists,
 * by direct differential runs.
 *
 * Build: gcc -std=c11 -O2 -ffp-contract=off (no FMA contraction: the reference's FP64
 * results depend on separately rounded multiplies and adds).
 */
#define _POSIX_C_SOURCE 200809L
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

const char* oracle_kind(void) { return "port"; }

/* config.hpp:25-43 defaults. */
void oracle_default_cfg(oracle_cfg* c) {
    c->base = -1;
    c->pop_threshold = 150;
    c->sigma_spatial = 8.0;
    c->sigma_range = 16.0;
    c->depth_block = 16;
    c->inpaint_block = 64;
    c->alpha = 0.7;
    c->beta = 0.3;
    c->mode = 0;
    c->formats = 1u;
}

static int set_msg(char* msg, size_t cap, const char* text) {
    if (msg && cap) {
        strncpy(msg, text, cap - 1);
        msg[cap - 1] = 0;
    }
    return 1;
}

/* config.cpp:8-25, same check order and messages. */
int oracle_validate(const oracle_cfg* c, char* msg, size_t cap) {
    if (c->base != -1) {
        if (c->base < 0) return set_msg(msg, cap, "base must be >= 0");
        if (c->base % 2 != 0) return set_msg(msg, cap, "base must be even");
    }
    if (c->pop_threshold < 0 || c->pop_threshold > 255)
        return set_msg(msg, cap, "pop_threshold must be in [0,255]");
    if (!(c->sigma_spatial > 0.0)) return set_msg(msg, cap, "sigma_spatial must be > 0");
    if (!(c->sigma_range > 0.0)) return set_msg(msg, cap, "sigma_range must be > 0");
    if (c->depth_block < 4) return set_msg(msg, cap, "depth_block must be >= 4");
    if (c->inpaint_block < 4) return set_msg(msg, cap, "inpaint_block must be >= 4");
    if (c->alpha < 0.0 || c->alpha > 1.0) return set_msg(msg, cap, "alpha must be in [0,1]");
    if (c->beta < 0.0 || c->beta > 1.0) return set_msg(msg, cap, "beta must be in [0,1]");
    if (c->alpha + c->beta > 1.0) return set_msg(msg, cap, "alpha + beta must be <= 1");
    if (c->formats == 0) return set_msg(msg, cap, "at least one output format is required");
    if ((c->formats & ~7u) != 0) return set_msg(msg, cap, "unknown output format bit");
    return 0;
}

/* config.cpp:27-31. */
int oracle_effective_base(const oracle_cfg* c, int width) {
    if (c->base != -1) return c->base;
    return 2 * (int)floor(width / 256.0 + 0.5);
}

/* ---- std::mt19937_64 (the C++ standard pins its parameters) ---- */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->idx = 312;
}

static uint64_t mt64_next(mt64* s) {
    if (s->idx >= 312) {
        const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (s->mt[i] & upper) | (s->mt[(i + 1) % 312] & lower);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
            s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
        }
        s->idx = 0;
    }
    uint64_t x = s->mt[s->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

/* bench.cpp:23-46: seed ^ (w<<32) ^ h, one draw per pixel in raster order. */
void oracle_synthetic_frame(int w, int h, uint64_t seed, uint8_t* r, uint8_t* g, uint8_t* b) {
    mt64 s;
    mt64_seed(&s, seed ^ ((uint64_t)w << 32) ^ (uint64_t)h);
    const int wd = w > 1 ? w - 1 : 1;
    const int hd = h > 1 ? h - 1 : 1;
    for (int y = 0; y < h; ++y) {
        for (int x = 0; x < w; ++x) {
            const uint64_t bits = mt64_next(&s);
            const size_t i = (size_t)y * w + x;
            const int gx = x * 255 / wd, gy = y * 255 / hd, gd = (x + y) * 255 / (wd + hd);
            r[i] = (uint8_t)((3 * gx + (int)(bits & 0xff)) / 4);
            g[i] = (uint8_t)((3 * gy + (int)((bits >> 8) & 0xff)) / 4);
            b[i] = (uint8_t)((3 * gd + (int)((bits >> 16) & 0xff)) / 4);
        }
    }
}

/* image.cpp:13-21. */
void oracle_luma(const uint8_t* r, const uint8_t* g, const uint8_t* b, size_t n, uint8_t* y) {
    for (size_t i = 0; i < n; ++i)
        y[i] = (uint8_t)((77u * r[i] + 150u * g[i] + 29u * b[i] + 128u) >> 8);
}

static inline int clampi(int v, int hi) { return v < 0 ? 0 : (v > hi ? hi : v); }

/* depth.cpp:21-41: clamp-to-edge 3x3 Sobel, (|gx|+|gy|)/4 truncated, capped at 255. */
void oracle_sobel(const uint8_t* p, int w, int h, uint8_t* out) {
    for (int y = 0; y < h; ++y) {
        const uint8_t* up = p + (size_t)clampi(y - 1, h - 1) * w;
        const uint8_t* mid = p + (size_t)y * w;
        const uint8_t* dn = p + (size_t)clampi(y + 1, h - 1) * w;
        for (int x = 0; x < w; ++x) {
            const int l = clampi(x - 1, w - 1), rr = clampi(x + 1, w - 1);
            const int gx = (up[rr] + 2 * mid[rr] + dn[rr]) - (up[l] + 2 * mid[l] + dn[l]);
            const int gy = (dn[l] + 2 * dn[x] + dn[rr]) - (up[l] + 2 * up[x] + up[rr]);
            const int m = (abs(gx) + abs(gy)) / 4;
            out[(size_t)y * w + x] = (uint8_t)(m < 255 ? m : 255);
        }
    }
}

/* depth.cpp:43-74: ramp from the block's centre row plus beta * mean edge. */
void oracle_block_depth(const uint8_t* e, int w, int h, const oracle_cfg* c, double* values) {
    const int blk = c->depth_block;
    const int bxn = (w + blk - 1) / blk, byn = (h + blk - 1) / blk;
    const double row_denom = h > 1 ? h - 1 : 1;
    for (int by = 0; by < byn; ++by) {
        const int y0 = by * blk, y1 = y0 + blk < h ? y0 + blk : h;
        const double centre = y0 + (y1 - 1 - y0) / 2.0;
        const double ramp = c->alpha * 255.0 * (centre / row_denom);
        for (int bx = 0; bx < bxn; ++bx) {
            const int x0 = bx * blk, x1 = x0 + blk < w ? x0 + blk : w;
            int64_t sum = 0;
            for (int y = y0; y < y1; ++y)
                for (int x = x0; x < x1; ++x) sum += e[(size_t)y * w + x];
            const double mean = (double)sum / ((y1 - y0) * (x1 - x0));
            values[(size_t)by * bxn + bx] = ramp + c->beta * mean;
        }
    }
}

static uint8_t round_half_up_u8(double v) {
    const double r = floor(v + 0.5);
    if (r <= 0.0) return 0;
    if (r >= 255.0) return 255;
    return (uint8_t)r;
}

/* depth.cpp:82-102: non-uniform centre list; v<=c0 -> (0,0), v>=last -> (last,0), else
 * the smallest i with v <= c[i+1] and frac (v-c[i])/(c[i+1]-c[i]). */
static void locate(const double* c, int n, double v, int* i, double* frac) {
    if (v <= c[0]) { *i = 0; *frac = 0.0; return; }
    if (v >= c[n - 1]) { *i = n - 1; *frac = 0.0; return; }
    int k = 0;
    while (v > c[k + 1]) ++k;
    *i = k;
    *frac = (v - c[k]) / (c[k + 1] - c[k]);
}

static double* centres(int count, int blocks, int blk) {
    double* c = (double*)malloc(sizeof(double) * (size_t)blocks);
    for (int i = 0; i < blocks; ++i) {
        const int lo = i * blk, hi = lo + blk < count ? lo + blk : count;
        c[i] = lo + (hi - 1 - lo) / 2.0;
    }
    return c;
}

/* depth.cpp:76-121: bilinear over block centres, round half up. */
void oracle_upsample(const double* g, int w, int h, int blk, uint8_t* out) {
    const int bxn = (w + blk - 1) / blk, byn = (h + blk - 1) / blk;
    double* cx = centres(w, bxn, blk);
    double* cy = centres(h, byn, blk);
    int* ixs = (int*)malloc(sizeof(int) * (size_t)w);
    double* fxs = (double*)malloc(sizeof(double) * (size_t)w);
    for (int x = 0; x < w; ++x) locate(cx, bxn, x, &ixs[x], &fxs[x]);
    for (int y = 0; y < h; ++y) {
        int iy;
        double fy;
        locate(cy, byn, y, &iy, &fy);
        const int iy1 = iy + 1 < byn - 1 ? iy + 1 : byn - 1;
        for (int x = 0; x < w; ++x) {
            const int ix = ixs[x], ix1 = ix + 1 < bxn - 1 ? ix + 1 : bxn - 1;
            const double fx = fxs[x];
            const double top = g[(size_t)iy * bxn + ix] * (1.0 - fx) + g[(size_t)iy * bxn + ix1] * fx;
            const double bot =
                g[(size_t)iy1 * bxn + ix] * (1.0 - fx) + g[(size_t)iy1 * bxn + ix1] * fx;
            out[(size_t)y * w + x] = round_half_up_u8(top * (1.0 - fy) + bot * fy);
        }
    }
    free(cx); free(cy); free(ixs); free(fxs);
}

/* depth.cpp:123-129 (luma -> sobel -> blocks -> upsample). */
void oracle_generate_depth(const uint8_t* r, const uint8_t* g, const uint8_t* b, int w, int h,
                           const oracle_cfg* c, uint8_t* depth) {
    const size_t n = (size_t)w * h;
    uint8_t* y = (uint8_t*)malloc(n);
    uint8_t* e = (uint8_t*)malloc(n);
    const int blk = c->depth_block;
    double* vals = (double*)malloc(sizeof(double) * (size_t)((w + blk - 1) / blk) *
                                   (size_t)((h + blk - 1) / blk));
    oracle_luma(r, g, b, n, y);
    oracle_sobel(y, w, h, e);
    oracle_block_depth(e, w, h, c, vals);
    oracle_upsample(vals, w, h, blk, depth);
    free(y); free(e); free(vals);
}

/* ---- cross-bilateral (bilateral.cpp) ---- */
typedef struct {
    int radius;
    double* spatial; /* (2r+1)^2 */
    double range[256];
} bkernel;

/* bilateral.cpp:22-35: libm exp on the integer-then-double exponent. */
static void build_kernel(const oracle_cfg* c, bkernel* k) {
    k->radius = (int)ceil(2.0 * c->sigma_spatial);
    const int r = k->radius, side = 2 * r + 1;
    k->spatial = (double*)malloc(sizeof(double) * (size_t)side * side);
    const double inv_s = 1.0 / (2.0 * c->sigma_spatial * c->sigma_spatial);
    for (int dy = -r; dy <= r; ++dy)
        for (int dx = -r; dx <= r; ++dx)
            k->spatial[(size_t)(dy + r) * side + (dx + r)] = exp(-(dx * dx + dy * dy) * inv_s);
    const double inv_r = 1.0 / (2.0 * c->sigma_range * c->sigma_range);
    for (int d = 0; d < 256; ++d) k->range[d] = exp(-(d * d) * inv_r);
}

/* bilateral.cpp:40-85: rows dy ascending over the clipped window; per row the centre tap,
 * then dx = 1..r as a mirrored pair (ws += wl+wr; vs += wl*dL + wr*dR) or one side. */
static double filter_pixel(const uint8_t* depth, const uint8_t* guide, int w, int h,
                           const bkernel* k, int x, int y) {
    const int r = k->radius, side = 2 * r + 1;
    const int gp = guide[(size_t)y * w + x];
    double ws = 0.0, vs = 0.0;
    const int dy0 = y - r < 0 ? -y : -r;
    const int dy1 = y + r >= h ? h - 1 - y : r;
    for (int dy = dy0; dy <= dy1; ++dy) {
        const size_t row = (size_t)(y + dy) * w;
        const double* s = k->spatial + (size_t)(dy + r) * side + r;
        {
            const double wc = s[0] * k->range[abs(gp - guide[row + x])];
            ws += wc;
            vs += wc * depth[row + x];
        }
        for (int dx = 1; dx <= r; ++dx) {
            const int lin = x - dx >= 0, rin = x + dx < w;
            if (lin && rin) {
                const double wl = s[dx] * k->range[abs(gp - guide[row + x - dx])];
                const double wr = s[dx] * k->range[abs(gp - guide[row + x + dx])];
                ws += wl + wr;
                vs += wl * depth[row + x - dx] + wr * depth[row + x + dx];
            } else if (lin) {
                const double wl = s[dx] * k->range[abs(gp - guide[row + x - dx])];
                ws += wl;
                vs += wl * depth[row + x - dx];
            } else if (rin) {
                const double wr = s[dx] * k->range[abs(gp - guide[row + x + dx])];
                ws += wr;
                vs += wr * depth[row + x + dx];
            }
        }
    }
    return vs / ws;
}

typedef struct {
    const uint8_t* depth;
    const uint8_t* guide;
    int w, h, y0, y1;
    const bkernel* k;
    double* raw;
    uint8_t* out;
} bil_job;

static void* bil_worker(void* arg) {
    bil_job* j = (bil_job*)arg;
    for (int y = j->y0; y < j->y1; ++y)
        for (int x = 0; x < j->w; ++x) {
            const double v = filter_pixel(j->depth, j->guide, j->w, j->h, j->k, x, y);
            if (j->raw) j->raw[(size_t)y * j->w + x] = v;
            if (j->out) j->out[(size_t)y * j->w + x] = round_half_up_u8(v);
        }
    return NULL;
}

/* Row ranges split like executor.cpp:62-83 (bytes are thread-count invariant anyway). */
static void bilateral_run(const uint8_t* depth, const uint8_t* guide, int w, int h,
                          const oracle_cfg* c, int threads, double* raw, uint8_t* out) {
    bkernel k;
    build_kernel(c, &k);
    if (threads < 1) threads = 1;
    if (threads > h) threads = h;
    pthread_t* tids = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    bil_job* jobs = (bil_job*)malloc(sizeof(bil_job) * (size_t)threads);
    for (int t = 0; t < threads; ++t) {
        jobs[t] = (bil_job){depth, guide, w, h, (int)((int64_t)h * t / threads),
                            (int)((int64_t)h * (t + 1) / threads), &k, raw, out};
        if (t > 0) pthread_create(&tids[t], NULL, bil_worker, &jobs[t]);
    }
    bil_worker(&jobs[0]);
    for (int t = 1; t < threads; ++t) pthread_join(tids[t], NULL);
    free(tids); free(jobs); free(k.spatial);
}

void oracle_cross_bilateral_raw(const uint8_t* depth, const uint8_t* guide, int w, int h,
                                const oracle_cfg* c, int threads, double* out) {
    bilateral_run(depth, guide, w, h, c, threads, out, NULL);
}

void oracle_cross_bilateral(const uint8_t* depth, const uint8_t* guide, int w, int h,
                            const oracle_cfg* c, int threads, uint8_t* out) {
    bilateral_run(depth, guide, w, h, c, threads, NULL, out);
}

/* ---- DIBR (dibr.cpp) ---- */

/* dibr.cpp:33-41. */
void oracle_shift_pair(int x, int d, int base, int T, double* left, double* right) {
    const double hb = base / 2.0;
    if (d > T) {
        const double s = hb * (d / 255.0);
        *left = x - s;
        *right = x + s;
    } else {
        const double s = hb * (1.0 - d / 255.0);
        *left = x + s;
        *right = x - s;
    }
}

/* dibr.cpp:43-104 (backward gather with fallback; forward per-row z-buffer, strict > in
 * ascending x keeps the smaller source column on depth ties; destination for the left
 * eye is trunc(right sample), for the right eye trunc(left sample); trunc toward 0). */
void oracle_reconstruct(const uint8_t* r, const uint8_t* g, const uint8_t* b,
                        const uint8_t* depth, int w, int h, const oracle_cfg* c, int threads,
                        uint8_t* lr, uint8_t* lg, uint8_t* lb, uint8_t* rr, uint8_t* rg,
                        uint8_t* rb, uint8_t* lmask, uint8_t* rmask) {
    (void)threads;
    const int base = oracle_effective_base(c, w);
    const size_t n = (size_t)w * h;
    if (c->mode == 1) {
        memset(lmask, 0, n);
        memset(rmask, 0, n);
        for (int y = 0; y < h; ++y) {
            const size_t row = (size_t)y * w;
            for (int x = 0; x < w; ++x) {
                double pl, pr;
                oracle_shift_pair(x, depth[row + x], base, c->pop_threshold, &pl, &pr);
                const int xl = (int)pl, xr = (int)pr;
                const size_t sl = row + (xl >= 0 && xl < w ? xl : x);
                const size_t sr = row + (xr >= 0 && xr < w ? xr : x);
                lr[row + x] = r[sl]; lg[row + x] = g[sl]; lb[row + x] = b[sl];
                rr[row + x] = r[sr]; rg[row + x] = g[sr]; rb[row + x] = b[sr];
            }
        }
        return;
    }
    memset(lr, 0, n); memset(lg, 0, n); memset(lb, 0, n);
    memset(rr, 0, n); memset(rg, 0, n); memset(rb, 0, n);
    memset(lmask, 1, n);
    memset(rmask, 1, n);
    int* bl = (int*)malloc(sizeof(int) * (size_t)w);
    int* br = (int*)malloc(sizeof(int) * (size_t)w);
    for (int y = 0; y < h; ++y) {
        const size_t row = (size_t)y * w;
        for (int x = 0; x < w; ++x) bl[x] = br[x] = -1;
        for (int x = 0; x < w; ++x) {
            const int d = depth[row + x];
            double pl, pr;
            oracle_shift_pair(x, d, base, c->pop_threshold, &pl, &pr);
            const int dl = (int)pr, dr = (int)pl;
            if (dl >= 0 && dl < w && d > bl[dl]) {
                bl[dl] = d;
                lr[row + dl] = r[row + x]; lg[row + dl] = g[row + x]; lb[row + dl] = b[row + x];
                lmask[row + dl] = 0;
            }
            if (dr >= 0 && dr < w && d > br[dr]) {
                br[dr] = d;
                rr[row + dr] = r[row + x]; rg[row + dr] = g[row + x]; rb[row + dr] = b[row + x];
                rmask[row + dr] = 0;
            }
        }
    }
    free(bl); free(br);
}

/* ---- inpaint (inpaint.cpp:29-130) ----
 * Jacobi passes against the pass-start snapshot: a damaged pixel with >= 2 intact
 * 8-neighbours takes the per-channel (2*sum+count)/(2*count) mean; a pass that repairs
 * nothing while damage remains fills the rest with 128. Tiles in the reference only
 * schedule work, so a raster-order list is equivalent. */
void oracle_inpaint(const uint8_t* r, const uint8_t* g, const uint8_t* b, const uint8_t* mask,
                    int w, int h, const oracle_cfg* c, int threads, uint8_t* outr,
                    uint8_t* outg, uint8_t* outb, int64_t* stats) {
    (void)c; (void)threads;
    const size_t n = (size_t)w * h;
    memcpy(outr, r, n); memcpy(outg, g, n); memcpy(outb, b, n);
    stats[0] = stats[1] = stats[2] = 0;
    size_t cnt = 0;
    for (size_t i = 0; i < n; ++i) cnt += mask[i] != 0;
    if (cnt == 0) return;
    uint8_t* dmg = (uint8_t*)malloc(n);
    for (size_t i = 0; i < n; ++i) dmg[i] = mask[i] != 0;
    /* two damaged-pixel lists, swapped each pass (current / still damaged) */
    size_t* bufs[2] = {(size_t*)malloc(sizeof(size_t) * cnt), (size_t*)malloc(sizeof(size_t) * cnt)};
    int cur = 0;
    size_t* list = bufs[0];
    uint8_t* rep = (uint8_t*)malloc(4 * cnt);
    size_t m = 0;
    for (size_t i = 0; i < n; ++i)
        if (dmg[i]) list[m++] = i;
    size_t remaining = m;
    while (remaining > 0) {
        size_t nrep = 0, nkeep = 0;
        size_t* keep = bufs[cur ^ 1];
        for (size_t k = 0; k < remaining; ++k) {
            const size_t idx = list[k];
            const int x = (int)(idx % (size_t)w), y = (int)(idx / (size_t)w);
            unsigned count = 0, sr = 0, sg = 0, sb = 0;
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    if (!dx && !dy) continue;
                    const int nx = x + dx, ny = y + dy;
                    if (nx < 0 || nx >= w || ny < 0 || ny >= h) continue;
                    const size_t ni = (size_t)ny * w + nx;
                    if (dmg[ni]) continue;
                    ++count; sr += outr[ni]; sg += outg[ni]; sb += outb[ni];
                }
            if (count >= 2) {
                rep[4 * k] = 1;
                rep[4 * k + 1] = (uint8_t)((2 * sr + count) / (2 * count));
                rep[4 * k + 2] = (uint8_t)((2 * sg + count) / (2 * count));
                rep[4 * k + 3] = (uint8_t)((2 * sb + count) / (2 * count));
                ++nrep;
            } else {
                rep[4 * k] = 0;
            }
        }
        for (size_t k = 0; k < remaining; ++k) {
            const size_t idx = list[k];
            if (rep[4 * k]) {
                outr[idx] = rep[4 * k + 1]; outg[idx] = rep[4 * k + 2]; outb[idx] = rep[4 * k + 3];
                dmg[idx] = 0;
            } else {
                keep[nkeep++] = idx;
            }
        }
        stats[0] += 1;
        stats[1] += (int64_t)nrep;
        cur ^= 1;
        list = bufs[cur];
        remaining = nkeep;
        if (nrep == 0 && remaining > 0) {
            for (size_t k = 0; k < remaining; ++k) {
                outr[list[k]] = outg[list[k]] = outb[list[k]] = 128;
                dmg[list[k]] = 0;
            }
            stats[2] += (int64_t)remaining;
            remaining = 0;
        }
    }
    free(dmg); free(bufs[0]); free(bufs[1]); free(rep);
}

/* stereo_format.cpp:8-21. */
void oracle_anaglyph(const uint8_t* lr, const uint8_t* lg, const uint8_t* lb, const uint8_t* rr,
                     const uint8_t* rg, const uint8_t* rb, int w, int h, uint8_t* outr,
                     uint8_t* outg, uint8_t* outb) {
    (void)lg; (void)lb; (void)rr;
    const size_t n = (size_t)w * h;
    memcpy(outr, lr, n); memcpy(outg, rg, n); memcpy(outb, rb, n);
}

/* stereo_format.cpp:23-73: FSBS concat (2w x h) or HSBS (a+b+1)/2 column-pair squeeze. */
int oracle_side_by_side(const uint8_t* lr, const uint8_t* lg, const uint8_t* lb,
                        const uint8_t* rr, const uint8_t* rg, const uint8_t* rb, int w, int h,
                        int half, uint8_t* outr, uint8_t* outg, uint8_t* outb) {
    const uint8_t* L[3] = {lr, lg, lb};
    const uint8_t* R[3] = {rr, rg, rb};
    uint8_t* O[3] = {outr, outg, outb};
    if (!half) {
        for (int ch = 0; ch < 3; ++ch)
            for (int y = 0; y < h; ++y) {
                memcpy(O[ch] + (size_t)y * 2 * w, L[ch] + (size_t)y * w, (size_t)w);
                memcpy(O[ch] + (size_t)y * 2 * w + w, R[ch] + (size_t)y * w, (size_t)w);
            }
        return 0;
    }
    if (w % 2 != 0) return 1;
    const int hw = w / 2;
    for (int ch = 0; ch < 3; ++ch)
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < hw; ++x) {
                const size_t s = (size_t)y * w + 2 * x;
                O[ch][(size_t)y * w + x] = (uint8_t)((L[ch][s] + L[ch][s + 1] + 1u) / 2u);
                O[ch][(size_t)y * w + hw + x] = (uint8_t)((R[ch][s] + R[ch][s + 1] + 1u) / 2u);
            }
    return 0;
}

static int64_t now_ns(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (int64_t)ts.tv_sec * 1000000000LL + ts.tv_nsec;
}

/* pipeline.cpp:29-78: fixed stage order; inpaint skipped when a mask is clean. */
int oracle_convert(const uint8_t* r, const uint8_t* g, const uint8_t* b, int w, int h,
                   const oracle_cfg* c, int threads, uint8_t* depth, uint8_t* filtered,
                   uint8_t* ana_r, uint8_t* ana_g, uint8_t* ana_b, uint8_t* hsbs_r,
                   uint8_t* hsbs_g, uint8_t* hsbs_b, uint8_t* fsbs_r, uint8_t* fsbs_g,
                   uint8_t* fsbs_b, int64_t* t, char* msg, size_t cap) {
    if (oracle_validate(c, msg, cap)) return 1;
    const size_t n = (size_t)w * h;
    for (int i = 0; i < 7; ++i) t[i] = 0;
    uint8_t* guide = (uint8_t*)malloc(n);
    uint8_t* e = (uint8_t*)malloc(n);
    uint8_t* buf = (uint8_t*)malloc(n * 14);
    uint8_t *lr = buf, *lg = buf + n, *lb = buf + 2 * n, *rr = buf + 3 * n, *rg = buf + 4 * n,
            *rb = buf + 5 * n, *lm = buf + 6 * n, *rm = buf + 7 * n, *pl = buf + 8 * n;
    uint8_t* pr = buf + 11 * n;
    const int blk = c->depth_block;
    double* vals = (double*)malloc(sizeof(double) * (size_t)((w + blk - 1) / blk) *
                                   (size_t)((h + blk - 1) / blk));
    int64_t t0 = now_ns();
    oracle_luma(r, g, b, n, guide);
    oracle_sobel(guide, w, h, e);
    oracle_block_depth(e, w, h, c, vals);
    oracle_upsample(vals, w, h, blk, depth);
    t[0] = now_ns() - t0;
    t0 = now_ns();
    oracle_cross_bilateral(depth, guide, w, h, c, threads, filtered);
    t[1] = now_ns() - t0;
    t0 = now_ns();
    oracle_reconstruct(r, g, b, filtered, w, h, c, threads, lr, lg, lb, rr, rg, rb, lm, rm);
    t[2] = now_ns() - t0;
    int64_t st[3];
    int any = 0;
    for (size_t i = 0; i < n && !any; ++i) any = lm[i];
    if (any) {
        t0 = now_ns();
        oracle_inpaint(lr, lg, lb, lm, w, h, c, threads, pl, pl + n, pl + 2 * n, st);
        memcpy(lr, pl, 3 * n);
        t[3] = now_ns() - t0;
    }
    any = 0;
    for (size_t i = 0; i < n && !any; ++i) any = rm[i];
    if (any) {
        t0 = now_ns();
        oracle_inpaint(rr, rg, rb, rm, w, h, c, threads, pr, pr + n, pr + 2 * n, st);
        memcpy(rr, pr, 3 * n);
        t[4] = now_ns() - t0;
    }
    int rc = 0;
    t0 = now_ns();
    if (c->formats & 1u) oracle_anaglyph(lr, lg, lb, rr, rg, rb, w, h, ana_r, ana_g, ana_b);
    if (c->formats & 2u) {
        if (oracle_side_by_side(lr, lg, lb, rr, rg, rb, w, h, 1, hsbs_r, hsbs_g, hsbs_b)) {
            set_msg(msg, cap, "side_by_side: half mode requires an even width");
            rc = 1;
        }
    }
    if (!rc && (c->formats & 4u))
        oracle_side_by_side(lr, lg, lb, rr, rg, rb, w, h, 0, fsbs_r, fsbs_g, fsbs_b);
    t[5] = now_ns() - t0;
    t[6] = t[1] + t[2] + t[3] + t[4] + t[5];
    free(guide); free(e); free(buf); free(vals);
    return rc;
}
