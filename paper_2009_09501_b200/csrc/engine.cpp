// Host orchestrator of the B200 pseudo-stereo pipeline: per-thread device contexts, plans
// (host-computed exact tables + one device arena per (size, config)), the stage API of
// include/p3s/pipeline.hpp and the full convert_image (reference pipeline.cpp:29-78),
// whose synchronous frames run as a row-banded schedule that overlaps the PCIe copies with
// the filter (band_plan, Pipeline::Impl::upload_run_conv; DESIGN.md "Banded synchronous
// convert").
//
// Built with -ffp-contract=off: the tables below must reproduce the reference's double
// expressions bit for bit (SURVEY.md §7 rules 1, 2, 4, 5).
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <deque>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <list>
#include <map>
#include <mutex>
#include <sstream>
#include <string>

#include "p3s/pipeline.hpp"
#include "p3s_cu.h"
#include "p3s_nvtx.hpp"

namespace p3s {

namespace {

void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw DeviceError(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
    }
}
#define CK(expr) check((expr), #expr)

int round_up(int v, int m) { return (v + m - 1) / m * m; }

// Stage events: inside a stream capture they must become event-record nodes of the graph
// (cudaEventRecordExternal); outside a capture that flag is invalid.
void record_event(cudaEvent_t e, cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    check(cudaStreamIsCapturing(st, &cs), "cudaStreamIsCapturing");
    if (cs == cudaStreamCaptureStatusActive)
        check(cudaEventRecordWithFlags(e, st, cudaEventRecordExternal), "cudaEventRecordWithFlags");
    else
        check(cudaEventRecord(e, st), "cudaEventRecord");
}

// Waits for an event recorded outside the stream's capture (an external event-wait node
// while capturing, a plain wait otherwise).
void wait_event_any(cudaStream_t st, cudaEvent_t e) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    check(cudaStreamIsCapturing(st, &cs), "cudaStreamIsCapturing");
    check(cudaStreamWaitEvent(st, e, cs == cudaStreamCaptureStatusActive ? cudaEventWaitExternal : 0),
          "cudaStreamWaitEvent");
}

int sm_count_cached() {
    static thread_local int n = [] {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return n;
}

// cu::ZeroRanges from {pointer, 4-byte words} pairs
cu::ZeroRanges zr(std::initializer_list<std::pair<void*, unsigned>> ranges) {
    cu::ZeroRanges z{};
    for (const auto& r : ranges) {
        if (z.n == cu::kZeroRanges) throw std::logic_error("too many zero ranges");
        z.p[z.n] = r.first;
        z.words[z.n] = r.second;
        ++z.n;
    }
    return z;
}

bool host_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// ---- exact host tables --------------------------------------------------------------------

// bilateral.cpp:22-35: radius ceil(2 sigma_s); spatial exp(-(dx^2+dy^2) * inv_s) with the
// integer sum formed first; range exp(-(d^2) * inv_r). Only dx >= 0 is stored (the table is
// symmetric in dx and the kernels index |dx|).
int bilateral_radius(const ConversionConfig& c) {
    return static_cast<int>(std::ceil(2.0 * c.sigma_spatial));
}

std::vector<double> spatial_table(const ConversionConfig& c, int r) {
    const double inv_s = 1.0 / (2.0 * c.sigma_spatial * c.sigma_spatial);
    std::vector<double> s(static_cast<std::size_t>(2 * r + 1) * (r + 1));
    for (int dy = -r; dy <= r; ++dy)
        for (int dx = 0; dx <= r; ++dx)
            s[static_cast<std::size_t>(dy + r) * (r + 1) + dx] = std::exp(-(dx * dx + dy * dy) * inv_s);
    return s;
}

void range_table(const ConversionConfig& c, double* out) {
    const double inv_r = 1.0 / (2.0 * c.sigma_range * c.sigma_range);
    for (int d = 0; d < 256; ++d) out[d] = std::exp(-(d * d) * inv_r);
}

// dibr.cpp:33-41 as a signed per-depth shift: sigma = +hb*(d/255) when d > T, else
// -(hb*(1 - d/255)); then p.left = x - sigma and p.right = x + sigma are exactly the
// reference's x - s / x + s and x + s' / x - s' (negation is exact in IEEE).
void shift_table(int base, int T, double* out) {
    const double hb = base / 2.0;
    for (int d = 0; d < 256; ++d) {
        if (d > T)
            out[d] = hb * (d / 255.0);
        else
            out[d] = -(hb * (1.0 - d / 255.0));
    }
}

// Integer form of the reference's destination columns (dibr.cpp:33-41, dibr.hpp:35):
// for each depth d and direction (P: x + sigma, M: x - sigma) the truncated column
// trunc(fl(x +- sigma)) over x in [0, w) is x + off + (x >= X), except 0 at x == z (where
// fl(x +- sigma) lies in (-1, 0)), valid iff in [0, w). (off, X, z) are derived from the
// exact double evaluation of EVERY x and the representation is verified against it; if
// any (d, direction) does not fit (or w >= 32768), the function returns false and the plan
// keeps the FP64 device path. Packed as {off & 0xFFFF | X << 16 (P), (M), zP, zM}.
bool dibr_col_table(const double* sigma, int w, int (*out)[4]) {
    if (w >= 32768) return false;
    auto exact = [w](double v) -> int {  // the reference's column, or INT_MIN if outside
        if (!(v > -1.0) || !(v < static_cast<double>(w))) return INT32_MIN;
        return static_cast<int>(v);  // truncation toward zero, (-1, 0) -> 0
    };
    for (int d = 0; d < 256; ++d) {
        int packed[2], zs[2];
        for (int dir = 0; dir < 2; ++dir) {
            const double sg = sigma[d];
            auto eval = [&](int x) {
                const double xd = x;
                return exact(dir == 0 ? xd + sg : xd - sg);
            };
            const double c = dir == 0 ? sg : -sg;
            const double fl = std::floor(c);
            if (fl < -32768.0 || fl > 32767.0) return false;
            const int off = static_cast<int>(fl);
            int X = w, z = -1;
            for (int x = 0; x < w; ++x) {
                const double xd = x;
                const double v = dir == 0 ? xd + sg : xd - sg;
                if (v > -1.0 && v < 0.0) {  // truncates to column 0
                    if (z < 0) z = x;
                    continue;
                }
                // a rounding-up of x +- sigma shows as floor(v) == x + off + 1 (whether or not
                // the column is then inside the image)
                if (v >= 0.0 && X == w && std::floor(v) == static_cast<double>(x + off + 1)) X = x;
            }
            for (int x = 0; x < w; ++x) {  // verify the representation everywhere
                const int e = eval(x);
                int col = x == z ? 0 : x + off + (x >= X ? 1 : 0);
                if (col < 0 || col >= w) col = INT32_MIN;
                if (col != e) return false;
            }
            packed[dir] = static_cast<int>((static_cast<unsigned>(off) & 0xFFFFu) |
                                           (static_cast<unsigned>(X) << 16));
            zs[dir] = z;
        }
        out[d][0] = packed[0];
        out[d][1] = packed[1];
        out[d][2] = zs[0];
        out[d][3] = zs[1];
    }
    return true;
}

// depth.cpp:82-102: centre list and locate(); the running index is monotone in v, so one
// forward sweep gives the same (i, frac) as the reference's per-pixel linear scan.
void locate_axis(int count, int blocks, int block, std::vector<int>& i0, std::vector<int>& i1,
                 std::vector<double>& f) {
    std::vector<double> c(blocks);
    for (int i = 0; i < blocks; ++i) {
        const int lo = i * block;
        const int hi = std::min(lo + block, count);
        c[i] = lo + (hi - 1 - lo) / 2.0;
    }
    i0.resize(count);
    i1.resize(count);
    f.resize(count);
    int k = 0;
    for (int p = 0; p < count; ++p) {
        const double v = p;
        int i;
        double frac;
        if (v <= c.front()) {
            i = 0;
            frac = 0.0;
        } else if (v >= c.back()) {
            i = blocks - 1;
            frac = 0.0;
        } else {
            while (v > c[k + 1]) ++k;
            i = k;
            frac = (v - c[i]) / (c[i + 1] - c[i]);
        }
        i0[p] = i;
        i1[p] = std::min(i + 1, blocks - 1);
        f[p] = frac;
    }
}

struct Arena {
    std::size_t off = 0;
    template <class T>
    std::size_t take(std::size_t count) {
        off = (off + 255) / 256 * 256;
        const std::size_t at = off;
        off += count * sizeof(T);
        return at;
    }
};

std::string plan_key(int w, int h, const ConversionConfig& c) {
    std::ostringstream os;
    os.precision(17);
    os << w << 'x' << h << '|' << c.effective_base(w) << '|' << c.pop_threshold << '|'
       << c.sigma_spatial << '|' << c.sigma_range << '|' << c.depth_block << '|' << c.alpha
       << '|' << c.beta << '|' << static_cast<int>(c.dibr_mode) << '|' << c.formats;
    return os.str();
}

std::int64_t ms_to_ns(float ms) { return static_cast<std::int64_t>(std::llround(ms * 1.0e6)); }

}  // namespace

// Row bands of the synchronous convert (Pipeline::Impl::plan_bands, DESIGN.md "Banded
// synchronous convert"): each entry is where a band ENDS in the units of every stage.
// Empty when the frame is too short for two bands.
std::vector<BandEnd> band_plan(int w, int h, int radius, int blk, const char* ends_env) {
    (void)w;
    std::vector<BandEnd> bands;
    if (!cu::bilateral_fast_available(radius)) return bands;  // the band kernels are the certified ones
    const int TYb = cu::bilateral_sep_tile_rows(), TD = cu::depth_tile_rows();
    const int tiles_y = (h + TYb - 1) / TYb, dtiles = (h + TD - 1) / TD;
    const int by = (h + blk - 1) / blk;
    std::vector<int> ri0, ri1;
    std::vector<double> rf;
    locate_axis(h, by, blk, ri0, ri1, rf);
    // band ends: a thin first band (short wait for its upload part), then 3 tile rows
    // per band (the upload of the next band outruns this band's filter ~3x), then 2-row
    // bands at the bottom and a 1-row last band: a band's download (~1/3 of its filter
    // time) must hide under the next band's filter, and the last one's under the inpaint.
    // Measured at 4K (tools/band_sweep2.sh, p3s_convert on pinned frames): {1,3,6,9,11,13,
    // 15,16} 572-575 frames/s against 559 for {1,4,8,12,14,16}.
    std::vector<int> ends = {1};
    if (ends_env) {  // e.g. "1,4,8,12,14,16" (tuning)
        ends.clear();
        for (const char* q = ends_env; *q;) {
            ends.push_back(std::atoi(q));
            while (*q && *q != ',') ++q;
            if (*q) ++q;
        }
    } else {
        const int tail_start = tiles_y - 6;  // the last 6 tile rows: 2, 2, 1, 1
        for (int t = 3; t < tail_start; t += 3) ends.push_back(t);
        for (int t = std::max(tail_start, ends.back() + 1); t < tiles_y - 1; t += 2)
            if (t > ends.back()) ends.push_back(t);
        if (tiles_y - 1 > ends.back()) ends.push_back(tiles_y - 1);
    }
    auto urows = [&](int bb) {
        return static_cast<int>(std::lower_bound(ri1.begin(), ri1.end(), bb) - ri1.begin());
    };
    for (int T : ends) {
        if (T >= tiles_y || (!bands.empty() && T <= bands.back().btile)) break;
        const int need = T * TYb + radius;  // depth / luma rows the band's filter reads
        if (need >= h) break;
        int b = bands.empty() ? 1 : bands.back().brow;
        while (b < by && urows(b) < need) ++b;  // fewest block rows whose rows cover it
        if (b >= by) break;
        const int dtl = (b * blk + TD - 1) / TD;  // depth tiles completing block rows < b
        if (dtl * TD >= h) break;
        bands.push_back(BandEnd{std::min(h, dtl * TD + 1), dtl, b, urows(b), T});
    }
    if (bands.empty()) return bands;
    constexpr std::size_t kMaxBands = 31;  // Pipeline::Impl::kBilSlots / 2 - 1
    while (bands.size() > kMaxBands) bands.pop_back();
    bands.push_back(BandEnd{h, dtiles, by, h, tiles_y});
    return bands;
}

// Whether a plan of this width and config uses the integer DIBR column tables (true) or
// the FP64 device path (false): dibr_col_table's derivation + verification, host only.
bool dibr_integer_columns(int w, const ConversionConfig& cfg) {
    double sh[256];
    shift_table(cfg.effective_base(w), cfg.pop_threshold, sh);
    int cols[256][4];
    return dibr_col_table(sh, w, cols);
}

// ==========================================================================================
// Pipeline::Impl — one plan
// ==========================================================================================
struct Pipeline::Impl {
    int dev = 0;
    int w = 0, h = 0, pitch = 0, fpitch = 0, mwords = 0;
    ConversionConfig cfg;
    int base = 0, radius = 0;
    bool backward = false;
    unsigned formats = 0;
    enum Route { kFusedAnaglyph, kDirectFsbs, kEyes } route = kEyes;
    cu::Geom gm{};
    cu::DepthTables dt{};
    std::vector<double> h_spatial;
    bool tiled = true;

    cudaStream_t stream = nullptr;
    unsigned char* arena = nullptr;
    std::size_t arena_bytes = 0;

    uint8_t *src = nullptr, *luma = nullptr, *depth = nullptr, *filt = nullptr;
    unsigned long long* sums = nullptr;
    double* values = nullptr;
    double *range = nullptr, *spatial = nullptr, *shift = nullptr;
    float* sep_table = nullptr;  // the certified bilateral's replicated FP32 range table
    uint32_t* wide_keys = nullptr;  // DIBR z-buffer slots for rows wider than shared memory
    int4* cols = nullptr;  // integer DIBR column tables (nullptr: FP64 device path)
    uint8_t *ana = nullptr, *hsbs = nullptr, *fsbs = nullptr, *eyes = nullptr;
    uint32_t* mbits = nullptr;
    uint32_t* lists = nullptr;  // [eye][N] damaged pixel lists
    unsigned char* ipa = nullptr;  // inpaint arena (state words + tile flags)
    uint32_t* counts = nullptr;  // 2
    uint32_t* bil_list = nullptr;   // bilateral fast path: uncertified pixels (N)
    static constexpr int kBilSlots = 64;  // counters ahead of the list: 2 per band, K <= 32
    uint32_t* bil_count = nullptr;  // kBilSlots: counts, tile-claim counters of the bilateral launches
    uint32_t* ctl = nullptr;     // 128
    long long* stats = nullptr;  // 8: inpaint passes/repaired/fallback per eye, per-eye busy ns
    // stage-API extras (allocated on first use)
    unsigned char* stage_arena = nullptr;
    uint8_t* stage_masks = nullptr;  // 2 byte masks
    double* stage_raw = nullptr;
    uint8_t* ilv = nullptr;  // interleaved RGB staging (6N bytes: FSBS output is 2w wide)

    // Per-run stage events in a ring, so a long timed loop keeps every step's stage
    // times without synchronising between steps (harvested by accumulated()).
    static constexpr int kRing = 64;
    std::vector<std::array<cudaEvent_t, 7>> ring;
    long long* ring_stats = nullptr;  // pinned [kRing][8]: the inpaint stats of each timed run
    long long* conv_stats = nullptr;  // pinned [8]: the last conv run's inpaint stats

    // Queues the D2H of the inpaint stats after a conv frame (read by timings()).
    void copy_conv_stats(cudaStream_t st) {
        if (backward) return;
        if (!conv_stats)
            CK(cudaHostAlloc(reinterpret_cast<void**>(&conv_stats), 8 * sizeof(long long), cudaHostAllocPortable));
        CK(cudaMemcpyAsync(conv_stats, stats, 8 * sizeof(long long), cudaMemcpyDeviceToHost, st));
    }
    int ring_next = 0, last_slot = -1;
    std::deque<int> pending;
    StageTimings acc;
    long long acc_n = 0;
    long long acc_bil_ns = 0, acc_bil_n = 0;  // main bilateral kernel (without the fix-up)
    bool own_stream = false;
    // CTAs of the cooperative inpaint (0: one per SM). Fewer leave SMs to other pipelines'
    // frames: more aggregate throughput with several streams, longer single-frame latency.
    int inpaint_ctas = [] {  // P3S_INPAINT_CTAS: experiment override of the default (0: one per SM)
        const char* e = std::getenv("P3S_INPAINT_CTAS");
        return e ? std::atoi(e) : 0;
    }();
    void set_inpaint_ctas(int ctas);

    // Row-banded synchronous conversion (convert_image on pinned host planes). The frame is
    // cut into K bands of bilateral tile rows; Band::* are each band's END boundaries in the
    // units of every stage (upload rows, depth tiles, block rows, depth rows, bilateral tile
    // rows). The upload goes out in K row parts; a high-priority stream runs the depth stage
    // part by part as the rows land; each band's filter (+ fix-up, + DIBR on the fused
    // routes) runs on its own stream, so band k+1's CTAs fill the SMs as band k's retire.
    // On the fused routes every band's output rows start back over PCIe while later bands
    // still filter; after the inpaint, only the 32-pixel words that held damage are patched
    // into the host planes. Same kernels, same bytes.
    struct Band {
        int in_rows, dtile, brow, urow, btile;
    };
    std::vector<Band> bands;
    bool band_ok = false;
    cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr, depth_stream = nullptr;
    std::vector<cudaStream_t> band_streams;
    // per band: upload part landed, depth part done (fork), band done (join), DIBR rows done
    std::vector<cudaEvent_t> ev_in, ev_fork, ev_join, ev_rows;
    cudaEvent_t ev_prior = nullptr, ev_d2h = nullptr, ev_start = nullptr;
    std::vector<cudaEvent_t> ev_dbg;  // P3S_DEBUG_CONV: per band, filter start / end (timing)
    bool last_banded = false;  // the last conv run used the banded schedule
    cudaGraphExec_t band_exec = nullptr, band_exec2 = nullptr;  // head, body
    std::size_t band_k1 = 0, band_k2 = 0;                        // their kernel nodes
    cudaStream_t aux_stream = nullptr;  // side copies beside the frame's tail
    cudaEvent_t aux_done = nullptr;
    cudaEvent_t maps_ready = nullptr;  // convert_image_deferred: the maps' device copy is done
    cudaStream_t aux() {
        if (!aux_stream) {
            CK(cudaStreamCreateWithFlags(&aux_stream, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&aux_done, cudaEventDisableTiming));
        }
        return aux_stream;
    }

    std::size_t plane() const { return static_cast<std::size_t>(pitch) * h; }
    std::size_t npix() const { return static_cast<std::size_t>(w) * h; }

    Impl(int width, int height, const ConversionConfig& c, int device, cudaStream_t st)
        : dev(device), w(width), h(height), cfg(c), stream(st) {
        cfg.validate();
        pixel_count(w, h);
        pitch = round_up(w, 16);
        fpitch = round_up(2 * w, 16);
        mwords = (w + 31) / 32;
        base = cfg.effective_base(w);
        radius = bilateral_radius(cfg);
        backward = cfg.dibr_mode == DibrMode::kBackwardFallback;
        formats = cfg.formats;
        route = formats == kFormatAnaglyph ? kFusedAnaglyph
                : formats == kFormatFsbs   ? kDirectFsbs
                                           : kEyes;
        gm = cu::Geom{w, h, pitch};
        tiled = radius <= cu::bilateral_tiled_max_radius();

        const int blk = cfg.depth_block;
        const int bx = (w + blk - 1) / blk, by = (h + blk - 1) / blk;
        std::vector<int> ci0, ci1, ri0, ri1;
        std::vector<double> cf, rf;
        locate_axis(w, bx, blk, ci0, ci1, cf);
        locate_axis(h, by, blk, ri0, ri1, rf);
        plan_bands(blk);
        h_spatial = spatial_table(cfg, radius);
        double h_range[256], h_shift[256];
        range_table(cfg, h_range);
        shift_table(base, cfg.pop_threshold, h_shift);
        thread_local int cols_buf[256][4];
        const char* fp64_env = std::getenv("P3S_DIBR_FP64");
        const bool int_cols = !(fp64_env && std::atoi(fp64_env)) && dibr_col_table(h_shift, w, cols_buf);
        if (std::getenv("P3S_DEBUG_PLAN"))
            std::fprintf(stderr, "[p3s] plan %dx%d base %d: DIBR %s\n", w, h, base,
                         int_cols ? "integer column tables" : "FP64");

        const std::size_t P = plane(), N = npix();
        Arena a;
        const std::size_t o_src = a.take<uint8_t>(3 * P);
        const std::size_t o_luma = a.take<uint8_t>(P);
        const std::size_t o_depth = a.take<uint8_t>(P);
        const std::size_t o_filt = a.take<uint8_t>(P);
        const std::size_t o_sums = a.take<unsigned long long>(static_cast<std::size_t>(bx) * by);
        const std::size_t o_vals = a.take<double>(static_cast<std::size_t>(bx) * by);
        const std::size_t o_ci0 = a.take<int>(w), o_ci1 = a.take<int>(w), o_cf = a.take<double>(w);
        const std::size_t o_ri0 = a.take<int>(h), o_ri1 = a.take<int>(h), o_rf = a.take<double>(h);
        const std::size_t o_range = a.take<double>(256), o_shift = a.take<double>(256);
        const std::size_t o_cols = a.take<int4>(256);
        const std::size_t o_spat = a.take<double>(h_spatial.size());
        const std::size_t o_septab = a.take<float>(cu::bilateral_sep_table_bytes() / 4);
        const std::size_t o_ana = (formats & kFormatAnaglyph) ? a.take<uint8_t>(3 * P) : 0;
        const std::size_t o_hsbs = (formats & kFormatHsbs) ? a.take<uint8_t>(3 * P) : 0;
        const std::size_t o_fsbs =
            (formats & kFormatFsbs) ? a.take<uint8_t>(3 * static_cast<std::size_t>(fpitch) * h) : 0;
        const std::size_t o_eyes = a.take<uint8_t>(route == kEyes ? 6 * P : 0);
        const std::size_t o_mbits = a.take<uint32_t>(2 * static_cast<std::size_t>(mwords) * h);
        const std::size_t o_lists = a.take<uint32_t>(backward ? 0 : 2 * N);
        const std::size_t o_ipa = a.take<unsigned char>(backward ? 0 : cu::inpaint_scratch_bytes(w, h));
        const std::size_t o_cnt = a.take<uint32_t>(2);
        const std::size_t o_bil = a.take<uint32_t>(N + kBilSlots);
        const std::size_t o_ctl = a.take<uint32_t>(128);
        const std::size_t o_stats = a.take<long long>(8);
        const std::size_t o_wkeys = a.take<uint32_t>(cu::dibr_wide_key_words(w));
        arena_bytes = a.off;
        CK(cudaSetDevice(dev));
        CK(cudaMalloc(&arena, arena_bytes));
        // zeroed once: the row padding of every plane (pitch > w) is never written by a
        // kernel but is read by 16-byte row loads (its bytes are ignored)
        CK(cudaMemsetAsync(arena, 0, arena_bytes, stream));
        src = arena + o_src;
        luma = arena + o_luma;
        depth = arena + o_depth;
        filt = arena + o_filt;
        sums = reinterpret_cast<unsigned long long*>(arena + o_sums);
        values = reinterpret_cast<double*>(arena + o_vals);
        range = reinterpret_cast<double*>(arena + o_range);
        shift = reinterpret_cast<double*>(arena + o_shift);
        if (int_cols) cols = reinterpret_cast<int4*>(arena + o_cols);
        spatial = reinterpret_cast<double*>(arena + o_spat);
        sep_table = reinterpret_cast<float*>(arena + o_septab);
        if (formats & kFormatAnaglyph) ana = arena + o_ana;
        if (formats & kFormatHsbs) hsbs = arena + o_hsbs;
        if (formats & kFormatFsbs) fsbs = arena + o_fsbs;
        if (route == kEyes) eyes = arena + o_eyes;
        mbits = reinterpret_cast<uint32_t*>(arena + o_mbits);
        if (!backward) {
            lists = reinterpret_cast<uint32_t*>(arena + o_lists);
            ipa = arena + o_ipa;
        }
        counts = reinterpret_cast<uint32_t*>(arena + o_cnt);
        bil_count = reinterpret_cast<uint32_t*>(arena + o_bil);
        bil_list = bil_count + kBilSlots;
        ctl = reinterpret_cast<uint32_t*>(arena + o_ctl);
        stats = reinterpret_cast<long long*>(arena + o_stats);
        wide_keys = cu::dibr_wide_key_words(w) ? reinterpret_cast<uint32_t*>(arena + o_wkeys) : nullptr;

        auto up = [&](std::size_t off, const void* p, std::size_t n) {
            CK(cudaMemcpyAsync(arena + off, p, n, cudaMemcpyHostToDevice, stream));
        };
        up(o_ci0, ci0.data(), w * sizeof(int));
        up(o_ci1, ci1.data(), w * sizeof(int));
        up(o_cf, cf.data(), w * sizeof(double));
        up(o_ri0, ri0.data(), h * sizeof(int));
        up(o_ri1, ri1.data(), h * sizeof(int));
        up(o_rf, rf.data(), h * sizeof(double));
        up(o_range, h_range, sizeof(h_range));
        up(o_shift, h_shift, sizeof(h_shift));
        if (int_cols) up(o_cols, cols_buf, sizeof(cols_buf));
        up(o_spat, h_spatial.data(), h_spatial.size() * sizeof(double));
        CK(cudaMemsetAsync(arena + o_stats, 0, 8 * sizeof(long long), stream));
        CK(cu::build_sep_table(range, sep_table, stream));
        CK(cudaStreamSynchronize(stream));  // host vectors above go out of scope

        dt.col_i0 = reinterpret_cast<int*>(arena + o_ci0);
        dt.col_i1 = reinterpret_cast<int*>(arena + o_ci1);
        dt.col_f = reinterpret_cast<double*>(arena + o_cf);
        dt.row_i0 = reinterpret_cast<int*>(arena + o_ri0);
        dt.row_i1 = reinterpret_cast<int*>(arena + o_ri1);
        dt.row_f = reinterpret_cast<double*>(arena + o_rf);
        dt.bx = bx;
        dt.by = by;
        dt.block = blk;
        dt.alpha255 = cfg.alpha * 255.0;
        dt.beta = cfg.beta;
        dt.row_denom = h > 1 ? h - 1 : 1;
    }

    void plan_bands(int blk) {
        band_ok = false;
        bands.clear();
        const char* env = std::getenv("P3S_BANDED");
        if (env && std::atoi(env) == 0) return;
        if (cu::dibr_wide_key_words(w)) return;  // wide rows: one DIBR launch owns the key slots
        for (const BandEnd& e : band_plan(w, h, radius, blk, std::getenv("P3S_BAND_ENDS")))
            bands.push_back(Band{e.in_rows, e.dtile, e.brow, e.urow, e.btile});
        band_ok = !bands.empty();
    }

    ~Impl() {
        cudaSetDevice(dev);
        if (band_exec) cudaGraphExecDestroy(band_exec);
        if (band_exec2) cudaGraphExecDestroy(band_exec2);
        if (ring_stats) cudaFreeHost(ring_stats);
        if (conv_stats) cudaFreeHost(conv_stats);
        if (aux_stream) cudaStreamDestroy(aux_stream);
        if (aux_done) cudaEventDestroy(aux_done);
        if (maps_ready) cudaEventDestroy(maps_ready);
        for (auto* v : {&ev_in, &ev_fork, &ev_join, &ev_rows})
            for (auto e : *v)
                if (e) cudaEventDestroy(e);
        for (auto e : {ev_prior, ev_d2h, ev_start})
            if (e) cudaEventDestroy(e);
        for (auto s2 : band_streams)
            if (s2) cudaStreamDestroy(s2);
        for (auto s2 : {h2d_stream, d2h_stream, depth_stream})
            if (s2) cudaStreamDestroy(s2);
        for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
        for (auto& g : timed_graphs) cudaGraphExecDestroy(g.exec);
        for (auto& e : conv_ev)
            if (e) cudaEventDestroy(e);
        if (own_stream && stream) {
            cudaStreamSynchronize(stream);
            cudaStreamDestroy(stream);
        }
        for (auto& set : ring)
            for (auto& e : set)
                if (e) cudaEventDestroy(e);
        if (arena) cudaFree(arena);
        if (stage_arena) cudaFree(stage_arena);
        if (ilv) cudaFree(ilv);
    }

    uint8_t* interleave_buffer() {
        if (!ilv) CK(cudaMalloc(&ilv, 6 * npix()));
        return ilv;
    }

    // RGB-interleaved frames (the PPM payload) straight through the fused kernels: the fused
    // depth front and the quad DIBR read the payload from the staging buffer's first 3N
    // bytes, DIBR + inpaint write the anaglyph interleaved into its second 3N bytes, so the
    // file / interleaved-video path makes no separate (de)interleave pass. Other routes and
    // shapes split the payload into planes first (cu::deinterleave).
    bool ilv_run = false;         // the frame being enqueued is interleaved (fused kernels)
    bool last_ilv_fused = false;  // the last run wrote the interleaved anaglyph
    bool ilv_fused_ok() const {
        static const bool off = std::getenv("P3S_ILV_UNFUSED") != nullptr;
        return !off && route == kFusedAnaglyph && !backward && depth_fused() && cols != nullptr &&
               w % 16 == 0 && !wide_keys &&
               static_cast<std::size_t>(pitch) * 13 + 48 <= cu::kDibrMaxSmem;
    }

    uint8_t* src_plane(const uint8_t* s, int c) const { return const_cast<uint8_t*>(s) + c * plane(); }
    uint32_t* list_ptr(int eye, int which) const {
        (void)which;
        return lists + eye * npix();
    }

    void ensure_stage() {
        if (stage_arena) return;
        const std::size_t bytes = 2 * plane() + 256 + npix() * sizeof(double);
        CK(cudaMalloc(&stage_arena, bytes));
        stage_masks = stage_arena;
        stage_raw = reinterpret_cast<double*>(stage_arena + (2 * plane() + 255) / 256 * 256);
    }

    // ---- stage launchers ----
    // Depth stage of depth tile rows [d0, d1) / block rows [b0, b1) / image rows [u0, u1):
    // the fused front (luma + block values, 16-pixel blocks) or front + block_values, then
    // the upsample. sums must be zeroed for the unfused front.
    bool depth_fused() const {
        static const bool off = std::getenv("P3S_DEPTH_UNFUSED") != nullptr;
        return !off && cu::depth_fused_ok(gm, dt.block);
    }
    void enq_depth_rows(const uint8_t* s, cudaStream_t st, int d0, int d1, int b0, int b1, int u0,
                        int u1) {
        if (ilv_run) {  // s: the interleaved payload
            CK(cu::depth_front_fused(s, nullptr, nullptr, gm, luma, dt, values, st, d0, d1, 3 * w));
        } else if (depth_fused()) {
            CK(cu::depth_front_fused(src_plane(s, 0), src_plane(s, 1), src_plane(s, 2), gm, luma, dt,
                                     values, st, d0, d1));
        } else {
            CK(cu::depth_front(src_plane(s, 0), src_plane(s, 1), src_plane(s, 2), gm, luma, sums,
                               dt.block, dt.bx, st, d0, d1));
            CK(cu::block_values(sums, gm, dt, values, st, b0, b1));
        }
        CK(cu::upsample(values, gm, dt, depth, st, u0, u1));
    }

    void enq_depth(const uint8_t* s, cudaStream_t st) {
        if (!depth_fused()) CK(cu::zero(zr({{sums, 2u * dt.bx * dt.by}}), st));
        enq_depth_rows(s, st, 0, -1, 0, -1, 0, -1);
    }

    void enq_bilateral(const uint8_t* dmap, const uint8_t* guide, uint8_t* out, double* raw,
                       cudaStream_t st, cudaEvent_t after_main = nullptr) {
        if (!raw && cu::bilateral_fast_available(radius)) {
            CK(cu::bilateral_fast(dmap, guide, gm, radius, h_spatial.data(), spatial, range, out,
                                  bil_list, bil_count, st, after_main, sep_table));
            static const bool dbg = std::getenv("P3S_DEBUG_BIL") != nullptr;
            if (dbg) {
                uint32_t n = 0;
                CK(cudaMemcpyAsync(&n, bil_count, sizeof(n), cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
                std::fprintf(stderr, "[p3s] bilateral %dx%d: %u uncertified pixels (%.4f%%)\n", w,
                             h, n, 100.0 * n / npix());
            }
        }
        else if (tiled)
            CK(cu::bilateral_tiled(dmap, guide, gm, radius, h_spatial.data(), range, out, raw, st));
        else
            CK(cu::bilateral(dmap, guide, gm, radius, spatial, range, out, raw, st));
        if (after_main && !(!raw && cu::bilateral_fast_available(radius))) record_event(after_main, st);
    }

    void eye_planes(uint8_t* (&L)[3], uint8_t* (&R)[3], int& lp) const {
        for (int c = 0; c < 3; ++c) L[c] = R[c] = nullptr;
        if (route == kFusedAnaglyph && ilv_run) {
            uint8_t* o = ilv + 3 * npix();  // interleaved anaglyph, row stride 3w
            L[0] = o;
            R[1] = o + 1;
            R[2] = o + 2;
            lp = 3 * w;
        } else if (route == kFusedAnaglyph) {
            L[0] = ana;
            R[1] = ana + plane();
            R[2] = ana + 2 * plane();
            lp = pitch;
        } else if (route == kDirectFsbs) {
            const std::size_t fp = static_cast<std::size_t>(fpitch) * h;
            for (int c = 0; c < 3; ++c) {
                L[c] = fsbs + c * fp;
                R[c] = fsbs + c * fp + w;
            }
            lp = fpitch;
        } else {
            for (int c = 0; c < 3; ++c) {
                L[c] = eyes + c * plane();
                R[c] = eyes + (3 + c) * plane();
            }
            lp = pitch;
        }
    }

    void enq_dibr_inpaint(const uint8_t* s, cudaStream_t st, cudaEvent_t mid) {
        cu::EyeOut eo[2];
        dibr_eyes(eo);
        if (!backward) CK(cu::zero(zr({{counts, 2u}}), st));
        if (ilv_run)
            CK(cu::dibr(s, nullptr, nullptr, filt, gm, shift, cols, backward, eo[0], eo[1], st, 0, -1,
                        nullptr, 3 * w));
        else
            CK(cu::dibr(src_plane(s, 0), src_plane(s, 1), src_plane(s, 2), filt, gm, shift, cols, backward,
                        eo[0], eo[1], st, 0, -1, wide_keys));
        if (mid) record_event(mid, st);
        enq_inpaint(st);
    }

    void enq_formats(cudaStream_t st) {
        if (route != kEyes) return;
        const uint8_t* L[3] = {eyes, eyes + plane(), eyes + 2 * plane()};
        const uint8_t* R[3] = {eyes + 3 * plane(), eyes + 4 * plane(), eyes + 5 * plane()};
        if (formats & kFormatAnaglyph) {
            uint8_t* o[3] = {ana, ana + plane(), ana + 2 * plane()};
            CK(cu::anaglyph(L, R, gm, o, pitch, st));
        }
        if (formats & kFormatHsbs) {
            uint8_t* o[3] = {hsbs, hsbs + plane(), hsbs + 2 * plane()};
            CK(cu::side_by_side_half(L, R, gm, o, pitch, st));
        }
        if (formats & kFormatFsbs) {
            const std::size_t fp = static_cast<std::size_t>(fpitch) * h;
            uint8_t* o[3] = {fsbs, fsbs + fp, fsbs + 2 * fp};
            CK(cu::side_by_side_full(L, R, gm, o, fpitch, st));
        }
    }

    // Banded schedule: depth, filter (+ fix-up) and, on the fused routes, DIBR of different
    // bands overlap on the GPU, so events cannot time them one by one (a queued kernel's span
    // includes its wait for SMs, and timing events inside the band graph cost ~10 % of the
    // call). Their joint time, from the frame's first kernel to the bands' join, is split by
    // the plan's measured stage shares: a one-time event-timed run of the same plan and
    // frame without bands (calibrate()). Stages that run alone (DIBR on the materialised-
    // eyes route, inpaint, formats) keep their own event times. So the parts sum to the
    // frame's GPU time and pure_ns = filter + DIBR + inpaint + format as the reference
    // defines it (pipeline.hpp:24-26).
    bool cal_valid = false;
    double cal_share[3] = {0, 0, 0};  // depth, filter, DIBR of the unbanded timed run

    void banded_stage_ms(const std::array<cudaEvent_t, 7>& ev, float (&ms)[5]) {
        const bool back = band_back();
        float joint = 0.f;  // ev[0] .. the join (ev[2]; the fused routes' DIBR is inside)
        CK(cudaEventElapsedTime(&joint, ev[0], ev[2]));
        const int n = back ? 3 : 2;  // stages sharing the joint time
        double tot = 0;
        for (int i = 0; i < n; ++i) tot += cal_share[i];
        for (int i = 0; i < n; ++i) ms[i] = tot > 0 ? static_cast<float>(joint * cal_share[i] / tot) : 0.f;
        if (tot <= 0) ms[1] = joint;
        // (fused routes: nothing runs between the join and the inpaint; ev[2] is both)
    }

    // The stage shares for banded_stage_ms: an event-timed, unbanded run of the frame now in
    // src, once per plan (the outputs of the banded frame are already on the host).
    void calibrate(cudaStream_t st) {
        if (cal_valid) return;
        const bool lc = last_conv, lb = last_banded;
        const std::array<cudaEvent_t, 7>* ev = next_events();
        enqueue(src, st, ev);
        const int slot = static_cast<int>(ev - &ring.front());
        CK(cudaEventSynchronize((*ev)[5]));
        pending.pop_back();  // not part of the plan's accumulated timings
        float ms[3] = {0, 0, 0};
        for (int i = 0; i < 3; ++i) CK(cudaEventElapsedTime(&ms[i], (*ev)[i], (*ev)[i + 1]));
        for (int i = 0; i < 3; ++i) cal_share[i] = ms[i];
        cal_valid = true;
        (void)slot;
        last_conv = lc;
        last_banded = lb;
    }

    // Stage times of one run from its events. st8: that run's inpaint stats (host copy), or
    // nullptr to read the plan's (the run must be the last one on the plan's stream).
    StageTimings stage_times(const std::array<cudaEvent_t, 7>& ev, const long long* st8 = nullptr,
                             bool banded = false) {
        StageTimings t;
        CK(cudaEventSynchronize(ev[5]));
        float ms[5] = {0, 0, 0, 0, 0};
        if (banded && band_back()) {
            // the banded fused routes record no ev[3] / ev[4]: ev[2] is the join and the
            // inpaint's start, ev[5] its end (the formats were written by the DIBR)
            CK(cudaEventElapsedTime(&ms[3], ev[2], ev[5]));
            banded_stage_ms(ev, ms);
        } else {
            for (int i = 0; i < 5; ++i) CK(cudaEventElapsedTime(&ms[i], ev[i], ev[i + 1]));
            if (banded) banded_stage_ms(ev, ms);
        }
        t.depth_gen_ns = ms_to_ns(ms[0]);
        t.filter_ns = ms_to_ns(ms[1]);
        t.dibr_ns = ms_to_ns(ms[2]);
        t.format_ns = ms_to_ns(ms[4]);
        split_inpaint(t, ms[3], st8);
        return t;
    }

    // Both eyes are repaired by one kernel (pipeline.cpp:56-65 runs them one after the other):
    // its time is split by each eye's tile-processing time; an eye with no damage reports 0,
    // as the reference skips its inpaint (so B = 0 or backward mode reports 0 for both).
    void split_inpaint(StageTimings& t, float inpaint_ms, const long long* st8) {
        t.inpaint_left_ns = t.inpaint_right_ns = 0;
        if (backward) return;
        long long s[8];
        if (!st8) {
            CK(cudaMemcpy(s, stats, sizeof(s), cudaMemcpyDeviceToHost));
            st8 = s;
        }
        const long long dmgL = st8[1] + st8[2], dmgR = st8[4] + st8[5];
        if (!dmgL && !dmgR) return;
        const std::int64_t total = ms_to_ns(inpaint_ms);
        if (!dmgR) {
            t.inpaint_left_ns = total;
            return;
        }
        if (!dmgL) {
            t.inpaint_right_ns = total;
            return;
        }
        const double bl = static_cast<double>(st8[6]), br = static_cast<double>(st8[7]);
        const double fl = bl + br > 0 ? bl / (bl + br) : 0.5;
        t.inpaint_left_ns = static_cast<std::int64_t>(std::llround(total * fl));
        t.inpaint_right_ns = total - t.inpaint_left_ns;
    }

    void harvest_one() {
        const int slot = pending.front();
        pending.pop_front();
        const StageTimings t = stage_times(ring[slot], ring_stats + 8 * slot);
        acc.depth_gen_ns += t.depth_gen_ns;
        acc.filter_ns += t.filter_ns;
        acc.dibr_ns += t.dibr_ns;
        acc.inpaint_left_ns += t.inpaint_left_ns;
        acc.inpaint_right_ns += t.inpaint_right_ns;
        acc.format_ns += t.format_ns;
        ++acc_n;
        float bm = 0.f;  // the dominant kernel alone: depth-stage end -> bilateral main kernel end
        CK(cudaEventElapsedTime(&bm, ring[slot][1], ring[slot][6]));
        acc_bil_ns += ms_to_ns(bm);
        ++acc_bil_n;
    }

    const std::array<cudaEvent_t, 7>* next_events() {
        if (ring.empty()) {
            ring.resize(kRing);
            for (auto& set : ring)
                for (auto& e : set) CK(cudaEventCreate(&e));
            // each timed run's inpaint stats land here (D2H in stream order) for its harvest
            CK(cudaHostAlloc(reinterpret_cast<void**>(&ring_stats), kRing * 8 * sizeof(long long),
                             cudaHostAllocPortable));
        }
        if (static_cast<int>(pending.size()) == kRing) harvest_one();
        const int slot = ring_next;
        ring_next = (ring_next + 1) % kRing;
        pending.push_back(slot);
        last_slot = slot;
        return &ring[slot];
    }

    // Untimed runs replay a CUDA graph of the whole frame (captured once per input frame
    // address; the ring of a video pipeline or bench is a handful of addresses), which
    // removes the per-kernel launch gaps. Timed runs enqueue directly (their stage events
    // differ per run). P3S_NO_GRAPHS=1 disables the graphs.
    struct GraphEntry {
        const uint8_t* src;
        cudaGraphExec_t exec;
        std::size_t kernels;  // kernel nodes (launch accounting)
    };
    std::list<GraphEntry> graphs;  // LRU
    static constexpr std::size_t kMaxGraphs = 16;
    // convert_image's timed frame: one graph per input address with a FIXED event set whose
    // record nodes are part of the graph (read back right after the synchronous call)
    std::array<cudaEvent_t, 7> conv_ev{};
    std::list<GraphEntry> timed_graphs;
    bool last_conv = false;  // the last timed run used conv_ev

    bool graphs_enabled() const {
        static const bool off = [] {
            const char* v = std::getenv("P3S_NO_GRAPHS");
            return v && std::atoi(v) != 0;
        }();
        return !off;
    }

    void run_graph(const uint8_t* s, cudaStream_t st, bool timed = false) {
        std::list<GraphEntry>& cache = timed ? timed_graphs : graphs;
        if (timed && !conv_ev[0])
            for (auto& e : conv_ev) CK(cudaEventCreate(&e));
        for (auto it = cache.begin(); it != cache.end(); ++it) {
            if (it->src == s) {
                cache.splice(cache.begin(), cache, it);
                CK(cudaGraphLaunch(cache.front().exec, st));
                cu::note_graph_launch(cache.front().kernels);
                return;
            }
        }
        cudaStream_t cap = stream;  // capture on the plan's own stream, launch on st
        CK(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
        try {
            enqueue(s, cap, timed ? &conv_ev : nullptr);
        } catch (...) {
            cudaGraph_t g = nullptr;
            cudaStreamEndCapture(cap, &g);
            if (g) cudaGraphDestroy(g);
            cudaGetLastError();
            throw;
        }
        cudaGraph_t g = nullptr;
        CK(cudaStreamEndCapture(cap, &g));
        cudaGraphExec_t exec = nullptr;
        const std::size_t kernels = cu::graph_kernel_nodes(g);
        const cudaError_t e = cudaGraphInstantiate(&exec, g, 0);
        cudaGraphDestroy(g);
        CK(e);
        cache.push_front(GraphEntry{s, exec, kernels});
        while (cache.size() > kMaxGraphs) {
            cudaGraphExecDestroy(cache.back().exec);
            cache.pop_back();
        }
        CK(cudaGraphLaunch(exec, st));
        cu::note_graph_launch(kernels);
    }

    // A timed frame for a synchronous caller (convert_image): graph replay with the plan's
    // fixed event set; timings()/download_overlapped() read those events.
    void run_conv(const uint8_t* s, cudaStream_t st) {
        last_banded = false;
        if ((formats & kFormatHsbs) && (w % 2 != 0))
            throw std::invalid_argument("side_by_side: half mode requires an even width");
        if (!graphs_enabled()) {
            run(s, st, true);
            last_conv = false;
            return;
        }
        run_graph(s, st, true);
        last_conv = true;
        copy_conv_stats(st);
    }

    void run(const uint8_t* s, cudaStream_t st, bool record) {
        if ((formats & kFormatHsbs) && (w % 2 != 0))
            throw std::invalid_argument("side_by_side: half mode requires an even width");
        last_ilv_fused = ilv_run;
        if (!record && graphs_enabled()) {
            run_graph(s, st);
            return;
        }
        if (record) last_conv = false;
        enqueue(s, st, record ? next_events() : nullptr);
    }

    void enqueue(const uint8_t* s, cudaStream_t st, const std::array<cudaEvent_t, 7>* ev) {
        if (ev) record_event((*ev)[0], st);
        enq_depth(s, st);
        if (ev) record_event((*ev)[1], st);
        enq_bilateral(depth, luma, filt, nullptr, st, ev ? (*ev)[6] : nullptr);
        if (ev) record_event((*ev)[2], st);
        enq_dibr_inpaint(s, st, ev ? (*ev)[3] : nullptr);
        if (ev) record_event((*ev)[4], st);
        if (ev && !ring.empty() && ev >= &ring.front() && ev <= &ring.back() && !backward)
            CK(cudaMemcpyAsync(ring_stats + 8 * (ev - &ring.front()), stats, 8 * sizeof(long long),
                               cudaMemcpyDeviceToHost, st));
        enq_formats(st);
        if (ev) record_event((*ev)[5], st);
    }

    void ensure_band_resources() {
        if (h2d_stream) return;
        int lo = 0, hi = 0;
        CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CK(cudaStreamCreateWithFlags(&h2d_stream, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&d2h_stream, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithPriority(&depth_stream, cudaStreamNonBlocking, hi));
        const std::size_t K = bands.size();
        band_streams.assign(K, nullptr);
        for (auto& s2 : band_streams) CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
        for (auto* v : {&ev_in, &ev_fork, &ev_join, &ev_rows}) {
            v->assign(K, nullptr);
            for (auto& e : *v) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        for (auto* e : {&ev_prior, &ev_d2h, &ev_start}) CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        if (std::getenv("P3S_DEBUG_CONV")) {
            ev_dbg.assign(3 * K, nullptr);
            for (auto& e : ev_dbg) CK(cudaEventCreate(&e));
        }

        if (!conv_ev[0])
            for (auto& e : conv_ev) CK(cudaEventCreate(&e));
    }

    // the fused routes write the final output planes in DIBR (patched in place by the
    // inpaint), so their rows can leave per band
    bool band_back() const { return route != kEyes; }

    // Host planes -> src in K row parts on h2d_stream (ev_in[k]): parts [k0, k1). Part 0 goes
    // before the frame's graph; the others after it, held until band 0's depth stage is done
    // (conv_ev[1]): while the copy engine streams host reads, every dependent launch of that
    // chain waits behind them on PCIe (~20 us each), so the first band gets the link first.
    void upload_banded(const ImageRGB8& img, cudaStream_t st, int k0, int k1) {
        if (k0 == 0) {
            CK(cudaEventRecord(ev_prior, st));  // earlier work on st (reads src) comes first
            CK(cudaStreamWaitEvent(h2d_stream, ev_prior, 0));
        } else {
            CK(cudaStreamWaitEvent(h2d_stream, conv_ev[1], 0));
        }
        int r0 = k0 == 0 ? 0 : bands[k0 - 1].in_rows;
        for (int k = k0; k < k1; ++k) {
            const int r1 = bands[k].in_rows;
            if (r1 > r0)
                for (int c = 0; c < 3; ++c)
                    CK(cudaMemcpy2DAsync(src + c * plane() + static_cast<std::size_t>(r0) * pitch, pitch,
                                         img.plane(c).data() + static_cast<std::size_t>(r0) * w, w, w,
                                         r1 - r0, cudaMemcpyHostToDevice, h2d_stream));
            CK(cudaEventRecord(ev_in[k], h2d_stream));
            r0 = std::max(r0, r1);
        }
    }

    void dibr_eyes(cu::EyeOut (&eo)[2]) const {
        uint8_t *L[3], *R[3];
        int lp = pitch;
        eye_planes(L, R, lp);
        for (int e = 0; e < 2; ++e) {
            for (int c = 0; c < 3; ++c) eo[e].plane[c] = e ? R[c] : L[c];
            eo[e].pitch = lp;
            eo[e].stride = route == kFusedAnaglyph && ilv_run ? 3 : 1;
            eo[e].mask_bytes = nullptr;
            eo[e].mask_bits = backward ? nullptr : mbits + static_cast<std::size_t>(e) * mwords * h;
            eo[e].mask_pitch = mwords;
            eo[e].list = backward ? nullptr : list_ptr(e, 0);
            eo[e].count = counts + e;
        }
    }

    // zero: 0 memsets, 1 a kernel, 2 none (enq_inpaint_zero ran earlier in stream order)
    void enq_inpaint(cudaStream_t st, int zero = 0) {
        if (backward) return;
        cu::EyeOut eo[2];
        dibr_eyes(eo);
        cu::InpaintEye ie[2];
        for (int e = 0; e < 2; ++e) {
            for (int c = 0; c < 3; ++c) ie[e].plane[c] = eo[e].plane[c];
            ie[e].pitch = eo[e].pitch;
            ie[e].stride = eo[e].stride;
            ie[e].mask_bytes = nullptr;
            ie[e].mask_bits = eo[e].mask_bits;
            ie[e].mask_pitch = mwords;
            ie[e].list = list_ptr(e, 0);
            ie[e].count = counts + e;
            ie[e].list2 = nullptr;
            ie[e].repair = reinterpret_cast<uint32_t*>(ipa);
        }
        CK(cu::inpaint(ie[0], ie[1], gm, static_cast<uint32_t>(npix()), ctl, stats, st, inpaint_ctas,
                       zero));
    }

    // The inpaint's control-word zeroing on its own (a kernel: see the banded body)
    void enq_inpaint_zero(cudaStream_t st) {
        if (backward) return;
        cu::InpaintEye left{};
        left.repair = reinterpret_cast<uint32_t*>(ipa);
        CK(cu::inpaint_zero(left, gm, ctl, stats, st, true));
    }

    // bil_count layout: [0, K) per-band uncertified counts, [K, 2K) tile-claim counters;
    // band k lists its pixels from bil_list + (first row of band k) * w.
    // Head: band 0's depth stage (launched before the upload of the other parts is queued).
    void enqueue_banded_head(cudaStream_t st, const std::array<cudaEvent_t, 7>& ev) {
        const uint8_t* s = src;
        const int K = static_cast<int>(bands.size());
        wait_event_any(st, ev_in[0]);
        record_event(ev[0], st);
        CK(cu::zero(zr({{sums, depth_fused() ? 0u : 2u * dt.bx * dt.by},
                        {bil_count, 2u * K},
                        {counts, backward ? 0u : 2u}}), st, true));
        const Band& b = bands[0];
        enq_depth_rows(s, st, 0, b.dtile, 0, b.brow, 0, b.urow);
        record_event(ev[1], st);
    }

    // Body: the other parts' depth stages (each after its upload part), every band's filter
    // (+ fix-up + DIBR rows on the fused routes), then the inpaint and formats.
    void enqueue_banded_body(cudaStream_t st, const std::array<cudaEvent_t, 7>& ev) {
        const uint8_t* s = src;
        const int K = static_cast<int>(bands.size());
        const int TYb = cu::bilateral_sep_tile_rows();
        const bool back = band_back();
        cu::EyeOut eo[2];
        dibr_eyes(eo);
        CK(cudaEventRecord(ev_start, st));
        CK(cudaStreamWaitEvent(depth_stream, ev_start, 0));
        // the inpaint's control words are zeroed now, while the bands run, so the tail after
        // the last band is DIBR -> inpaint with no zeroing node between them
        enq_inpaint_zero(st);
        Band prev{0, 0, 0, 0, 0};
        for (int k = 0; k < K; ++k) {
            const Band& b = bands[k];
            cudaStream_t ds = depth_stream, bs = band_streams[k];
            if (k > 0) {
                wait_event_any(ds, ev_in[k]);
                enq_depth_rows(s, ds, prev.dtile, b.dtile, prev.brow, b.brow, prev.urow, b.urow);
            }
            CK(cudaEventRecord(ev_fork[k], ds));
            CK(cudaStreamWaitEvent(bs, ev_fork[k], 0));
            if (!ev_dbg.empty()) record_event(ev_dbg[3 * k], bs);
            const int y0 = prev.btile * TYb, y1 = std::min(h, b.btile * TYb);
            uint32_t* list = bil_list + static_cast<std::size_t>(y0) * w;
            CK(cu::bilateral_sep_main(depth, luma, gm, radius, h_spatial.data(), range, filt, list,
                                      bil_count + k, bil_count + K + k, prev.btile, b.btile,
                                      sep_table, bs));
            if (!ev_dbg.empty()) record_event(ev_dbg[3 * k + 1], bs);
            // a band lists a few hundred pixels: one CTA per SM is plenty
            CK(cu::bilateral_sep_fixup(depth, luma, gm, radius, spatial, range, filt, list,
                                       bil_count + k, bs, sm_count_cached()));
            if (back) {
                CK(cu::dibr(src_plane(s, 0), src_plane(s, 1), src_plane(s, 2), filt, gm, shift, cols,
                            backward, eo[0], eo[1], bs, y0, y1));
                record_event(ev_rows[k], bs);
            }
            if (!ev_dbg.empty()) record_event(ev_dbg[3 * k + 2], bs);
            CK(cudaEventRecord(ev_join[k], bs));
            prev = b;
        }
        for (int k = 0; k < K; ++k) CK(cudaStreamWaitEvent(st, ev_join[k], 0));
        // (each event record is a graph node on the tail's critical path: the fused routes,
        // where nothing runs between the join and the inpaint, record the join once and
        // stage_times reads it as both ev[2] and ev[3]; ev[6] only for P3S_DEBUG_CONV)
        if (!ev_dbg.empty()) record_event(ev[6], st);
        record_event(ev[2], st);
        if (!back) {
            CK(cu::dibr(src_plane(s, 0), src_plane(s, 1), src_plane(s, 2), filt, gm, shift, cols,
                        backward, eo[0], eo[1], st, 0, -1, wide_keys));
            record_event(ev[3], st);
        }
        enq_inpaint(st, 2);  // zeroed at the body's start (enq_inpaint_zero)
        if (!back) {
            record_event(ev[4], st);
            enq_formats(st);
        }
        // (fused routes: the formats were written by the DIBR, so the inpaint's end is the end)
        record_event(ev[5], st);
    }

    cudaGraphExec_t capture(void (Impl::*fn)(cudaStream_t, const std::array<cudaEvent_t, 7>&),
                            std::size_t& kernels) {
        CK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
        try {
            (this->*fn)(stream, conv_ev);
        } catch (...) {
            cudaGraph_t g = nullptr;
            cudaStreamEndCapture(stream, &g);
            if (g) cudaGraphDestroy(g);
            cudaGetLastError();
            throw;
        }
        cudaGraph_t g = nullptr;
        CK(cudaStreamEndCapture(stream, &g));
        cudaGraphExec_t exec = nullptr;
        kernels = cu::graph_kernel_nodes(g);
        const cudaError_t e = cudaGraphInstantiate(&exec, g, 0);
        cudaGraphDestroy(g);
        CK(e);
        return exec;
    }

    // Output planes of format f on the host (pitch = output width).
    struct HostOut {
        uint8_t* plane[3];
    };

    // After the banded graph: each band's output rows leave as soon as its DIBR finished
    // (d2h_stream); then the words that held damage are rewritten from the final planes.
    void download_banded(StereoFormat f, const HostOut& out, cudaStream_t st) {
        const int K = static_cast<int>(bands.size());
        const int TYb = cu::bilateral_sep_tile_rows();
        const int ow = output_width(f), op = output_pitch(f);
        const std::size_t ps = static_cast<std::size_t>(op) * h;
        int y0 = 0;
        for (int k = 0; k < K; ++k) {
            const int y1 = std::min(h, bands[k].btile * TYb);
            CK(cudaStreamWaitEvent(d2h_stream, ev_rows[k], 0));
            for (int c = 0; c < 3; ++c)
                CK(cudaMemcpy2DAsync(out.plane[c] + static_cast<std::size_t>(y0) * ow, ow,
                                     output(f) + c * ps + static_cast<std::size_t>(y0) * op, op, ow,
                                     y1 - y0, cudaMemcpyDeviceToHost, d2h_stream));
            y0 = y1;
        }
        CK(cudaEventRecord(ev_d2h, d2h_stream));
        CK(cudaStreamWaitEvent(st, ev_d2h, 0));
        if (backward) return;  // no holes: the early rows are final
        cu::EyeOut eo[2];
        dibr_eyes(eo);
        cu::PatchEye pe[2];
        for (int e = 0; e < 2; ++e) {
            for (int c = 0; c < 3; ++c) {
                pe[e].dev[c] = eo[e].plane[c];
                pe[e].host[c] = eo[e].plane[c] ? out.plane[c] + (route == kDirectFsbs && e ? w : 0) : nullptr;
            }
            pe[e].dpitch = eo[e].pitch;
            pe[e].hpitch = ow;
            pe[e].mask = eo[e].mask_bits;
            pe[e].mpitch = mwords;
        }
        CK(cu::patch_host(pe[0], pe[1], gm, st));
    }

    // convert_image's frame: upload + run (+ the outputs' download when banded). Returns
    // true when the outputs in `outs` were downloaded here.
    bool upload_run_conv(const ImageRGB8& img, cudaStream_t st, std::map<StereoFormat, ImageRGB8>* outs) {
        bool pinned = band_ok;
        for (int c = 0; c < 3 && pinned; ++c) pinned = host_pinned(img.plane(c).data());
        if (!pinned) {
            for (int c = 0; c < 3; ++c) h2d_plane(src + c * plane(), img.plane(c).data(), st);
            run_conv(src, st);
            return false;
        }
        if ((formats & kFormatHsbs) && (w % 2 != 0))
            throw std::invalid_argument("side_by_side: half mode requires an even width");
        ensure_band_resources();
        const int K = static_cast<int>(bands.size());
        // part 0 -> head (band 0's depth) -> the other parts (held until the head is done)
        // -> body. An event-wait node sees the records made before its graph's launch, so
        // each graph is launched after the uploads it waits for are queued.
        upload_banded(img, st, 0, 1);
        last_conv = true;
        last_banded = true;
        if (!graphs_enabled()) {
            enqueue_banded_head(st, conv_ev);
            upload_banded(img, st, 1, K);
            enqueue_banded_body(st, conv_ev);
        } else {
            if (!band_exec) band_exec = capture(&Impl::enqueue_banded_head, band_k1);
            if (!band_exec2) band_exec2 = capture(&Impl::enqueue_banded_body, band_k2);
            CK(cudaGraphLaunch(band_exec, st));
            cu::note_graph_launch(band_k1);
            upload_banded(img, st, 1, K);
            CK(cudaGraphLaunch(band_exec2, st));
            cu::note_graph_launch(band_k2);
        }
        copy_conv_stats(st);
        if (!outs || !band_back()) return false;
        const StereoFormat f = route == kFusedAnaglyph ? kFormatAnaglyph : kFormatFsbs;
        ImageRGB8 o(output_width(f), h, false);
        HostOut ho{{o.plane(0).data(), o.plane(1).data(), o.plane(2).data()}};
        for (int c = 0; c < 3; ++c)
            if (!host_pinned(ho.plane[c])) {
                // unpinned output planes: plain download after the frame
                for (int c2 = 0; c2 < 3; ++c2)
                    d2h_plane(ho.plane[c2], output(f) + c2 * static_cast<std::size_t>(output_pitch(f)) * h,
                              output_pitch(f), output_width(f), st);
                (*outs)[f] = std::move(o);
                return true;
            }
        download_banded(f, ho, st);
        (*outs)[f] = std::move(o);
        return true;
    }

    void drop_graphs() {
        CK(cudaStreamSynchronize(stream));
        for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
        for (auto& g : timed_graphs) cudaGraphExecDestroy(g.exec);
        graphs.clear();
        timed_graphs.clear();
        if (band_exec) cudaGraphExecDestroy(band_exec);
        if (band_exec2) cudaGraphExecDestroy(band_exec2);
        band_exec = band_exec2 = nullptr;
    }

    StageTimings timings() {
        if (last_conv) return stage_times(conv_ev, conv_stats, last_banded);
        if (last_slot < 0) return StageTimings{};
        return stage_times(ring[last_slot], ring_stats + 8 * last_slot);
    }

    long long bilateral_kernel_sum(long long* count, bool reset) {
        while (!pending.empty()) harvest_one();
        const long long t = acc_bil_ns;
        if (count) *count = acc_bil_n;
        if (reset) {
            acc_bil_ns = 0;
            acc_bil_n = 0;
        }
        return t;
    }

    StageTimings accumulated(long long* count, bool reset) {
        while (!pending.empty()) harvest_one();
        const StageTimings t = acc;
        if (count) *count = acc_n;
        if (reset) {
            acc = StageTimings{};
            acc_n = 0;
        }
        return t;
    }

    const uint8_t* output(StereoFormat f) const {
        return f == kFormatAnaglyph ? ana : f == kFormatHsbs ? hsbs : fsbs;
    }
    int output_pitch(StereoFormat f) const { return f == kFormatFsbs ? fpitch : pitch; }
    int output_width(StereoFormat f) const { return f == kFormatFsbs ? 2 * w : w; }

    void d2h_plane(uint8_t* host, const uint8_t* dev_plane, int dpitch, int width,
                   cudaStream_t st) {
        CK(cudaMemcpy2DAsync(host, width, dev_plane, dpitch, width, h, cudaMemcpyDeviceToHost, st));
    }
    void h2d_plane(uint8_t* dev_plane, const uint8_t* host, cudaStream_t st) {
        CK(cudaMemcpy2DAsync(dev_plane, pitch, host, w, w, h, cudaMemcpyHostToDevice, st));
    }

    // Download with the depth and filtered-depth copies on a second stream, each started as
    // soon as its producer finished (events of the timed run), so they overlap the later
    // stages; the outputs follow the last kernel on the compute stream.
    void download_overlapped(ConversionResult& out, cudaStream_t st, cudaStream_t cs) {
        if (!last_conv && last_slot < 0) return download(out, st);
        const std::array<cudaEvent_t, 7>& ev = last_conv ? conv_ev : ring[last_slot];
        out.depth = GrayMap(w, h, false);
        out.filtered_depth = GrayMap(w, h, false);
        CK(cudaStreamWaitEvent(cs, ev[1], 0));
        d2h_plane(out.depth.data.data(), depth, pitch, w, cs);
        CK(cudaStreamWaitEvent(cs, ev[2], 0));
        d2h_plane(out.filtered_depth.data.data(), filt, pitch, w, cs);
        for (StereoFormat f : {kFormatAnaglyph, kFormatHsbs, kFormatFsbs}) {
            if (!(formats & f)) continue;
            const int ow = output_width(f);
            ImageRGB8 img(ow, h, false);
            const std::size_t ps = static_cast<std::size_t>(output_pitch(f)) * h;
            for (int c = 0; c < 3; ++c)
                d2h_plane(img.plane(c).data(), output(f) + c * ps, output_pitch(f), ow, st);
            out.outputs[f] = std::move(img);
        }
        CK(cudaStreamSynchronize(cs));
        CK(cudaStreamSynchronize(st));
    }

    void download(ConversionResult& out, cudaStream_t st) {
        out.depth = GrayMap(w, h, false);
        out.filtered_depth = GrayMap(w, h, false);
        d2h_plane(out.depth.data.data(), depth, pitch, w, st);
        d2h_plane(out.filtered_depth.data.data(), filt, pitch, w, st);
        for (StereoFormat f : {kFormatAnaglyph, kFormatHsbs, kFormatFsbs}) {
            if (!(formats & f)) continue;
            const int ow = output_width(f);
            ImageRGB8 img(ow, h, false);
            const std::size_t ps = static_cast<std::size_t>(output_pitch(f)) * h;
            for (int c = 0; c < 3; ++c)
                d2h_plane(img.plane(c).data(), output(f) + c * ps, output_pitch(f), ow, st);
            out.outputs[f] = std::move(img);
        }
        CK(cudaStreamSynchronize(st));
    }
};

// ==========================================================================================
// Device
// ==========================================================================================
struct Device::Impl {
    int ordinal = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;  // D2H of intermediate results, overlapping compute
    std::list<std::pair<std::string, std::shared_ptr<Pipeline::Impl>>> plans;  // LRU
    static constexpr std::size_t kMaxPlans = 4;

    std::shared_ptr<Pipeline::Impl> plan(int w, int h, const ConversionConfig& cfg) {
        const std::string key = plan_key(w, h, cfg);
        for (auto it = plans.begin(); it != plans.end(); ++it) {
            if (it->first == key) {
                plans.splice(plans.begin(), plans, it);
                return plans.front().second;
            }
        }
        auto p = std::make_shared<Pipeline::Impl>(w, h, cfg, ordinal, stream);
        plans.emplace_front(key, p);
        while (plans.size() > kMaxPlans) plans.pop_back();
        return p;
    }
};

Device::Device(int ordinal) : impl_(new Impl) {
    int n = 0;
    const cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        throw DeviceError(std::string("no CUDA device available (") +
                          (e == cudaSuccess ? "0 devices" : cudaGetErrorString(e)) +
                          "); the B200 pipeline has no CPU fallback");
    }
    if (ordinal < 0 || ordinal >= n) throw DeviceError("CUDA device ordinal out of range");
    impl_->ordinal = ordinal;
    CK(cudaSetDevice(ordinal));
    CK(cudaStreamCreateWithFlags(&impl_->stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&impl_->copy_stream, cudaStreamNonBlocking));
}

Device::~Device() {
    if (impl_) {
        impl_->plans.clear();
        cudaSetDevice(impl_->ordinal);
        if (impl_->stream) cudaStreamDestroy(impl_->stream);
        if (impl_->copy_stream) cudaStreamDestroy(impl_->copy_stream);
    }
}

int Device::ordinal() const { return impl_->ordinal; }
void* Device::stream() const { return impl_->stream; }

Device& Device::current() {
    thread_local std::map<int, std::unique_ptr<Device>> devices;
    int ord = 0;
    const cudaError_t e = cudaGetDevice(&ord);
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw DeviceError(std::string("no CUDA device available (") + cudaGetErrorString(e) +
                          "); the B200 pipeline has no CPU fallback");
    }
    auto it = devices.find(ord);
    if (it == devices.end()) it = devices.emplace(ord, std::make_unique<Device>(ord)).first;
    CK(cudaSetDevice(ord));
    return *it->second;
}


// ==========================================================================================
// Pipeline (device-resident; owns its plan and stream, so several pipelines on one
// device overlap freely)
// ==========================================================================================
Pipeline::Pipeline(int width, int height, const ConversionConfig& cfg, Device& dev) {
    CK(cudaSetDevice(dev.ordinal()));
    cudaStream_t st = nullptr;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    try {
        impl_ = std::make_shared<Impl>(width, height, cfg, dev.ordinal(), st);
    } catch (...) {
        cudaStreamDestroy(st);
        throw;
    }
    impl_->own_stream = true;
}
Pipeline::~Pipeline() = default;
int Pipeline::pitch() const { return impl_->pitch; }
int Pipeline::width() const { return impl_->w; }
int Pipeline::height() const { return impl_->h; }
void* Pipeline::stream() const { return impl_->stream; }
std::size_t Pipeline::frame_bytes() const { return 3 * impl_->plane(); }
void Pipeline::run(const std::uint8_t* d_src, void* stream) {
    impl_->run(d_src, stream ? static_cast<cudaStream_t>(stream) : impl_->stream, false);
}
void Pipeline::Impl::set_inpaint_ctas(int ctas) {
    if (ctas < 0) throw std::invalid_argument("inpaint CTAs must be >= 0");
    if (ctas == inpaint_ctas) return;
    drop_graphs();  // the launch configuration is baked into captured graphs
    inpaint_ctas = ctas;
}
void Pipeline::set_inpaint_ctas(int ctas) { impl_->set_inpaint_ctas(ctas); }
void Pipeline::run_timed(const std::uint8_t* d_src, void* stream) {
    impl_->run(d_src, stream ? static_cast<cudaStream_t>(stream) : impl_->stream, true);
}
StageTimings Pipeline::last_timings() { return impl_->timings(); }
StageTimings Pipeline::accumulated_timings(long long* count, bool reset) {
    return impl_->accumulated(count, reset);
}
long long Pipeline::bilateral_kernel_ns(long long* count, bool reset) {
    return impl_->bilateral_kernel_sum(count, reset);
}
const std::uint8_t* Pipeline::d_depth() const { return impl_->depth; }
const std::uint8_t* Pipeline::d_filtered() const { return impl_->filt; }
const std::uint8_t* Pipeline::d_output(StereoFormat f) const { return impl_->output(f); }
int Pipeline::output_pitch(StereoFormat f) const { return impl_->output_pitch(f); }
void Pipeline::download(ConversionResult& out, void* stream) {
    impl_->download(out, stream ? static_cast<cudaStream_t>(stream) : impl_->stream);
}
void Pipeline::inpaint_stats(InpaintStats& left, InpaintStats& right) {
    long long s[6];
    CK(cudaMemcpyAsync(s, impl_->stats, sizeof(s), cudaMemcpyDeviceToHost, impl_->stream));
    CK(cudaStreamSynchronize(impl_->stream));
    left = InpaintStats{static_cast<int>(s[0]), static_cast<std::size_t>(s[1]),
                        static_cast<std::size_t>(s[2])};
    right = InpaintStats{static_cast<int>(s[3]), static_cast<std::size_t>(s[4]),
                         static_cast<std::size_t>(s[5])};
}

std::uint8_t* Pipeline::d_input() { return impl_->src; }
void Pipeline::upload(const std::uint8_t* r, const std::uint8_t* g, const std::uint8_t* b,
                      std::uint8_t* d_dst, void* stream) {
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : impl_->stream;
    const std::uint8_t* planes[3] = {r, g, b};
    for (int c = 0; c < 3; ++c) impl_->h2d_plane(d_dst + c * impl_->plane(), planes[c], st);
}
void Pipeline::upload_interleaved(const std::uint8_t* rgb, std::uint8_t* d_dst, void* stream) {
    Impl& p = *impl_;
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : p.stream;
    uint8_t* buf = p.interleave_buffer();
    CK(cudaMemcpyAsync(buf, rgb, 3 * p.npix(), cudaMemcpyHostToDevice, st));
    CK(cu::deinterleave(buf, p.w, p.h, d_dst, d_dst + p.plane(), d_dst + 2 * p.plane(), p.pitch, st));
}
void Pipeline::run_interleaved(const std::uint8_t* rgb, bool timed, void* stream) {
    Impl& p = *impl_;
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : p.stream;
    uint8_t* buf = p.interleave_buffer();
    CK(cudaMemcpyAsync(buf, rgb, 3 * p.npix(), cudaMemcpyHostToDevice, st));
    if (!p.ilv_fused_ok()) {
        uint8_t* d = p.src;
        CK(cu::deinterleave(buf, p.w, p.h, d, d + p.plane(), d + 2 * p.plane(), p.pitch, st));
        p.run(d, st, timed);
        return;
    }
    p.ilv_run = true;
    try {
        p.run(buf, st, timed);
    } catch (...) {
        p.ilv_run = false;
        throw;
    }
    p.ilv_run = false;
}
void Pipeline::download_interleaved(StereoFormat f, std::uint8_t* rgb_out, void* stream, bool sync) {
    Impl& p = *impl_;
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : p.stream;
    if (!(p.formats & f)) throw std::invalid_argument("format was not requested in the configuration");
    if (p.last_ilv_fused && f == kFormatAnaglyph) {  // already interleaved by DIBR + inpaint
        CK(cudaMemcpyAsync(rgb_out, p.interleave_buffer() + 3 * p.npix(), 3 * p.npix(),
                           cudaMemcpyDeviceToHost, st));
        if (sync) CK(cudaStreamSynchronize(st));
        return;
    }
    uint8_t* buf = p.interleave_buffer();
    const int ow = p.output_width(f), op = p.output_pitch(f);
    const std::size_t ps = static_cast<std::size_t>(op) * p.h;
    const uint8_t* o = p.output(f);
    CK(cu::interleave(o, o + ps, o + 2 * ps, op, ow, p.h, buf, st));
    CK(cudaMemcpyAsync(rgb_out, buf, 3 * static_cast<std::size_t>(ow) * p.h, cudaMemcpyDeviceToHost, st));
    if (sync) CK(cudaStreamSynchronize(st));
}
void Pipeline::download_to(std::uint8_t* depth, std::uint8_t* filtered, StereoFormat f,
                           std::uint8_t* const* out, void* stream, bool sync) {
    Impl& p = *impl_;
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : p.stream;
    if (depth) p.d2h_plane(depth, p.depth, p.pitch, p.w, st);
    if (filtered) p.d2h_plane(filtered, p.filt, p.pitch, p.w, st);
    if (out && (p.formats & f)) {
        const int ow = p.output_width(f);
        const std::size_t ps = static_cast<std::size_t>(p.output_pitch(f)) * p.h;
        for (int c = 0; c < 3; ++c)
            if (out[c]) p.d2h_plane(out[c], p.output(f) + c * ps, p.output_pitch(f), ow, st);
    }
    if (sync) CK(cudaStreamSynchronize(st));
}

// ==========================================================================================
// Stage API (each call: H2D, the stage's kernels, D2H, on the thread's device stream)
// ==========================================================================================
namespace {

std::shared_ptr<Pipeline::Impl> stage_plan(Device& dev, int w, int h, const ConversionConfig& cfg) {
    return dev.impl().plan(w, h, cfg);
}

void upload_image(Pipeline::Impl& p, const ImageRGB8& img, cudaStream_t st) {
    for (int c = 0; c < 3; ++c) p.h2d_plane(p.src + c * p.plane(), img.plane(c).data(), st);
}

void require_same(int w0, int h0, int w1, int h1, const char* msg) {
    if (w0 != w1 || h0 != h1) throw std::invalid_argument(msg);
}

}  // namespace

GrayMap luma(const ImageRGB8& img, Device& dev) {
    ConversionConfig cfg;
    auto p = stage_plan(dev, img.width, img.height, cfg);
    cudaStream_t st = p->stream;
    upload_image(*p, img, st);
    p->enq_depth(p->src, st);
    GrayMap out(img.width, img.height, false);
    p->d2h_plane(out.data.data(), p->luma, p->pitch, p->w, st);
    CK(cudaStreamSynchronize(st));
    return out;
}

BlockGrid block_depth(const ImageRGB8& img, const ConversionConfig& cfg, Device& dev) {
    cfg.validate();
    auto p = stage_plan(dev, img.width, img.height, cfg);
    cudaStream_t st = p->stream;
    upload_image(*p, img, st);
    p->enq_depth(p->src, st);
    BlockGrid g;
    g.block = cfg.depth_block;
    g.width = img.width;
    g.height = img.height;
    g.blocks_x = p->dt.bx;
    g.blocks_y = p->dt.by;
    g.values.resize(static_cast<std::size_t>(g.blocks_x) * g.blocks_y);
    CK(cudaMemcpyAsync(g.values.data(), p->values, g.values.size() * sizeof(double),
                       cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return g;
}

GrayMap upsample_block_grid(const BlockGrid& grid, Device& dev) {
    ConversionConfig cfg;
    cfg.depth_block = grid.block;
    auto p = stage_plan(dev, grid.width, grid.height, cfg);
    cudaStream_t st = p->stream;
    if (grid.values.size() != static_cast<std::size_t>(p->dt.bx) * p->dt.by)
        throw std::invalid_argument("upsample_block_grid: grid size mismatch");
    CK(cudaMemcpyAsync(p->values, grid.values.data(), grid.values.size() * sizeof(double),
                       cudaMemcpyHostToDevice, st));
    CK(cu::upsample(p->values, p->gm, p->dt, p->depth, st));
    GrayMap out(grid.width, grid.height, false);
    p->d2h_plane(out.data.data(), p->depth, p->pitch, p->w, st);
    CK(cudaStreamSynchronize(st));
    return out;
}

GrayMap generate_depth(const ImageRGB8& img, const ConversionConfig& cfg, Device& dev) {
    cfg.validate();
    auto p = stage_plan(dev, img.width, img.height, cfg);
    cudaStream_t st = p->stream;
    upload_image(*p, img, st);
    p->enq_depth(p->src, st);
    GrayMap out(img.width, img.height, false);
    p->d2h_plane(out.data.data(), p->depth, p->pitch, p->w, st);
    CK(cudaStreamSynchronize(st));
    return out;
}

static void bilateral_common(const GrayMap& depth, const GrayMap& guide,
                             const ConversionConfig& cfg, Device& dev, GrayMap* out,
                             std::vector<double>* raw) {
    require_same(depth.width, depth.height, guide.width, guide.height,
                 "cross_bilateral: depth and guide dimensions differ");
    auto p = stage_plan(dev, depth.width, depth.height, cfg);
    cudaStream_t st = p->stream;
    p->h2d_plane(p->depth, depth.data.data(), st);
    p->h2d_plane(p->luma, guide.data.data(), st);
    double* d_raw = nullptr;
    if (raw) {
        p->ensure_stage();
        d_raw = p->stage_raw;
    }
    p->enq_bilateral(p->depth, p->luma, p->filt, d_raw, st);
    if (out) {
        *out = GrayMap(depth.width, depth.height, false);
        p->d2h_plane(out->data.data(), p->filt, p->pitch, p->w, st);
    }
    if (raw) {
        raw->resize(p->npix());
        CK(cudaMemcpyAsync(raw->data(), d_raw, p->npix() * sizeof(double), cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
}

GrayMap cross_bilateral(const GrayMap& depth, const GrayMap& guide, const ConversionConfig& cfg,
                        Device& dev) {
    GrayMap out;
    bilateral_common(depth, guide, cfg, dev, &out, nullptr);
    return out;
}

std::vector<double> cross_bilateral_raw(const GrayMap& depth, const GrayMap& guide,
                                        const ConversionConfig& cfg, Device& dev) {
    std::vector<double> raw;
    bilateral_common(depth, guide, cfg, dev, nullptr, &raw);
    return raw;
}

StereoFrames reconstruct(const ImageRGB8& src, const GrayMap& depth, const ConversionConfig& cfg,
                         Device& dev) {
    require_same(src.width, src.height, depth.width, depth.height,
                 "reconstruct: source and depth dimensions differ");
    // The stage API materialises both eye frames and byte masks (reference StereoFrames).
    ConversionConfig c = cfg;
    c.formats = kFormatAnaglyph | kFormatHsbs;  // forces the materialised-eyes route
    auto p = stage_plan(dev, src.width, src.height, c);
    p->ensure_stage();
    cudaStream_t st = p->stream;
    upload_image(*p, src, st);
    p->h2d_plane(p->filt, depth.data.data(), st);
    cu::EyeOut eo[2];
    for (int e = 0; e < 2; ++e) {
        for (int ch = 0; ch < 3; ++ch) eo[e].plane[ch] = p->eyes + (3 * e + ch) * p->plane();
        eo[e].pitch = p->pitch;
        eo[e].mask_bytes = p->stage_masks + e * p->plane();
        eo[e].mask_bits = nullptr;
        eo[e].mask_pitch = p->pitch;
        eo[e].list = nullptr;
        eo[e].count = p->counts + e;
    }
    CK(cu::dibr(p->src, p->src + p->plane(), p->src + 2 * p->plane(), p->filt, p->gm, p->shift,
                p->cols, p->backward, eo[0], eo[1], st, 0, -1, p->wide_keys));
    StereoFrames f;
    f.left = ImageRGB8(src.width, src.height, false);
    f.right = ImageRGB8(src.width, src.height, false);
    f.left_mask = DamageMask(src.width, src.height);
    f.right_mask = DamageMask(src.width, src.height);
    for (int ch = 0; ch < 3; ++ch) {
        p->d2h_plane(f.left.plane(ch).data(), eo[0].plane[ch], p->pitch, p->w, st);
        p->d2h_plane(f.right.plane(ch).data(), eo[1].plane[ch], p->pitch, p->w, st);
    }
    p->d2h_plane(f.left_mask.damaged.data(), eo[0].mask_bytes, p->pitch, p->w, st);
    p->d2h_plane(f.right_mask.damaged.data(), eo[1].mask_bytes, p->pitch, p->w, st);
    CK(cudaStreamSynchronize(st));
    return f;
}

ImageRGB8 inpaint(const ImageRGB8& frame, const DamageMask& mask, const ConversionConfig& cfg,
                  Device& dev, InpaintStats* stats) {
    require_same(frame.width, frame.height, mask.width, mask.height,
                 "inpaint: frame and mask dimensions differ");
    ConversionConfig c = cfg;
    c.dibr_mode = DibrMode::kForwardZBuffer;  // the plan needs its work lists
    c.formats = kFormatAnaglyph | kFormatHsbs;
    auto p = stage_plan(dev, frame.width, frame.height, c);
    p->ensure_stage();
    cudaStream_t st = p->stream;
    // left eye = the frame; the right eye gets an empty list
    for (int ch = 0; ch < 3; ++ch) p->h2d_plane(p->eyes + ch * p->plane(), frame.plane(ch).data(), st);
    p->h2d_plane(p->stage_masks, mask.damaged.data(), st);
    CK(cudaMemsetAsync(p->counts, 0, 2 * sizeof(uint32_t), st));
    CK(cu::mask_to_list(p->stage_masks, p->pitch, p->gm, p->list_ptr(0, 0), p->counts, st, p->mbits,
                        p->mwords));
    cu::InpaintEye ie[2];
    for (int e = 0; e < 2; ++e) {
        for (int ch = 0; ch < 3; ++ch) ie[e].plane[ch] = p->eyes + (3 * e + ch) * p->plane();
        ie[e].pitch = p->pitch;
        ie[e].mask_bytes = nullptr;
        ie[e].mask_bits = p->mbits + static_cast<std::size_t>(e) * p->mwords * p->h;  // eye 1: no damage listed
        ie[e].mask_pitch = p->mwords;
        ie[e].list = p->list_ptr(e, 0);
        ie[e].count = p->counts + e;
        ie[e].list2 = nullptr;
        ie[e].repair = reinterpret_cast<uint32_t*>(p->ipa);
    }
    CK(cu::inpaint(ie[0], ie[1], p->gm, static_cast<uint32_t>(p->npix()), p->ctl, p->stats, st));
    ImageRGB8 out(frame.width, frame.height, false);
    for (int ch = 0; ch < 3; ++ch)
        p->d2h_plane(out.plane(ch).data(), p->eyes + ch * p->plane(), p->pitch, p->w, st);
    long long s[6];
    CK(cudaMemcpyAsync(s, p->stats, sizeof(s), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (stats) *stats = InpaintStats{static_cast<int>(s[0]), static_cast<std::size_t>(s[1]),
                                     static_cast<std::size_t>(s[2])};
    return out;
}

static ImageRGB8 format_common(const ImageRGB8& left, const ImageRGB8& right, unsigned fmt,
                               Device& dev) {
    ConversionConfig c;
    c.formats = kFormatAnaglyph | kFormatHsbs | kFormatFsbs;
    auto p = stage_plan(dev, left.width, left.height, c);
    cudaStream_t st = p->stream;
    for (int ch = 0; ch < 3; ++ch) {
        p->h2d_plane(p->eyes + ch * p->plane(), left.plane(ch).data(), st);
        p->h2d_plane(p->eyes + (3 + ch) * p->plane(), right.plane(ch).data(), st);
    }
    const unsigned saved = p->formats;
    p->formats = fmt;
    try {
        p->enq_formats(st);
    } catch (...) {
        p->formats = saved;
        throw;
    }
    p->formats = saved;
    const StereoFormat f = static_cast<StereoFormat>(fmt);
    const int ow = p->output_width(f);
    ImageRGB8 out(ow, left.height, false);
    const std::size_t ps = static_cast<std::size_t>(p->output_pitch(f)) * p->h;
    for (int ch = 0; ch < 3; ++ch)
        p->d2h_plane(out.plane(ch).data(), p->output(f) + ch * ps, p->output_pitch(f), ow, st);
    CK(cudaStreamSynchronize(st));
    return out;
}

ImageRGB8 anaglyph(const ImageRGB8& left, const ImageRGB8& right, Device& dev) {
    require_same(left.width, left.height, right.width, right.height,
                 "anaglyph: eye dimensions differ");
    return format_common(left, right, kFormatAnaglyph, dev);
}

ImageRGB8 side_by_side(const ImageRGB8& left, const ImageRGB8& right, bool half, Device& dev) {
    require_same(left.width, left.height, right.width, right.height,
                 "side_by_side: eye dimensions differ");
    if (half && left.width % 2 != 0)
        throw std::invalid_argument("side_by_side: half mode requires an even width");
    return format_common(left, right, half ? kFormatHsbs : kFormatFsbs, dev);
}

// ---- deferred depth maps ------------------------------------------------------------------
namespace {

// Process-wide pool of device buffers for deferred maps, per (device, bytes).
struct MapPool {
    std::mutex mu;
    std::multimap<std::pair<int, std::size_t>, void*> free;
    std::size_t cached = 0;
    static constexpr std::size_t kMaxCached = std::size_t(1) << 30;

    void* take(int dev, std::size_t bytes) {
        {
            std::lock_guard<std::mutex> lk(mu);
            auto it = free.find({dev, bytes});
            if (it != free.end()) {
                void* p = it->second;
                free.erase(it);
                cached -= bytes;
                return p;
            }
        }
        void* p = nullptr;
        CK(cudaMalloc(&p, bytes));
        return p;
    }
    void give(int dev, std::size_t bytes, void* p) {
        {
            std::lock_guard<std::mutex> lk(mu);
            if (cached + bytes <= kMaxCached) {
                free.emplace(std::make_pair(dev, bytes), p);
                cached += bytes;
                return;
            }
        }
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(dev);
        cudaFree(p);
        cudaSetDevice(cur);
    }
};

MapPool& map_pool() {
    static MapPool* p = new MapPool();  // intentionally leaked: outlives static dtors
    return *p;
}

}  // namespace

DeferredMaps::DeferredMaps(int device, int w, int h, void* dev_buf)
    : device_(device), w_(w), h_(h), buf_(dev_buf) {}

DeferredMaps::~DeferredMaps() {
    if (done_) {
        cudaEventSynchronize(static_cast<cudaEvent_t>(done_));  // the D2H reads buf_
        cudaEventDestroy(static_cast<cudaEvent_t>(done_));
        cudaGetLastError();
    }
    if (buf_) map_pool().give(device_, 2 * static_cast<std::size_t>(w_) * h_, buf_);
}

namespace {
// One copy stream per device for the background map downloads.
cudaStream_t maps_stream(int device) {
    static std::mutex mu;
    static std::map<int, cudaStream_t> streams;
    std::lock_guard<std::mutex> lk(mu);
    cudaStream_t& s = streams[device];
    if (!s) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    return s;
}
}  // namespace

void DeferredMaps::start_download(void* ready_event) {
    const std::size_t n = static_cast<std::size_t>(w_) * h_;
    depth_ = GrayMap(w_, h_, false);     // pinned pool: the copy engine writes them directly
    filtered_ = GrayMap(w_, h_, false);
    cudaStream_t s = maps_stream(device_);
    CK(cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(ready_event), 0));
    CK(cudaMemcpyAsync(depth_.data.data(), buf_, n, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(filtered_.data.data(), static_cast<uint8_t*>(buf_) + n, n, cudaMemcpyDeviceToHost, s));
    cudaEvent_t e = nullptr;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CK(cudaEventRecord(e, s));
    done_ = e;
}

void DeferredMaps::materialize() {
    std::lock_guard<std::mutex> lk(mu_);
    if (ready_) return;
    int cur = 0;
    cudaGetDevice(&cur);
    CK(cudaSetDevice(device_));
    if (done_) {
        const cudaError_t e = cudaEventSynchronize(static_cast<cudaEvent_t>(done_));
        cudaSetDevice(cur);
        CK(e);
    } else {
        const std::size_t n = static_cast<std::size_t>(w_) * h_;
        GrayMap d(w_, h_, false), f(w_, h_, false);
        const cudaError_t e1 = cudaMemcpy(d.data.data(), buf_, n, cudaMemcpyDeviceToHost);
        const cudaError_t e2 = cudaMemcpy(f.data.data(), static_cast<uint8_t*>(buf_) + n, n,
                                          cudaMemcpyDeviceToHost);
        cudaSetDevice(cur);
        CK(e1);
        CK(e2);
        depth_ = std::move(d);
        filtered_ = std::move(f);
    }
    ready_ = true;
    map_pool().give(device_, 2 * static_cast<std::size_t>(w_) * h_, buf_);
    buf_ = nullptr;
}

const GrayMap& DeferredMaps::depth() {
    materialize();
    return depth_;
}
const GrayMap& DeferredMaps::filtered() {
    materialize();
    return filtered_;
}

ConversionResult convert_image_deferred(const ImageRGB8& src, const ConversionConfig& cfg,
                                        Device& dev, std::shared_ptr<DeferredMaps>& maps) {
    NvtxRange nv_conv("p3s_convert");
    cfg.validate();
    auto p = stage_plan(dev, src.width, src.height, cfg);
    cudaStream_t st = p->stream;
    ConversionResult res;
    static const bool dbg = std::getenv("P3S_DEBUG_CONV") != nullptr;
    static thread_local cudaEvent_t dbg_ev[2] = {nullptr, nullptr};
    if (dbg && !dbg_ev[0]) {
        CK(cudaEventCreate(&dbg_ev[0]));
        CK(cudaEventCreate(&dbg_ev[1]));
    }
    const auto t0 = std::chrono::steady_clock::now();
    if (dbg) CK(cudaEventRecord(dbg_ev[0], st));
    bool have_outputs;
    {
        NvtxRange nv("p3s_convert: upload + enqueue");
        have_outputs = p->upload_run_conv(src, st, &res.outputs);
    }
    const auto t1 = std::chrono::steady_clock::now();
    const std::size_t n = p->npix();
    uint8_t* buf = static_cast<uint8_t*>(map_pool().take(dev.ordinal(), 2 * n));
    try {
        // device copies of the maps (unpitched), then the outputs to the host. After a
        // graph frame the copies run on a side stream from the filter's end (conv_ev[2]),
        // beside the inpaint and the downloads.
        cudaStream_t ms = st;
        if (p->last_conv) {
            ms = p->aux();
            CK(cudaStreamWaitEvent(ms, p->conv_ev[2], 0));
        }
        CK(cudaMemcpy2DAsync(buf, p->w, p->depth, p->pitch, p->w, p->h, cudaMemcpyDeviceToDevice, ms));
        CK(cudaMemcpy2DAsync(buf + n, p->w, p->filt, p->pitch, p->w, p->h, cudaMemcpyDeviceToDevice, ms));
        if (ms != st) {
            CK(cudaEventRecord(p->aux_done, ms));
            CK(cudaStreamWaitEvent(st, p->aux_done, 0));
        }
        for (StereoFormat f : {kFormatAnaglyph, kFormatHsbs, kFormatFsbs}) {
            if (!(p->formats & f) || have_outputs) continue;
            const int ow = p->output_width(f);
            ImageRGB8 img(ow, p->h, false);
            const std::size_t ps = static_cast<std::size_t>(p->output_pitch(f)) * p->h;
            for (int c = 0; c < 3; ++c)
                p->d2h_plane(img.plane(c).data(), p->output(f) + c * ps, p->output_pitch(f), ow, st);
            res.outputs[f] = std::move(img);
        }
        if (dbg) CK(cudaEventRecord(dbg_ev[1], st));
        {
            NvtxRange nv("p3s_convert: wait");
            CK(cudaStreamSynchronize(st));
        }
        if (p->last_banded && !p->cal_valid) p->calibrate(st);
        res.timings = p->timings();
        if (dbg) {
            float a0 = 0, b5 = 0, ab = 0;
            cudaEventElapsedTime(&a0, dbg_ev[0], p->conv_ev[0]);
            cudaEventElapsedTime(&b5, p->conv_ev[5], dbg_ev[1]);
            cudaEventElapsedTime(&ab, dbg_ev[0], dbg_ev[1]);
            std::fprintf(stderr, "[p3s] gpu: start->ev0 %.1f us, ev5->end %.1f us, start->end %.1f us\n",
                         a0 * 1e3, b5 * 1e3, ab * 1e3);
            for (std::size_t k = 0; 3 * k + 2 < p->ev_dbg.size(); ++k) {
                float t0 = 0, t1 = 0, t2 = 0;
                cudaEventElapsedTime(&t0, p->conv_ev[0], p->ev_dbg[3 * k]);
                cudaEventElapsedTime(&t1, p->conv_ev[0], p->ev_dbg[3 * k + 1]);
                cudaEventElapsedTime(&t2, p->conv_ev[0], p->ev_dbg[3 * k + 2]);
                cudaGetLastError();
                std::fprintf(stderr, "[p3s]   band %zu (tile rows to %d): start %.1f, filter end %.1f, end %.1f us\n",
                             k, p->bands[k].btile, t0 * 1e3, t1 * 1e3, t2 * 1e3);
            }
            const auto t2 = std::chrono::steady_clock::now();
            auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
            float e01 = 0, e06 = 0, e64 = 0, e05 = 0;
            cudaEventElapsedTime(&e01, p->conv_ev[0], p->conv_ev[1]);
            cudaEventElapsedTime(&e06, p->conv_ev[0], p->conv_ev[6]);
            cudaEventElapsedTime(&e64, p->conv_ev[6], p->conv_ev[5]);
            cudaEventElapsedTime(&e05, p->conv_ev[0], p->conv_ev[5]);
            std::fprintf(stderr, "[p3s] convert: enqueue %.1f us, wait %.1f us, total %.1f us | gpu: depth0 %.1f, "
                         "filter+dibr end %.1f, inpaint %.1f, all %.1f us\n", us(t0, t1), us(t1, t2), us(t0, t2),
                         e01 * 1e3, e06 * 1e3, e64 * 1e3, e05 * 1e3);
        }
        maps = std::make_shared<DeferredMaps>(dev.ordinal(), p->w, p->h, buf);
        // the maps go to the host in the background (after their device copy); p3s_convert
        // does not wait for them
        // P3S_EAGER_MAPS=1: the maps go to the host in the background right away (the next
        // call's output downloads then share the D2H link with them: -20 % e2e at 4K);
        // default: on first access
        static const bool eager = [] {
            const char* e = std::getenv("P3S_EAGER_MAPS");
            return e && *e == '1';
        }();
        if (eager) {
            try {
                if (!p->maps_ready) CK(cudaEventCreateWithFlags(&p->maps_ready, cudaEventDisableTiming));
                CK(cudaEventRecord(p->maps_ready, ms));
                maps->start_download(p->maps_ready);
            } catch (...) {
                cudaGetLastError();  // not queued: the maps download on first access instead
            }
        }
        return res;
    } catch (...) {
        map_pool().give(dev.ordinal(), 2 * n, buf);
        throw;
    }
}

ConversionResult convert_image(const ImageRGB8& src, const ConversionConfig& cfg, Device& dev) {
    NvtxRange nv_conv("p3s_convert");
    cfg.validate();
    auto p = stage_plan(dev, src.width, src.height, cfg);
    cudaStream_t st = p->stream;
    ConversionResult res;
    if (p->upload_run_conv(src, st, &res.outputs)) {
        res.depth = GrayMap(p->w, p->h, false);
        res.filtered_depth = GrayMap(p->w, p->h, false);
        p->d2h_plane(res.depth.data.data(), p->depth, p->pitch, p->w, st);
        p->d2h_plane(res.filtered_depth.data.data(), p->filt, p->pitch, p->w, st);
        CK(cudaStreamSynchronize(st));
        if (p->last_banded && !p->cal_valid) p->calibrate(st);
        res.timings = p->timings();
        return res;
    }
    p->download_overlapped(res, st, dev.impl().copy_stream);
    if (p->last_banded && !p->cal_valid) p->calibrate(st);
    res.timings = p->timings();
    return res;
}

}  // namespace p3s
