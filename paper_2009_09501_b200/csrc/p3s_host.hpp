// Internal host-side declarations shared by the C-ABI implementation (capi.cpp), the
// sequence driver and the bench harness. Not installed.
#pragma once

#include <cstdint>
#include <optional>
#include <string>
#include <vector>

#include "p3s/core.hpp"
#include "p3s/pipeline.hpp"

namespace p3s {

// ---- PNM and files (reference pnm.cpp, io.cpp) ----
// A validated P6 file viewed in place: dimensions and the interleaved RGB payload (same
// checks and PnmError messages as decode_ppm, no copy).
struct PpmView {
    int width, height;
    const std::uint8_t* payload;
};
PpmView ppm_view(const std::uint8_t* data, std::size_t size);
std::string ppm_header(int w, int h);
ImageRGB8 decode_ppm(const std::uint8_t* data, std::size_t size);
std::vector<std::uint8_t> encode_ppm(const ImageRGB8& img);
GrayMap decode_pgm(const std::uint8_t* data, std::size_t size);
std::vector<std::uint8_t> encode_pgm(const GrayMap& map);
void deinterleave_rgb(const std::uint8_t* src, std::size_t n, std::uint8_t* r, std::uint8_t* g,
                      std::uint8_t* b);
void interleave_rgb(const std::uint8_t* r, const std::uint8_t* g, const std::uint8_t* b,
                    std::size_t n, std::uint8_t* dst);
std::vector<std::uint8_t> read_file(const std::string& path);
void write_file(const std::string& path, const std::uint8_t* data, std::size_t size);

// ---- sequences (reference sequence.hpp) ----
struct FrameTiming {
    std::int64_t index = 0;
    int width = 0, height = 0;
    StageTimings timings;
};

struct SequenceReport {
    std::vector<FrameTiming> frames;
    std::int64_t wall_ns = 0;
    std::int64_t pure_sum_ns() const;
    std::int64_t pure_min_ns() const;
    std::int64_t pure_max_ns() const;
    double pure_mean_ns() const;
    std::string to_csv(int threads) const;
};

class FramePattern {
public:
    static FramePattern parse(const std::string& pattern);
    std::string filename(std::int64_t index) const;
    std::string stem(std::int64_t index) const;

private:
    std::string prefix_, suffix_;
    int pad_ = 0;
};

SequenceReport convert_sequence_dir(const std::string& in_dir, const std::string& pattern,
                                    const std::string& out_dir, const ConversionConfig& cfg,
                                    int threads);

// ---- bench (reference bench.hpp) ----
ImageRGB8 synthetic_frame(int w, int h, std::uint64_t seed);

struct BenchRow {
    int width = 0, height = 0, threads = 0, rep = 0;
    std::int64_t depth_ns = 0, filter_ns = 0, dibr_ns = 0, inpaint_l_ns = 0, inpaint_r_ns = 0,
                 format_ns = 0, pure_ns = 0;
};

struct BenchReport {
    std::vector<BenchRow> rows;
    double speedup(int width, int height, int threads) const;
    std::string to_csv() const;
};

BenchReport run_bench(const std::vector<std::pair<int, int>>& sizes,
                      const std::vector<int>& thread_counts, int reps, std::uint64_t seed,
                      const ConversionConfig& cfg);

int resolve_threads(int threads);

}  // namespace p3s
