// p3s/core.hpp — host-side value types and configuration of the B200 pseudo-stereo library.
//
// Mirrors the reference's C++ stage API types (reference include/pseudo3d/image.hpp:12-77,
// config.hpp:8-51) so code written against p3s:: reads the same, with one B200-first
// change: pixel planes are allocated from a pinned (page-locked) host pool, so every
// host<->device copy of an image is a direct DMA with no staging buffer.
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>

namespace p3s {

// ---- pinned host memory ---------------------------------------------------------------
// Size-bucketed cache of cudaHostAlloc blocks; falls back to ordinary aligned memory when
// no CUDA driver is present (host-only uses such as PNM decoding still work; GPU entry
// points then fail loudly instead of computing on the CPU).
void* pinned_alloc(std::size_t bytes);
void pinned_free(void* p) noexcept;
bool pinned_is_page_locked(const void* p);
// NUMA placement for multi-GPU hosts: the node of a CUDA device (-1 unknown), a fresh pinned
// block whose pages sit on that node (released with pinned_free), and binding the calling
// thread to the node's CPUs.
int device_numa_node(int device);
void* pinned_alloc_near(int device, std::size_t bytes);
bool bind_thread_to_device_node(int device);

// A byte array backed by the pinned pool (the reference uses std::vector<uint8_t>).
class Plane {
public:
    Plane() = default;
    explicit Plane(std::size_t n, bool zero = true);
    Plane(const Plane& o);
    Plane& operator=(const Plane& o);
    Plane(Plane&&) noexcept = default;
    Plane& operator=(Plane&&) noexcept = default;

    std::uint8_t* data() { return p_.get(); }
    const std::uint8_t* data() const { return p_.get(); }
    std::size_t size() const { return n_; }
    std::uint8_t& operator[](std::size_t i) { return p_.get()[i]; }
    std::uint8_t operator[](std::size_t i) const { return p_.get()[i]; }

private:
    struct Free {
        void operator()(std::uint8_t* p) const noexcept { pinned_free(p); }
    };
    std::unique_ptr<std::uint8_t, Free> p_;
    std::size_t n_ = 0;
};

std::size_t pixel_count(int w, int h);  // throws std::invalid_argument on w<1 || h<1

// Planar 8-bit RGB, row-major, index = y*width + x (reference image.hpp:12-35).
struct ImageRGB8 {
    int width = 0;
    int height = 0;
    Plane r, g, b;

    ImageRGB8() = default;
    ImageRGB8(int w, int h, bool zero = true)
        : width(w), height(h), r(pixel_count(w, h), zero), g(pixel_count(w, h), zero),
          b(pixel_count(w, h), zero) {}
    std::size_t size() const { return static_cast<std::size_t>(width) * height; }
    std::size_t index(int x, int y) const { return static_cast<std::size_t>(y) * width + x; }
    Plane& plane(int c) { return c == 0 ? r : (c == 1 ? g : b); }
    const Plane& plane(int c) const { return c == 0 ? r : (c == 1 ? g : b); }
};

// Single-channel 8-bit map (reference image.hpp:37-49).
struct GrayMap {
    int width = 0;
    int height = 0;
    Plane data;

    GrayMap() = default;
    GrayMap(int w, int h, bool zero = true) : width(w), height(h), data(pixel_count(w, h), zero) {}
    std::size_t size() const { return static_cast<std::size_t>(width) * height; }
    std::size_t index(int x, int y) const { return static_cast<std::size_t>(y) * width + x; }
    std::uint8_t at(int x, int y) const { return data[index(x, y)]; }
};

// Byte-per-pixel damage flags, 1 = damaged (reference image.hpp:51-77).
struct DamageMask {
    int width = 0;
    int height = 0;
    Plane damaged;

    DamageMask() = default;
    DamageMask(int w, int h, bool all_damaged = false);
    std::size_t size() const { return static_cast<std::size_t>(width) * height; }
    bool any_damaged() const;
    std::size_t damaged_count() const;
};

// ---- configuration (reference config.hpp:8-51, config.cpp:8-31) -----------------------
enum class DibrMode { kForwardZBuffer, kBackwardFallback };

enum StereoFormat : unsigned {
    kFormatAnaglyph = 1u << 0,
    kFormatHsbs = 1u << 1,
    kFormatFsbs = 1u << 2,
};

struct ConversionConfig {
    int base = kAutoBase;  // even >= 0, or kAutoBase: 2 * round(width / 256)
    int pop_threshold = 150;
    double sigma_spatial = 8.0;
    double sigma_range = 16.0;
    int depth_block = 16;
    int inpaint_block = 64;  // scheduling-only in the reference; accepted and validated
    double alpha = 0.7;
    double beta = 0.3;
    DibrMode dibr_mode = DibrMode::kForwardZBuffer;
    unsigned formats = kFormatAnaglyph;

    static constexpr int kAutoBase = -1;

    void validate() const;  // throws std::invalid_argument, reference messages
    int effective_base(int width) const;
};

const char* format_name(StereoFormat format);

// ---- error taxonomy (reference pnm.hpp, io.hpp, sequence.hpp) --------------------------
class PnmError : public std::runtime_error {
    using std::runtime_error::runtime_error;
};
class IoError : public std::runtime_error {
    using std::runtime_error::runtime_error;
};
class SequenceError : public std::runtime_error {
public:
    SequenceError(std::int64_t frame, std::int64_t written, const std::string& what)
        : std::runtime_error(what), frame_index_(frame), frames_written_(written) {}
    std::int64_t frame_index() const { return frame_index_; }
    std::int64_t frames_written() const { return frames_written_; }

private:
    std::int64_t frame_index_;
    std::int64_t frames_written_;
};
// CUDA failures (no device, OOM, launch errors) — mapped to P3S_ERR_INTERNAL.
class DeviceError : public std::runtime_error {
    using std::runtime_error::runtime_error;
};

}  // namespace p3s
