// Host-side PNM codec and whole-file I/O (reference proj/src/pnm.cpp, io.cpp): the
// on-disk formats around the GPU path, with the reference's rules and error messages.
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <limits>
#include <memory>
#include <string>
#include <vector>

#include "p3s/core.hpp"
#include "p3s_host.hpp"

namespace p3s {

namespace {

bool pnm_space(std::uint8_t c) {
    return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f';
}

// Header cursor: whitespace and '#'-to-end-of-line comments separate the fields.
struct Cursor {
    const std::uint8_t* p;
    std::size_t n;
    std::size_t at = 0;

    void skip() {
        while (at < n) {
            if (pnm_space(p[at])) {
                ++at;
            } else if (p[at] == '#') {
                while (at < n && p[at] != '\n') ++at;
            } else {
                return;
            }
        }
    }
    long number(const char* field) {
        skip();
        if (at >= n || p[at] < '0' || p[at] > '9')
            throw PnmError(std::string("missing or malformed ") + field + " in header");
        long v = 0;
        while (at < n && p[at] >= '0' && p[at] <= '9') {
            v = v * 10 + (p[at] - '0');
            if (v > 1000000000L) throw PnmError(std::string(field) + " out of supported range");
            ++at;
        }
        return v;
    }
};

struct Header {
    int w, h;
    const std::uint8_t* payload;
    std::size_t payload_size;
};

Header parse(const std::uint8_t* data, std::size_t size, char digit) {
    if (size < 2 || data[0] != 'P' || data[1] != digit)
        throw PnmError(std::string("not a binary P") + digit + " file");
    Cursor c{data, size, 2};
    const long w = c.number("width");
    const long h = c.number("height");
    const long maxval = c.number("maxval");
    if (w < 1 || h < 1) throw PnmError("image dimensions must be >= 1");
    if (maxval != 255)
        throw PnmError("unsupported maxval " + std::to_string(maxval) + " (only 255)");
    if (static_cast<unsigned long>(w) * static_cast<unsigned long>(h) >
        std::numeric_limits<std::size_t>::max() / 3)
        throw PnmError("image dimensions overflow");
    if (c.at >= size || !pnm_space(data[c.at]))
        throw PnmError("missing whitespace before pixel data");
    ++c.at;
    return Header{static_cast<int>(w), static_cast<int>(h), data + c.at, size - c.at};
}

void check_payload(std::size_t got, std::size_t expected) {
    if (got < expected)
        throw PnmError("pixel data truncated: expected " + std::to_string(expected) +
                       " bytes, got " + std::to_string(got));
    if (got > expected) throw PnmError("trailing bytes after pixel data");
}

std::string header_text(const char* magic, int w, int h) {
    return std::string(magic) + "\n" + std::to_string(w) + " " + std::to_string(h) + "\n255\n";
}

}  // namespace

PpmView ppm_view(const std::uint8_t* data, std::size_t size) {
    const Header hd = parse(data, size, '6');
    check_payload(hd.payload_size, 3 * static_cast<std::size_t>(hd.w) * hd.h);
    return PpmView{hd.w, hd.h, hd.payload};
}

std::string ppm_header(int w, int h) { return header_text("P6", w, h); }

ImageRGB8 decode_ppm(const std::uint8_t* data, std::size_t size) {
    const Header hd = parse(data, size, '6');
    const std::size_t n = static_cast<std::size_t>(hd.w) * hd.h;
    check_payload(hd.payload_size, 3 * n);
    ImageRGB8 img(hd.w, hd.h, false);
    deinterleave_rgb(hd.payload, n, img.r.data(), img.g.data(), img.b.data());
    return img;
}

std::vector<std::uint8_t> encode_ppm(const ImageRGB8& img) {
    const std::string head = header_text("P6", img.width, img.height);
    std::vector<std::uint8_t> out(head.size() + 3 * img.size());
    std::memcpy(out.data(), head.data(), head.size());
    interleave_rgb(img.r.data(), img.g.data(), img.b.data(), img.size(), out.data() + head.size());
    return out;
}

GrayMap decode_pgm(const std::uint8_t* data, std::size_t size) {
    const Header hd = parse(data, size, '5');
    const std::size_t n = static_cast<std::size_t>(hd.w) * hd.h;
    check_payload(hd.payload_size, n);
    GrayMap m(hd.w, hd.h, false);
    std::memcpy(m.data.data(), hd.payload, n);
    return m;
}

std::vector<std::uint8_t> encode_pgm(const GrayMap& map) {
    const std::string head = header_text("P5", map.width, map.height);
    std::vector<std::uint8_t> out(head.size() + map.size());
    std::memcpy(out.data(), head.data(), head.size());
    std::memcpy(out.data() + head.size(), map.data.data(), map.size());
    return out;
}

void deinterleave_rgb(const std::uint8_t* src, std::size_t n, std::uint8_t* r, std::uint8_t* g,
                      std::uint8_t* b) {
    for (std::size_t i = 0; i < n; ++i) {
        r[i] = src[3 * i];
        g[i] = src[3 * i + 1];
        b[i] = src[3 * i + 2];
    }
}

void interleave_rgb(const std::uint8_t* r, const std::uint8_t* g, const std::uint8_t* b,
                    std::size_t n, std::uint8_t* dst) {
    for (std::size_t i = 0; i < n; ++i) {
        dst[3 * i] = r[i];
        dst[3 * i + 1] = g[i];
        dst[3 * i + 2] = b[i];
    }
}

std::vector<std::uint8_t> read_file(const std::string& path) {
    std::unique_ptr<std::FILE, int (*)(std::FILE*)> f(std::fopen(path.c_str(), "rb"), &std::fclose);
    if (!f) throw IoError("cannot open for reading: " + path);
    std::vector<std::uint8_t> bytes;
    std::uint8_t chunk[1 << 16];
    std::size_t got;
    while ((got = std::fread(chunk, 1, sizeof(chunk), f.get())) > 0)
        bytes.insert(bytes.end(), chunk, chunk + got);
    if (std::ferror(f.get())) throw IoError("read failed: " + path);
    return bytes;
}

void write_file(const std::string& path, const std::uint8_t* data, std::size_t size) {
    std::unique_ptr<std::FILE, int (*)(std::FILE*)> f(std::fopen(path.c_str(), "wb"), &std::fclose);
    if (!f) throw IoError("cannot open for writing: " + path);
    if (size && std::fwrite(data, 1, size, f.get()) != size) throw IoError("write failed: " + path);
    if (std::fflush(f.get()) != 0) throw IoError("write failed: " + path);
}

}  // namespace p3s
