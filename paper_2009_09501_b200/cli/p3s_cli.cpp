// p3s — command-line front end over the C ABI (include/pseudo3d.h), as specified by the
// reference's SPEC.md "[MODULE] cli" (the reference ships no CLI).
//
//   p3s convert <in.ppm> --out <dir> [--format anaglyph|hsbs|fsbs]... [--emit-depth]
//   p3s depth   <in.ppm> --out <file.pgm>
//   p3s video   --in <dir> --pattern 'frame_%06d.ppm' --out <dir> [--timing-csv <file>]
//   p3s bench   --sizes 1920x1080,3840x2160 --threads 1,4,8 --reps 5 --csv <file|-> [--seed S]
//
// Shared flags: --base, --pop-threshold, --sigma-spatial, --sigma-range, --depth-block,
// --inpaint-block, --mode forward|backward, --threads (accepted; the GPU path ignores it).
// Exit codes: 0 success, 1 usage / invalid argument, 2 I/O error, 3 decode error
// (p3s_status values), 4 internal (GPU) error. Diagnostics go to stderr; data to files or
// stdout. The CLI is a thin mapping: every operation is one C-ABI call.
#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "pseudo3d.h"

namespace {

constexpr int kUsage = 1, kIo = 2, kInternal = 4;

const char* kHelp =
    "usage: p3s <convert|depth|video|bench> [options]\n"
    "  convert <in.ppm> --out <dir> [--format anaglyph|hsbs|fsbs]... [--emit-depth]\n"
    "  depth <in.ppm> --out <file.pgm>\n"
    "  video --in <dir> --pattern 'frame_%06d.ppm' --out <dir> [--timing-csv <file>]\n"
    "  bench --sizes WxH[,WxH...] --threads N[,N...] --reps N --csv <file|-> [--seed S]\n"
    "shared: --base N --pop-threshold N --sigma-spatial X --sigma-range X --depth-block N\n"
    "        --inpaint-block N --mode forward|backward --threads N\n";

struct UsageError {
    std::string msg;
};

// exit code for a failed C-ABI call, with the library's message on stderr
int fail(p3s_status st, const char* what) {
    std::fprintf(stderr, "p3s: %s: %s\n", what, p3s_last_error());
    return st == P3S_ERR_INTERNAL ? kInternal : static_cast<int>(st);
}

long parse_int(const std::string& flag, const char* v) {
    char* end = nullptr;
    errno = 0;
    const long x = std::strtol(v, &end, 10);
    if (errno || end == v || *end) throw UsageError{flag + " expects an integer, got '" + v + "'"};
    return x;
}

double parse_double(const std::string& flag, const char* v) {
    char* end = nullptr;
    errno = 0;
    const double x = std::strtod(v, &end);
    if (errno || end == v || *end) throw UsageError{flag + " expects a number, got '" + v + "'"};
    return x;
}

std::vector<std::string> split(const std::string& s, char sep) {
    std::vector<std::string> out;
    std::size_t a = 0;
    for (;;) {
        const std::size_t b = s.find(sep, a);
        out.push_back(s.substr(a, b == std::string::npos ? std::string::npos : b - a));
        if (b == std::string::npos) return out;
        a = b + 1;
    }
}

struct Options {
    std::vector<std::string> positional;
    std::string out, in, pattern, timing_csv, csv = "-", sizes = "1920x1080", threads_list = "1";
    unsigned formats = 0;
    bool emit_depth = false;
    int reps = 5;
    unsigned long long seed = 1;
    // config overrides (applied in order through the C ABI setters, which validate)
    bool has_base = false, has_pop = false, has_ss = false, has_sr = false, has_db = false,
         has_ib = false, has_mode = false, has_threads = false;
    int base = 0, pop = 0, depth_block = 0, inpaint_block = 0, threads = 0;
    double sigma_s = 0, sigma_r = 0;
    p3s_dibr_mode mode = P3S_MODE_FORWARD_ZBUFFER;
};

Options parse(int argc, char** argv, int first) {
    Options o;
    for (int i = first; i < argc; ++i) {
        const std::string a = argv[i];
        if (a.rfind("--", 0) != 0) {
            o.positional.push_back(a);
            continue;
        }
        auto value = [&]() -> const char* {
            if (i + 1 >= argc) throw UsageError{a + " needs a value"};
            return argv[++i];
        };
        if (a == "--out") o.out = value();
        else if (a == "--in") o.in = value();
        else if (a == "--pattern") o.pattern = value();
        else if (a == "--timing-csv") o.timing_csv = value();
        else if (a == "--csv") o.csv = value();
        else if (a == "--sizes") o.sizes = value();
        else if (a == "--reps") o.reps = static_cast<int>(parse_int(a, value()));
        else if (a == "--seed") o.seed = static_cast<unsigned long long>(parse_int(a, value()));
        else if (a == "--emit-depth") o.emit_depth = true;
        else if (a == "--format") {
            const std::string f = value();
            if (f == "anaglyph") o.formats |= P3S_FORMAT_ANAGLYPH;
            else if (f == "hsbs") o.formats |= P3S_FORMAT_HSBS;
            else if (f == "fsbs") o.formats |= P3S_FORMAT_FSBS;
            else throw UsageError{"unknown format '" + f + "'"};
        } else if (a == "--base") { o.has_base = true; o.base = static_cast<int>(parse_int(a, value())); }
        else if (a == "--pop-threshold") { o.has_pop = true; o.pop = static_cast<int>(parse_int(a, value())); }
        else if (a == "--sigma-spatial") { o.has_ss = true; o.sigma_s = parse_double(a, value()); }
        else if (a == "--sigma-range") { o.has_sr = true; o.sigma_r = parse_double(a, value()); }
        else if (a == "--depth-block") { o.has_db = true; o.depth_block = static_cast<int>(parse_int(a, value())); }
        else if (a == "--inpaint-block") { o.has_ib = true; o.inpaint_block = static_cast<int>(parse_int(a, value())); }
        else if (a == "--mode") {
            const std::string m = value();
            o.has_mode = true;
            if (m == "forward") o.mode = P3S_MODE_FORWARD_ZBUFFER;
            else if (m == "backward") o.mode = P3S_MODE_BACKWARD_FALLBACK;
            else throw UsageError{"--mode expects forward or backward"};
        } else if (a == "--threads") {
            o.has_threads = true;
            o.threads_list = value();
            o.threads = static_cast<int>(parse_int(a, split(o.threads_list, ',')[0].c_str()));
        } else {
            throw UsageError{"unknown flag " + a};
        }
    }
    return o;
}

struct Config {
    p3s_config* c = p3s_config_create();
    ~Config() { p3s_config_free(c); }
};

// Applies the shared flags; returns 0 or the exit code of the rejected setter.
int configure(const Options& o, p3s_config* c, unsigned default_formats) {
    struct Step {
        bool on;
        p3s_status st;
        const char* what;
    };
    const Step steps[] = {
        {o.has_base, o.has_base ? p3s_config_set_base(c, o.base) : P3S_OK, "--base"},
        {o.has_pop, o.has_pop ? p3s_config_set_pop_threshold(c, o.pop) : P3S_OK, "--pop-threshold"},
        {o.has_ss, o.has_ss ? p3s_config_set_sigma_spatial(c, o.sigma_s) : P3S_OK, "--sigma-spatial"},
        {o.has_sr, o.has_sr ? p3s_config_set_sigma_range(c, o.sigma_r) : P3S_OK, "--sigma-range"},
        {o.has_db, o.has_db ? p3s_config_set_depth_block(c, o.depth_block) : P3S_OK, "--depth-block"},
        {o.has_ib, o.has_ib ? p3s_config_set_inpaint_block(c, o.inpaint_block) : P3S_OK, "--inpaint-block"},
        {o.has_mode, o.has_mode ? p3s_config_set_mode(c, o.mode) : P3S_OK, "--mode"},
        {o.has_threads, o.has_threads ? p3s_config_set_threads(c, o.threads) : P3S_OK, "--threads"},
    };
    for (const Step& s : steps)
        if (s.on && s.st != P3S_OK) return fail(s.st, s.what);
    const unsigned f = o.formats ? o.formats : default_formats;
    const p3s_status st = p3s_config_set_formats(c, f);
    return st == P3S_OK ? 0 : fail(st, "--format");
}

std::string stem_of(const std::string& path) {
    const std::size_t slash = path.find_last_of('/');
    std::string name = slash == std::string::npos ? path : path.substr(slash + 1);
    const std::size_t dot = name.find_last_of('.');
    return dot == std::string::npos || dot == 0 ? name : name.substr(0, dot);
}

int write_buffer(const std::string& path, const p3s_buffer* buf) {
    if (path == "-") {
        std::fwrite(p3s_buffer_data(buf), 1, p3s_buffer_size(buf), stdout);
        return 0;
    }
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) {
        std::fprintf(stderr, "p3s: cannot write %s: %s\n", path.c_str(), std::strerror(errno));
        return kIo;
    }
    const std::size_t n = std::fwrite(p3s_buffer_data(buf), 1, p3s_buffer_size(buf), f);
    const bool ok = n == p3s_buffer_size(buf) && std::fclose(f) == 0;
    if (!ok) {
        std::fprintf(stderr, "p3s: short write to %s\n", path.c_str());
        return kIo;
    }
    return 0;
}

int cmd_convert(const Options& o) {
    if (o.positional.size() != 1) throw UsageError{"convert needs exactly one input file"};
    if (o.out.empty()) throw UsageError{"convert needs --out <dir>"};
    Config cfg;
    if (const int rc = configure(o, cfg.c, P3S_FORMAT_ANAGLYPH)) return rc;
    p3s_image* img = nullptr;
    p3s_status st = p3s_image_load_ppm(o.positional[0].c_str(), &img);
    if (st != P3S_OK) return fail(st, o.positional[0].c_str());
    p3s_result* res = nullptr;
    st = p3s_convert(img, cfg.c, &res);
    p3s_image_free(img);
    if (st != P3S_OK) return fail(st, "convert");
    const std::string stem = o.out + "/" + stem_of(o.positional[0]);
    int rc = 0;
    const struct {
        p3s_format f;
        const char* name;
    } outs[] = {{P3S_FORMAT_ANAGLYPH, "anaglyph"}, {P3S_FORMAT_HSBS, "hsbs"}, {P3S_FORMAT_FSBS, "fsbs"}};
    const unsigned want = o.formats ? o.formats : static_cast<unsigned>(P3S_FORMAT_ANAGLYPH);
    for (const auto& e : outs) {
        if (!(want & e.f) || rc) continue;
        const p3s_image* out = nullptr;
        st = p3s_result_output(res, e.f, &out);
        if (st == P3S_OK) st = p3s_image_save_ppm((stem + "_" + e.name + ".ppm").c_str(), out);
        if (st != P3S_OK) rc = fail(st, e.name);
    }
    if (!rc && o.emit_depth) {
        const p3s_graymap* d = p3s_result_depth(res);
        st = d ? p3s_graymap_save_pgm((stem + "_depth.pgm").c_str(), d) : static_cast<p3s_status>(P3S_ERR_INTERNAL);
        if (st != P3S_OK) rc = fail(st, "depth");
    }
    p3s_result_free(res);
    return rc;
}

int cmd_depth(const Options& o) {
    if (o.positional.size() != 1) throw UsageError{"depth needs exactly one input file"};
    if (o.out.empty()) throw UsageError{"depth needs --out <file.pgm>"};
    Config cfg;
    if (const int rc = configure(o, cfg.c, P3S_FORMAT_ANAGLYPH)) return rc;
    p3s_image* img = nullptr;
    p3s_status st = p3s_image_load_ppm(o.positional[0].c_str(), &img);
    if (st != P3S_OK) return fail(st, o.positional[0].c_str());
    p3s_graymap* map = nullptr;
    st = p3s_depth_map(img, cfg.c, &map);
    p3s_image_free(img);
    if (st != P3S_OK) return fail(st, "depth");
    st = p3s_graymap_save_pgm(o.out.c_str(), map);
    p3s_graymap_free(map);
    return st == P3S_OK ? 0 : fail(st, o.out.c_str());
}

int cmd_video(const Options& o) {
    if (!o.positional.empty()) throw UsageError{"video takes no positional arguments"};
    if (o.in.empty() || o.pattern.empty() || o.out.empty())
        throw UsageError{"video needs --in <dir> --pattern <fmt> --out <dir>"};
    Config cfg;
    if (const int rc = configure(o, cfg.c, P3S_FORMAT_ANAGLYPH)) return rc;
    p3s_sequence_summary sum{};
    p3s_buffer* csv = nullptr;
    const p3s_status st = p3s_convert_sequence(o.in.c_str(), o.pattern.c_str(), o.out.c_str(), cfg.c,
                                               &sum, o.timing_csv.empty() ? nullptr : &csv);
    if (st != P3S_OK) return fail(st, "video");
    std::printf("frames=%lld pure_sum_ns=%lld pure_min_ns=%lld pure_max_ns=%lld pure_mean_ns=%.1f wall_ns=%lld\n",
                static_cast<long long>(sum.frames), static_cast<long long>(sum.pure_sum_ns),
                static_cast<long long>(sum.pure_min_ns), static_cast<long long>(sum.pure_max_ns),
                sum.pure_mean_ns, static_cast<long long>(sum.wall_ns));
    int rc = 0;
    if (csv) {
        rc = write_buffer(o.timing_csv, csv);
        p3s_buffer_free(csv);
    }
    return rc;
}

int cmd_bench(const Options& o) {
    if (!o.positional.empty()) throw UsageError{"bench takes no positional arguments"};
    std::vector<int> ws, hs, ts;
    for (const std::string& s : split(o.sizes, ',')) {
        const std::vector<std::string> wh = split(s, 'x');
        if (wh.size() != 2) throw UsageError{"--sizes expects WxH[,WxH...], got '" + s + "'"};
        ws.push_back(static_cast<int>(parse_int("--sizes", wh[0].c_str())));
        hs.push_back(static_cast<int>(parse_int("--sizes", wh[1].c_str())));
    }
    for (const std::string& t : split(o.threads_list, ','))
        ts.push_back(static_cast<int>(parse_int("--threads", t.c_str())));
    if (o.reps < 1) throw UsageError{"--reps must be >= 1"};
    Options shared = o;
    shared.has_threads = false;  // thread counts are the bench's CSV labels
    Config cfg;
    if (const int rc = configure(shared, cfg.c, P3S_FORMAT_ANAGLYPH)) return rc;
    p3s_bench_report* rep = nullptr;
    p3s_status st = p3s_bench(ws.data(), hs.data(), ws.size(), ts.data(), ts.size(), o.reps,
                              static_cast<uint64_t>(o.seed), cfg.c, &rep);
    if (st != P3S_OK) return fail(st, "bench");
    p3s_buffer* csv = nullptr;
    st = p3s_bench_report_csv(rep, &csv);
    p3s_bench_report_free(rep);
    if (st != P3S_OK) return fail(st, "bench csv");
    const int rc = write_buffer(o.csv, csv);
    p3s_buffer_free(csv);
    return rc;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2 || !std::strcmp(argv[1], "--help") || !std::strcmp(argv[1], "-h")) {
        std::fputs(kHelp, argc < 2 ? stderr : stdout);
        return argc < 2 ? kUsage : 0;
    }
    const std::string cmd = argv[1];
    try {
        const Options o = parse(argc, argv, 2);
        if (cmd == "convert") return cmd_convert(o);
        if (cmd == "depth") return cmd_depth(o);
        if (cmd == "video") return cmd_video(o);
        if (cmd == "bench") return cmd_bench(o);
        throw UsageError{"unknown subcommand '" + cmd + "'"};
    } catch (const UsageError& e) {
        std::fprintf(stderr, "p3s: %s\n%s", e.msg.c_str(), kHelp);
        return kUsage;
    }
}
