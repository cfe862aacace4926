// Frame-sequence driver (reference proj/src/sequence.cpp:13-145) around the GPU pipeline.
//
// Same contract: frames <pattern> from index 0 (or 1 when frame 0 is missing) up to the
// first gap, outputs <stem>_<format>.ppm, one CSV row per frame, SequenceError naming the
// failing frame with every earlier output already on disk. Unlike the reference's strictly
// serial loop, file read + PPM decode of frame i+1 and encode + write of frame i-1 run on
// host threads while frame i is on the GPU, so disk/codec time hides behind the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <exception>
#include <filesystem>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <thread>

#include "p3s_host.hpp"
#include "p3s_nvtx.hpp"

namespace p3s {

std::int64_t SequenceReport::pure_sum_ns() const {
    std::int64_t s = 0;
    for (const auto& f : frames) s += f.timings.pure_ns();
    return s;
}
std::int64_t SequenceReport::pure_min_ns() const {
    std::int64_t best = 0;
    for (std::size_t i = 0; i < frames.size(); ++i) {
        const std::int64_t v = frames[i].timings.pure_ns();
        if (i == 0 || v < best) best = v;
    }
    return best;
}
std::int64_t SequenceReport::pure_max_ns() const {
    std::int64_t best = 0;
    for (const auto& f : frames) best = std::max(best, f.timings.pure_ns());
    return best;
}
double SequenceReport::pure_mean_ns() const {
    return frames.empty() ? 0.0 : static_cast<double>(pure_sum_ns()) / frames.size();
}
std::string SequenceReport::to_csv(int threads) const {
    std::ostringstream os;
    os << "frame,width,height,threads,depth_ns,filter_ns,dibr_ns,inpaint_l_ns,inpaint_r_ns,"
          "format_ns,pure_ns\n";
    for (const auto& f : frames) {
        const StageTimings& t = f.timings;
        os << f.index << ',' << f.width << ',' << f.height << ',' << threads << ','
           << t.depth_gen_ns << ',' << t.filter_ns << ',' << t.dibr_ns << ',' << t.inpaint_left_ns
           << ',' << t.inpaint_right_ns << ',' << t.format_ns << ',' << t.pure_ns() << '\n';
    }
    return os.str();
}

// sequence.cpp:85-117
FramePattern FramePattern::parse(const std::string& pattern) {
    const std::size_t pct = pattern.find('%');
    if (pct == std::string::npos)
        throw std::invalid_argument("frame pattern needs one %d or %0Nd field: " + pattern);
    std::size_t pos = pct + 1;
    int pad = 0;
    while (pos < pattern.size() && pattern[pos] >= '0' && pattern[pos] <= '9')
        pad = pad * 10 + (pattern[pos++] - '0');
    if (pos >= pattern.size() || pattern[pos] != 'd')
        throw std::invalid_argument("frame pattern needs one %d or %0Nd field: " + pattern);
    if (pattern.find('%', pos) != std::string::npos)
        throw std::invalid_argument("frame pattern must contain exactly one % field: " + pattern);
    FramePattern fp;
    fp.prefix_ = pattern.substr(0, pct);
    fp.suffix_ = pattern.substr(pos + 1);
    fp.pad_ = pad;
    return fp;
}

std::string FramePattern::filename(std::int64_t index) const {
    std::string digits = std::to_string(index);
    if (static_cast<int>(digits.size()) < pad_) digits.insert(0, pad_ - digits.size(), '0');
    return prefix_ + digits + suffix_;
}

std::string FramePattern::stem(std::int64_t index) const {
    const std::string name = filename(index);
    const std::size_t dot = name.rfind('.');
    return dot == std::string::npos ? name : name.substr(0, dot);
}

int resolve_threads(int threads) {
    if (threads > 0) return threads;
    const unsigned hw = std::thread::hardware_concurrency();
    return hw > 0 ? static_cast<int>(hw) : 1;
}

namespace {

// Single-producer single-consumer bounded queue of tasks.
class Worker {
public:
    explicit Worker(std::size_t cap) : cap_(cap), th_([this] { loop(); }) {}
    ~Worker() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        th_.join();
    }
    void push(std::function<void()> f) {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return q_.size() < cap_ || err_; });
        q_.push_back(std::move(f));
        cv_.notify_all();
    }
    void drain() {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return q_.empty() && !busy_; });
    }
    // Drops the queued tasks (the running one finishes): an error path must not write
    // outputs after it has been raised.
    void cancel() {
        std::lock_guard<std::mutex> lk(mu_);
        q_.clear();
        cv_.notify_all();
    }
    std::exception_ptr error() {
        std::lock_guard<std::mutex> lk(mu_);
        return err_;
    }

private:
    void loop() {
        for (;;) {
            std::function<void()> f;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || !q_.empty(); });
                if (q_.empty()) return;
                f = std::move(q_.front());
                q_.pop_front();
                busy_ = true;
            }
            try {
                if (!err_) f();
            } catch (...) {
                std::lock_guard<std::mutex> lk(mu_);
                err_ = std::current_exception();
            }
            {
                std::lock_guard<std::mutex> lk(mu_);
                busy_ = false;
            }
            cv_.notify_all();
        }
    }
    std::size_t cap_;
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<std::function<void()>> q_;
    bool stop_ = false, busy_ = false;
    std::exception_ptr err_;
    std::thread th_;
};

struct Loaded {
    std::int64_t index = 0;
    bool present = false;
    std::vector<std::uint8_t> bytes;
    std::exception_ptr read_error;
};

}  // namespace

SequenceReport convert_sequence_dir(const std::string& in_dir, const std::string& pattern,
                                    const std::string& out_dir, const ConversionConfig& cfg,
                                    int threads) {
    (void)threads;
    cfg.validate();
    namespace fs = std::filesystem;
    const FramePattern in_pat = FramePattern::parse(pattern);
    const FramePattern out_pat = FramePattern::parse(pattern);
    SequenceReport report;
    const auto wall0 = std::chrono::steady_clock::now();

    std::int64_t next = 0;
    if (!fs::exists(fs::path(in_dir) / in_pat.filename(0)) &&
        fs::exists(fs::path(in_dir) / in_pat.filename(1)))
        next = 1;
    auto load = [&](std::int64_t idx) {
        Loaded l;
        l.index = idx;
        const fs::path path = fs::path(in_dir) / in_pat.filename(idx);
        if (!fs::exists(path)) return l;
        l.present = true;
        try {
            l.bytes = read_file(path.string());
        } catch (...) {
            l.read_error = std::current_exception();
        }
        return l;
    };

    // Frames go to the GPU as raw PPM payload (read interleaved by the fused kernels, or
    // de-interleaved on the device) and come back as ready-to-write interleaved payload
    // (written interleaved by DIBR + inpaint, or interleaved on the device): the host never
    // touches pixels. One plan per frame size (two alternating); file reads of frame i+1
    // and writes of frame i-1 run on host threads while frame i is on the device.
    Device& dev = Device::current();
    struct Plan {
        std::unique_ptr<Pipeline> pipe[2];
    };
    std::map<std::pair<int, int>, Plan> plans;
    // declared before the writer: its destructor runs (and drains queued writes) first
    std::int64_t written = 0;
    std::mutex written_mu;
    Worker writer(2);
    struct CancelOnError {
        Worker& w;
        int n = std::uncaught_exceptions();
        ~CancelOnError() {
            if (std::uncaught_exceptions() > n) w.cancel();
        }
    } cancel_on_error{writer};
    std::int64_t ordinal = 0;
    Loaded cur = load(next);
    while (cur.present) {
        // prefetch the next frame's bytes while this one converts
        Loaded nxt;
        std::thread pre([&] { nxt = load(cur.index + 1); });
        struct Join {
            std::thread& t;
            ~Join() {
                if (t.joinable()) t.join();
            }
        } join{pre};
        if (cur.read_error) {
            writer.drain();
            std::rethrow_exception(cur.read_error);
        }
        PpmView view{};
        try {
            view = ppm_view(cur.bytes.data(), cur.bytes.size());
        } catch (const PnmError& e) {
            writer.drain();
            if (auto err = writer.error()) std::rethrow_exception(err);
            std::lock_guard<std::mutex> lk(written_mu);
            throw SequenceError(cur.index, written,
                                "frame " + std::to_string(cur.index) + ": " + e.what());
        }
        if ((cfg.formats & kFormatHsbs) && view.width % 2 != 0) {
            writer.drain();
            throw std::invalid_argument("side_by_side: half mode requires an even width");
        }
        Plan& plan = plans[{view.width, view.height}];
        std::unique_ptr<Pipeline>& slot = plan.pipe[ordinal & 1];
        if (!slot) slot = std::make_unique<Pipeline>(view.width, view.height, cfg, dev);
        Pipeline& pipe = *slot;
        {
            NvtxRange nv("p3s_convert_sequence frame");
            pipe.run_interleaved(view.payload, true);
        }
        struct Out {
            StereoFormat fmt;
            Plane bytes;
        };
        auto outs = std::make_shared<std::vector<Out>>();
        for (StereoFormat f : {kFormatAnaglyph, kFormatHsbs, kFormatFsbs}) {
            if (!(cfg.formats & f)) continue;
            const int ow = f == kFormatFsbs ? 2 * view.width : view.width;
            const std::string head = ppm_header(ow, view.height);
            Out o{f, Plane(head.size() + 3 * static_cast<std::size_t>(ow) * view.height, false)};
            std::memcpy(o.bytes.data(), head.data(), head.size());
            pipe.download_interleaved(f, o.bytes.data() + head.size(), nullptr, false);
            outs->push_back(std::move(o));
        }
        report.frames.push_back({cur.index, view.width, view.height, pipe.last_timings()});
        {  // the outputs must be on the host before the writer sees them
            const cudaError_t e = cudaStreamSynchronize(static_cast<cudaStream_t>(pipe.stream()));
            if (e != cudaSuccess) throw DeviceError(std::string("CUDA error: ") + cudaGetErrorString(e));
        }
        ++ordinal;
        if (auto err = writer.error()) std::rethrow_exception(err);
        const std::int64_t idx = cur.index;
        writer.push([&, outs, idx] {
            for (const Out& o : *outs) {
                const std::string name = out_pat.stem(idx) + "_" + format_name(o.fmt) + ".ppm";
                write_file((fs::path(out_dir) / name).string(), o.bytes.data(), o.bytes.size());
                std::lock_guard<std::mutex> lk(written_mu);
                ++written;
            }
        });
        pre.join();
        cur = std::move(nxt);
    }
    writer.drain();
    if (auto err = writer.error()) std::rethrow_exception(err);
    report.wall_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(
                         std::chrono::steady_clock::now() - wall0)
                         .count();
    return report;
}

}  // namespace p3s
