// Host value types, configuration validation and the pinned host-memory pool.
#include <cuda_runtime.h>
#include <pthread.h>
#include <sched.h>

#include <atomic>
#include <cctype>
#include <fstream>
#include <sstream>
#include <string>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <unordered_map>

#include "p3s/core.hpp"

namespace p3s {

// ---- pinned pool ------------------------------------------------------------------------
namespace {

struct Block {
    std::size_t bytes;
    bool pinned;
};

class PinnedPool {
public:
    void* alloc(std::size_t n) {
        const std::size_t bytes = round(n);
        {
            std::lock_guard<std::mutex> lk(mu_);
            auto it = free_.find(bytes);
            if (it != free_.end()) {
                void* p = it->second;
                free_.erase(it);
                cached_ -= bytes;
                return p;
            }
        }
        void* p = nullptr;
        bool pinned = false;
        if (cuda_usable()) {
            if (cudaHostAlloc(&p, bytes, cudaHostAllocPortable) == cudaSuccess) {
                pinned = true;
            } else {
                cudaGetLastError();
                p = nullptr;
            }
        }
        if (!p) {
            p = std::aligned_alloc(4096, bytes);
            if (!p) throw std::bad_alloc();
        }
        std::lock_guard<std::mutex> lk(mu_);
        live_[p] = Block{bytes, pinned};
        return p;
    }

    // a new allocation (never a cached block: the caller wants pages placed now)
    void* alloc_fresh(std::size_t n) {
        const std::size_t bytes = round(n);
        void* p = nullptr;
        bool pinned = false;
        if (cuda_usable() && cudaHostAlloc(&p, bytes, cudaHostAllocPortable) == cudaSuccess) {
            pinned = true;
        } else {
            cudaGetLastError();
            p = std::aligned_alloc(4096, bytes);
            if (!p) throw std::bad_alloc();
        }
        std::lock_guard<std::mutex> lk(mu_);
        live_[p] = Block{bytes, pinned};
        return p;
    }

    void release(void* p) noexcept {
        if (!p) return;
        std::lock_guard<std::mutex> lk(mu_);
        auto it = live_.find(p);
        if (it == live_.end()) return;
        const Block b = it->second;
        if (cached_ + b.bytes <= kMaxCached) {
            free_.emplace(b.bytes, p);
            cached_ += b.bytes;
            return;
        }
        live_.erase(it);
        if (b.pinned)
            cudaFreeHost(p);
        else
            std::free(p);
    }

    bool pinned(const void* p) {
        std::lock_guard<std::mutex> lk(mu_);
        auto it = live_.find(const_cast<void*>(p));
        return it != live_.end() && it->second.pinned;
    }

private:
    static constexpr std::size_t kMaxCached = std::size_t(4) << 30;
    static std::size_t round(std::size_t n) {
        if (n == 0) n = 1;
        const std::size_t g = n <= (std::size_t(1) << 20) ? 4096 : (std::size_t(1) << 20);
        return (n + g - 1) / g * g;
    }
    static bool cuda_usable() {
        static const bool ok = [] {
            int n = 0;
            const bool good = cudaGetDeviceCount(&n) == cudaSuccess && n > 0;
            if (!good) cudaGetLastError();
            return good;
        }();
        return ok;
    }

    std::mutex mu_;
    std::multimap<std::size_t, void*> free_;
    std::unordered_map<void*, Block> live_;
    std::size_t cached_ = 0;
};

PinnedPool& pool() {
    static PinnedPool* p = new PinnedPool();  // intentionally leaked: outlives static dtors
    return *p;
}

}  // namespace

void* pinned_alloc(std::size_t bytes) { return pool().alloc(bytes); }

// NUMA node of a CUDA device (sysfs numa_node of its PCI function; -1 when unknown).
int device_numa_node(int device) {
    char bus[64] = {0};
    if (cudaDeviceGetPCIBusId(bus, sizeof(bus), device) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    std::string id(bus);
    for (auto& c : id) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
    std::ifstream f("/sys/bus/pci/devices/" + id + "/numa_node");
    int node = -1;
    if (!(f >> node)) return -1;
    return node;
}

namespace {
// CPUs of a NUMA node from sysfs ("0-55,112-167").
bool node_cpus(int node, cpu_set_t& set) {
    std::ifstream f("/sys/devices/system/node/node" + std::to_string(node) + "/cpulist");
    std::string list;
    if (node < 0 || !std::getline(f, list)) return false;
    CPU_ZERO(&set);
    std::stringstream ss(list);
    std::string part;
    int n = 0;
    while (std::getline(ss, part, ',')) {
        const auto dash = part.find('-');
        const int a = std::atoi(part.c_str());
        const int b = dash == std::string::npos ? a : std::atoi(part.c_str() + dash + 1);
        for (int c = a; c <= b && c < CPU_SETSIZE; ++c) {
            CPU_SET(c, &set);
            ++n;
        }
    }
    return n > 0;
}
}  // namespace

// Runs f with the calling thread bound to the CPUs of `device`'s NUMA node (first-touch and
// cudaHostAlloc pages then come from that node), restoring the affinity afterwards.
template <class F>
static void on_device_node(int device, F&& f) {
    cpu_set_t old, want;
    const bool saved = pthread_getaffinity_np(pthread_self(), sizeof(old), &old) == 0;
    const bool bind = saved && node_cpus(device_numa_node(device), want) &&
                      pthread_setaffinity_np(pthread_self(), sizeof(want), &want) == 0;
    try {
        f();
    } catch (...) {
        if (bind) pthread_setaffinity_np(pthread_self(), sizeof(old), &old);
        throw;
    }
    if (bind) pthread_setaffinity_np(pthread_self(), sizeof(old), &old);
}

void* pinned_alloc_near(int device, std::size_t bytes) {
    void* p = nullptr;
    on_device_node(device, [&] {
        p = pool().alloc_fresh(bytes);
        std::memset(p, 0, bytes);  // fault the pages in while bound to the node
    });
    return p;
}

bool bind_thread_to_device_node(int device) {
    cpu_set_t want;
    return node_cpus(device_numa_node(device), want) &&
           pthread_setaffinity_np(pthread_self(), sizeof(want), &want) == 0;
}
void pinned_free(void* p) noexcept { pool().release(p); }
bool pinned_is_page_locked(const void* p) { return pool().pinned(p); }

Plane::Plane(std::size_t n, bool zero) : n_(n) {
    p_.reset(static_cast<std::uint8_t*>(pinned_alloc(n)));
    if (zero) std::memset(p_.get(), 0, n);
}

Plane::Plane(const Plane& o) : n_(o.n_) {
    if (o.p_) {
        p_.reset(static_cast<std::uint8_t*>(pinned_alloc(n_)));
        std::memcpy(p_.get(), o.p_.get(), n_);
    }
}

Plane& Plane::operator=(const Plane& o) {
    if (this != &o) {
        Plane t(o);
        *this = std::move(t);
    }
    return *this;
}

std::size_t pixel_count(int w, int h) {
    if (w < 1 || h < 1) throw std::invalid_argument("image dimensions must be >= 1");
    return static_cast<std::size_t>(w) * h;
}

DamageMask::DamageMask(int w, int h, bool all_damaged)
    : width(w), height(h), damaged(pixel_count(w, h), false) {
    std::memset(damaged.data(), all_damaged ? 1 : 0, damaged.size());
}

bool DamageMask::any_damaged() const {
    const std::uint8_t* p = damaged.data();
    for (std::size_t i = 0; i < size(); ++i)
        if (p[i]) return true;
    return false;
}

std::size_t DamageMask::damaged_count() const {
    std::size_t n = 0;
    const std::uint8_t* p = damaged.data();
    for (std::size_t i = 0; i < size(); ++i) n += p[i] != 0;
    return n;
}

// ---- configuration: reference config.cpp:8-31 (same bounds, order and messages) --------
void ConversionConfig::validate() const {
    if (base != kAutoBase) {
        if (base < 0) throw std::invalid_argument("base must be >= 0");
        if (base % 2 != 0) throw std::invalid_argument("base must be even");
    }
    if (pop_threshold < 0 || pop_threshold > 255)
        throw std::invalid_argument("pop_threshold must be in [0,255]");
    if (!(sigma_spatial > 0.0)) throw std::invalid_argument("sigma_spatial must be > 0");
    if (!(sigma_range > 0.0)) throw std::invalid_argument("sigma_range must be > 0");
    if (depth_block < 4) throw std::invalid_argument("depth_block must be >= 4");
    if (inpaint_block < 4) throw std::invalid_argument("inpaint_block must be >= 4");
    if (alpha < 0.0 || alpha > 1.0) throw std::invalid_argument("alpha must be in [0,1]");
    if (beta < 0.0 || beta > 1.0) throw std::invalid_argument("beta must be in [0,1]");
    if (alpha + beta > 1.0) throw std::invalid_argument("alpha + beta must be <= 1");
    if (formats == 0) throw std::invalid_argument("at least one output format is required");
    if ((formats & ~(kFormatAnaglyph | kFormatHsbs | kFormatFsbs)) != 0)
        throw std::invalid_argument("unknown output format bit");
}

int ConversionConfig::effective_base(int width) const {
    if (base != kAutoBase) return base;
    return 2 * static_cast<int>(std::floor(width / 256.0 + 0.5));
}

const char* format_name(StereoFormat format) {
    switch (format) {
        case kFormatAnaglyph: return "anaglyph";
        case kFormatHsbs: return "hsbs";
        case kFormatFsbs: return "fsbs";
    }
    return "unknown";
}

}  // namespace p3s
