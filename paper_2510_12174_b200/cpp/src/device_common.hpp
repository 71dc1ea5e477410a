// msplat C++ drop-in: shared device-side helpers (internal).  The context,
// device buffers and the AoS/HWC <-> SoA/planar marshalling used by the render
// path (device_path.cpp) and the trainer (trainer_path.cpp).
#pragma once

#include <cuda_runtime.h>
#include <malloc.h>

#include <limits>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <unordered_map>
#include <vector>

#include "msplat/normals.hpp"
#include "msplat/rasterizer.hpp"
#include "msplat/scene.hpp"
#include "msplat_b200.h"
#include "parallel.hpp"

namespace msplat {
namespace dropin {

inline void rethrow(msplat_status st) {
    if (st == MSPLAT_OK) return;
    const std::string m = msplat_last_error();
    if (st == MSPLAT_ERR_INVALID_ARGUMENT) throw std::invalid_argument(m);
    if (st == MSPLAT_ERR_LOGIC) throw std::logic_error(m);
    throw std::runtime_error(m);
}

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

// MSPLAT_DROPIN_PROFILE=1: wall-clock of the marshalling phases on stderr.
struct PhaseTimer {
    bool on;
    std::chrono::steady_clock::time_point t;
    const char* fn;
    explicit PhaseTimer(const char* f) : fn(f) {
        const char* e = std::getenv("MSPLAT_DROPIN_PROFILE");
        on = e && e[0] == '1';
        t = std::chrono::steady_clock::now();
    }
    void mark(const char* what) {
        if (!on) return;
        cudaDeviceSynchronize();
        const auto n = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[dropin] %s %-24s %8.2f ms\n", fn, what,
                     std::chrono::duration<double, std::milli>(n - t).count());
        t = n;
    }
    ~PhaseTimer() { mark("teardown"); }  // the locals' destructors (device frees) run before this one
};

inline bool use_fp32() {
    const char* p = std::getenv("MSPLAT_PRECISION");
    return p && std::string(p) == "32";
}

// Host allocation reuse.  The reference API hands frames, gradients and the
// ReplayState's host fields back as fresh std::vectors (~1.5 GB per fwd+bwd
// call pair at cfg3); glibc serves blocks that large with fresh mmap'd pages,
// and their first-touch faults dominated the marshalling (FP64 call pair
// 1.2 s -> 0.4 s with reuse).  Large blocks are therefore kept on the heap and
// reused (mallopt M_MMAP_MAX = 0, no trimming).  Process-wide:
// MSPLAT_DROPIN_HOST_REUSE=0 keeps glibc's defaults.
inline void tune_host_allocator() {
    static const bool done = [] {
        const char* e = std::getenv("MSPLAT_DROPIN_HOST_REUSE");
        if (e && e[0] == '0') return false;
        mallopt(M_MMAP_MAX, 0);
        mallopt(M_TRIM_THRESHOLD, std::numeric_limits<int>::max());
        mallopt(M_TOP_PAD, 64 << 20);
        return true;
    }();
    (void)done;
}

inline msplat_context* context() {
    thread_local std::unique_ptr<msplat_context, void (*)(msplat_context*)> ctx(nullptr, msplat_context_destroy);
    if (!ctx) {
        tune_host_allocator();
        const char* d = std::getenv("MSPLAT_DEVICE");
        msplat_context* c = nullptr;
        rethrow(msplat_context_create(d ? std::atoi(d) : 0, nullptr, &c));
        // The reference's accumulation is reproducible at a fixed thread count
        // (tests/test_rasterizer.cpp:386-419): fixed-order reduction, no atomics.
        // MSPLAT_DETERMINISTIC=0 selects the (faster) atomic accumulation.
        const char* det = std::getenv("MSPLAT_DETERMINISTIC");
        rethrow(msplat_context_set_deterministic(c, (det && std::string(det) == "0") ? 0 : 1));
        ctx.reset(c);
    }
    return ctx.get();
}

// Pinned host staging (per thread, grown on demand): transfers at full link
// speed, filled / read by parallel loops in the kernel precision.
inline void* pinned_staging(size_t bytes, int slot = 0) {
    struct Pin {
        void* p = nullptr;
        size_t bytes = 0;
        ~Pin() {
            if (p) cudaFreeHost(p);
        }
    };
    thread_local Pin pins[2];
    Pin& s = pins[slot & 1];
    if (bytes > s.bytes) {
        if (s.p) cudaFreeHost(s.p);
        s.p = nullptr;
        s.bytes = 0;
        cuda_check(cudaHostAlloc(&s.p, bytes, cudaHostAllocDefault), "cudaHostAlloc");
        s.bytes = bytes;
    }
    return s.p;
}

// Device buffer holding host doubles converted to the kernel precision.
// Device block reuse.  Every reference-API call allocates its device arrays
// afresh (the same sizes call after call); cudaFree of GB-sized blocks
// measured 3-550 ms per call on the B200 box, so freed blocks are kept, keyed
// by their size rounded to 2 MiB, and handed to the next request of that size.
// Reuse is safe because every eager msplat_* call synchronizes its stream
// before returning and the drop-in's copies are synchronous.  Capped at
// MSPLAT_DROPIN_DEVICE_CACHE_MB (default 16384; 0 disables); dropped entirely
// when a cudaMalloc fails.
class DeviceBlockCache {
  public:
    static DeviceBlockCache& get() {
        static DeviceBlockCache c;
        return c;
    }
    static size_t rounded(size_t bytes) { return (std::max<size_t>(bytes, 1) + kGrain - 1) / kGrain * kGrain; }
    void* take(size_t bytes) {
        {
            std::lock_guard<std::mutex> lk(mu_);
            auto it = free_.find(bytes);
            if (it != free_.end()) {
                void* p = it->second;
                free_.erase(it);
                held_ -= bytes;
                return p;
            }
        }
        void* p = nullptr;
        if (cudaMalloc(&p, bytes) != cudaSuccess) {
            (void)cudaGetLastError();
            release_all();
            cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
        }
        return p;
    }
    void give(void* p, size_t bytes) {
        {
            std::lock_guard<std::mutex> lk(mu_);
            if (held_ + bytes <= cap_) {
                free_.emplace(bytes, p);
                held_ += bytes;
                return;
            }
        }
        cudaFree(p);
    }
    void release_all() {
        std::lock_guard<std::mutex> lk(mu_);
        for (auto& kv : free_) cudaFree(kv.second);
        free_.clear();
        held_ = 0;
    }

  private:
    static constexpr size_t kGrain = size_t(2) << 20;
    DeviceBlockCache() {
        const char* e = std::getenv("MSPLAT_DROPIN_DEVICE_CACHE_MB");
        cap_ = size_t(e ? std::atoll(e) : 16384) << 20;
    }
    ~DeviceBlockCache() = default;  // process exit: the driver reclaims the blocks
    std::mutex mu_;
    std::unordered_multimap<size_t, void*> free_;
    size_t held_ = 0, cap_ = 0;
};

struct DBuf {
    void* p = nullptr;
    size_t n = 0;
    bool f32 = false;
    size_t block = 0;  // bytes of the (cached) device block
    DBuf() = default;
    // zero = false: the caller overwrites every element (upload / kernel output).
    DBuf(size_t count, bool fp32, bool zero = true) : n(count), f32(fp32) {
        block = DeviceBlockCache::rounded(count * (fp32 ? 4 : 8));
        p = DeviceBlockCache::get().take(block);
        if (zero) cuda_check(cudaMemset(p, 0, std::max<size_t>(count, 1) * (fp32 ? 4 : 8)), "cudaMemset");
    }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() {
        if (p) DeviceBlockCache::get().give(p, block);
    }
    void upload(const std::vector<double>& h) {
        if (h.empty()) return;
        if (f32) {
            std::vector<float> t(h.size());
            parallel_for(h.size(), [&](size_t b, size_t e) {
                for (size_t i = b; i < e; ++i) t[i] = float(h[i]);
            }, 1 << 18);
            cuda_check(cudaMemcpy(p, t.data(), t.size() * 4, cudaMemcpyHostToDevice), "upload");
        } else {
            cuda_check(cudaMemcpy(p, h.data(), h.size() * 8, cudaMemcpyHostToDevice), "upload");
        }
    }
    // fill(T* dst) writes the n values (T = float or double, the buffer's
    // precision) into pinned staging; one copy to the device.
    template <class F>
    void upload_fill(F&& fill) {
        if (!n) return;
        void* st = pinned_staging(n * (f32 ? 4 : 8));
        if (f32) fill(static_cast<float*>(st));
        else fill(static_cast<double*>(st));
        cuda_check(cudaMemcpy(p, st, n * (f32 ? 4 : 8), cudaMemcpyHostToDevice), "upload");
    }
    // one copy to pinned staging, then use(const T* src)
    template <class F>
    void download_with(F&& use) const {
        if (!n) return;
        void* st = pinned_staging(n * (f32 ? 4 : 8));
        cuda_check(cudaMemcpy(st, p, n * (f32 ? 4 : 8), cudaMemcpyDeviceToHost), "download");
        if (f32) use(static_cast<const float*>(st));
        else use(static_cast<const double*>(st));
    }
    std::vector<double> download() const {
        std::vector<double> h(n);
        if (!n) return h;
        if (f32) {
            std::vector<float> t(n);
            cuda_check(cudaMemcpy(t.data(), p, n * 4, cudaMemcpyDeviceToHost), "download");
            parallel_for(n, [&](size_t b, size_t e) {
                for (size_t i = b; i < e; ++i) h[i] = double(t[i]);
            }, 1 << 18);
        } else {
            cuda_check(cudaMemcpy(h.data(), p, n * 8, cudaMemcpyDeviceToHost), "download");
        }
        return h;
    }
};

// Scene -> SoA device buffers (scene.hpp layout; sh rows per colour channel):
// one device allocation, filled in parallel straight into pinned staging in
// the kernel precision, one copy.
struct DeviceScene {
    bool f32;
    int64_t n;
    int C, deg, K;
    size_t off[8];
    DBuf all;
    static size_t total(int64_t n, int C, int K) { return size_t(n) * size_t(12 + 3 * K + C); }
    DeviceScene(const Scene& s, bool fp32)
        : f32(fp32), n(int64_t(s.size())), C(s.num_classes), deg(s.sh_degree), K(s.sh_coeff_count()),
          all(total(n, C, K), fp32, false) {
        const size_t N = size_t(n);
        const size_t len[7] = {3 * N, 4 * N, 3 * N, N, N, size_t(3 * K) * N, size_t(C) * N};
        off[0] = 0;
        for (int i = 0; i < 7; ++i) off[i + 1] = off[i] + len[i];
        all.upload_fill([&](auto* d) {
            using T = std::remove_pointer_t<decltype(d)>;
            T *m = d + off[0], *q = d + off[1], *ls = d + off[2], *o = d + off[3], *kk = d + off[4], *shv = d + off[5],
              *se = d + off[6];
            parallel_for(N, [&](size_t b, size_t e) {
                for (size_t i = b; i < e; ++i) {
                    const GaussianPrimitive& g = s.gaussians[i];
                    for (int j = 0; j < 3; ++j) {
                        m[3 * i + j] = T(g.position[j]);
                        ls[3 * i + j] = T(g.log_scale[j]);
                    }
                    for (int j = 0; j < 4; ++j) q[4 * i + j] = T(g.rotation[j]);
                    o[i] = T(g.opacity_logit);
                    kk[i] = T(g.gradient_factor);
                    for (int c = 0; c < 3; ++c)
                        for (int j = 0; j < K; ++j) shv[(i * 3 + c) * K + j] = T(g.sh(c, j));
                    for (int c = 0; c < C; ++c) se[i * C + c] = T(g.semantic_logits[c]);
                }
            }, 4096);
        });
    }
    void* ptr(int i) const { return static_cast<char*>(all.p) + off[i] * (f32 ? 4 : 8); }
    msplat_scene abi() const {
        return msplat_scene{n, C, deg, f32 ? MSPLAT_F32 : MSPLAT_F64, ptr(0), ptr(1), ptr(2), ptr(3),
                            ptr(4), ptr(5), C ? ptr(6) : nullptr};
    }
};

inline msplat_camera to_abi(const CameraView& v) {
    msplat_camera c{};
    c.fx = v.fx;
    c.fy = v.fy;
    c.cx = v.cx;
    c.cy = v.cy;
    c.width = v.width;
    c.height = v.height;
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) c.R_c2w[i * 3 + j] = v.R_cam_to_world(i, j);
        c.t_c2w[i] = v.t_cam_to_world[i];
    }
    return c;
}

inline msplat_render_config to_abi(const RenderConfig& r) {
    return msplat_render_config{r.sigma_scale, {r.background.x(), r.background.y(), r.background.z()},
                                r.early_stop_transmittance, r.early_termination ? 1 : 0, r.threads};
}

inline msplat_normal_config to_abi(const NormalConfig& n) {
    return msplat_normal_config{n.step1, n.step2, n.fuse_lambda, n.mask_threshold};
}

// HWC grid <-> planar [C][H][W] device buffer, through pinned staging.
inline void upload_planar(DBuf& d, const GridF& g) {
    const int W = g.width(), H = g.height(), C = g.channels();
    d.upload_fill([&](auto* out) {
        using T = std::remove_pointer_t<decltype(out)>;
        parallel_for(size_t(H), [&](size_t y0, size_t y1) {
            for (int y = int(y0); y < int(y1); ++y)
                for (int x = 0; x < W; ++x) {
                    const double* px = g.row(y) + size_t(x) * C;
                    for (int c = 0; c < C; ++c) out[(size_t(c) * H + y) * W + x] = T(px[c]);
                }
        }, 4);
    });
}

inline GridF download_planar(const DBuf& d, int W, int H, int C) {
    GridF g(W, H, C, 0.0);
    d.download_with([&](const auto* v) {
        parallel_for(size_t(H), [&](size_t y0, size_t y1) {
            for (int y = int(y0); y < int(y1); ++y)
                for (int x = 0; x < W; ++x) {
                    double* px = g.row(y) + size_t(x) * C;
                    for (int c = 0; c < C; ++c) px[c] = double(v[(size_t(c) * H + y) * W + x]);
                }
        }, 4);
    });
    return g;
}

// HWC grid <-> planar [C][H][W] host vectors.
inline std::vector<double> to_planar(const GridF& g) {
    const int W = g.width(), H = g.height(), C = g.channels();
    std::vector<double> out(size_t(W) * H * C);
    parallel_for(size_t(H), [&](size_t y0, size_t y1) {
        for (int y = int(y0); y < int(y1); ++y)
            for (int x = 0; x < W; ++x)
                for (int c = 0; c < C; ++c) out[(size_t(c) * H + y) * W + x] = g.at(x, y, c);
    }, 8);
    return out;
}

inline GridF from_planar(const std::vector<double>& v, int W, int H, int C) {
    GridF g(W, H, C, 0.0);
    parallel_for(size_t(H), [&](size_t y0, size_t y1) {
        for (int y = int(y0); y < int(y1); ++y)
            for (int x = 0; x < W; ++x)
                for (int c = 0; c < C; ++c) g.at(x, y, c) = v[(size_t(c) * H + y) * W + x];
    }, 8);
    return g;
}


}  // namespace dropin
}  // namespace msplat
