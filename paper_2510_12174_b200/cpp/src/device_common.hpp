// msplat C++ drop-in: shared device-side helpers (internal).  The context,
// device buffers and the AoS/HWC <-> SoA/planar marshalling used by the render
// path (device_path.cpp) and the trainer (trainer_path.cpp).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "msplat/normals.hpp"
#include "msplat/rasterizer.hpp"
#include "msplat/scene.hpp"
#include "msplat_b200.h"

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

inline bool use_fp32() {
    const char* p = std::getenv("MSPLAT_PRECISION");
    return p && std::string(p) == "32";
}

inline msplat_context* context() {
    thread_local std::unique_ptr<msplat_context, void (*)(msplat_context*)> ctx(nullptr, msplat_context_destroy);
    if (!ctx) {
        const char* d = std::getenv("MSPLAT_DEVICE");
        msplat_context* c = nullptr;
        rethrow(msplat_context_create(d ? std::atoi(d) : 0, nullptr, &c));
        // The reference's accumulation is reproducible at a fixed thread count
        // (tests/test_rasterizer.cpp:386-419): fixed-order reduction, no atomics.
        rethrow(msplat_context_set_deterministic(c, 1));
        ctx.reset(c);
    }
    return ctx.get();
}

// Device buffer holding host doubles converted to the kernel precision.
struct DBuf {
    void* p = nullptr;
    size_t n = 0;
    bool f32 = false;
    DBuf() = default;
    DBuf(size_t count, bool fp32) : n(count), f32(fp32) {
        cuda_check(cudaMalloc(&p, std::max<size_t>(count, 1) * (fp32 ? 4 : 8)), "cudaMalloc");
        cuda_check(cudaMemset(p, 0, std::max<size_t>(count, 1) * (fp32 ? 4 : 8)), "cudaMemset");
    }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() {
        if (p) cudaFree(p);
    }
    void upload(const std::vector<double>& h) {
        if (h.empty()) return;
        if (f32) {
            std::vector<float> t(h.begin(), h.end());
            cuda_check(cudaMemcpy(p, t.data(), t.size() * 4, cudaMemcpyHostToDevice), "upload");
        } else {
            cuda_check(cudaMemcpy(p, h.data(), h.size() * 8, cudaMemcpyHostToDevice), "upload");
        }
    }
    std::vector<double> download() const {
        std::vector<double> h(n);
        if (!n) return h;
        if (f32) {
            std::vector<float> t(n);
            cuda_check(cudaMemcpy(t.data(), p, n * 4, cudaMemcpyDeviceToHost), "download");
            h.assign(t.begin(), t.end());
        } else {
            cuda_check(cudaMemcpy(h.data(), p, n * 8, cudaMemcpyDeviceToHost), "download");
        }
        return h;
    }
};

// Scene -> SoA device buffers (scene.hpp layout; sh rows per colour channel).
struct DeviceScene {
    bool f32;
    int64_t n;
    int C, deg, K;
    DBuf means, quats, log_scales, opac, k, sh, sem;
    DeviceScene(const Scene& s, bool fp32)
        : f32(fp32), n(int64_t(s.size())), C(s.num_classes), deg(s.sh_degree), K(s.sh_coeff_count()),
          means(3 * n, fp32), quats(4 * n, fp32), log_scales(3 * n, fp32), opac(n, fp32), k(n, fp32),
          sh(size_t(3 * K) * n, fp32), sem(size_t(C) * n, fp32) {
        std::vector<double> m(3 * n), q(4 * n), ls(3 * n), o(n), kk(n), shv(size_t(3 * K) * n), se(size_t(C) * n);
        for (int64_t i = 0; i < n; ++i) {
            const GaussianPrimitive& g = s.gaussians[size_t(i)];
            for (int j = 0; j < 3; ++j) {
                m[3 * i + j] = g.position[j];
                ls[3 * i + j] = g.log_scale[j];
            }
            for (int j = 0; j < 4; ++j) q[4 * i + j] = g.rotation[j];
            o[i] = g.opacity_logit;
            kk[i] = g.gradient_factor;
            for (int c = 0; c < 3; ++c)
                for (int j = 0; j < K; ++j) shv[(i * 3 + c) * K + j] = g.sh(c, j);
            for (int c = 0; c < C; ++c) se[i * C + c] = g.semantic_logits[c];
        }
        means.upload(m);
        quats.upload(q);
        log_scales.upload(ls);
        opac.upload(o);
        k.upload(kk);
        sh.upload(shv);
        sem.upload(se);
    }
    msplat_scene abi() const {
        return msplat_scene{n, C, deg, f32 ? MSPLAT_F32 : MSPLAT_F64, means.p, quats.p, log_scales.p, opac.p,
                            k.p, sh.p, C ? sem.p : nullptr};
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

// HWC grid <-> planar [C][H][W] host vectors.
inline std::vector<double> to_planar(const GridF& g) {
    const int W = g.width(), H = g.height(), C = g.channels();
    std::vector<double> out(size_t(W) * H * C);
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x)
            for (int c = 0; c < C; ++c) out[(size_t(c) * H + y) * W + x] = g.at(x, y, c);
    return out;
}

inline GridF from_planar(const std::vector<double>& v, int W, int H, int C) {
    GridF g(W, H, C, 0.0);
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x)
            for (int c = 0; c < C; ++c) g.at(x, y, c) = v[(size_t(c) * H + y) * W + x];
    return g;
}


}  // namespace dropin
}  // namespace msplat
