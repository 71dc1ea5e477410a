// msplat C++ drop-in: the render path on the B200.
//
// rasterize / rasterize_backward / estimate_normals / normals_backward /
// chain_activations / bin_and_sort keep the reference signatures
// (msplat/rasterizer.hpp:52-83, normals.hpp:33-43, scene.hpp:74) and run
// through the C ABI of include/msplat_b200.h.  This file only marshals: AoS
// Eigen doubles <-> SoA device buffers, HWC host grids <-> planar device grids,
// and msplat_status -> the reference's exception types and messages.
//
// Precision: MSPLAT_F64 unless MSPLAT_PRECISION=32 is set in the environment.
#include <cuda_runtime.h>

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
#include "device_common.hpp"

namespace msplat {

using namespace dropin;

// Device replays are pooled per thread: the reference API makes a fresh
// ReplayState for every forward, and a fresh msplat_replay would allocate and
// free its device buffers (GBs at cfg3: the event log and the FP32 weight
// rows) on every call.  A replay goes back to the pool of the thread (and
// context) that made it, else it is destroyed.
struct ReplayPool {
    std::vector<msplat_replay*> free;
    ~ReplayPool() {
        for (msplat_replay* r : free) msplat_replay_destroy(r);
    }
};
inline ReplayPool& replay_pool() {
    thread_local ReplayPool pool;  // constructed after (destroyed before) the thread's context
    return pool;
}

struct DeviceReplay {
    msplat_replay* handle = nullptr;
    bool f32 = false;
    ReplayPool* owner = nullptr;
    explicit DeviceReplay(bool fp32) : f32(fp32) {
        msplat_context* ctx = context();
        owner = &replay_pool();
        if (!owner->free.empty()) {
            handle = owner->free.back();
            owner->free.pop_back();
        } else {
            rethrow(msplat_replay_create(ctx, &handle));
        }
        rethrow(msplat_replay_set_capture(handle, 3));
    }
    ~DeviceReplay() {
        if (owner == &replay_pool() && owner->free.size() < 2)
            owner->free.push_back(handle);
        else
            msplat_replay_destroy(handle);
    }
};

PixelGradients PixelGradients::zero(int width, int height, int num_classes) {
    PixelGradients pg;
    pg.dcolor = GridF(width, height, 3, 0.0);
    pg.ddepth = GridF(width, height, 1, 0.0);
    pg.dsemantics = GridF(width, height, num_classes, 0.0);
    pg.dkmap = GridF(width, height, 1, 0.0);
    return pg;
}

// bin_and_sort -- core/src/rasterizer.cpp:14-45, on the device radix sort.
TileBins bin_and_sort(const std::vector<std::optional<Splat2D>>& splats, int width, int height) {
    const int64_t n = int64_t(splats.size());
    std::vector<uint8_t> vis(n);
    std::vector<double> center(2 * n), radius(n), depth(n);
    for (int64_t i = 0; i < n; ++i) {
        vis[i] = splats[i].has_value();
        if (!vis[i]) continue;
        center[2 * i] = splats[i]->center.x();
        center[2 * i + 1] = splats[i]->center.y();
        radius[i] = splats[i]->radius;
        depth[i] = splats[i]->sort_depth;
    }
    TileBins out;
    out.tiles_x = (width + TileBins::kTileSize - 1) / TileBins::kTileSize;
    out.tiles_y = (height + TileBins::kTileSize - 1) / TileBins::kTileSize;
    const size_t tiles = size_t(out.tiles_x) * out.tiles_y;
    std::vector<int64_t> off(tiles + 1);
    std::vector<int32_t> vals(std::max<int64_t>(n, 1) * 4);
    int64_t count = 0;
    for (;;) {
        rethrow(msplat_bin_and_sort_host(context(), n, vis.data(), center.data(), radius.data(), depth.data(), width,
                                         height, off.data(), vals.data(), int64_t(vals.size()), &count));
        if (count <= int64_t(vals.size())) break;
        vals.resize(size_t(count));
    }
    out.bins.resize(tiles);
    for (size_t t = 0; t < tiles; ++t) out.bins[t].assign(vals.begin() + off[t], vals.begin() + off[t + 1]);
    return out;
}

// rasterize -- core/src/rasterizer.cpp:87-205
MultimodalFrame rasterize(const Scene& scene, const CameraView& view, const RenderConfig& cfg, ReplayState* replay) {
    PhaseTimer pt("rasterize");
    scene.validate();
    pt.mark("validate");
    const bool f32 = use_fp32();
    const int W = view.width, H = view.height, C = scene.num_classes;
    const size_t HW = size_t(W) * H;
    DeviceScene ds(scene, f32);
    pt.mark("scene upload");
    DBuf color(3 * HW, f32, false), depth(HW, f32, false), sem(size_t(C) * HW, f32, false), kmap(HW, f32, false),
        T(HW, f32, false);
    DBuf contrib_buf(HW, true, false);  // int32 per pixel
    int32_t* contrib = static_cast<int32_t*>(contrib_buf.p);
    msplat_frame fr{color.p, depth.p, C ? sem.p : nullptr, kmap.p, T.p, nullptr, contrib};
    auto dev = replay ? std::make_shared<DeviceReplay>(f32) : nullptr;
    const msplat_scene s = ds.abi();
    const msplat_camera c = to_abi(view);
    const msplat_render_config rc = to_abi(cfg);
    pt.mark("buffers");
    rethrow(msplat_rasterize(context(), &s, &c, &rc, &fr, dev ? dev->handle : nullptr));
    pt.mark("msplat_rasterize");

    MultimodalFrame f;
    f.width = W;
    f.height = H;
    f.num_classes = C;
    f.color = download_planar(color, W, H, 3);
    f.depth = download_planar(depth, W, H, 1);
    f.semantics = C ? download_planar(sem, W, H, C) : GridF(W, H, 0, 0.0);
    f.kmap = download_planar(kmap, W, H, 1);
    f.transmittance = download_planar(T, W, H, 1);
    f.normals = GridF(W, H, 3, 0.0);  // filled by estimate_normals, as in the reference
    f.contributors = Grid<int>(W, H, 1, 0);
    cuda_check(cudaMemcpy(f.contributors.data(), contrib, HW * 4, cudaMemcpyDeviceToHost), "download");
    pt.mark("frame download");

    if (replay) {
        const size_t n = scene.size();
        replay->device = dev;
        // activate_scene (borrows from `scene`, like the reference), in parallel
        replay->activated.assign(n, ActivatedGaussian{});
        parallel_for(n, [&](size_t b, size_t e) {
            for (size_t i = b; i < e; ++i) replay->activated[i] = activate(scene.gaussians[i], i);
        });
        pt.mark("replay activated");
        std::vector<uint8_t> vis(n), cl(3 * n);
        std::vector<double> center(2 * n), conic(3 * n), sdepth(n), radius(n), rgb(3 * n);
        rethrow(msplat_replay_splats(dev->handle, vis.data(), center.data(), conic.data(), sdepth.data(),
                                     radius.data(), rgb.data(), cl.data()));
        replay->splats.assign(n, std::nullopt);
        replay->colors.assign(n, ShColor{});
        parallel_for(n, [&](size_t b, size_t e) {
          for (size_t i = b; i < e; ++i) {
            if (!vis[i]) continue;
            Splat2D sp;
            sp.center = Vec2(center[2 * i], center[2 * i + 1]);
            sp.conic << conic[3 * i], conic[3 * i + 1], conic[3 * i + 1], conic[3 * i + 2];
            const Scalar det = conic[3 * i] * conic[3 * i + 2] - conic[3 * i + 1] * conic[3 * i + 1];
            sp.cov << conic[3 * i + 2] / det, -conic[3 * i + 1] / det, -conic[3 * i + 1] / det, conic[3 * i] / det;
            sp.sort_depth = sdepth[i];
            sp.radius = radius[i];
            replay->splats[i] = sp;
            for (int ch = 0; ch < 3; ++ch) {
                replay->colors[i].rgb[ch] = rgb[3 * i + ch];
                replay->colors[i].clamped[ch] = cl[3 * i + ch] != 0;
            }
          }
        });
        pt.mark("replay splats");
        msplat_counters cn{};
        rethrow(msplat_replay_counters(dev->handle, &cn));
        std::vector<int64_t> off(size_t(cn.tiles) + 1);
        std::vector<int32_t> vals(size_t(std::max<int64_t>(cn.instances, 1)));
        rethrow(msplat_replay_bins(dev->handle, off.data(), vals.data(), int64_t(vals.size())));
        replay->bins.tiles_x = (W + TileBins::kTileSize - 1) / TileBins::kTileSize;
        replay->bins.tiles_y = (H + TileBins::kTileSize - 1) / TileBins::kTileSize;
        replay->bins.bins.assign(size_t(cn.tiles), {});
        parallel_for(size_t(cn.tiles), [&](size_t b, size_t e) {
            for (size_t t = b; t < e; ++t) replay->bins.bins[t].assign(vals.begin() + off[t], vals.begin() + off[t + 1]);
        }, 64);
        replay->terminus = Grid<int>(W, H, 1, 0);
        rethrow(msplat_replay_terminus(dev->handle, replay->terminus.data()));
        replay->weight_sums.assign(n, 0.0);
        if (n) rethrow(msplat_replay_weight_sums(dev->handle, replay->weight_sums.data()));
        replay->num_gaussians = n;
        replay->sh_degree = scene.sh_degree;
        replay->num_classes = scene.num_classes;
        replay->cfg = cfg;
        pt.mark("replay bins/terminus/ws");
    }
    return f;
}

namespace {

// The gradient arrays as one device allocation (the packed order of
// DeviceScene), downloaded once and scattered into the AoS GradientBuffer
// (GradientBuffer::resize_zero's shapes, scene.cpp:70-95) in parallel.
struct DeviceGrads {
    size_t off[8];
    DBuf all;
    DeviceGrads(const Scene& scene, bool f32)
        : all(DeviceScene::total(int64_t(scene.size()), scene.num_classes, scene.sh_coeff_count()), f32, false) {
        const size_t N = scene.size();
        const int K = scene.sh_coeff_count(), C = scene.num_classes;
        const size_t len[7] = {3 * N, 4 * N, 3 * N, N, N, size_t(3 * K) * N, size_t(C) * N};
        off[0] = 0;
        for (int i = 0; i < 7; ++i) off[i + 1] = off[i] + len[i];
    }
    void* ptr(int i) const { return static_cast<char*>(all.p) + off[i] * (all.f32 ? 4 : 8); }
    // buffer order: position, rotation, scale, opacity, k, sh, semantics
    msplat_grads abi(int C) const { return msplat_grads{ptr(0), ptr(1), ptr(2), ptr(3), ptr(4), ptr(5), C ? ptr(6) : nullptr}; }
    void to_host(GradientBuffer& g, const Scene& scene) const {
        const size_t n = scene.size();
        const int K = scene.sh_coeff_count(), C = scene.num_classes;
        g.dposition.resize(n);
        g.drotation.resize(n);
        g.dscale.resize(n);
        g.dopacity.resize(n);
        g.dk.resize(n);
        g.dsh.resize(n);
        g.dsemantics.resize(n);
        g.raw_space = false;
        all.download_with([&](const auto* d) {
            const auto *p = d + off[0], *r = d + off[1], *s = d + off[2], *o = d + off[3], *k = d + off[4],
                       *h = d + off[5], *e = d + off[6];
            parallel_for(n, [&](size_t b, size_t e_) {
                for (size_t i = b; i < e_; ++i) {
                    g.dposition[i] = Vec3(p[3 * i], p[3 * i + 1], p[3 * i + 2]);
                    g.drotation[i] = Vec4(r[4 * i], r[4 * i + 1], r[4 * i + 2], r[4 * i + 3]);
                    g.dscale[i] = Vec3(s[3 * i], s[3 * i + 1], s[3 * i + 2]);
                    g.dopacity[i] = o[i];
                    g.dk[i] = k[i];
                    g.dsh[i].resize(3, K);
                    for (int c = 0; c < 3; ++c)
                        for (int j = 0; j < K; ++j) g.dsh[i](c, j) = h[(i * 3 + c) * K + j];
                    g.dsemantics[i].resize(C);
                    for (int c = 0; c < C; ++c) g.dsemantics[i][c] = e[i * C + c];
                }
            }, 4096);
        });
    }
};

}  // namespace

// rasterize_backward -- core/src/rasterizer_backward.cpp:127-264 (check_replay :35-53)
GradientBuffer rasterize_backward(const Scene& scene, const CameraView& view, const MultimodalFrame& frame,
                                  const ReplayState& replay, const PixelGradients& pix) {
    PhaseTimer pt("backward");
    if (replay.num_gaussians != scene.size() || replay.sh_degree != scene.sh_degree ||
        replay.num_classes != scene.num_classes || !replay.device)
        throw std::runtime_error("rasterize_backward: replay state does not match the scene");
    // check_replay's scan (rasterizer_backward.cpp:40-44) in parallel chunks; the
    // lowest chunk's exception is rethrown, so the message names the first
    // modified primitive, as the sequential loop does.
    parallel_for(scene.size(), [&](size_t b, size_t e) {
        for (size_t i = b; i < e; ++i)
            if ((replay.activated[i].position.array() != scene.gaussians[i].position.array()).any() ||
                replay.activated[i].k != scene.gaussians[i].gradient_factor)
                throw std::runtime_error("rasterize_backward: scene modified since forward (primitive " +
                                         std::to_string(i) + ")");
    }, 1 << 14);
    if (frame.width != view.width || frame.height != view.height)
        throw std::runtime_error("rasterize_backward: frame/view size mismatch");
    const bool ok = pix.dcolor.width() == frame.width && pix.dcolor.height() == frame.height &&
                    pix.dcolor.channels() == 3 && pix.ddepth.same_shape(frame.depth) &&
                    pix.dsemantics.same_shape(frame.semantics) && pix.dkmap.same_shape(frame.kmap);
    if (!ok) throw std::runtime_error("rasterize_backward: pixel-gradient shape mismatch");

    pt.mark("checks");
    const bool f32 = replay.device->f32;
    const int W = frame.width, H = frame.height, C = scene.num_classes;
    const size_t HW = size_t(W) * H;
    DeviceScene ds(scene, f32);
    pt.mark("scene upload");
    DBuf T(HW, f32, false), dC(3 * HW, f32, false), dD(HW, f32, false), dO(size_t(C) * HW, f32, false),
        dK(HW, f32, false);
    upload_planar(T, frame.transmittance);
    upload_planar(dC, pix.dcolor);
    upload_planar(dD, pix.ddepth);
    if (C) upload_planar(dO, pix.dsemantics);
    upload_planar(dK, pix.dkmap);
    DeviceGrads dg(scene, f32);  // zeroed by the backward
    msplat_frame fr{nullptr, nullptr, nullptr, nullptr, T.p, nullptr, nullptr};
    msplat_pixel_grads pg{dC.p, dD.p, C ? dO.p : nullptr, dK.p, nullptr};
    msplat_grads g = dg.abi(C);
    const msplat_scene s = ds.abi();
    const msplat_camera c = to_abi(view);
    pt.mark("pixel-grad upload");
    rethrow(msplat_rasterize_backward(context(), &s, &c, &fr, replay.device->handle, &pg, &g));
    pt.mark("msplat_rasterize_backward");
    GradientBuffer out;
    dg.to_host(out, scene);
    pt.mark("grads download");
    return out;
}

// chain_activations -- core/src/scene.cpp:108-129, on the device.
void chain_activations(GradientBuffer& buf, const Scene& scene) {
    if (buf.size() != scene.size()) throw std::invalid_argument("chain_activations: buffer/scene size mismatch");
    if (buf.raw_space) throw std::logic_error("chain_activations: buffer already in raw-parameter space");
    const bool f32 = use_fp32();
    const size_t n = scene.size();
    DeviceScene ds(scene, f32);
    DBuf grot(4 * n, f32), gsc(3 * n, f32), gop(n, f32);
    std::vector<double> r(4 * n), sc(3 * n), op(n);
    for (size_t i = 0; i < n; ++i) {
        for (int j = 0; j < 4; ++j) r[4 * i + j] = buf.drotation[i][j];
        for (int j = 0; j < 3; ++j) sc[3 * i + j] = buf.dscale[i][j];
        op[i] = buf.dopacity[i];
    }
    grot.upload(r);
    gsc.upload(sc);
    gop.upload(op);
    msplat_grads g{nullptr, grot.p, gsc.p, gop.p, nullptr, nullptr, nullptr};
    const msplat_scene s = ds.abi();
    rethrow(msplat_chain_activations(context(), &s, &g));
    rethrow(msplat_context_check(context()));
    r = grot.download();
    sc = gsc.download();
    op = gop.download();
    for (size_t i = 0; i < n; ++i) {
        buf.drotation[i] = Vec4(r[4 * i], r[4 * i + 1], r[4 * i + 2], r[4 * i + 3]);
        buf.dscale[i] = Vec3(sc[3 * i], sc[3 * i + 1], sc[3 * i + 2]);
        buf.dopacity[i] = op[i];
    }
    buf.raw_space = true;
}

// estimate_normals -- core/src/normals.cpp:28-101, on the device.
NormalState estimate_normals(const GridF& depth, const GridF& transmittance, const CameraView& view,
                             const NormalConfig& cfg, GridF& normals) {
    if (cfg.step1 >= cfg.step2) throw std::invalid_argument("estimate_normals: step1 must be smaller than step2");
    if (cfg.fuse_lambda < 0 || cfg.fuse_lambda > 1)
        throw std::invalid_argument("estimate_normals: fuse weight must be in [0,1]");
    NormalState st;
    st.p_world = backproject(depth, view);  // also validates the depth shape
    const int W = view.width, H = view.height;
    const size_t HW = size_t(W) * H;
    const bool f32 = use_fp32();
    DBuf d(HW, f32), t(HW, f32), nrm(3 * HW, f32);
    d.upload(depth.storage());
    t.upload(transmittance.storage());
    const msplat_camera c = to_abi(view);
    const msplat_normal_config nc = to_abi(cfg);
    rethrow(msplat_estimate_normals(context(), f32 ? MSPLAT_F32 : MSPLAT_F64, d.p, t.p, &c, &nc, nrm.p));
    rethrow(msplat_context_check(context()));
    normals = from_planar(nrm.download(), W, H, 3);
    st.width = W;
    st.height = H;
    st.cfg = cfg;
    st.valid = Grid<std::uint8_t>(W, H, 1, 0);
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x)
            st.valid.at(x, y) = normals.at(x, y, 0) != 0 || normals.at(x, y, 1) != 0 || normals.at(x, y, 2) != 0;
    st.depth = depth;
    st.transmittance = transmittance;
    return st;
}

// normals_backward -- core/src/normals.cpp:103-152, gather form on the device.
GridF normals_backward(const GridF& dL_dnormals, const NormalState& state, const CameraView& view) {
    const int W = state.width, H = state.height;
    if (dL_dnormals.width() != W || dL_dnormals.height() != H || dL_dnormals.channels() != 3)
        throw std::invalid_argument("normals_backward: gradient shape mismatch");
    const size_t HW = size_t(W) * H;
    const bool f32 = use_fp32();
    DBuf g(3 * HW, f32), d(HW, f32), t(HW, f32), dD(HW, f32);
    g.upload(to_planar(dL_dnormals));
    d.upload(state.depth.storage());
    t.upload(state.transmittance.storage());
    const msplat_camera c = to_abi(view);
    const msplat_normal_config nc = to_abi(state.cfg);
    rethrow(msplat_normals_backward(context(), f32 ? MSPLAT_F32 : MSPLAT_F64, g.p, d.p, t.p, &c, &nc, 1.0, dD.p));
    rethrow(msplat_context_check(context()));
    return from_planar(dD.download(), W, H, 1);
}

}  // namespace msplat
