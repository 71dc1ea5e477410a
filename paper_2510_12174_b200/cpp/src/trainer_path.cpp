// msplat C++ drop-in: training (reference API msplat/trainer.hpp,
// core/src/trainer.cpp) over the B200 C ABI.
//
// train() keeps everything on the device: the packed parameters (layout of
// msplat_param_layout), both Adam moments, the last finite scene, every
// training frame's ground truth (uploaded once) and the per-iteration frame,
// pixel-gradient and gradient buffers.  One iteration is the reference's
// (trainer.cpp:289-328): rasterize, estimate_normals, evaluate_frame_losses,
// non-finite halt, rasterize_backward, chain_activations, adam_step and every
// prune_interval iterations the prune mask + compaction of parameters and
// moments.  The host reads only the 18-double loss report per iteration.
#include <chrono>
#include <cmath>
#include <random>

#include "device_common.hpp"
#include "msplat/trainer.hpp"

namespace msplat {

using namespace dropin;

// core/src/dataset.cpp:19-33: frames whose split is not / is "test".
std::vector<int> SceneDataset::train_indices() const {
    std::vector<int> out;
    for (int i = 0; i < int(frames.size()); ++i)
        if (frames[i].split != "test") out.push_back(i);
    return out;
}

std::vector<int> SceneDataset::test_indices() const {
    std::vector<int> out;
    for (int i = 0; i < int(frames.size()); ++i)
        if (frames[i].split == "test") out.push_back(i);
    return out;
}

// trainer.cpp:14-32
void TrainConfig::validate() const {
    if (iterations < 0) throw std::invalid_argument("TrainConfig: iterations must be >= 0");
    for (Scalar lr : {lr_position, lr_rotation, lr_scale, lr_opacity, lr_sh, lr_semantics, lr_k})
        if (!(lr > 0)) throw std::invalid_argument("TrainConfig: learning rates must be positive");
    if (prune_interval < 1) throw std::invalid_argument("TrainConfig: prune_interval must be >= 1");
    if (!(prune_threshold > 0)) throw std::invalid_argument("TrainConfig: prune_threshold must be positive");
    if (step1 >= step2 || step1 < 1) throw std::invalid_argument("TrainConfig: need 1 <= step1 < step2");
    if (lambda_fuse < 0 || lambda_fuse > 1) throw std::invalid_argument("TrainConfig: lambda_fuse must be in [0,1]");
    if (sh_degree < 0 || sh_degree > 3) throw std::invalid_argument("TrainConfig: sh_degree must be in [0,3]");
    if (!(sigma_scale > 0)) throw std::invalid_argument("TrainConfig: sigma_scale must be positive");
}

OptimizerState OptimizerState::init(const Scene& scene) {
    OptimizerState st;
    st.m.resize_zero(scene);
    st.v.resize_zero(scene);
    st.step = 0;
    return st;
}

// losses.cpp:285-313 (host scalar arithmetic; the training loop uses the
// device combine inside msplat_frame_losses).
LossReport combine(Scalar l1, Scalar ssim, Scalar normal, Scalar depth, Scalar seg, Scalar k,
                   const std::array<Scalar, 6>& lambdas) {
    LossReport r;
    r.l1 = l1;
    r.ssim = ssim;
    r.normal = normal;
    r.depth = depth;
    r.seg = seg;
    r.k = k;
    const Scalar mag = std::abs(l1);
    auto ratio = [&](Scalar v) { return std::abs(v) < 1e-12 ? 0.0 : mag / std::abs(v); };
    r.ratio_ssim = ratio(ssim);
    r.ratio_normal = ratio(normal);
    r.ratio_depth = ratio(depth);
    r.ratio_seg = ratio(seg);
    r.ratio_k = ratio(k);
    r.seed_l1 = lambdas[0];
    r.seed_ssim = lambdas[1] * r.ratio_ssim;
    r.seed_normal = lambdas[2] * r.ratio_normal;
    r.seed_depth = lambdas[3] * r.ratio_depth;
    r.seed_seg = lambdas[4] * r.ratio_seg;
    r.seed_k = lambdas[5] * r.ratio_k;
    r.combined = lambdas[0] * l1 + r.seed_ssim * ssim + r.seed_normal * normal + r.seed_depth * depth +
                 r.seed_seg * seg + r.seed_k * k;
    return r;
}

namespace {

// ---- packed parameter layout (msplat_param_layout): host <-> device
struct Layout {
    int64_t n = 0;
    int C = 0, deg = 0, K = 1;
    int64_t off[8] = {};
    Layout(int64_t n_, int C_, int deg_) : n(n_), C(C_), deg(deg_), K((deg_ + 1) * (deg_ + 1)) {
        rethrow(msplat_param_layout(n, C, deg, off));
    }
    size_t total() const { return size_t(off[7]); }
};

std::vector<double> pack_scene(const Scene& s, const Layout& L) {
    std::vector<double> f(L.total());
    for (size_t i = 0; i < s.size(); ++i) {
        const GaussianPrimitive& g = s.gaussians[i];
        for (int j = 0; j < 3; ++j) {
            f[L.off[0] + 3 * i + j] = g.position[j];
            f[L.off[2] + 3 * i + j] = g.log_scale[j];
        }
        for (int j = 0; j < 4; ++j) f[L.off[1] + 4 * i + j] = g.rotation[j];
        f[L.off[3] + i] = g.opacity_logit;
        f[L.off[4] + i] = g.gradient_factor;
        for (int c = 0; c < 3; ++c)
            for (int j = 0; j < L.K; ++j) f[L.off[5] + (3 * i + c) * L.K + j] = g.sh(c, j);
        for (int c = 0; c < L.C; ++c) f[L.off[6] + i * L.C + c] = g.semantic_logits[c];
    }
    return f;
}

Scene unpack_scene(const std::vector<double>& f, const Layout& L) {
    Scene s;
    s.num_classes = L.C;
    s.sh_degree = L.deg;
    s.gaussians.resize(size_t(L.n));
    for (size_t i = 0; i < size_t(L.n); ++i) {
        GaussianPrimitive& g = s.gaussians[i];
        g.position = Vec3(f[L.off[0] + 3 * i], f[L.off[0] + 3 * i + 1], f[L.off[0] + 3 * i + 2]);
        g.rotation = Vec4(f[L.off[1] + 4 * i], f[L.off[1] + 4 * i + 1], f[L.off[1] + 4 * i + 2], f[L.off[1] + 4 * i + 3]);
        g.log_scale = Vec3(f[L.off[2] + 3 * i], f[L.off[2] + 3 * i + 1], f[L.off[2] + 3 * i + 2]);
        g.opacity_logit = f[L.off[3] + i];
        g.gradient_factor = f[L.off[4] + i];
        g.sh = ShMatrix::Zero(3, L.K);
        for (int c = 0; c < 3; ++c)
            for (int j = 0; j < L.K; ++j) g.sh(c, j) = f[L.off[5] + (3 * i + c) * L.K + j];
        g.semantic_logits = VecX::Zero(L.C);
        for (int c = 0; c < L.C; ++c) g.semantic_logits[c] = f[L.off[6] + i * L.C + c];
    }
    return s;
}

std::vector<double> pack_grads(const GradientBuffer& b, const Layout& L) {
    std::vector<double> f(L.total());
    for (size_t i = 0; i < size_t(L.n); ++i) {
        for (int j = 0; j < 3; ++j) {
            f[L.off[0] + 3 * i + j] = b.dposition[i][j];
            f[L.off[2] + 3 * i + j] = b.dscale[i][j];
        }
        for (int j = 0; j < 4; ++j) f[L.off[1] + 4 * i + j] = b.drotation[i][j];
        f[L.off[3] + i] = b.dopacity[i];
        f[L.off[4] + i] = b.dk[i];
        for (int c = 0; c < 3; ++c)
            for (int j = 0; j < L.K; ++j) f[L.off[5] + (3 * i + c) * L.K + j] = b.dsh[i](c, j);
        for (int c = 0; c < L.C; ++c) f[L.off[6] + i * L.C + c] = b.dsemantics[i][c];
    }
    return f;
}

void unpack_grads(const std::vector<double>& f, const Layout& L, GradientBuffer& b) {
    for (size_t i = 0; i < size_t(L.n); ++i) {
        b.dposition[i] = Vec3(f[L.off[0] + 3 * i], f[L.off[0] + 3 * i + 1], f[L.off[0] + 3 * i + 2]);
        b.drotation[i] = Vec4(f[L.off[1] + 4 * i], f[L.off[1] + 4 * i + 1], f[L.off[1] + 4 * i + 2], f[L.off[1] + 4 * i + 3]);
        b.dscale[i] = Vec3(f[L.off[2] + 3 * i], f[L.off[2] + 3 * i + 1], f[L.off[2] + 3 * i + 2]);
        b.dopacity[i] = f[L.off[3] + i];
        b.dk[i] = f[L.off[4] + i];
        for (int c = 0; c < 3; ++c)
            for (int j = 0; j < L.K; ++j) b.dsh[i](c, j) = f[L.off[5] + (3 * i + c) * L.K + j];
        for (int c = 0; c < L.C; ++c) b.dsemantics[i][c] = f[L.off[6] + i * L.C + c];
    }
}

size_t real_size(bool f32) { return f32 ? 4 : 8; }

// Views of a packed device buffer as the ABI's scene / gradient structs.
msplat_scene scene_view(void* p, const Layout& L, bool f32) {
    char* b = static_cast<char*>(p);
    const size_t R = real_size(f32);
    return msplat_scene{L.n, L.C, L.deg, f32 ? MSPLAT_F32 : MSPLAT_F64, b + L.off[0] * R, b + L.off[1] * R,
                        b + L.off[2] * R, b + L.off[3] * R, b + L.off[4] * R, b + L.off[5] * R,
                        L.C ? b + L.off[6] * R : nullptr};
}
msplat_grads grads_view(void* p, const Layout& L, bool f32) {
    char* b = static_cast<char*>(p);
    const size_t R = real_size(f32);
    return msplat_grads{b + L.off[0] * R, b + L.off[1] * R, b + L.off[2] * R, b + L.off[3] * R,
                        b + L.off[4] * R, b + L.off[5] * R, L.C ? b + L.off[6] * R : nullptr};
}

std::array<double, 7> packed_lrs(const TrainConfig& c) {  // layout order: means quats scales opacity k sh sem
    return {c.lr_position, c.lr_rotation, c.lr_scale, c.lr_opacity, c.lr_k, c.lr_sh, c.lr_semantics};
}

void require_gt(const FrameRecord& gt, const TrainConfig& cfg) {  // trainer.cpp:181-224
    auto missing = [](const std::string& p) { return p.empty() ? std::string("<missing>") : p; };
    if ((cfg.lambdas[0] > 0 || cfg.lambdas[1] > 0) && gt.rgb.empty())
        throw std::runtime_error("rgb loss enabled but the frame has no rgb ground truth (" + missing(gt.rgb_path) + ")");
    if (cfg.lambdas[2] > 0 && gt.normal.empty())
        throw std::runtime_error("normal loss enabled but the frame has no normal ground truth (" +
                                 missing(gt.normal_path) + ")");
    if (cfg.lambdas[3] > 0 && gt.depth.empty())
        throw std::runtime_error("depth loss enabled but the frame has no depth ground truth (" +
                                 missing(gt.depth_path) + ")");
    if (cfg.lambdas[4] > 0 && gt.labels.empty())
        throw std::runtime_error("segmentation loss enabled but the frame has no label ground truth (" +
                                 missing(gt.sem_path) + ")");
}

// Raw device bytes (labels).
struct ByteBuf {
    void* p = nullptr;
    explicit ByteBuf(size_t n) { cuda_check(cudaMalloc(&p, std::max<size_t>(n, 1)), "cudaMalloc"); }
    ByteBuf(const ByteBuf&) = delete;
    ByteBuf& operator=(const ByteBuf&) = delete;
    ~ByteBuf() {
        if (p) cudaFree(p);
    }
};

// One frame's ground truth on the device, planar.
struct DeviceGT {
    std::unique_ptr<DBuf> rgb, depth, normal;
    std::unique_ptr<ByteBuf> labels;
    msplat_ground_truth abi{};
    DeviceGT(const FrameRecord& f, bool f32) {
        if (!f.rgb.empty()) {
            rgb = std::make_unique<DBuf>(f.rgb.size(), f32);
            rgb->upload(to_planar(f.rgb));
            abi.rgb = rgb->p;
        }
        if (!f.depth.empty()) {
            depth = std::make_unique<DBuf>(f.depth.size(), f32);
            depth->upload(f.depth.storage());
            abi.depth = depth->p;
        }
        if (!f.normal.empty()) {
            normal = std::make_unique<DBuf>(f.normal.size(), f32);
            normal->upload(to_planar(f.normal));
            abi.normal = normal->p;
        }
        if (!f.labels.empty()) {
            labels = std::make_unique<ByteBuf>(f.labels.size());
            cuda_check(cudaMemcpy(labels->p, f.labels.data(), f.labels.size(), cudaMemcpyHostToDevice), "upload");
            abi.labels = static_cast<const uint8_t*>(labels->p);
        }
    }
};

LossReport from_abi(const msplat_loss_report& r) {
    LossReport o;
    o.l1 = r.l1;
    o.ssim = r.ssim;
    o.depth = r.depth;
    o.normal = r.normal;
    o.seg = r.seg;
    o.k = r.k;
    o.combined = r.combined;
    o.ratio_ssim = r.ratio_ssim;
    o.ratio_normal = r.ratio_normal;
    o.ratio_depth = r.ratio_depth;
    o.ratio_seg = r.ratio_seg;
    o.ratio_k = r.ratio_k;
    o.seed_l1 = r.seed_l1;
    o.seed_ssim = r.seed_ssim;
    o.seed_depth = r.seed_depth;
    o.seed_normal = r.seed_normal;
    o.seed_seg = r.seed_seg;
    o.seed_k = r.seed_k;
    return o;
}

[[noreturn]] void throw_prune_all(const TrainConfig& cfg) {  // trainer.cpp:146-148
    throw std::runtime_error("prune: threshold " + std::to_string(cfg.prune_threshold) +
                             " would remove every gaussian");
}

}  // namespace

// init_scene (trainer.cpp:42-86): the neighbour search runs on the device.
Scene init_scene(const std::vector<Vec3>& points, const std::vector<Vec3>& colors, int num_classes,
                 const TrainConfig& cfg) {
    if (points.empty()) throw std::invalid_argument("init_scene: empty point list");
    if (colors.size() != points.size()) throw std::invalid_argument("init_scene: point/color count mismatch");
    const Layout L(int64_t(points.size()), num_classes, cfg.sh_degree);
    std::vector<double> pts(3 * points.size()), cols(3 * points.size());
    for (size_t i = 0; i < points.size(); ++i)
        for (int j = 0; j < 3; ++j) {
            pts[3 * i + j] = points[i][j];
            cols[3 * i + j] = colors[i][j];
        }
    DBuf params(L.total(), false);
    rethrow(msplat_init_scene(context(), MSPLAT_F64, L.n, pts.data(), cols.data(), num_classes, cfg.sh_degree,
                              cfg.k_reset, params.p));
    return unpack_scene(params.download(), L);
}

// adam_step (trainer.cpp:98-133) on the device.
void adam_step(Scene& scene, const GradientBuffer& grads, OptimizerState& state, const TrainConfig& cfg) {
    if (!grads.raw_space) throw std::logic_error("adam_step: gradients not chained to raw parameters");
    if (grads.size() != scene.size() || state.m.size() != scene.size())
        throw std::invalid_argument("adam_step: size mismatch");
    state.step += 1;
    const bool f32 = use_fp32();
    const Layout L(int64_t(scene.size()), scene.num_classes, scene.sh_degree);
    DBuf p(L.total(), f32), g(L.total(), f32), m(L.total(), f32), v(L.total(), f32);
    p.upload(pack_scene(scene, L));
    g.upload(pack_grads(grads, L));
    m.upload(pack_grads(state.m, L));
    v.upload(pack_grads(state.v, L));
    const auto lr = packed_lrs(cfg);
    rethrow(msplat_adam_step(context(), f32 ? MSPLAT_F32 : MSPLAT_F64, L.n, L.C, L.deg, p.p, g.p, m.p, v.p,
                             state.step, lr.data()));
    Scene out = unpack_scene(p.download(), L);
    scene.gaussians.swap(out.gaussians);
    unpack_grads(m.download(), L, state.m);
    unpack_grads(v.download(), L, state.v);
}

// prune (trainer.cpp:135-169): device mask + stable compaction.
size_t prune(Scene& scene, OptimizerState& state, const TrainConfig& cfg) {
    const bool f32 = use_fp32();
    const Layout L(int64_t(scene.size()), scene.num_classes, scene.sh_degree);
    DBuf p(L.total(), f32), m(L.total(), f32), v(L.total(), f32);
    p.upload(pack_scene(scene, L));
    m.upload(pack_grads(state.m, L));
    v.upload(pack_grads(state.v, L));
    ByteBuf keep(size_t(L.n));
    int64_t kept = 0;
    const msplat_scene s = scene_view(p.p, L, f32);
    const msplat_status st = msplat_prune_mask(context(), s.dtype, L.n, s.k, cfg.prune_threshold,
                                               cfg.prune_keep_small ? 1 : 0, static_cast<uint8_t*>(keep.p), &kept);
    if (st == MSPLAT_ERR_RUNTIME && kept == 0) throw_prune_all(cfg);
    rethrow(st);
    const Layout K(kept, L.C, L.deg);
    DBuf p2(K.total(), f32), m2(K.total(), f32), v2(K.total(), f32);
    const void* const in[3] = {p.p, m.p, v.p};
    void* const out[3] = {p2.p, m2.p, v2.p};
    rethrow(msplat_prune_compact(context(), s.dtype, L.n, L.C, L.deg, static_cast<const uint8_t*>(keep.p), kept, in,
                                 out, cfg.k_reset));
    const size_t removed = scene.size() - size_t(kept);
    scene = unpack_scene(p2.download(), K);
    Scene shape = scene;
    state.m.resize_zero(shape);
    state.v.resize_zero(shape);
    unpack_grads(m2.download(), K, state.m);
    unpack_grads(v2.download(), K, state.v);
    return removed;
}

// evaluate_frame_losses (trainer.cpp:171-264) on the device.
FrameLossResult evaluate_frame_losses(const MultimodalFrame& frame, const NormalState& nstate, const FrameRecord& gt,
                                      const CameraView& view, const TrainConfig& cfg) {
    require_gt(gt, cfg);
    const bool f32 = use_fp32();
    const int W = frame.width, H = frame.height, C = frame.num_classes;
    const size_t HW = size_t(W) * H;
    DBuf color(3 * HW, f32), depth(HW, f32), sem(size_t(C) * HW, f32), kmap(HW, f32), T(HW, f32), nrm(3 * HW, f32);
    color.upload(to_planar(frame.color));
    depth.upload(frame.depth.storage());
    if (C) sem.upload(to_planar(frame.semantics));
    kmap.upload(frame.kmap.storage());
    T.upload(frame.transmittance.storage());
    nrm.upload(to_planar(frame.normals));
    DeviceGT dgt(gt, f32);
    DBuf dC(3 * HW, f32), dD(HW, f32), dO(size_t(C) * HW, f32), dK(HW, f32);
    msplat_frame fr{color.p, depth.p, C ? sem.p : nullptr, kmap.p, T.p, nrm.p, nullptr};
    msplat_pixel_grads pg{dC.p, dD.p, C ? dO.p : nullptr, dK.p, nullptr};
    const msplat_camera cam = to_abi(view);
    const msplat_normal_config nc = to_abi(cfg.normal_config());
    msplat_loss_report rep{};
    rethrow(msplat_frame_losses(context(), f32 ? MSPLAT_F32 : MSPLAT_F64, C, &cam, &nc, &fr, &dgt.abi,
                                cfg.lambdas.data(), &pg, &rep));
    FrameLossResult out;
    out.report = from_abi(rep);
    out.pixel_grads.dcolor = from_planar(dC.download(), W, H, 3);
    out.pixel_grads.ddepth = from_planar(dD.download(), W, H, 1);
    out.pixel_grads.dsemantics = C ? from_planar(dO.download(), W, H, C) : GridF(W, H, 0, 0.0);
    out.pixel_grads.dkmap = from_planar(dK.download(), W, H, 1);
    out.normal_mask = Grid<std::uint8_t>(W, H, 1, 0);
    if (cfg.lambdas[2] > 0 && !gt.normal.empty())
        for (int y = 0; y < H; ++y)
            for (int x = 0; x < W; ++x)
                out.normal_mask.at(x, y) = nstate.valid.at(x, y) &&
                                           (gt.normal.at(x, y, 0) != 0 || gt.normal.at(x, y, 1) != 0 ||
                                            gt.normal.at(x, y, 2) != 0);
    return out;
}

// train (trainer.cpp:266-331), device-resident.
TrainResult train(const SceneDataset& dataset, const TrainConfig& cfg) {
    cfg.validate();
    const auto train_views = dataset.train_indices();
    if (train_views.size() < 2) throw std::invalid_argument("train: need at least 2 training views");
    if (dataset.points.empty()) throw std::invalid_argument("train: dataset has no initial points");
    if (dataset.point_colors.size() != dataset.points.size())
        throw std::invalid_argument("init_scene: point/color count mismatch");

    const bool f32 = use_fp32();
    const int dtype = f32 ? MSPLAT_F32 : MSPLAT_F64;
    const int C = dataset.num_classes;
    msplat_context* ctx = context();
    Layout L(int64_t(dataset.points.size()), C, cfg.sh_degree);
    const size_t cap = L.total();

    // init_scene straight into the device parameter buffer
    auto params = std::make_unique<DBuf>(cap, f32);
    {
        std::vector<double> pts(3 * size_t(L.n)), cols(3 * size_t(L.n));
        for (size_t i = 0; i < size_t(L.n); ++i)
            for (int j = 0; j < 3; ++j) {
                pts[3 * i + j] = dataset.points[i][j];
                cols[3 * i + j] = dataset.point_colors[i][j];
            }
        rethrow(msplat_init_scene(ctx, dtype, L.n, pts.data(), cols.data(), C, cfg.sh_degree, cfg.k_reset, params->p));
    }
    auto m = std::make_unique<DBuf>(cap, f32), v = std::make_unique<DBuf>(cap, f32);  // zero-initialised
    DBuf grads(cap, f32), last_good(cap, f32);
    Layout last_L = L;
    int64_t step = 0;

    // view schedule: round-robin over a seed-shuffled order (trainer.cpp:278-281)
    std::vector<int> order = train_views;
    std::mt19937_64 rng(cfg.seed);
    std::shuffle(order.begin(), order.end(), rng);

    // ground truth of the training frames, uploaded once
    std::vector<std::unique_ptr<DeviceGT>> gts(dataset.frames.size());
    for (int vi : train_views) gts[size_t(vi)] = std::make_unique<DeviceGT>(dataset.frames[size_t(vi)], f32);

    const msplat_render_config rc = to_abi(cfg.render_config());
    const msplat_normal_config nc = to_abi(cfg.normal_config());
    const auto lr = packed_lrs(cfg);
    // frame / pixel-gradient buffers sized for the largest view
    int Wm = 0, Hm = 0;
    for (int vi : train_views) {
        Wm = std::max(Wm, dataset.frames[size_t(vi)].view.width);
        Hm = std::max(Hm, dataset.frames[size_t(vi)].view.height);
    }
    const size_t HWm = size_t(Wm) * Hm;
    DBuf color(3 * HWm, f32), depth(HWm, f32), sem(size_t(C) * HWm, f32), kmap(HWm, f32), T(HWm, f32),
        nrm(3 * HWm, f32), dC(3 * HWm, f32), dD(HWm, f32), dO(size_t(C) * HWm, f32), dK(HWm, f32);
    ByteBuf contrib(HWm * 4), keep(size_t(L.n));
    msplat_replay* replay = nullptr;
    rethrow(msplat_replay_create(ctx, &replay));
    std::unique_ptr<msplat_replay, void (*)(msplat_replay*)> replay_guard(replay, msplat_replay_destroy);
    msplat_frame fr{color.p, depth.p, C ? sem.p : nullptr, kmap.p, T.p, nrm.p, static_cast<int32_t*>(contrib.p)};
    msplat_pixel_grads pg{dC.p, dD.p, C ? dO.p : nullptr, dK.p, nullptr};

    TrainResult result;
    result.log.reserve(size_t(cfg.iterations));
    const size_t R = f32 ? 4 : 8;
    for (int it = 1; it <= cfg.iterations; ++it) {
        const auto t0 = std::chrono::steady_clock::now();
        const int vi = order[size_t(it - 1) % order.size()];
        const FrameRecord& gt = dataset.frames[size_t(vi)];
        require_gt(gt, cfg);
        const msplat_camera cam = to_abi(gt.view);
        msplat_scene s = scene_view(params->p, L, f32);
        rethrow(msplat_rasterize(ctx, &s, &cam, &rc, &fr, replay));
        rethrow(msplat_estimate_normals(ctx, dtype, depth.p, T.p, &cam, &nc, nrm.p));
        msplat_loss_report rep{};
        rethrow(msplat_frame_losses(ctx, dtype, C, &cam, &nc, &fr, &gts[size_t(vi)]->abi, cfg.lambdas.data(), &pg,
                                    &rep));
        if (!std::isfinite(rep.combined)) {  // trainer.cpp:300-305: keep the last finite scene
            cuda_check(cudaMemcpy(params->p, last_good.p, last_L.total() * R, cudaMemcpyDeviceToDevice), "restore");
            L = last_L;
            result.halted_non_finite = true;
            break;
        }
        cuda_check(cudaMemcpy(last_good.p, params->p, L.total() * R, cudaMemcpyDeviceToDevice), "snapshot");
        last_L = L;
        msplat_grads g = grads_view(grads.p, L, f32);
        rethrow(msplat_rasterize_backward(ctx, &s, &cam, &fr, replay, &pg, &g));
        rethrow(msplat_chain_activations(ctx, &s, &g));
        ++step;
        rethrow(msplat_adam_step(ctx, dtype, L.n, L.C, L.deg, params->p, grads.p, m->p, v->p, step, lr.data()));
        if (cfg.prune_enabled && it % cfg.prune_interval == 0) {
            int64_t kept = 0;
            s = scene_view(params->p, L, f32);
            const msplat_status st = msplat_prune_mask(ctx, dtype, L.n, s.k, cfg.prune_threshold,
                                                       cfg.prune_keep_small ? 1 : 0, static_cast<uint8_t*>(keep.p),
                                                       &kept);
            if (st == MSPLAT_ERR_RUNTIME && kept == 0) throw_prune_all(cfg);
            rethrow(st);
            const Layout K(kept, L.C, L.deg);
            auto p2 = std::make_unique<DBuf>(K.total(), f32), m2 = std::make_unique<DBuf>(K.total(), f32),
                 v2 = std::make_unique<DBuf>(K.total(), f32);
            const void* const in[3] = {params->p, m->p, v->p};
            void* const out[3] = {p2->p, m2->p, v2->p};
            rethrow(msplat_prune_compact(ctx, dtype, L.n, L.C, L.deg, static_cast<const uint8_t*>(keep.p), kept, in,
                                         out, cfg.k_reset));
            params = std::move(p2);
            m = std::move(m2);
            v = std::move(v2);
            L = K;
        }
        rethrow(msplat_context_check(ctx));
        IterationLog entry;
        entry.iteration = it;
        entry.view_index = vi;
        entry.losses = from_abi(rep);
        entry.gaussian_count = size_t(L.n);
        entry.wall_ms = cfg.deterministic
                            ? 0.0
                            : std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        result.log.push_back(entry);
        result.completed_iterations = it;
    }
    std::vector<double> flat(L.total());
    if (L.total()) {
        if (f32) {
            std::vector<float> t(L.total());
            cuda_check(cudaMemcpy(t.data(), params->p, t.size() * 4, cudaMemcpyDeviceToHost), "download");
            flat.assign(t.begin(), t.end());
        } else {
            cuda_check(cudaMemcpy(flat.data(), params->p, flat.size() * 8, cudaMemcpyDeviceToHost), "download");
        }
    }
    result.scene = unpack_scene(flat, L);
    return result;
}

}  // namespace msplat
