// ref_adapter.cpp -- implements oracle/msplat_oracle.h on top of the
// reference's own C++ sources (compiled unmodified from
// /root/reference/proj/core/src with -Dmsplat=msplat_ref against
// third_party/eigen_subset).  TEST INFRASTRUCTURE ONLY: it lets the pytest
// parity suite and bench.py's reference arm call the real reference through a
// flat C ABI.  Every entry point marshals the flat arrays into the reference's
// AoS Eigen types, calls the reference function named in the comment, and
// marshals back.
#include "msplat_oracle.h"

#include "msplat/io_ply.hpp"
#include "msplat/metrics.hpp"
#include "msplat/normals.hpp"
#include "msplat/rasterizer.hpp"
#include "msplat/scene.hpp"
#include "msplat/trainer.hpp"

#include <chrono>
#include <cstring>
#include <stdexcept>
#include <string>

using namespace msplat;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

Scene to_scene(const mo_scene* s) {
    Scene sc;
    sc.num_classes = s->num_classes;
    sc.sh_degree = s->sh_degree;
    const int K = sc.sh_coeff_count(), C = s->num_classes;
    sc.gaussians.resize(size_t(s->n));
    for (int64_t i = 0; i < s->n; ++i) {
        auto& g = sc.gaussians[size_t(i)];
        g.position = Vec3(s->means[3 * i], s->means[3 * i + 1], s->means[3 * i + 2]);
        g.rotation = Vec4(s->quats[4 * i], s->quats[4 * i + 1], s->quats[4 * i + 2],
                          s->quats[4 * i + 3]);
        g.log_scale = Vec3(s->log_scales[3 * i], s->log_scales[3 * i + 1], s->log_scales[3 * i + 2]);
        g.opacity_logit = s->opacity_logits[i];
        g.sh = ShMatrix::Zero(3, K);
        for (int c = 0; c < 3; ++c)
            for (int j = 0; j < K; ++j)
                g.sh(c, j) = s->sh[(i * 3 + c) * K + j];
        g.semantic_logits = VecX::Zero(C);
        for (int c = 0; c < C; ++c)
            g.semantic_logits[c] = s->semantics[i * C + c];
        g.gradient_factor = s->k[i];
    }
    return sc;
}

CameraView to_camera(const mo_camera* c) {
    Mat3 R;
    R << c->R_c2w[0], c->R_c2w[1], c->R_c2w[2], c->R_c2w[3], c->R_c2w[4], c->R_c2w[5],
        c->R_c2w[6], c->R_c2w[7], c->R_c2w[8];
    return make_camera(c->fx, c->fy, c->cx, c->cy, c->width, c->height, R,
                       Vec3(c->t_c2w[0], c->t_c2w[1], c->t_c2w[2]));
}

RenderConfig to_cfg(const mo_render_cfg* c) {
    RenderConfig rc;
    rc.sigma_scale = c->sigma_scale;
    rc.background = Vec3(c->background[0], c->background[1], c->background[2]);
    rc.early_stop_transmittance = c->early_stop_transmittance;
    rc.early_termination = c->early_termination != 0;
    rc.threads = c->threads;
    return rc;
}

NormalConfig to_ncfg(const mo_normal_cfg* c) {
    NormalConfig nc;
    nc.step1 = c->step1;
    nc.step2 = c->step2;
    nc.fuse_lambda = c->fuse_lambda;
    nc.mask_threshold = c->mask_threshold;
    return nc;
}

GridF grid_from(const double* p, int W, int H, int C) {
    GridF g(W, H, C, 0.0);
    std::memcpy(g.data(), p, sizeof(double) * size_t(W) * H * C);
    return g;
}

void grid_to(const GridF& g, double* p) {
    if (p)
        std::memcpy(p, g.data(), sizeof(double) * g.size());
}

PixelGradients pix_from(int W, int H, int C, const double* dc, const double* dd, const double* ds,
                        const double* dk) {
    PixelGradients pg = PixelGradients::zero(W, H, C);
    std::memcpy(pg.dcolor.data(), dc, sizeof(double) * pg.dcolor.size());
    std::memcpy(pg.ddepth.data(), dd, sizeof(double) * pg.ddepth.size());
    if (C)
        std::memcpy(pg.dsemantics.data(), ds, sizeof(double) * pg.dsemantics.size());
    std::memcpy(pg.dkmap.data(), dk, sizeof(double) * pg.dkmap.size());
    return pg;
}

void grads_to(const GradientBuffer& b, int K, int C, mo_grads* o) {
    for (size_t i = 0; i < b.size(); ++i) {
        for (int j = 0; j < 3; ++j) {
            o->dposition[3 * i + j] = b.dposition[i][j];
            o->dscale[3 * i + j] = b.dscale[i][j];
        }
        for (int j = 0; j < 4; ++j)
            o->drotation[4 * i + j] = b.drotation[i][j];
        o->dopacity[i] = b.dopacity[i];
        for (int c = 0; c < 3; ++c)
            for (int j = 0; j < K; ++j)
                o->dsh[(i * 3 + c) * K + j] = b.dsh[i](c, j);
        for (int c = 0; c < C; ++c)
            o->dsemantics[i * C + c] = b.dsemantics[i][c];
        o->dk[i] = b.dk[i];
    }
}

GradientBuffer grads_from(const mo_grads* g, const Scene& sc, bool raw) {
    GradientBuffer b;
    b.resize_zero(sc);
    const int K = sc.sh_coeff_count(), C = sc.num_classes;
    for (size_t i = 0; i < sc.size(); ++i) {
        b.dposition[i] = Vec3(g->dposition[3 * i], g->dposition[3 * i + 1], g->dposition[3 * i + 2]);
        b.drotation[i] = Vec4(g->drotation[4 * i], g->drotation[4 * i + 1], g->drotation[4 * i + 2],
                              g->drotation[4 * i + 3]);
        b.dscale[i] = Vec3(g->dscale[3 * i], g->dscale[3 * i + 1], g->dscale[3 * i + 2]);
        b.dopacity[i] = g->dopacity[i];
        for (int c = 0; c < 3; ++c)
            for (int j = 0; j < K; ++j)
                b.dsh[i](c, j) = g->dsh[(i * 3 + c) * K + j];
        for (int c = 0; c < C; ++c)
            b.dsemantics[i][c] = g->dsemantics[i * C + c];
        b.dk[i] = g->dk[i];
    }
    b.raw_space = raw;
    return b;
}

} // namespace

extern "C" {

const char* mo_last_error(void) { return g_err.c_str(); }
const char* mo_impl_name(void) { return "reference"; }

// activate_scene + project_gaussian + eval_sh_color as prepare_view does
// (core/src/rasterizer.cpp:55-74).
int mo_preprocess(const mo_scene* s, const mo_camera* cam, uint8_t* visible, double* center,
                  double* cov, double* conic, double* sort_depth, double* radius, double* rgb,
                  uint8_t* clamped) {
    return guarded([&] {
        const Scene sc = to_scene(s);
        const CameraView view = to_camera(cam);
        sc.validate();
        const auto act = activate_scene(sc);
        for (size_t i = 0; i < sc.size(); ++i) {
            const auto sp = project_gaussian(act[i], view);
            if (visible)
                visible[i] = sp.has_value();
            if (!sp)
                continue;
            if (center) {
                center[2 * i] = sp->center.x();
                center[2 * i + 1] = sp->center.y();
            }
            if (cov)
                for (int r = 0; r < 2; ++r)
                    for (int c = 0; c < 2; ++c)
                        cov[4 * i + 2 * r + c] = sp->cov(r, c);
            if (conic) {
                conic[3 * i] = sp->conic(0, 0);
                conic[3 * i + 1] = sp->conic(0, 1);
                conic[3 * i + 2] = sp->conic(1, 1);
            }
            if (sort_depth)
                sort_depth[i] = sp->sort_depth;
            if (radius)
                radius[i] = sp->radius;
            const Vec3 to_g = act[i].position - view.t_cam_to_world;
            const Scalar norm = to_g.norm();
            const Vec3 dir = norm > 1e-12 ? Vec3(to_g / norm) : Vec3(0, 0, 1);
            const ShColor col = eval_sh_color(*act[i].sh, sc.sh_degree, dir);
            for (int c = 0; c < 3; ++c) {
                if (rgb)
                    rgb[3 * i + c] = col.rgb[c];
                if (clamped)
                    clamped[3 * i + c] = col.clamped[c];
            }
        }
    });
}

// bin_and_sort (core/src/rasterizer.cpp:14-45)
int64_t mo_bin(int64_t n, const uint8_t* visible, const double* center, const double* radius,
               const double* sort_depth, int width, int height, int64_t* tile_offsets,
               int32_t* values, int64_t capacity) {
    int64_t count = 0;
    const int st = guarded([&] {
        std::vector<std::optional<Splat2D>> splats(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) {
            if (!visible[i])
                continue;
            Splat2D sp;
            sp.center = Vec2(center[2 * i], center[2 * i + 1]);
            sp.radius = radius[i];
            sp.sort_depth = sort_depth[i];
            splats[size_t(i)] = sp;
        }
        const TileBins bins = bin_and_sort(splats, width, height);
        int64_t off = 0;
        for (size_t t = 0; t < bins.bins.size(); ++t) {
            if (tile_offsets)
                tile_offsets[t] = off;
            off += int64_t(bins.bins[t].size());
        }
        if (tile_offsets)
            tile_offsets[bins.bins.size()] = off;
        count = off;
        if (values && capacity >= count) {
            int64_t k = 0;
            for (const auto& b : bins.bins)
                for (int v : b)
                    values[k++] = v;
        }
    });
    return st ? -st : count;
}

// rasterize (core/src/rasterizer.cpp:87-205)
int mo_render(const mo_scene* s, const mo_camera* cam, const mo_render_cfg* cfg, double* color,
              double* depth, double* semantics, double* kmap, double* transmittance,
              int32_t* contributors, int32_t* terminus, double* weight_sums) {
    return guarded([&] {
        const Scene sc = to_scene(s);
        ReplayState replay;
        const MultimodalFrame f = rasterize(sc, to_camera(cam), to_cfg(cfg), &replay);
        grid_to(f.color, color);
        grid_to(f.depth, depth);
        if (s->num_classes)
            grid_to(f.semantics, semantics);
        grid_to(f.kmap, kmap);
        grid_to(f.transmittance, transmittance);
        if (contributors)
            std::memcpy(contributors, f.contributors.data(), sizeof(int) * f.contributors.size());
        if (terminus)
            std::memcpy(terminus, replay.terminus.data(), sizeof(int) * replay.terminus.size());
        if (weight_sums)
            for (size_t i = 0; i < sc.size(); ++i)
                weight_sums[i] = replay.weight_sums[i];
    });
}

// estimate_normals (core/src/normals.cpp:28-101)
int mo_normals(const double* depth, const double* transmittance, const mo_camera* cam,
               const mo_normal_cfg* ncfg, double* normals, uint8_t* valid, uint8_t* flipped) {
    return guarded([&] {
        const CameraView view = to_camera(cam);
        const int W = view.width, H = view.height;
        GridF nrm;
        const NormalState st = estimate_normals(grid_from(depth, W, H, 1),
                                                grid_from(transmittance, W, H, 1), view,
                                                to_ncfg(ncfg), nrm);
        grid_to(nrm, normals);
        if (valid)
            std::memcpy(valid, st.valid.data(), st.valid.size());
        if (flipped)
            std::memcpy(flipped, st.flipped.data(), st.flipped.size());
    });
}

// normals_backward (core/src/normals.cpp:103-152)
int mo_normals_backward(const double* dL_dnormals, const double* depth,
                        const double* transmittance, const mo_camera* cam,
                        const mo_normal_cfg* ncfg, double* dD) {
    return guarded([&] {
        const CameraView view = to_camera(cam);
        const int W = view.width, H = view.height;
        GridF nrm;
        const NormalState st = estimate_normals(grid_from(depth, W, H, 1),
                                                grid_from(transmittance, W, H, 1), view,
                                                to_ncfg(ncfg), nrm);
        grid_to(normals_backward(grid_from(dL_dnormals, W, H, 3), st, view), dD);
    });
}

// rasterize + rasterize_backward (core/src/rasterizer_backward.cpp:127-264)
int mo_backward(const mo_scene* s, const mo_camera* cam, const mo_render_cfg* cfg,
                const double* dcolor, const double* ddepth, const double* dsemantics,
                const double* dkmap, mo_grads* out) {
    return guarded([&] {
        const Scene sc = to_scene(s);
        const CameraView view = to_camera(cam);
        ReplayState replay;
        const MultimodalFrame f = rasterize(sc, view, to_cfg(cfg), &replay);
        const PixelGradients pg =
            pix_from(view.width, view.height, sc.num_classes, dcolor, ddepth, dsemantics, dkmap);
        const GradientBuffer g = rasterize_backward(sc, view, f, replay, pg);
        grads_to(g, sc.sh_coeff_count(), sc.num_classes, out);
    });
}

// chain_activations (core/src/scene.cpp:108-129)
int mo_chain(const mo_scene* s, mo_grads* g) {
    return guarded([&] {
        const Scene sc = to_scene(s);
        GradientBuffer b = grads_from(g, sc, false);
        chain_activations(b, sc);
        grads_to(b, sc.sh_coeff_count(), sc.num_classes, g);
    });
}

// The benchmark unit, exactly the calls train() makes per iteration minus the
// losses (trainer.cpp:295-309): rasterize, estimate_normals,
// normals_backward merged into ddepth (seed 1), rasterize_backward,
// chain_activations.  Marshalling is outside the timed stages.
int mo_fwd_bwd(const mo_scene* s, const mo_camera* cam, const mo_render_cfg* cfg,
               const mo_normal_cfg* ncfg, const double* dcolor, const double* ddepth,
               const double* dsemantics, const double* dkmap, const double* dnormals,
               double* color, double* depth, double* semantics, double* kmap,
               double* transmittance, double* normals, mo_grads* out, double* ms_out) {
    return guarded([&] {
        using clk = std::chrono::steady_clock;
        auto ms = [](clk::time_point a, clk::time_point b) {
            return std::chrono::duration<double, std::milli>(b - a).count();
        };
        const Scene sc = to_scene(s);
        const CameraView view = to_camera(cam);
        const int W = view.width, H = view.height, C = sc.num_classes;
        PixelGradients pg = pix_from(W, H, C, dcolor, ddepth, dsemantics, dkmap);
        const GridF dN = grid_from(dnormals, W, H, 3);
        const RenderConfig rc = to_cfg(cfg);
        const NormalConfig nc = to_ncfg(ncfg);

        const auto t0 = clk::now();
        ReplayState replay;
        MultimodalFrame f = rasterize(sc, view, rc, &replay);
        const auto t1 = clk::now();
        const NormalState nst = estimate_normals(f.depth, f.transmittance, view, nc, f.normals);
        const auto t2 = clk::now();
        const GridF dD = normals_backward(dN, nst, view);
        for (size_t i = 0; i < pg.ddepth.size(); ++i)
            pg.ddepth.storage()[i] += 1.0 * dD.storage()[i];
        const auto t3 = clk::now();
        GradientBuffer g = rasterize_backward(sc, view, f, replay, pg);
        const auto t4 = clk::now();
        chain_activations(g, sc);
        const auto t5 = clk::now();
        if (ms_out) {
            ms_out[0] = ms(t0, t1);
            ms_out[1] = ms(t1, t2);
            ms_out[2] = ms(t2, t3);
            ms_out[3] = ms(t3, t4);
            ms_out[4] = ms(t4, t5);
        }
        grid_to(f.color, color);
        grid_to(f.depth, depth);
        if (C)
            grid_to(f.semantics, semantics);
        grid_to(f.kmap, kmap);
        grid_to(f.transmittance, transmittance);
        grid_to(f.normals, normals);
        if (out)
            grads_to(g, sc.sh_coeff_count(), C, out);
    });
}

// adam_step (core/src/trainer.cpp:98-133)
int mo_adam(int64_t n, int num_classes, int sh_degree, double* means, double* quats,
            double* log_scales, double* opacity_logits, double* sh, double* semantics, double* k,
            const mo_grads* g, mo_grads* m, mo_grads* v, int64_t step, const double* lr) {
    return guarded([&] {
        mo_scene s{n, num_classes, sh_degree, means, quats, log_scales, opacity_logits, sh,
                   semantics, k};
        Scene sc = to_scene(&s);
        OptimizerState st;
        st.m = grads_from(m, sc, true);
        st.v = grads_from(v, sc, true);
        st.step = step - 1;
        TrainConfig tc;
        tc.lr_position = lr[0];
        tc.lr_rotation = lr[1];
        tc.lr_scale = lr[2];
        tc.lr_opacity = lr[3];
        tc.lr_sh = lr[4];
        tc.lr_semantics = lr[5];
        tc.lr_k = lr[6];
        adam_step(sc, grads_from(g, sc, true), st, tc);
        const int K = sc.sh_coeff_count();
        for (int64_t i = 0; i < n; ++i) {
            const auto& p = sc.gaussians[size_t(i)];
            for (int j = 0; j < 3; ++j) {
                means[3 * i + j] = p.position[j];
                log_scales[3 * i + j] = p.log_scale[j];
            }
            for (int j = 0; j < 4; ++j)
                quats[4 * i + j] = p.rotation[j];
            opacity_logits[i] = p.opacity_logit;
            for (int c = 0; c < 3; ++c)
                for (int j = 0; j < K; ++j)
                    sh[(i * 3 + c) * K + j] = p.sh(c, j);
            for (int c = 0; c < num_classes; ++c)
                semantics[i * num_classes + c] = p.semantic_logits[c];
            k[i] = p.gradient_factor;
        }
        grads_to(st.m, K, num_classes, m);
        grads_to(st.v, K, num_classes, v);
    });
}

// prune keep mask (core/src/trainer.cpp:135-147): run prune() on a scene whose
// only payload is k, then recover which indices survived from the compaction.
int64_t mo_prune_mask(int64_t n, const double* k, double threshold, int keep_small,
                      uint8_t* keep) {
    int64_t kept = 0;
    const int st = guarded([&] {
        Scene sc;
        sc.sh_degree = 0;
        sc.num_classes = 0;
        sc.gaussians.resize(size_t(n));
        for (int64_t i = 0; i < n; ++i) {
            auto& g = sc.gaussians[size_t(i)];
            g.sh = ShMatrix::Zero(3, 1);
            g.semantic_logits = VecX::Zero(0);
            g.gradient_factor = k[i];
            g.opacity_logit = double(i); // tag to recover survivors
        }
        OptimizerState os = OptimizerState::init(sc);
        TrainConfig tc;
        tc.prune_threshold = threshold;
        tc.prune_keep_small = keep_small != 0;
        prune(sc, os, tc);
        std::memset(keep, 0, size_t(n));
        for (const auto& g : sc.gaussians)
            keep[int64_t(g.opacity_logit)] = 1;
        kept = int64_t(sc.size());
    });
    return st ? -st : kept;
}

} // extern "C"

// evaluate_frame_losses (core/src/trainer.cpp:171-264) on a given frame, with
// the normals estimated first as train() does (trainer.cpp:296-297).
extern "C" int mo_frame_losses(int W, int H, int C, const mo_camera* cam, const mo_normal_cfg* ncfg,
                               const double* color, const double* depth, const double* semantics,
                               const double* kmap, const double* transmittance, const double* gt_rgb,
                               const double* gt_depth, const double* gt_normal, const uint8_t* gt_labels,
                               const double* lambdas, double* report, double* dcolor, double* ddepth,
                               double* dsemantics, double* dkmap, double* normals_out) {
    return guarded([&] {
        const CameraView view = to_camera(cam);
        MultimodalFrame f;
        f.width = W;
        f.height = H;
        f.num_classes = C;
        f.color = grid_from(color, W, H, 3);
        f.depth = grid_from(depth, W, H, 1);
        f.semantics = C ? grid_from(semantics, W, H, C) : GridF(W, H, 0, 0.0);
        f.kmap = grid_from(kmap, W, H, 1);
        f.transmittance = grid_from(transmittance, W, H, 1);
        const NormalState ns = estimate_normals(f.depth, f.transmittance, view, to_ncfg(ncfg), f.normals);
        if (normals_out)
            grid_to(f.normals, normals_out);
        FrameRecord gt;
        if (gt_rgb)
            gt.rgb = grid_from(gt_rgb, W, H, 3);
        if (gt_depth)
            gt.depth = grid_from(gt_depth, W, H, 1);
        if (gt_normal)
            gt.normal = grid_from(gt_normal, W, H, 3);
        if (gt_labels) {
            gt.labels = GridU8(W, H, 1, 0);
            std::memcpy(gt.labels.data(), gt_labels, size_t(W) * H);
        }
        TrainConfig cfg;
        for (int i = 0; i < 6; ++i)
            cfg.lambdas[size_t(i)] = lambdas[i];
        const FrameLossResult r = evaluate_frame_losses(f, ns, gt, view, cfg);
        const LossReport& q = r.report;
        const double rep[18] = {q.l1, q.ssim, q.depth, q.normal, q.seg, q.k, q.combined, q.ratio_ssim,
                                q.ratio_normal, q.ratio_depth, q.ratio_seg, q.ratio_k, q.seed_l1, q.seed_ssim,
                                q.seed_depth, q.seed_normal, q.seed_seg, q.seed_k};
        if (report)
            std::memcpy(report, rep, sizeof rep);
        grid_to(r.pixel_grads.dcolor, dcolor);
        grid_to(r.pixel_grads.ddepth, ddepth);
        if (C && dsemantics)
            grid_to(r.pixel_grads.dsemantics, dsemantics);
        grid_to(r.pixel_grads.dkmap, dkmap);
    });
}

// train (core/src/trainer.cpp:266-331) on flat arrays; the same contract as the
// drop-in's msplat_train_flat (cfg: 32 doubles, see there; log rows of 21).
extern "C" int mo_train(int n_points, const double* points, const double* colors, int num_classes, int n_frames,
                        const mo_camera* cams, const double* rgb, const double* depth, const double* normal,
                        const uint8_t* labels, const uint8_t* is_test, const double* c, double* params_out,
                        int64_t* n_out, double* log_out, int* completed, int* halted) {
    return guarded([&] {
        SceneDataset ds;
        ds.num_classes = num_classes;
        for (int i = 0; i < n_points; ++i) {
            ds.points.emplace_back(points[3 * i], points[3 * i + 1], points[3 * i + 2]);
            ds.point_colors.emplace_back(colors[3 * i], colors[3 * i + 1], colors[3 * i + 2]);
        }
        size_t o3 = 0, o1 = 0;
        for (int f = 0; f < n_frames; ++f) {
            FrameRecord fr;
            fr.view = to_camera(&cams[f]);
            fr.split = is_test && is_test[f] ? "test" : "train";
            const int W = cams[f].width, H = cams[f].height;
            const size_t HW = size_t(W) * H;
            fr.rgb = grid_from(rgb + o3, W, H, 3);
            fr.depth = grid_from(depth + o1, W, H, 1);
            fr.normal = grid_from(normal + o3, W, H, 3);
            fr.labels = GridU8(W, H, 1, 0);
            std::memcpy(fr.labels.data(), labels + o1, HW);
            o3 += 3 * HW;
            o1 += HW;
            ds.frames.push_back(std::move(fr));
            ds.width = W;
            ds.height = H;
        }
        TrainConfig t;
        t.iterations = int(c[0]);
        t.lr_position = c[1];
        t.lr_rotation = c[2];
        t.lr_scale = c[3];
        t.lr_opacity = c[4];
        t.lr_sh = c[5];
        t.lr_semantics = c[6];
        t.lr_k = c[7];
        for (int i = 0; i < 6; ++i)
            t.lambdas[size_t(i)] = c[8 + i];
        t.prune_interval = int(c[14]);
        t.prune_threshold = c[15];
        t.prune_enabled = c[16] != 0;
        t.prune_keep_small = c[17] != 0;
        t.k_reset = c[18];
        t.step1 = int(c[19]);
        t.step2 = int(c[20]);
        t.lambda_fuse = c[21];
        t.mask_threshold = c[22];
        t.sigma_scale = c[23];
        t.early_stop_transmittance = c[24];
        t.background = Vec3(c[25], c[26], c[27]);
        t.sh_degree = int(c[28]);
        t.seed = uint64_t(c[29]);
        t.threads = int(c[30]);
        t.deterministic = c[31] != 0;
        const TrainResult r = train(ds, t);
        const Scene& s = r.scene;
        const int K = s.sh_coeff_count(), C = s.num_classes;
        const int64_t n = int64_t(s.size());
        const int64_t sizes[7] = {3, 4, 3, 1, 1, 3 * K, C};
        int64_t off[8];
        off[0] = 0;
        for (int i = 0; i < 7; ++i)
            off[i + 1] = off[i] + n * sizes[i];
        for (int64_t i = 0; i < n; ++i) {
            const GaussianPrimitive& g = s.gaussians[size_t(i)];
            for (int j = 0; j < 3; ++j) {
                params_out[off[0] + 3 * i + j] = g.position[j];
                params_out[off[2] + 3 * i + j] = g.log_scale[j];
            }
            for (int j = 0; j < 4; ++j)
                params_out[off[1] + 4 * i + j] = g.rotation[j];
            params_out[off[3] + i] = g.opacity_logit;
            params_out[off[4] + i] = g.gradient_factor;
            for (int ch = 0; ch < 3; ++ch)
                for (int j = 0; j < K; ++j)
                    params_out[off[5] + (3 * i + ch) * K + j] = g.sh(ch, j);
            for (int ch = 0; ch < C; ++ch)
                params_out[off[6] + i * C + ch] = g.semantic_logits[ch];
        }
        *n_out = n;
        for (size_t it = 0; it < r.log.size(); ++it) {
            const IterationLog& e = r.log[it];
            const LossReport& q = e.losses;
            const double vals[21] = {double(e.iteration), double(e.view_index), double(e.gaussian_count), q.l1,
                                     q.ssim, q.depth, q.normal, q.seg, q.k, q.combined, q.ratio_ssim,
                                     q.ratio_normal, q.ratio_depth, q.ratio_seg, q.ratio_k, q.seed_l1, q.seed_ssim,
                                     q.seed_depth, q.seed_normal, q.seed_seg, q.seed_k};
            std::memcpy(log_out + it * 21, vals, sizeof vals);
        }
        *completed = r.completed_iterations;
        *halted = r.halted_non_finite ? 1 : 0;
    });
}

// metrics.cpp:68-187 through the reference's own functions.
extern "C" int mo_metrics(int W, int H, int C, const double* color, const double* gt_rgb, const double* depth,
                          const double* gt_depth, const uint8_t* depth_mask, const double* normals,
                          const double* gt_normal, const uint8_t* normal_mask, const double* semantics,
                          const uint8_t* gt_labels, const uint8_t* label_mask, double* vals, int* has) {
    return guarded([&] {
        for (int i = 0; i < 6; ++i) {
            vals[i] = 0;
            has[i] = 0;
        }
        auto mask_of = [&](const uint8_t* m) {
            GridU8 g(W, H, 1, 0);
            std::memcpy(g.data(), m, size_t(W) * H);
            return g;
        };
        auto set = [&](int i, std::optional<Scalar> v) {
            if (v) {
                vals[i] = *v;
                has[i] = 1;
            }
        };
        if (color && gt_rgb) {
            const GridF a = grid_from(color, W, H, 3), b = grid_from(gt_rgb, W, H, 3);
            set(0, psnr(a, b));
            set(1, ssim_metric(a, b));
        }
        if (depth && gt_depth && depth_mask) {
            const GridF d = grid_from(depth, W, H, 1), g = grid_from(gt_depth, W, H, 1);
            const GridU8 m = mask_of(depth_mask);
            set(2, abs_rel(d, g, m));
            set(3, rmse(d, g, m));
        }
        if (normals && gt_normal && normal_mask)
            set(4, cos_simi(grid_from(normals, W, H, 3), grid_from(gt_normal, W, H, 3), mask_of(normal_mask)));
        if (semantics && gt_labels && label_mask && C > 0)
            set(5, miou(argmax_labels(grid_from(semantics, W, H, C)), mask_of(gt_labels), mask_of(label_mask), C));
    });
}

// io_ply.cpp through the reference (save_scene_ply / load_scene_ply).
extern "C" int mo_ply_save(const char* path, const mo_scene* s) {
    return guarded([&] { save_scene_ply(path, to_scene(s)); });
}

// Loads into the packed layout (means quats log_scales opacity k sh sem).
extern "C" int mo_ply_load(const char* path, int64_t cap, double* packed, int64_t* n_out, int* C_out, int* deg_out) {
    return guarded([&] {
        const Scene s = load_scene_ply(path);
        const int K = s.sh_coeff_count(), C = s.num_classes;
        const int64_t n = int64_t(s.size());
        const int64_t sizes[7] = {3, 4, 3, 1, 1, 3 * K, C};
        int64_t off[8];
        off[0] = 0;
        for (int i = 0; i < 7; ++i)
            off[i + 1] = off[i] + n * sizes[i];
        *n_out = n;
        *C_out = C;
        *deg_out = s.sh_degree;
        if (off[7] > cap)
            return;
        for (int64_t i = 0; i < n; ++i) {
            const GaussianPrimitive& g = s.gaussians[size_t(i)];
            for (int j = 0; j < 3; ++j) {
                packed[off[0] + 3 * i + j] = g.position[j];
                packed[off[2] + 3 * i + j] = g.log_scale[j];
            }
            for (int j = 0; j < 4; ++j)
                packed[off[1] + 4 * i + j] = g.rotation[j];
            packed[off[3] + i] = g.opacity_logit;
            packed[off[4] + i] = g.gradient_factor;
            for (int ch = 0; ch < 3; ++ch)
                for (int j = 0; j < K; ++j)
                    packed[off[5] + (3 * i + ch) * K + j] = g.sh(ch, j);
            for (int ch = 0; ch < C; ++ch)
                packed[off[6] + i * C + ch] = g.semantic_logits[ch];
        }
    });
}
