// msplat C++ drop-in: a flat C entry point for train() (non-C++ callers: the
// Python binding, the parity tests).  Arrays in, arrays out; no C++ types
// cross it.  Parameters come back in the msplat_param_layout order.
#include <cstring>
#include <stdexcept>

#include "msplat/trainer.hpp"
#include "msplat_b200.h"

namespace {

// TrainConfig from 32 doubles: iterations, lr x7 (position rotation scale
// opacity sh semantics k), lambdas x6, prune_interval, prune_threshold,
// prune_enabled, prune_keep_small, k_reset, step1, step2, lambda_fuse,
// mask_threshold, sigma_scale, early_stop_transmittance, background x3,
// sh_degree, seed, threads, deterministic.
msplat::TrainConfig config_from(const double* c) {
    msplat::TrainConfig t;
    t.iterations = int(c[0]);
    t.lr_position = c[1];
    t.lr_rotation = c[2];
    t.lr_scale = c[3];
    t.lr_opacity = c[4];
    t.lr_sh = c[5];
    t.lr_semantics = c[6];
    t.lr_k = c[7];
    for (int i = 0; i < 6; ++i) t.lambdas[size_t(i)] = c[8 + i];
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
    t.background = msplat::Vec3(c[25], c[26], c[27]);
    t.sh_degree = int(c[28]);
    t.seed = uint64_t(c[29]);
    t.threads = int(c[30]);
    t.deterministic = c[31] != 0;
    return t;
}

thread_local std::string g_err;

}  // namespace

extern "C" __attribute__((visibility("default"))) const char* msplat_train_last_error() { return g_err.c_str(); }

// Returns 0, or 1 invalid_argument / 2 runtime_error / 3 logic_error.
extern "C" __attribute__((visibility("default"))) int msplat_train_flat(
    int n_points, const double* points, const double* colors, int num_classes, int n_frames,
    const msplat_camera* cams, const double* rgb, const double* depth, const double* normal, const uint8_t* labels,
    const uint8_t* is_test, const double* cfg, double* params_out, int64_t* n_out, double* log_out,
    int* completed, int* halted) {
    try {
        using namespace msplat;
        SceneDataset ds;
        ds.num_classes = num_classes;
        for (int i = 0; i < n_points; ++i) {
            ds.points.emplace_back(points[3 * i], points[3 * i + 1], points[3 * i + 2]);
            ds.point_colors.emplace_back(colors[3 * i], colors[3 * i + 1], colors[3 * i + 2]);
        }
        size_t o3 = 0, o1 = 0;
        for (int f = 0; f < n_frames; ++f) {
            const msplat_camera& c = cams[f];
            Mat3 R;
            R << c.R_c2w[0], c.R_c2w[1], c.R_c2w[2], c.R_c2w[3], c.R_c2w[4], c.R_c2w[5], c.R_c2w[6], c.R_c2w[7],
                c.R_c2w[8];
            FrameRecord fr;
            fr.view = make_camera(c.fx, c.fy, c.cx, c.cy, c.width, c.height, R, Vec3(c.t_c2w[0], c.t_c2w[1], c.t_c2w[2]));
            fr.split = is_test && is_test[f] ? "test" : "train";
            const int W = c.width, H = c.height;
            const size_t HW = size_t(W) * H;
            fr.rgb = GridF(W, H, 3, 0.0);
            std::memcpy(fr.rgb.data(), rgb + o3, HW * 3 * 8);
            fr.depth = GridF(W, H, 1, 0.0);
            std::memcpy(fr.depth.data(), depth + o1, HW * 8);
            fr.normal = GridF(W, H, 3, 0.0);
            std::memcpy(fr.normal.data(), normal + o3, HW * 3 * 8);
            fr.labels = GridU8(W, H, 1, 0);
            std::memcpy(fr.labels.data(), labels + o1, HW);
            o3 += 3 * HW;
            o1 += HW;
            ds.frames.push_back(std::move(fr));
            ds.width = W;
            ds.height = H;
        }
        const TrainResult r = train(ds, config_from(cfg));
        const Scene& s = r.scene;
        const int K = s.sh_coeff_count(), C = s.num_classes;
        const int64_t n = int64_t(s.size());
        int64_t off[8];
        msplat_param_layout(n, C, s.sh_degree, off);
        for (int64_t i = 0; i < n; ++i) {
            const GaussianPrimitive& g = s.gaussians[size_t(i)];
            for (int j = 0; j < 3; ++j) {
                params_out[off[0] + 3 * i + j] = g.position[j];
                params_out[off[2] + 3 * i + j] = g.log_scale[j];
            }
            for (int j = 0; j < 4; ++j) params_out[off[1] + 4 * i + j] = g.rotation[j];
            params_out[off[3] + i] = g.opacity_logit;
            params_out[off[4] + i] = g.gradient_factor;
            for (int c = 0; c < 3; ++c)
                for (int j = 0; j < K; ++j) params_out[off[5] + (3 * i + c) * K + j] = g.sh(c, j);
            for (int c = 0; c < C; ++c) params_out[off[6] + i * C + c] = g.semantic_logits[c];
        }
        *n_out = n;
        for (size_t it = 0; it < r.log.size(); ++it) {
            const IterationLog& e = r.log[it];
            double* row = log_out + it * 21;
            const LossReport& q = e.losses;
            const double vals[21] = {double(e.iteration), double(e.view_index), double(e.gaussian_count), q.l1,
                                     q.ssim, q.depth, q.normal, q.seg, q.k, q.combined, q.ratio_ssim,
                                     q.ratio_normal, q.ratio_depth, q.ratio_seg, q.ratio_k, q.seed_l1, q.seed_ssim,
                                     q.seed_depth, q.seed_normal, q.seed_seg, q.seed_k};
            std::memcpy(row, vals, sizeof vals);
        }
        *completed = r.completed_iterations;
        *halted = r.halted_non_finite ? 1 : 0;
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}
