/*
 * msplat_oracle.h -- flat C interface of the CPU parity oracle.
 *
 * TEST INFRASTRUCTURE ONLY.  Two libraries implement exactly this interface:
 *   oracle/liboracle.so          -- msplat_oracle.c, a plain-C double-precision
 *                                   restatement of the reference hot path;
 *   oracle/_ref/libmsplat_ref.so -- the reference's own C++ sources
 *                                   (/root/reference/proj/core/src) compiled
 *                                   unmodified against third_party/eigen_subset,
 *                                   behind ref_adapter.cpp.
 * tests/ check the two against each other (bit-exact binning, <=1e-12 floats)
 * and then use them as the checker for the CUDA path.  Nothing in the product
 * (paper_2510_12174_b200/) links or calls this.
 *
 * Conventions (all host memory, double unless noted):
 *   scene:  means[n][3], quats[n][4] (w,x,y,z, raw), log_scales[n][3],
 *           opacity_logits[n], sh[n][3][K] (row per colour channel, K=(d+1)^2),
 *           semantics[n][C], k[n]   (reference msplat/scene.hpp:14-22)
 *   camera: pinhole + cam->world pose, R row-major (msplat/camera.hpp:8-32)
 *   pixel grids: HWC like the reference Grid (msplat/types.hpp:40-41)
 *   status: 0 ok, 1 invalid_argument, 2 runtime_error, 3 logic_error;
 *           mo_last_error() holds the message (reference exception text).
 */
#ifndef MSPLAT_ORACLE_H
#define MSPLAT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int64_t n;
    int num_classes;
    int sh_degree;
    const double* means;
    const double* quats;
    const double* log_scales;
    const double* opacity_logits;
    const double* sh;
    const double* semantics;
    const double* k;
} mo_scene;

typedef struct {
    double fx, fy, cx, cy;
    int width, height;
    double R_c2w[9];
    double t_c2w[3];
} mo_camera;

typedef struct {
    double sigma_scale;
    double background[3];
    double early_stop_transmittance;
    int early_termination;
    int threads; /* reference RenderConfig::threads (only the _ref build uses it) */
} mo_render_cfg;

typedef struct {
    int step1, step2;
    double fuse_lambda;
    double mask_threshold;
} mo_normal_cfg;

typedef struct {
    double* dposition; /* [n][3] */
    double* drotation; /* [n][4] */
    double* dscale;    /* [n][3] */
    double* dopacity;  /* [n]    */
    double* dsh;       /* [n][3][K] */
    double* dsemantics;/* [n][C] */
    double* dk;        /* [n]    */
} mo_grads;

const char* mo_last_error(void);
const char* mo_impl_name(void);

/* Per-Gaussian preprocess (activate + project_gaussian + eval_sh_color). */
int mo_preprocess(const mo_scene* s, const mo_camera* cam, uint8_t* visible, double* center,
                  double* cov /*[n][4] row-major*/, double* conic /*[n][3] xx,xy,yy*/,
                  double* sort_depth, double* radius, double* rgb, uint8_t* clamped);

/* bin_and_sort on explicit splats.  Writes tile_offsets[tiles+1]; writes the
 * concatenated per-tile lists into values when capacity suffices.  Returns the
 * instance count I (>= 0) or a negative status. */
int64_t mo_bin(int64_t n, const uint8_t* visible, const double* center, const double* radius,
               const double* sort_depth, int width, int height, int64_t* tile_offsets,
               int32_t* values, int64_t capacity);

/* rasterize(): any output pointer may be NULL. */
int mo_render(const mo_scene* s, const mo_camera* cam, const mo_render_cfg* cfg, double* color,
              double* depth, double* semantics, double* kmap, double* transmittance,
              int32_t* contributors, int32_t* terminus, double* weight_sums);

/* estimate_normals(): normals [H][W][3], valid/flipped [H][W] (may be NULL). */
int mo_normals(const double* depth, const double* transmittance, const mo_camera* cam,
               const mo_normal_cfg* ncfg, double* normals, uint8_t* valid, uint8_t* flipped);

/* normals_backward() after an estimate_normals on the same depth/T. */
int mo_normals_backward(const double* dL_dnormals, const double* depth,
                        const double* transmittance, const mo_camera* cam,
                        const mo_normal_cfg* ncfg, double* dD);

/* rasterize() + rasterize_backward(); gradients in activated space. */
int mo_backward(const mo_scene* s, const mo_camera* cam, const mo_render_cfg* cfg,
                const double* dcolor, const double* ddepth, const double* dsemantics,
                const double* dkmap, mo_grads* out);

/* chain_activations() in place. */
int mo_chain(const mo_scene* s, mo_grads* g);

/* The benchmark unit: rasterize, estimate_normals, normals_backward(dN) merged
 * into ddepth with seed 1, rasterize_backward, chain_activations.  Frame
 * outputs may be NULL.  ms_out[5] (optional) = per-stage wall milliseconds. */
int mo_fwd_bwd(const mo_scene* s, const mo_camera* cam, const mo_render_cfg* cfg,
               const mo_normal_cfg* ncfg, const double* dcolor, const double* ddepth,
               const double* dsemantics, const double* dkmap, const double* dnormals,
               double* color, double* depth, double* semantics, double* kmap,
               double* transmittance, double* normals, mo_grads* out, double* ms_out);

/* evaluate_frame_losses (trainer.cpp:171-264) on a rendered frame: normals are
 * estimated from depth/T first (estimate_normals), exactly as the trainer does,
 * then l1_rgb, ssim_loss, normal_cosine, depth_l1, cross_entropy_seg,
 * gradient_factor_loss and combine (losses.cpp).  All maps HWC; ground truth
 * NULL = absent; lambdas[6] = (l1, ssim, normal, depth, seg, k).  report[18] in
 * LossReport order; pixel gradients HWC (dsemantics may be NULL when C = 0);
 * normals_out (optional) receives the estimated normals. */
int mo_frame_losses(int width, int height, int num_classes, const mo_camera* cam, const mo_normal_cfg* ncfg,
                    const double* color, const double* depth, const double* semantics, const double* kmap,
                    const double* transmittance, const double* gt_rgb, const double* gt_depth,
                    const double* gt_normal, const uint8_t* gt_labels, const double* lambdas, double* report,
                    double* dcolor, double* ddepth, double* dsemantics, double* dkmap, double* normals_out);

/* Image metrics (core/src/metrics.cpp:68-187), HWC inputs; a metric whose
 * inputs are NULL is skipped.  vals[6] = psnr, ssim, abs_rel, rmse, cos_simi,
 * miou; has[6] = 0 for nullopt / skipped. */
int mo_metrics(int width, int height, int num_classes, const double* color, const double* gt_rgb,
               const double* depth, const double* gt_depth, const uint8_t* depth_mask, const double* normals,
               const double* gt_normal, const uint8_t* normal_mask, const double* semantics,
               const uint8_t* gt_labels, const uint8_t* label_mask, double* vals, int* has);

/* Adam on raw parameters (trainer.cpp:90-133).  params/grads/m/v share the
 * scene layout; lr[7] = position, rotation, scale, opacity, sh, semantics, k. */
int mo_adam(int64_t n, int num_classes, int sh_degree, double* means, double* quats,
            double* log_scales, double* opacity_logits, double* sh, double* semantics,
            double* k, const mo_grads* g, mo_grads* m, mo_grads* v, int64_t step,
            const double* lr);

/* prune() keep mask (trainer.cpp:135-147); returns kept count or -status. */
int64_t mo_prune_mask(int64_t n, const double* k, double threshold, int keep_small,
                      uint8_t* keep);

#ifdef __cplusplus
}
#endif
#endif
