// Kernel argument structs and launchers shared by the msplat CUDA translation
// units (preprocess.cu, binning.cu, forward.cu, normals.cu, backward.cu,
// optim.cu) and the C-ABI layer (cabi.cu).
#pragma once

#include <atomic>

#include <string>

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "blend_common.cuh"

namespace msplat_cuda {

// Process-wide kernel launch counter (msplat_kernel_launches); every launch
// site calls count_launches with the number of kernels it enqueued.
void count_launches(int n);

// cudaFuncAttributeMaxDynamicSharedMemorySize belongs to the device context:
// opt a kernel in once per (kernel, device id), thread-safely.  `done` is the
// kernel's bitmask of configured devices (a function-local static).
inline cudaError_t opt_in_smem(const void* fn, std::atomic<unsigned long long>& done, int bytes = 227 * 1024) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const unsigned long long bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}

// SM count of the current device (cached per device id; persistent-grid sizing).
inline int device_sm_count() {
    static std::atomic<int> cache[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    int v = cache[dev & 63].load(std::memory_order_relaxed);
    if (v == 0) {
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        cache[dev & 63].store(v, std::memory_order_relaxed);
    }
    return v;
}

template <typename Real>
struct PreprocessArgs {
    int64_t n;
    int C, deg, K;
    const Real *means, *quats, *log_scales, *opacity_logits, *k, *sh, *semantics;
    Cam cam;
    double sigma;
    int W, H;
    // outputs
    uint64_t* depth_key;
    uint32_t* order;
    uint32_t* tile_count;
    uint2* tile_rect;
    uint8_t* visible;
    uint8_t* clamped_bits;
    AlphaRec<Real>* arec;
    BlendRec<Real>* brec;  // null: not written (FP32 atomic path: no reader)
    DepthRec* drec;  // FP32 only (the forward's depth flush); may be null
    double *cap_center, *cap_conic, *cap_depth, *cap_radius, *cap_rgb;  // optional
    unsigned long long* visible_count;
    DeviceError* err;
};

template <typename Real>
void launch_preprocess(const PreprocessArgs<Real>& a, cudaStream_t s);

// Binning (K2-K5).  Workspace is owned by the replay (cabi.cu).
struct BinningBuffers {
    int64_t n;            // Gaussians
    int tiles_x, tiles_y;
    int64_t inst_cap;     // capacity of the instance arrays
    int depth_key_bits;   // 63 for K1 keys (z > 0.01), 64 for explicit splats
    // per Gaussian
    uint64_t *depth_key, *depth_key_alt;
    uint32_t *order, *order_alt;
    uint32_t* tile_count;  // by Gaussian id (K1 output)
    uint2* tile_rect;      // by Gaussian id (K1 output)
    uint32_t* count_sorted;  // tile_count in depth order
    uint32_t* offset_sorted; // exclusive scan of count_sorted
    // per instance
    uint32_t *inst_tile, *inst_tile_alt;
    uint32_t *inst_gauss, *inst_gauss_alt;
    // per tile
    uint2* tile_range;  // [start, end) into the sorted instance list
    // scalars (device)
    int64_t* d_inst_count;
    uint32_t* d_inst_total32;  // [0] instance total, [1] longest tile list (per-tile path)
    // per-tile path: per-tile counters and cursors, per-instance depth keys,
    // shared-memory capacity (entries) of the tile sort
    uint32_t *tile_cnt, *tile_cur;
    uint64_t* inst_key;     // per-instance sort items (depth-key high word, Gaussian id)
    uint32_t* big_tiles;    // [0] = count, then the tiles whose list exceeds one CTA's register sort
    unsigned long long* key_range;  // [0] max ~key, [1] max key over the binned Gaussians
    // scratch
    uint32_t *hist, *hist_scanned, *scan_tiles;
    DeviceError* err;
    // results (which ping-pong buffer holds the final list)
    uint32_t* sorted_gauss;  // per-instance Gaussian ids, tile-major (set by run_binning)
};

void run_binning(BinningBuffers& b, cudaStream_t s);

// bin_and_sort on explicit splats: tile rects / counts / depth keys from
// centre, radius, depth (rasterizer.cpp:30-39).
void launch_rects_from_splats(int64_t n, const uint8_t* visible, const double* center,
                              const double* radius, const double* depth, int W, int H,
                              uint64_t* depth_key, uint32_t* order, uint32_t* tile_count,
                              uint2* tile_rect, cudaStream_t s);
size_t binning_scratch_elems(int64_t n_cap, int64_t inst_cap);

// Forward blend (K6).
template <typename Real>
struct ForwardArgs {
    int W, H, tiles_x, C;
    Cam cam;
    RenderParams rp;
    const uint2* tile_range;
    const uint32_t* inst_gauss;
    const AlphaRec<Real>* arec;
    const BlendRec<Real>* brec;
    const DepthRec* drec;   // FP32: the depth flush's quadratic forms
    const Real* semantics;  // [n][C] scene parameters
    RawParams<Real> raw;    // means/quats/log_scales for the FP64 re-decision
    Real *color, *depth, *sem_out, *kmap, *T;  // planar outputs (T required)
    int32_t* contributors;
    int32_t* terminus;
    Real* weight_sums;  // optional
    // Blend-event log for the backward (optional): per (tile, warp) the events
    // in which some lane blended, front to back, as (list position, lane mask),
    // in the region [8 * range.x + warp * len, + len) of a buffer of 8 I
    // entries; ev_count[tile * 8 + warp] = number of events.
    uint4* ev_list;    // (list position, lane mask, Gaussian id, 0)
    uint32_t* ev_count;
    uint32_t* ev_npairs;  // blended pairs per (tile, warp): the backward's pair-record segments
    // FP32 split forward (forward_split.cu): per event one row of 32 blend
    // weights (0 for lanes that did not blend, negated where alpha was clamped
    // at 0.99), in the region [32 (8 range.x +
    // warp len), + 32 len) -- the event log's region scaled by 32 -- and the
    // optional longest-first segment order of its per-pair kernel.
    float* ev_w;
    int64_t ev_w_cap;  // floats
    int sem_vec;       // semantic rows may be staged in 8-byte pieces (C even, 8-byte aligned)
    const uint32_t* work_order;
    int nseg;          // (tile, warp) segments (set by the launcher)
    DeviceError* err;
};
template <typename Real>
void launch_forward(const ForwardArgs<Real>& a, int ntiles, cudaStream_t s);
// The fused blend without semantics (colour, k, depth, T, the event log and
// the weight rows), for the split FP32 forward.
void launch_forward_blend_split(const ForwardArgs<float>& a, int ntiles, cudaStream_t s);
// The split FP32 forward (blend pass + tensor-core semantic pass) handles C <= 64.
bool forward_split_supported(int C);
void launch_forward_split(const ForwardArgs<float>& a, int ntiles, cudaStream_t s, const uint32_t* seg_order,
                          uint32_t* order_scratch);

// Longest-first order of the nseg = 8 * tiles (tile, warp) segments for the
// FP32 backward, cost = seg_cost[i] (the forward's per-warp event counts):
// a two-kernel counting sort into 1024 buckets (count, clamped), arbitrary
// order inside a bucket (scheduling only: results do not depend on it).
// scratch: 2048 uint32 (bucket sizes and cursors, zeroed here).
void launch_work_order(const uint32_t* seg_cost, int nseg, uint32_t* order, uint32_t* scratch, cudaStream_t s);

// K12: frame losses + seed assembly (core/src/trainer.cpp:171-264, losses.cpp).
template <typename Real>
struct LossArgs {
    int W, H, C;
    int en[6];          // lambda > 0, order (l1, ssim, normal, depth, seg, k)
    double lambdas[6];
    double ssim_w[11];  // normalised Gaussian window (losses.cpp:24-35)
    double ssim_inv_count;
    const Real *color, *depth, *sem, *kmap, *normals;  // rendered frame, planar
    const Real *gt_rgb, *gt_depth, *gt_normal;         // ground truth, planar
    const uint8_t* labels;
    double* acc;        // [8] reduced sums / counts
    double* report;     // [20] msplat_loss_report + 2 counts
    Real* ssim_maps;    // [3 maps][3][Hv][Wv]
    Real* ssim_grad;    // [3][H][W]
    Real* ce_stats;     // [2][H][W] per-pixel softmax max and normaliser (loss_pixel -> assemble)
    Real *dcolor, *ddepth, *dsem, *dkmap, *dN;  // outputs (dN: seeded normal-loss gradient)
    DeviceError* err;
};
template <typename Real>
void launch_frame_losses(const LossArgs<Real>& a, cudaStream_t s);

// Evaluation metrics (core/src/metrics.cpp:68-187); NULL inputs skip a metric.
template <typename Real>
struct MetricArgs {
    int W, H, C;
    double ssim_w[11];
    const Real *color, *gt_rgb;                       // psnr, ssim_metric
    const Real *depth, *gt_depth;                     // abs_rel, rmse
    const uint8_t* depth_mask;
    const Real *normals, *gt_normal;                  // cos_simi
    const uint8_t* normal_mask;
    const Real* sem;                                  // argmax_labels + miou
    const uint8_t *labels, *label_mask;
    double* acc;                                      // [9]
    unsigned long long* hist;                         // [3][C]
    DeviceError* err;
};
template <typename Real>
void launch_frame_metrics(const MetricArgs<Real>& a, cudaStream_t s);

// K13: trainer support (core/src/trainer.cpp:42-86, 150-168).
template <typename Real>
void launch_init_scene(int64_t n, int C, int deg, const double* pts_dev, const double* cols_dev, double* log_scale_dev,
                       double k_reset, Real* params, cudaStream_t s);
template <typename Real>
void launch_prune_compact(int64_t n, int C, int deg, const uint8_t* keep, int64_t kept, const Real* const in[3],
                          Real* const out[3], double k_reset, uint32_t* k32, uint32_t* newidx, uint32_t* scan_tiles,
                          uint32_t* d_total, cudaStream_t s);

// Extended-PLY scene I/O (core/src/io_ply.cpp) to / from the packed layout.
// code: 0 ok, 1 invalid_argument, 2 runtime_error, 4 CUDA error.
struct IoResult {
    int code = 0;
    std::string msg;
};
IoResult ply_scene_info(const char* path, int64_t* n, int* C, int* deg);
template <typename Real>
IoResult ply_load_scene(const char* path, Real* packed, cudaStream_t s, DeviceError* err);
template <typename Real>
IoResult ply_save_scene(const char* path, int64_t n, int C, int deg, const Real* packed, cudaStream_t s);

// Normals (K7, K8).
template <typename Real>
struct NormalArgs {
    int W, H;
    Cam cam;
    int step1, step2;
    double lambda, mask_threshold;
    const Real* depth;
    const Real* T;
    Real* normals;           // K7 output [3][H][W]
    const Real* dN;          // K8 input [3][H][W]
    Real* dv;                // K8 scratch [12][H][W] (per-centre adjoints)
    Real* dD;                // K8 output (accumulated with seed)
    double seed;
};
template <typename Real>
void launch_normals_forward(const NormalArgs<Real>& a, cudaStream_t s);
template <typename Real>
void launch_normals_backward(const NormalArgs<Real>& a, cudaStream_t s);

// Backward blend (K9) and per-Gaussian backward (K10).
template <typename Real>
struct BackwardArgs {
    int W, H, tiles_x, C;
    int64_t n;
    Cam cam;
    RenderParams rp;
    const uint2* tile_range;
    const uint32_t* inst_gauss;
    const AlphaRec<Real>* arec;
    const BlendRec<Real>* brec;
    const DepthRec* drec;     // FP32 phase B: the depth moments (DepthRec)
    const Real* semantics;
    RawParams<Real> raw;
    const uint4* ev_list;     // the forward's blend-event log (ForwardArgs::ev_list)
    const uint32_t* ev_count;
    // FP32 split backward: per-(tile, warp) pair-record segments written by the
    // tensor-core phase A and consumed by the phase-B kernel: one 16-byte
    // record per blended pair {gid, pixel lane, G dalpha (0 when alpha was
    // clamped), dD w}, pair_cap records in all.
    const uint32_t* pair_off;  // [tiles * 8] exclusive scan of ev_npairs
    uint32_t* pair_n;          // [tiles * 8] pairs phase A wrote
    uint4* pr;
    int64_t pair_cap;
    const Real* T_final;
    const int32_t* terminus;
    const Real *dcolor, *ddepth, *dsem, *dkmap;  // planar pixel grads
    // accumulation targets (zeroed before K9)
    Real *g_pos, *g_rot, *g_scale, *g_opac, *g_k, *g_sem;  // output gradient buffer
    Real* acc_dcolor;  // scratch [n][3]
    // scratch [n][16]: the per-pair geometric sums of K9 in one 64-byte row,
    // [opacity, dmean2, dconic3, dposition3, drotation4, dscale3]; K10 folds
    // it into the gradient buffer.  FP32 phase B (ProjBackwardArgs::
    // depth_moments) instead keeps the depth chain as camera-space moments
    // [.., u3, S6, miss] that K10 turns into dposition / drotation / dscale.
    Real* acc16;
    // Deterministic mode (null = atomics): per-(instance, warp) slots of V =
    // 20 + C values [opac, dmean2, dconic3, pos3, rot4, scale3, dcolor3, k, sem C].
    Real* partial;
    int V;
    // The split forward's per-event weight rows (null when the forward ran
    // fused): phase A then replays without alpha tests.
    const float* ev_w;
    // Segment schedule of the FP32 split backward (optional): warp w of CTA b
    // replays segment work_order[8 b + w] = tile * 8 + block (longest first,
    // launch_work_order), and phase B takes segments in the same order.  Null:
    // warp w of CTA b replays block w of tile b.
    const uint32_t* work_order;
    int nseg;  // (tile, warp) segments of the FP32 phase A (set by the launcher)
    // FP32: semantic rows may be moved in 8-byte pieces (C even and both the
    // scene's and the gradient buffer's semantic arrays 8-byte aligned).
    int sem_vec;
    DeviceError* err;
};
template <typename Real>
void launch_backward_blend(const BackwardArgs<Real>& a, int ntiles, cudaStream_t s);

// Deterministic reduction of BackwardArgs::partial into the targets: instances
// stably sorted by Gaussian id, then each Gaussian sums its slots in (list
// position, warp) order -- bitwise reproducible run to run.
struct DetScratch {
    uint32_t *keys, *keys_alt, *vals, *vals_alt;  // >= count each
    uint2* gid_range;                             // [n]
    uint32_t *hist, *hist_scanned, *scan_tiles;   // radix-sort scratch for count items
};
// Zeroes the first (*d_count) x per_item slots of the deterministic partial
// buffer (capacity cap items); raises kErrPairOverflow when *d_count > cap.
template <typename Real>
void launch_zero_det_slots(Real* partial, const int64_t* d_count, int64_t cap, int per_item, DeviceError* err,
                           cudaStream_t s);
template <typename Real>
void launch_deterministic_reduce(const BackwardArgs<Real>& a, const DetScratch& d, const int64_t* d_count,
                                 int64_t count, cudaStream_t s);

template <typename Real>
struct ProjBackwardArgs {
    int64_t n;
    int C, deg, K;
    Cam cam;
    const Real *means, *quats, *log_scales, *opacity_logits, *sh;
    const uint8_t* visible;
    const uint8_t* clamped_bits;
    const Real *acc_dcolor, *acc16;
    Real *g_pos, *g_rot, *g_scale, *g_opac, *g_sh, *g_k, *g_sem;
    int chain;  // fuse chain_activations (scene.cpp:108-129); only for single-view buffers
    // acc16[6..15] holds the FP32 phase B's depth moments (u_c[3], S_c[6]
    // = xx yy zz xy xz yz, miss sum) instead of dposition / drotation / dscale
    int depth_moments;
    double sigma;  // RenderConfig::sigma_scale (axes = sigma * scale)
    DeviceError* err;
};
template <typename Real>
void launch_projection_backward(const ProjBackwardArgs<Real>& a, cudaStream_t s);

template <typename Real>
void launch_chain(int64_t n, const Real* quats, const Real* log_scales, const Real* opac,
                  Real* g_rot, Real* g_scale, Real* g_opac, cudaStream_t s);

template <typename Real>
void launch_check_replay(int64_t n, const Real* means, const Real* k, const Real* saved_means,
                         const Real* saved_k, DeviceError* err, cudaStream_t s);

// Optimizer (K11).
// Elements [base, base + total) of the packed buffer; the pointers address
// element `base` (a shard of a sharded optimizer step, or base = 0 for all).
template <typename Real>
void launch_adam(int64_t base, int64_t total, const int64_t* seg_starts /*host, 8*/, const double* lr /*7*/,
                 Real* params, const Real* grads, Real* m, Real* v, double bc1, double bc2,
                 cudaStream_t s);
// dst += src over total packed values (multi-lane gradient sums).
template <typename Real>
void launch_accumulate(int64_t total, Real* dst, const Real* src, cudaStream_t s);
template <typename Real>
void launch_prune_mask(int64_t n, const Real* k, double threshold, int keep_small, uint8_t* keep,
                       unsigned long long* kept, cudaStream_t s);

}  // namespace msplat_cuda
