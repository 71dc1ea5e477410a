// C ABI (include/msplat_b200.h): context / replay lifetime, device buffer
// management, precision dispatch and the error contract.  No kernels here.
#include <cstdlib>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/msplat_b200.h"
#include "kernels.h"
#include "radix_sort.cuh"

using namespace msplat_cuda;

namespace {

thread_local std::string g_error;

msplat_status set_error(msplat_status st, const std::string& msg) {
    g_error = msg;
    return st;
}

#define CUDA_TRY(expr)                                                                         \
    do {                                                                                       \
        cudaError_t e_ = (expr);                                                               \
        if (e_ != cudaSuccess)                                                                 \
            return set_error(e_ == cudaErrorMemoryAllocation ? MSPLAT_ERR_OUT_OF_MEMORY        \
                                                             : MSPLAT_ERR_CUDA,                \
                             std::string("CUDA error: ") + cudaGetErrorString(e_) + " (" #expr ")"); \
    } while (0)

// Makes a context's device current for the duration of an entry point and
// restores the caller's device afterwards (dev < 0: no-op).
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (dev < 0) return;
        int cur = -1;
        if (cudaGetDevice(&cur) != cudaSuccess) return;
        if (cur != dev && cudaSetDevice(dev) == cudaSuccess) prev = cur;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;
};
#define CTX_DEVICE_GUARD(c) DeviceGuard device_guard_((c) ? (c)->device : -1)
#define REPLAY_DEVICE_GUARD(r) DeviceGuard device_guard_((r) && (r)->ctx ? (r)->ctx->device : -1)

// Grow-only device allocation.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaError_t ensure(size_t want) {
        if (want <= bytes) return cudaSuccess;
        if (const char* e = std::getenv("MSPLAT_DEBUG_CAPTURE"); e && e[0] == '1')
            std::fprintf(stderr, "[msplat debug] DevBuf grow %zu -> %zu\n", bytes, want);
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        size_t b = std::max<size_t>(want, 256);
        cudaError_t e = cudaMalloc(&p, b);
        if (e == cudaSuccess) bytes = b;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

int64_t sh_coeffs(int deg) { return int64_t(deg + 1) * (deg + 1); }
size_t real_size(int dtype) { return dtype == MSPLAT_F64 ? 8 : 4; }

std::atomic<long long> g_launches{0};

// CUDA-event brackets per stage (msplat_context_set_timing).  Events come from
// a grow-only pool; elapsed times are summed when the caller asks.
struct StageTimer {
    bool enabled = false;
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    struct Mark {
        int stage;
        cudaEvent_t a, b;
    };
    std::vector<Mark> marks;
    int open_stage = -1;
    cudaEvent_t open_ev = nullptr;

    cudaEvent_t next() {
        if (used == pool.size()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            pool.push_back(e);
        }
        return pool[used++];
    }
    // Inside CUDA-graph capture a plain record is only a dependency edge; an
    // external record becomes an event-record node that timestamps each replay.
    static void record(cudaEvent_t e, cudaStream_t s) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(s, &cs);
        if (cs == cudaStreamCaptureStatusActive)
            cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
        else
            cudaEventRecord(e, s);
    }
    // MSPLAT_DEBUG_CAPTURE=1: report, at every stage boundary, a capture
    // that has been invalidated or a pending launch error (debugging aid).
    static void debug_check(int stage, const char* where, cudaStream_t s) {
        static const bool on = [] {
            const char* e = std::getenv("MSPLAT_DEBUG_CAPTURE");
            return e && e[0] == '1';
        }();
        if (!on) return;
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        const cudaError_t e1 = cudaStreamIsCapturing(s, &cs);
        const cudaError_t e2 = cudaPeekAtLastError();
        if (cs == cudaStreamCaptureStatusInvalidated || e1 != cudaSuccess || e2 != cudaSuccess)
            std::fprintf(stderr, "[msplat debug] stage %d %s: capture status %d, %s / %s\n", stage, where, int(cs),
                         cudaGetErrorString(e1), cudaGetErrorString(e2));
    }
    void begin(int stage, cudaStream_t s) {
        debug_check(stage, "begin", s);
        if (!enabled) return;
        open_stage = stage;
        open_ev = next();
        record(open_ev, s);
    }
    void end(cudaStream_t s) {
        debug_check(open_stage, "end", s);
        if (!enabled || open_stage < 0) return;
        cudaEvent_t e = next();
        record(e, s);
        marks.push_back({open_stage, open_ev, e});
        open_stage = -1;
    }
    void collect(double* ms, int64_t* calls) {
        for (int i = 0; i < MSPLAT_STAGE_COUNT; ++i) {
            ms[i] = 0;
            if (calls) calls[i] = 0;
        }
        for (const Mark& m : marks) {
            // A bracket captured into a graph that was never replayed has no
            // timestamps: skip it (and clear the non-sticky error it raises).
            float t = 0;
            if (cudaEventSynchronize(m.b) != cudaSuccess || cudaEventElapsedTime(&t, m.a, m.b) != cudaSuccess) {
                (void)cudaGetLastError();
                continue;
            }
            ms[m.stage] += t;
            if (calls) calls[m.stage] += 1;
        }
        marks.clear();
        used = 0;
    }
    ~StageTimer() {
        for (cudaEvent_t e : pool) cudaEventDestroy(e);
    }
};

}  // namespace

namespace msplat_cuda {
void count_launches(int n) {
    g_launches.fetch_add(n, std::memory_order_relaxed);
    // MSPLAT_DEBUG_CAPTURE=1: report launch errors as they happen (inside a
    // graph capture they only surface at the end of the capture otherwise)
    static const bool dbg = [] {
        const char* e = std::getenv("MSPLAT_DEBUG_CAPTURE");
        return e && e[0] == '1';
    }();
    if (dbg) {
        const cudaError_t e = cudaPeekAtLastError();
        if (e != cudaSuccess)
            std::fprintf(stderr, "[msplat debug] launch error after launch #%lld: %s\n", (long long)g_launches.load(),
                         cudaGetErrorString(e));
    }
}
}  // namespace msplat_cuda

struct msplat_context {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    DeviceError* d_err = nullptr;
    DeviceError* h_err = nullptr;  // pinned
    unsigned long long* h_u64 = nullptr;  // pinned scratch
    // scratch owned by the context (shared by calls on its stream)
    DevBuf acc_dcolor, acc16, ddepth_total, normal_dv, kept;
    // frame losses (msplat_frame_losses)
    DevBuf loss_acc, loss_report, ssim_maps, ssim_grad, loss_dN, loss_ce;
    DevBuf metric_acc, metric_hist;
    // trainer support (msplat_init_scene, msplat_prune_compact)
    DevBuf init_pts, init_cols, init_logs, cmp_k32, cmp_idx, cmp_tiles, cmp_total;
    // deterministic backward (msplat_context_set_deterministic)
    int deterministic = 0;
    DevBuf det_partial, det_keys, det_keys_alt, det_vals, det_vals_alt, det_range;
    int64_t det_cap = 0;  // instances the deterministic slots hold (grown by eager calls)
    StageTimer timer;
};

struct msplat_replay {
    msplat_context* ctx = nullptr;
    bool valid = false;
    int capture = 0;
    int dtype = 0;
    int64_t n = 0;
    int C = 0, deg = 0, W = 0, H = 0, tiles_x = 0, tiles_y = 0;
    Cam cam{};
    RenderParams rp{};
    int64_t inst_cap = 0;
    bool binned_explicit = false;
    DevBuf arec, brec, drec, visible, clamped, depth_key, depth_key_alt, order, order_alt, tile_count, tile_rect,
        count_sorted, offset_sorted, inst_tile, inst_tile_alt, inst_gauss, inst_gauss_alt, tile_range,
        d_inst_count, d_inst_total32, hist, hist_scanned, scan_tiles, terminus, weight_sums, saved_means,
        saved_k, cap_center, cap_conic, cap_depth, cap_radius, cap_rgb, visible_count, ev_list, ev_count, ev_npairs,
        pair_off, pair_n, pair_scan, pair_total, pair_rec, wq_order, wq_scratch, ev_w, tile_cnt, tile_cur, inst_key, big_tiles, key_range;
    bool split_fwd = false;  // the last forward ran split: its weight rows are valid
    bool brec_written = false;  // K1 wrote the BlendRecs (FP64 or deterministic mode; the FP32 atomic path has no reader)
    bool order_valid = false;   // wq_order holds the last forward's longest-first segment order (reused by the backward)
    int64_t pair_cap = 0;  // pair-record capacity of the FP32 split backward
    uint32_t* sorted_gauss = nullptr;

    void release_all() {
        for (DevBuf* b : {&arec, &brec, &drec, &visible, &clamped, &depth_key, &depth_key_alt, &order, &order_alt,
                          &tile_count, &tile_rect, &count_sorted, &offset_sorted, &inst_tile, &inst_tile_alt,
                          &inst_gauss, &inst_gauss_alt, &tile_range, &d_inst_count, &d_inst_total32, &hist,
                          &hist_scanned, &scan_tiles, &terminus, &weight_sums, &saved_means, &saved_k,
                          &cap_center, &cap_conic, &cap_depth, &cap_radius, &cap_rgb, &visible_count, &ev_list,
                          &ev_count, &ev_npairs, &pair_off, &pair_n, &pair_scan, &pair_total, &pair_rec,
                          &wq_order, &wq_scratch, &ev_w, &tile_cnt, &tile_cur, &inst_key, &big_tiles, &key_range})
            b->release();
    }
};

namespace {

// FP32 backward over a longest-first segment order (default); the environment
// variable MSPLAT_STATIC_SCHEDULE=1 restores tile order (A/B timing).
bool dynamic_schedule() {
    static const bool on = [] {
        const char* e = std::getenv("MSPLAT_STATIC_SCHEDULE");
        return !(e && e[0] == '1');
    }();
    return on;
}

// CameraView::finalize (core/src/camera.cpp:8-21).
msplat_status make_cam(const msplat_camera* c, Cam& o) {
    if (!c) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "CameraView: null camera");
    if (c->width < 1 || c->height < 1)
        return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "CameraView: width and height must be >= 1");
    if (!(c->fx > 0) || !(c->fy > 0))
        return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "CameraView: focal lengths must be positive");
    const double* R = c->R_c2w;
    double worst = 0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = R[0 * 3 + i] * R[0 * 3 + j];
            s += R[1 * 3 + i] * R[1 * 3 + j];
            s += R[2 * 3 + i] * R[2 * 3 + j];
            worst = std::max(worst, std::fabs(s - (i == j ? 1.0 : 0.0)));
        }
    if (worst > 1e-6)
        return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "CameraView: rotation is not orthonormal (tol 1e-6)");
    const double det = R[0] * (R[4] * R[8] - R[7] * R[5]) - R[3] * (R[1] * R[8] - R[7] * R[2]) +
                       R[6] * (R[1] * R[5] - R[4] * R[2]);
    if (std::fabs(det - 1.0) > 1e-6)
        return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "CameraView: rotation determinant is not +1 (tol 1e-6)");
    o.fx = c->fx;
    o.fy = c->fy;
    o.cx = c->cx;
    o.cy = c->cy;
    o.W = c->width;
    o.H = c->height;
    for (int i = 0; i < 9; ++i) o.Rc2w[i] = R[i];
    for (int i = 0; i < 3; ++i) o.tc2w[i] = c->t_c2w[i];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) o.Rw2c[i * 3 + j] = R[j * 3 + i];
    for (int i = 0; i < 3; ++i) {
        double s = o.Rw2c[i * 3 + 0] * o.tc2w[0];
        s += o.Rw2c[i * 3 + 1] * o.tc2w[1];
        s += o.Rw2c[i * 3 + 2] * o.tc2w[2];
        o.tw2c[i] = -s;
    }
    return MSPLAT_OK;
}

msplat_status check_scene(const msplat_scene* s) {
    if (!s) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "Scene: null scene");
    if (s->sh_degree < 0 || s->sh_degree > 3)
        return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "Scene: sh_degree must be in [0,3]");
    if (s->num_classes < 0) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "Scene: num_classes must be >= 0");
    if (s->n < 0) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "Scene: negative size");
    if (s->dtype != MSPLAT_F32 && s->dtype != MSPLAT_F64)
        return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "Scene: dtype must be MSPLAT_F32 or MSPLAT_F64");
    if (s->n > 0 && (!s->means || !s->quats || !s->log_scales || !s->opacity_logits || !s->k || !s->sh ||
                     (s->num_classes > 0 && !s->semantics)))
        return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "Scene: null parameter array");
    if (s->n >= (int64_t(1) << 31)) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "Scene: too many Gaussians");
    return MSPLAT_OK;
}

// Reads (and clears) the latched device error.  Synchronizes the stream.
msplat_status drain_device_error(msplat_context* ctx, int W) {
    CUDA_TRY(cudaMemcpyAsync(ctx->h_err, ctx->d_err, sizeof(DeviceError), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    DeviceError e = *ctx->h_err;
    if (e.code == kErrNone) return MSPLAT_OK;
    if (e.min_b != 0) e.b = static_cast<long long>(~e.min_b);  // raise_error_ordered: lowest primitive
    CUDA_TRY(cudaMemsetAsync(ctx->d_err, 0, sizeof(DeviceError), ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    char buf[256];
    const int w = W > 0 ? W : 1;
    switch (e.code) {
        case kErrNonFiniteBlend:
            snprintf(buf, sizeof buf, "rasterize: non-finite blend at pixel (%lld,%lld), primitive %lld",
                     e.a % w, e.a / w, e.b);
            return set_error(MSPLAT_ERR_RUNTIME, buf);
        case kErrNonFiniteOutput:
            snprintf(buf, sizeof buf, "rasterize: non-finite output at pixel (%lld,%lld)", e.a % w, e.a / w);
            return set_error(MSPLAT_ERR_RUNTIME, buf);
        case kErrSceneModified:
            snprintf(buf, sizeof buf, "rasterize_backward: scene modified since forward (primitive %lld)", e.b);
            return set_error(MSPLAT_ERR_RUNTIME, buf);
        case kErrNonFiniteGrad:
            snprintf(buf, sizeof buf, "rasterize_backward: non-finite gradient for primitive %lld", e.b);
            return set_error(MSPLAT_ERR_RUNTIME, buf);
        case kErrZeroQuat:
            snprintf(buf, sizeof buf, "activate: primitive %lld has a zero quaternion", e.b);
            return set_error(MSPLAT_ERR_INVALID_ARGUMENT, buf);
        case kErrNonFiniteParam:
            snprintf(buf, sizeof buf, "Scene: primitive %lld has non-finite fields", e.b);
            return set_error(MSPLAT_ERR_INVALID_ARGUMENT, buf);
        case kErrInstanceOverflow:
            snprintf(buf, sizeof buf, "internal: tile-instance capacity %lld exceeded (needed %lld)", e.b, e.a);
            return set_error(MSPLAT_ERR_RUNTIME, buf);
        case kErrPairOverflow:
            snprintf(buf, sizeof buf, "internal: pair-record capacity %lld exceeded", e.b);
            return set_error(MSPLAT_ERR_RUNTIME, buf);
        case kErrMiouLabel:
            return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "miou: label out of range");
        case kErrLabelRange:
            snprintf(buf, sizeof buf, "cross_entropy_seg: label %lld out of range at pixel (%lld,%lld)", e.b, e.a % w,
                     e.a / w);
            return set_error(MSPLAT_ERR_INVALID_ARGUMENT, buf);
        default:
            snprintf(buf, sizeof buf, "device error %d", e.code);
            return set_error(MSPLAT_ERR_RUNTIME, buf);
    }
}

// Allocates per-Gaussian / per-pixel / per-tile replay storage for a view.
msplat_status size_replay(msplat_replay* r, int dtype, int64_t n, int C, int deg, int W, int H) {
    const size_t R = real_size(dtype);
    r->dtype = dtype;
    r->n = n;
    r->C = C;
    r->deg = deg;
    r->W = W;
    r->H = H;
    r->tiles_x = (W + kTile - 1) / kTile;
    r->tiles_y = (H + kTile - 1) / kTile;
    const int64_t tiles = int64_t(r->tiles_x) * r->tiles_y;
    const size_t nn = size_t(std::max<int64_t>(n, 1));
    if (r->inst_cap == 0) r->inst_cap = std::max<int64_t>(int64_t(1) << 20, 4 * n);
    CUDA_TRY(r->arec.ensure(nn * sizeof(AlphaRec<double>) / 8 * R));
    CUDA_TRY(r->brec.ensure(nn * 32 * R));
    if (dtype != MSPLAT_F64) CUDA_TRY(r->drec.ensure(nn * sizeof(DepthRec)));  // (FP32 only)
    CUDA_TRY(r->visible.ensure(nn));
    CUDA_TRY(r->clamped.ensure(nn));
    CUDA_TRY(r->depth_key.ensure(nn * 8));
    CUDA_TRY(r->depth_key_alt.ensure(nn * 8));
    CUDA_TRY(r->order.ensure(nn * 4));
    CUDA_TRY(r->order_alt.ensure(nn * 4));
    CUDA_TRY(r->tile_count.ensure(nn * 4));
    CUDA_TRY(r->tile_rect.ensure(nn * 8));
    CUDA_TRY(r->count_sorted.ensure(nn * 4));
    CUDA_TRY(r->offset_sorted.ensure(nn * 4));
    const size_t ic = size_t(r->inst_cap);
    CUDA_TRY(r->inst_tile.ensure(ic * 4));
    CUDA_TRY(r->inst_tile_alt.ensure(ic * 4));
    CUDA_TRY(r->inst_key.ensure(ic * 8));
    CUDA_TRY(r->ev_list.ensure(ic * 8 * sizeof(uint4)));  // 8 warps x (position, mask, id) per instance

    CUDA_TRY(r->ev_count.ensure(size_t(tiles) * 8 * 4));
    CUDA_TRY(r->ev_npairs.ensure(size_t(tiles) * 8 * 4));
    CUDA_TRY(r->wq_order.ensure(size_t(tiles) * 8 * 4));
    CUDA_TRY(r->wq_scratch.ensure(2048 * 4));
    CUDA_TRY(r->inst_gauss.ensure(ic * 4));
    CUDA_TRY(r->inst_gauss_alt.ensure(ic * 4));
    CUDA_TRY(r->tile_range.ensure(size_t(tiles) * 8));
    CUDA_TRY(r->tile_cnt.ensure(size_t(tiles) * 4));
    CUDA_TRY(r->tile_cur.ensure(size_t(tiles) * 4));
    CUDA_TRY(r->big_tiles.ensure(size_t(tiles + 1) * 4));
    CUDA_TRY(r->key_range.ensure(16));
    CUDA_TRY(r->d_inst_count.ensure(8));
    CUDA_TRY(r->d_inst_total32.ensure(8));
    CUDA_TRY(r->visible_count.ensure(8));
    const size_t hist = binning_scratch_elems(int64_t(nn), r->inst_cap);
    CUDA_TRY(r->hist.ensure(hist * 4));
    CUDA_TRY(r->hist_scanned.ensure((hist + 512) * 4));  // + the radix digit totals
    const size_t scan_tiles = (std::max(hist, nn) + kScanTile - 1) / kScanTile + 1;
    CUDA_TRY(r->scan_tiles.ensure(scan_tiles * 4));
    CUDA_TRY(r->terminus.ensure(size_t(W) * H * 4));
    CUDA_TRY(r->saved_means.ensure(nn * 3 * R));
    CUDA_TRY(r->saved_k.ensure(nn * R));
    if (r->capture & 1) {
        CUDA_TRY(r->cap_center.ensure(nn * 2 * 8));
        CUDA_TRY(r->cap_conic.ensure(nn * 3 * 8));
        CUDA_TRY(r->cap_depth.ensure(nn * 8));
        CUDA_TRY(r->cap_radius.ensure(nn * 8));
        CUDA_TRY(r->cap_rgb.ensure(nn * 3 * 8));
    }
    if (r->capture & 2) CUDA_TRY(r->weight_sums.ensure(nn * R));
    return MSPLAT_OK;
}

BinningBuffers binning_view(msplat_replay* r) {
    BinningBuffers b{};
    b.n = r->n;
    b.tiles_x = r->tiles_x;
    b.tiles_y = r->tiles_y;
    b.inst_cap = r->inst_cap;
    b.depth_key_bits = r->binned_explicit ? 64 : 63;
    b.depth_key = r->depth_key.as<uint64_t>();
    b.depth_key_alt = r->depth_key_alt.as<uint64_t>();
    b.order = r->order.as<uint32_t>();
    b.order_alt = r->order_alt.as<uint32_t>();
    b.tile_count = r->tile_count.as<uint32_t>();
    b.tile_rect = r->tile_rect.as<uint2>();
    b.count_sorted = r->count_sorted.as<uint32_t>();
    b.offset_sorted = r->offset_sorted.as<uint32_t>();
    b.inst_tile = r->inst_tile.as<uint32_t>();
    b.inst_tile_alt = r->inst_tile_alt.as<uint32_t>();
    b.inst_gauss = r->inst_gauss.as<uint32_t>();
    b.inst_gauss_alt = r->inst_gauss_alt.as<uint32_t>();
    b.tile_range = r->tile_range.as<uint2>();
    b.d_inst_count = r->d_inst_count.as<int64_t>();
    b.d_inst_total32 = r->d_inst_total32.as<uint32_t>();
    b.tile_cnt = r->tile_cnt.as<uint32_t>();
    b.tile_cur = r->tile_cur.as<uint32_t>();
    b.inst_key = r->inst_key.as<uint64_t>();
    b.big_tiles = r->big_tiles.as<uint32_t>();
    b.key_range = r->key_range.as<unsigned long long>();
    b.hist = r->hist.as<uint32_t>();
    b.hist_scanned = r->hist_scanned.as<uint32_t>();
    b.scan_tiles = r->scan_tiles.as<uint32_t>();
    b.err = r->ctx->d_err;
    return b;
}

// Binning with capacity management: if the device reports more instances
// than the buffers hold, grow and redo.  When `sync` is false the capacity is
// trusted (graph-capturable path) and an overflow surfaces as a latched error.
msplat_status binning_with_capacity(msplat_replay* r, bool sync) {
    msplat_context* ctx = r->ctx;
    for (int attempt = 0; attempt < 3; ++attempt) {
        BinningBuffers b = binning_view(r);
        run_binning(b, ctx->stream);
        r->sorted_gauss = b.sorted_gauss;
        CUDA_TRY(cudaGetLastError());
        if (!sync) return MSPLAT_OK;
        CUDA_TRY(cudaMemcpyAsync(ctx->h_u64, b.d_inst_total32, 8, cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        const int64_t need = int64_t(reinterpret_cast<uint32_t*>(ctx->h_u64)[0]);
        if (need <= r->inst_cap) {
            // split FP32 forward: <= 32 compacted blend weights per event-log
            // entry (8 per instance), sized from this render's instances (a
            // captured replay keeps the capacity; K6a checks it)
            if (r->dtype != MSPLAT_F64 && forward_split_supported(r->C)) {
                const size_t want = size_t(need + need / 4 + 1024) * 8 * 32 * sizeof(float);
                if (r->ev_w.bytes < size_t(need) * 8 * 32 * sizeof(float)) CUDA_TRY(r->ev_w.ensure(want));
            }
            return MSPLAT_OK;
        }
        // clear the latched overflow, grow, retry
        CUDA_TRY(cudaMemsetAsync(ctx->d_err, 0, sizeof(DeviceError), ctx->stream));
        r->inst_cap = need + need / 4 + 1024;
        msplat_status st = size_replay(r, r->dtype, r->n, r->C, r->deg, r->W, r->H);
        if (st != MSPLAT_OK) return st;
    }
    return set_error(MSPLAT_ERR_RUNTIME, "internal: instance capacity did not converge");
}

template <typename Real>
PreprocessArgs<Real> preprocess_args(msplat_replay* r, const msplat_scene* s, const msplat_render_config* cfg) {
    PreprocessArgs<Real> a{};
    a.n = s->n;
    a.C = s->num_classes;
    a.deg = s->sh_degree;
    a.K = int(sh_coeffs(s->sh_degree));
    a.means = static_cast<const Real*>(s->means);
    a.quats = static_cast<const Real*>(s->quats);
    a.log_scales = static_cast<const Real*>(s->log_scales);
    a.opacity_logits = static_cast<const Real*>(s->opacity_logits);
    a.k = static_cast<const Real*>(s->k);
    a.sh = static_cast<const Real*>(s->sh);
    a.semantics = static_cast<const Real*>(s->semantics);
    a.cam = r->cam;
    a.sigma = cfg->sigma_scale;
    a.W = r->W;
    a.H = r->H;
    a.depth_key = r->depth_key.as<uint64_t>();
    a.order = r->order.as<uint32_t>();
    a.tile_count = r->tile_count.as<uint32_t>();
    a.tile_rect = r->tile_rect.as<uint2>();
    a.visible = r->visible.as<uint8_t>();
    a.clamped_bits = r->clamped.as<uint8_t>();
    a.arec = r->arec.as<AlphaRec<Real>>();
    // the BlendRecs feed the FP64 kernels and the deterministic backward only
    a.brec = (sizeof(Real) == 8 || r->ctx->deterministic) ? r->brec.as<BlendRec<Real>>() : nullptr;
    a.drec = sizeof(Real) == 4 ? r->drec.as<DepthRec>() : nullptr;
    if (r->capture & 1) {
        a.cap_center = r->cap_center.as<double>();
        a.cap_conic = r->cap_conic.as<double>();
        a.cap_depth = r->cap_depth.as<double>();
        a.cap_radius = r->cap_radius.as<double>();
        a.cap_rgb = r->cap_rgb.as<double>();
    }
    a.visible_count = r->visible_count.as<unsigned long long>();
    a.err = r->ctx->d_err;
    return a;
}

template <typename Real>
msplat_status rasterize_impl(msplat_context* ctx, const msplat_scene* s, const msplat_render_config* cfg,
                             const msplat_frame* f, msplat_replay* r, bool sync) {
    const size_t R = sizeof(Real);
    CUDA_TRY(cudaMemsetAsync(r->visible_count.p, 0, 8, ctx->stream));
    ctx->timer.begin(MSPLAT_STAGE_PREPROCESS, ctx->stream);
    {
        const PreprocessArgs<Real> pa = preprocess_args<Real>(r, s, cfg);
        launch_preprocess<Real>(pa, ctx->stream);
        r->brec_written = pa.brec != nullptr;
    }
    ctx->timer.end(ctx->stream);
    CUDA_TRY(cudaGetLastError());
    r->binned_explicit = false;
    ctx->timer.begin(MSPLAT_STAGE_BINNING, ctx->stream);
    msplat_status st = binning_with_capacity(r, sync);
    ctx->timer.end(ctx->stream);
    if (st != MSPLAT_OK) return st;
    // snapshot for check_replay (rasterizer_backward.cpp:40-44)
    if (s->n > 0) {
        CUDA_TRY(cudaMemcpyAsync(r->saved_means.p, s->means, size_t(s->n) * 3 * R, cudaMemcpyDeviceToDevice,
                                 ctx->stream));
        CUDA_TRY(cudaMemcpyAsync(r->saved_k.p, s->k, size_t(s->n) * R, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    if (r->capture & 2) CUDA_TRY(cudaMemsetAsync(r->weight_sums.p, 0, size_t(std::max<int64_t>(s->n, 1)) * R, ctx->stream));
    ForwardArgs<Real> a{};
    a.W = r->W;
    a.H = r->H;
    a.tiles_x = r->tiles_x;
    a.C = s->num_classes;
    a.cam = r->cam;
    a.rp = r->rp;
    a.tile_range = r->tile_range.as<uint2>();
    a.inst_gauss = r->sorted_gauss;
    a.arec = r->arec.as<AlphaRec<Real>>();
    a.brec = r->brec.as<BlendRec<Real>>();
    a.drec = sizeof(Real) == 4 ? r->drec.as<DepthRec>() : nullptr;
    a.semantics = static_cast<const Real*>(s->semantics);
    a.raw = RawParams<Real>{static_cast<const Real*>(s->means), static_cast<const Real*>(s->quats),
                            static_cast<const Real*>(s->log_scales), cfg->sigma_scale};
    a.color = static_cast<Real*>(f->color);
    a.depth = static_cast<Real*>(f->depth);
    a.sem_out = static_cast<Real*>(f->semantics);
    a.kmap = static_cast<Real*>(f->kmap);
    a.T = static_cast<Real*>(f->transmittance);
    a.contributors = f->contributors;
    a.terminus = r->terminus.as<int32_t>();
    a.weight_sums = (r->capture & 2) ? r->weight_sums.as<Real>() : nullptr;
    a.ev_list = r->ev_list.as<uint4>();
    a.ev_count = r->ev_count.as<uint32_t>();
    a.ev_npairs = r->ev_npairs.as<uint32_t>();
    a.err = ctx->d_err;
    ctx->timer.begin(MSPLAT_STAGE_FORWARD, ctx->stream);
    if constexpr (sizeof(Real) == 4) {
        if (forward_split_supported(a.C) && r->ev_w.p) {
            a.ev_w = r->ev_w.as<float>();
            a.ev_w_cap = int64_t(r->ev_w.bytes / sizeof(float));
            a.sem_vec = (a.C % 2 == 0) && (reinterpret_cast<uintptr_t>(s->semantics) % 8 == 0);
            launch_forward_split(a, r->tiles_x * r->tiles_y, ctx->stream,
                                 dynamic_schedule() ? r->wq_order.as<uint32_t>() : nullptr, r->wq_scratch.as<uint32_t>());
            r->split_fwd = true;
            r->order_valid = dynamic_schedule() && a.C > 0;  // the semantic pass ordered the segments
        } else {
            launch_forward<Real>(a, r->tiles_x * r->tiles_y, ctx->stream);
            r->split_fwd = false;
            r->order_valid = false;
        }
    } else {
        launch_forward<Real>(a, r->tiles_x * r->tiles_y, ctx->stream);
        r->order_valid = false;
    }
    ctx->timer.end(ctx->stream);
    CUDA_TRY(cudaGetLastError());
    r->valid = true;
    return MSPLAT_OK;
}

template <typename Real>
NormalArgs<Real> normal_args(const Cam& cam, const msplat_normal_config* n, const void* depth, const void* T) {
    NormalArgs<Real> a{};
    a.W = cam.W;
    a.H = cam.H;
    a.cam = cam;
    a.step1 = n->step1;
    a.step2 = n->step2;
    a.lambda = n->fuse_lambda;
    a.mask_threshold = n->mask_threshold;
    a.depth = static_cast<const Real*>(depth);
    a.T = static_cast<const Real*>(T);
    return a;
}

msplat_status check_ncfg(const msplat_normal_config* n) {
    if (!n) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "estimate_normals: null config");
    if (n->step1 >= n->step2)
        return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "estimate_normals: step1 must be smaller than step2");
    if (n->fuse_lambda < 0 || n->fuse_lambda > 1)
        return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "estimate_normals: fuse weight must be in [0,1]");
    return MSPLAT_OK;
}

template <typename Real>
msplat_status backward_impl(msplat_context* ctx, const msplat_scene* s, const msplat_frame* f,
                            const msplat_replay* r, const msplat_pixel_grads* pix, const void* ddepth,
                            msplat_grads* g, int chain, int accumulate) {
    const size_t R = sizeof(Real);
    const int64_t n = s->n;
    const int C = s->num_classes, K = int(sh_coeffs(s->sh_degree));
    const size_t nn = size_t(std::max<int64_t>(n, 1));
    CUDA_TRY(ctx->acc_dcolor.ensure(nn * 3 * R));
    CUDA_TRY(ctx->acc16.ensure(nn * 16 * R));
    cudaStream_t st = ctx->stream;
    CUDA_TRY(cudaMemsetAsync(ctx->acc_dcolor.p, 0, nn * 3 * R, st));
    CUDA_TRY(cudaMemsetAsync(ctx->acc16.p, 0, nn * 16 * R, st));
    if (!accumulate && n > 0) {
        CUDA_TRY(cudaMemsetAsync(g->dposition, 0, size_t(n) * 3 * R, st));
        CUDA_TRY(cudaMemsetAsync(g->drotation, 0, size_t(n) * 4 * R, st));
        CUDA_TRY(cudaMemsetAsync(g->dscale, 0, size_t(n) * 3 * R, st));
        CUDA_TRY(cudaMemsetAsync(g->dopacity, 0, size_t(n) * R, st));
        CUDA_TRY(cudaMemsetAsync(g->dk, 0, size_t(n) * R, st));
        CUDA_TRY(cudaMemsetAsync(g->dsh, 0, size_t(n) * 3 * K * R, st));
        if (C > 0) CUDA_TRY(cudaMemsetAsync(g->dsemantics, 0, size_t(n) * C * R, st));
    }
    launch_check_replay<Real>(n, static_cast<const Real*>(s->means), static_cast<const Real*>(s->k),
                              r->saved_means.as<Real>(), r->saved_k.as<Real>(), ctx->d_err, st);
    if (ctx->deterministic && !r->brec_written && n > 0) {
        // deterministic mode switched on after an FP32 forward: K1 again for
        // the BlendRecs (its other outputs are rewritten with the same values)
        msplat_replay* rw = const_cast<msplat_replay*>(r);
        msplat_render_config rc{};
        rc.sigma_scale = r->rp.sigma_scale;
        CUDA_TRY(cudaMemsetAsync(rw->visible_count.p, 0, 8, st));
        const PreprocessArgs<Real> pa = preprocess_args<Real>(rw, s, &rc);
        launch_preprocess<Real>(pa, st);
        rw->brec_written = true;
        CUDA_TRY(cudaGetLastError());
    }
    BackwardArgs<Real> a{};
    a.W = r->W;
    a.H = r->H;
    a.tiles_x = r->tiles_x;
    a.C = C;
    a.n = n;
    a.cam = r->cam;
    a.rp = r->rp;
    a.tile_range = r->tile_range.as<uint2>();
    a.inst_gauss = r->sorted_gauss;
    a.arec = r->arec.as<AlphaRec<Real>>();
    a.brec = r->brec.as<BlendRec<Real>>();
    a.drec = sizeof(Real) == 4 ? r->drec.as<DepthRec>() : nullptr;
    a.semantics = static_cast<const Real*>(s->semantics);
    a.raw = RawParams<Real>{static_cast<const Real*>(s->means), static_cast<const Real*>(s->quats),
                            static_cast<const Real*>(s->log_scales), r->rp.sigma_scale};
    a.ev_list = r->ev_list.as<uint4>();
    a.ev_count = r->ev_count.as<uint32_t>();
    a.T_final = static_cast<const Real*>(f->transmittance);
    a.terminus = r->terminus.as<int32_t>();
    a.dcolor = static_cast<const Real*>(pix->dcolor);
    a.ddepth = static_cast<const Real*>(ddepth);
    a.dsem = static_cast<const Real*>(pix->dsemantics);
    a.dkmap = static_cast<const Real*>(pix->dkmap);
    a.g_pos = static_cast<Real*>(g->dposition);
    a.g_rot = static_cast<Real*>(g->drotation);
    a.g_scale = static_cast<Real*>(g->dscale);
    a.g_opac = static_cast<Real*>(g->dopacity);
    a.g_k = static_cast<Real*>(g->dk);
    a.g_sem = static_cast<Real*>(g->dsemantics);
    a.acc_dcolor = ctx->acc_dcolor.as<Real>();
    a.acc16 = ctx->acc16.as<Real>();
    a.err = ctx->d_err;
    int64_t det_count = 0;
    DetScratch det{};
    if (ctx->deterministic) {
        // The partial slots are sized by a CAPACITY of instances, grown whenever
        // the stream is not being captured (one synchronizing read of the
        // instance count), so the deterministic backward is graph-capturable;
        // the kernels bound themselves by the device-side count.
        a.V = 20 + C;
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        CUDA_TRY(cudaStreamIsCapturing(st, &cs));
        if (cs == cudaStreamCaptureStatusNone) {
            CUDA_TRY(cudaMemcpyAsync(ctx->h_u64, r->d_inst_count.p, 8, cudaMemcpyDeviceToHost, st));
            CUDA_TRY(cudaStreamSynchronize(st));
            const int64_t need = int64_t(*ctx->h_u64);
            if (need > ctx->det_cap || size_t(ctx->det_cap) * 8 * size_t(a.V) * R > ctx->det_partial.bytes) {
                const int64_t cap = std::max<int64_t>(need + need / 4 + 4096, ctx->det_cap);
                CUDA_TRY(ctx->det_partial.ensure(size_t(cap) * 8 * size_t(a.V) * R));
                CUDA_TRY(ctx->det_keys.ensure(size_t(cap) * 4));
                CUDA_TRY(ctx->det_keys_alt.ensure(size_t(cap) * 4));
                CUDA_TRY(ctx->det_vals.ensure(size_t(cap) * 4));
                CUDA_TRY(ctx->det_vals_alt.ensure(size_t(cap) * 4));
                ctx->det_cap = cap;
            }
        }
        if (ctx->det_cap == 0)
            return set_error(MSPLAT_ERR_RUNTIME, "rasterize_backward: deterministic capture before any eager call");
        det_count = std::min<int64_t>(ctx->det_cap, r->inst_cap);
        CUDA_TRY(ctx->det_range.ensure(nn * 8));
        a.partial = ctx->det_partial.as<Real>();
        a.pair_cap = ctx->det_cap;  // slot capacity (instances)
        launch_zero_det_slots<Real>(a.partial, r->d_inst_count.as<int64_t>(), ctx->det_cap, 8 * a.V, ctx->d_err, st);
        // the replay's radix scratch is sized for inst_cap >= det_count items
        det = DetScratch{ctx->det_keys.as<uint32_t>(), ctx->det_keys_alt.as<uint32_t>(),
                         ctx->det_vals.as<uint32_t>(), ctx->det_vals_alt.as<uint32_t>(),
                         ctx->det_range.as<uint2>(), r->hist.as<uint32_t>(), r->hist_scanned.as<uint32_t>(),
                         r->scan_tiles.as<uint32_t>()};
    }
    if (sizeof(Real) == 4 && !ctx->deterministic) {
        // FP32 split backward: segment offsets of the pair records (scan of the
        // forward's per-warp pair counts) and their capacity, grown whenever
        // the stream is not being captured.
        msplat_replay* rw = const_cast<msplat_replay*>(r);  // device scratch of the replay
        const int64_t nseg = int64_t(r->tiles_x) * r->tiles_y * 8;
        CUDA_TRY(rw->pair_off.ensure(size_t(nseg) * 4));
        CUDA_TRY(rw->pair_n.ensure(size_t(nseg) * 4));
        CUDA_TRY(rw->pair_scan.ensure((size_t(nseg) + kScanTile - 1) / kScanTile * 4 + 8));
        CUDA_TRY(rw->pair_total.ensure(8));
        device_exclusive_scan<uint32_t>(r->ev_npairs.as<uint32_t>(), rw->pair_off.as<uint32_t>(), nullptr, nseg,
                                        rw->pair_scan.as<uint32_t>(), rw->pair_total.as<uint32_t>(), st);
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        CUDA_TRY(cudaStreamIsCapturing(st, &cs));
        if (cs == cudaStreamCaptureStatusNone) {
            CUDA_TRY(cudaMemcpyAsync(ctx->h_u64, rw->pair_total.p, 4, cudaMemcpyDeviceToHost, st));
            CUDA_TRY(cudaStreamSynchronize(st));
            const int64_t need = int64_t(*reinterpret_cast<uint32_t*>(ctx->h_u64));
            if (need > rw->pair_cap) {
                const int64_t cap = need + need / 4 + 4096;
                CUDA_TRY(rw->pair_rec.ensure(size_t(cap) * sizeof(uint4)));
                rw->pair_cap = cap;
            }
        }
        if (rw->pair_cap == 0) return set_error(MSPLAT_ERR_RUNTIME, "rasterize_backward: capture before any eager call");
        BackwardArgs<float>& af = reinterpret_cast<BackwardArgs<float>&>(a);
        af.pair_off = rw->pair_off.as<uint32_t>();
        af.pair_n = rw->pair_n.as<uint32_t>();
        if (r->split_fwd) af.ev_w = r->ev_w.as<float>();
        af.pr = rw->pair_rec.as<uint4>();
        af.pair_cap = rw->pair_cap;
        if (dynamic_schedule()) af.work_order = rw->wq_order.as<uint32_t>();
        af.sem_vec = (C % 2 == 0) && (reinterpret_cast<uintptr_t>(s->semantics) % 8 == 0) &&
                     (reinterpret_cast<uintptr_t>(g->dsemantics) % 8 == 0);
    }
    ctx->timer.begin(MSPLAT_STAGE_BACKWARD, st);
    if (sizeof(Real) == 4 && !ctx->deterministic && dynamic_schedule() && !r->order_valid)  // else the forward's
        launch_work_order(r->ev_count.as<uint32_t>(), r->tiles_x * r->tiles_y * 8, r->wq_order.as<uint32_t>(),
                          r->wq_scratch.as<uint32_t>(), st);
    launch_backward_blend<Real>(a, r->tiles_x * r->tiles_y, st);
    if (ctx->deterministic)
        launch_deterministic_reduce<Real>(a, det, r->d_inst_count.as<int64_t>(), det_count, st);
    ctx->timer.end(st);
    ProjBackwardArgs<Real> p{};
    p.n = n;
    p.C = C;
    p.deg = s->sh_degree;
    p.K = K;
    p.cam = r->cam;
    p.means = static_cast<const Real*>(s->means);
    p.quats = static_cast<const Real*>(s->quats);
    p.log_scales = static_cast<const Real*>(s->log_scales);
    p.opacity_logits = static_cast<const Real*>(s->opacity_logits);
    p.sh = static_cast<const Real*>(s->sh);
    p.visible = r->visible.as<uint8_t>();
    p.clamped_bits = r->clamped.as<uint8_t>();
    p.acc_dcolor = a.acc_dcolor;
    p.acc16 = a.acc16;
    p.g_pos = a.g_pos;
    p.g_rot = a.g_rot;
    p.g_scale = a.g_scale;
    p.g_opac = a.g_opac;
    p.g_sh = static_cast<Real*>(g->dsh);
    p.g_k = a.g_k;
    p.g_sem = a.g_sem;
    // chain_activations is linear per Gaussian, so a multi-view sum is chained
    // once by the caller (msplat_chain_activations) after the last view.
    p.chain = chain && !accumulate;
    p.depth_moments = sizeof(Real) == 4 && !a.partial;  // the FP32 phase B (backward_pairs_kernel)
    p.sigma = r->rp.sigma_scale;
    p.err = ctx->d_err;
    ctx->timer.begin(MSPLAT_STAGE_PROJ_BWD, st);
    launch_projection_backward<Real>(p, st);
    ctx->timer.end(st);
    CUDA_TRY(cudaGetLastError());
    return MSPLAT_OK;
}

}  // namespace

// =====================================================================  ABI
namespace {

template <typename Real>
msplat_status frame_losses_impl(msplat_context* ctx, int C, const Cam& cam, const msplat_normal_config* ncfg,
                                const msplat_frame* f, const msplat_ground_truth* gt, const double lambdas[6],
                                msplat_pixel_grads* out) {
    const size_t HW = size_t(cam.W) * cam.H, R = sizeof(Real);
    LossArgs<Real> a{};
    a.W = cam.W;
    a.H = cam.H;
    a.C = C;
    for (int i = 0; i < 6; ++i) {
        a.lambdas[i] = lambdas[i];
        a.en[i] = lambdas[i] > 0;
    }
    // losses.cpp:24-35: normalised Gaussian window, sigma 1.5
    double wsum = 0;
    for (int i = 0; i < 11; ++i) {
        const double d = i - 5.0;
        a.ssim_w[i] = std::exp(-d * d / (2.0 * 1.5 * 1.5));
        wsum += a.ssim_w[i];
    }
    for (int i = 0; i < 11; ++i) a.ssim_w[i] /= wsum;
    const size_t nv = a.en[1] ? size_t(cam.W - 10) * (cam.H - 10) : 0;
    a.ssim_inv_count = a.en[1] ? 1.0 / (double(nv) * 3) : 0;
    a.color = static_cast<const Real*>(f->color);
    a.depth = static_cast<const Real*>(f->depth);
    a.sem = static_cast<const Real*>(f->semantics);
    a.kmap = static_cast<const Real*>(f->kmap);
    a.normals = static_cast<const Real*>(f->normals);
    a.gt_rgb = static_cast<const Real*>(gt->rgb);
    a.gt_depth = static_cast<const Real*>(gt->depth);
    a.gt_normal = static_cast<const Real*>(gt->normal);
    a.labels = gt->labels;
    CUDA_TRY(ctx->loss_acc.ensure(8 * sizeof(double)));
    CUDA_TRY(ctx->loss_report.ensure(20 * sizeof(double)));
    a.acc = ctx->loss_acc.as<double>();
    a.report = ctx->loss_report.as<double>();
    if (a.en[1]) {
        CUDA_TRY(ctx->ssim_maps.ensure(9 * nv * R));
        CUDA_TRY(ctx->ssim_grad.ensure(3 * HW * R));
        a.ssim_maps = ctx->ssim_maps.as<Real>();
        a.ssim_grad = ctx->ssim_grad.as<Real>();
    }
    a.dcolor = static_cast<Real*>(const_cast<void*>(out->dcolor));
    a.ddepth = static_cast<Real*>(const_cast<void*>(out->ddepth));
    a.dsem = C > 0 ? static_cast<Real*>(const_cast<void*>(out->dsemantics)) : nullptr;
    a.dkmap = static_cast<Real*>(const_cast<void*>(out->dkmap));
    if (a.en[2]) {
        CUDA_TRY(ctx->loss_dN.ensure(3 * HW * R));
        a.dN = ctx->loss_dN.as<Real>();
    }
    if (a.en[4] && C > 0) {
        CUDA_TRY(ctx->loss_ce.ensure(2 * HW * R));
        a.ce_stats = ctx->loss_ce.as<Real>();
    }
    a.err = ctx->d_err;
    launch_frame_losses<Real>(a, ctx->stream);
    CUDA_TRY(cudaGetLastError());
    return MSPLAT_OK;
}

}  // namespace

extern "C" {

const char* msplat_last_error(void) { return g_error.c_str(); }
int msplat_abi_version(void) { return MSPLAT_ABI_VERSION; }

msplat_status msplat_context_create(int device, void* cuda_stream, msplat_context** out) {
    if (!out) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "null output");
    *out = nullptr;
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "context: no such device");
    DeviceGuard device_guard_(device);  // the caller's current device is restored on return
    auto* ctx = new msplat_context();
    ctx->device = device;
    if (cuda_stream) {
        ctx->stream = static_cast<cudaStream_t>(cuda_stream);
    } else {
        cudaError_t e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            delete ctx;
            CUDA_TRY(e);
        }
        ctx->own_stream = true;
    }
    CUDA_TRY(cudaMalloc(&ctx->d_err, sizeof(DeviceError)));
    CUDA_TRY(cudaMemset(ctx->d_err, 0, sizeof(DeviceError)));
    CUDA_TRY(cudaMallocHost(&ctx->h_err, sizeof(DeviceError)));
    CUDA_TRY(cudaMallocHost(&ctx->h_u64, 64));
    *out = ctx;
    return MSPLAT_OK;
}

void msplat_context_destroy(msplat_context* ctx) {
    CTX_DEVICE_GUARD(ctx);
    if (!ctx) return;
    cudaStreamSynchronize(ctx->stream);
    for (DevBuf* b : {&ctx->acc_dcolor, &ctx->acc16, &ctx->loss_acc, &ctx->loss_report, &ctx->metric_acc, &ctx->metric_hist, &ctx->ssim_maps, &ctx->ssim_grad, &ctx->loss_dN, &ctx->loss_ce, &ctx->init_pts,
                       &ctx->init_cols, &ctx->init_logs, &ctx->cmp_k32, &ctx->cmp_idx, &ctx->cmp_tiles, &ctx->cmp_total,
                       &ctx->ddepth_total, &ctx->normal_dv, &ctx->kept, &ctx->det_partial, &ctx->det_keys,
                       &ctx->det_keys_alt, &ctx->det_vals, &ctx->det_vals_alt, &ctx->det_range})
        b->release();
    cudaFree(ctx->d_err);
    cudaFreeHost(ctx->h_err);
    cudaFreeHost(ctx->h_u64);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

msplat_status msplat_context_set_stream(msplat_context* ctx, void* cuda_stream) {
    CTX_DEVICE_GUARD(ctx);
    if (!ctx) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "null context");
    if (ctx->own_stream) {
        cudaStreamSynchronize(ctx->stream);
        cudaStreamDestroy(ctx->stream);
        ctx->own_stream = false;
    }
    ctx->stream = static_cast<cudaStream_t>(cuda_stream);
    return MSPLAT_OK;
}

msplat_status msplat_context_check(msplat_context* ctx) {
    CTX_DEVICE_GUARD(ctx);
    if (!ctx) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "null context");
    CUDA_TRY(cudaGetLastError());
    return drain_device_error(ctx, 0);
}

msplat_status msplat_replay_create(msplat_context* ctx, msplat_replay** out) {
    CTX_DEVICE_GUARD(ctx);
    if (!ctx || !out) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "null argument");
    *out = new msplat_replay();
    (*out)->ctx = ctx;
    return MSPLAT_OK;
}

void msplat_replay_destroy(msplat_replay* r) {
    REPLAY_DEVICE_GUARD(r);
    if (!r) return;
    cudaStreamSynchronize(r->ctx->stream);
    r->release_all();
    delete r;
}

msplat_status msplat_replay_set_capture(msplat_replay* r, int flags) {
    REPLAY_DEVICE_GUARD(r);
    if (!r) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "null replay");
    r->capture = flags;
    return MSPLAT_OK;
}

msplat_status msplat_param_layout(int64_t n, int C, int deg, int64_t off[8]) {
    if (n < 0 || C < 0 || deg < 0 || deg > 3) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "bad layout query");
    const int64_t sizes[7] = {3, 4, 3, 1, 1, 3 * sh_coeffs(deg), C};
    off[0] = 0;
    for (int i = 0; i < 7; ++i) off[i + 1] = off[i] + n * sizes[i];
    return MSPLAT_OK;
}

static msplat_status rasterize_entry(msplat_context* ctx, const msplat_scene* s, const msplat_camera* cam,
                                     const msplat_render_config* cfg, const msplat_frame* f, msplat_replay* replay,
                                     bool sync) {
    if (!ctx || !cfg || !f) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "rasterize: null argument");
    msplat_status st = check_scene(s);
    if (st != MSPLAT_OK) return st;
    Cam c;
    if ((st = make_cam(cam, c)) != MSPLAT_OK) return st;
    if (!f->transmittance) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "rasterize: transmittance buffer required");
    msplat_replay local;
    local.ctx = ctx;
    msplat_replay* r = replay ? replay : &local;
    r->cam = c;
    r->rp.sigma_scale = cfg->sigma_scale;
    for (int i = 0; i < 3; ++i) r->rp.bg[i] = cfg->background[i];
    r->rp.early_stop_T = cfg->early_stop_transmittance;
    r->rp.early_termination = cfg->early_termination;
    if ((st = size_replay(r, s->dtype, s->n, s->num_classes, s->sh_degree, c.W, c.H)) != MSPLAT_OK) return st;
    st = s->dtype == MSPLAT_F64 ? rasterize_impl<double>(ctx, s, cfg, f, r, sync)
                                : rasterize_impl<float>(ctx, s, cfg, f, r, sync);
    if (st == MSPLAT_OK && (sync || !replay)) st = drain_device_error(ctx, c.W);
    if (!replay) {
        cudaStreamSynchronize(ctx->stream);
        local.release_all();
    }
    return st;
}

msplat_status msplat_rasterize(msplat_context* ctx, const msplat_scene* s, const msplat_camera* cam,
                               const msplat_render_config* cfg, const msplat_frame* f, msplat_replay* replay) {
    CTX_DEVICE_GUARD(ctx);
    // Inside a CUDA-graph capture the call stays asynchronous (no capacity
    // read-back, errors latched for the next synchronizing call); the replay
    // must have been sized by an eager call first.
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (ctx) CUDA_TRY(cudaStreamIsCapturing(ctx->stream, &cs));
    const bool capturing = cs != cudaStreamCaptureStatusNone;
    if (capturing && (!replay || replay->inst_cap == 0 || !replay->valid))
        return set_error(MSPLAT_ERR_RUNTIME, "rasterize: capture before any eager call with this replay");
    return rasterize_entry(ctx, s, cam, cfg, f, replay, !capturing);
}

msplat_status msplat_estimate_normals(msplat_context* ctx, int dtype, const void* depth, const void* T,
                                      const msplat_camera* cam, const msplat_normal_config* ncfg, void* normals) {
    CTX_DEVICE_GUARD(ctx);
    if (!ctx || !depth || !T || !normals) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "estimate_normals: null argument");
    msplat_status st = check_ncfg(ncfg);
    if (st != MSPLAT_OK) return st;
    Cam c;
    if ((st = make_cam(cam, c)) != MSPLAT_OK) return st;
    ctx->timer.begin(MSPLAT_STAGE_NORMALS, ctx->stream);
    if (dtype == MSPLAT_F64) {
        auto a = normal_args<double>(c, ncfg, depth, T);
        a.normals = static_cast<double*>(normals);
        launch_normals_forward<double>(a, ctx->stream);
    } else {
        auto a = normal_args<float>(c, ncfg, depth, T);
        a.normals = static_cast<float*>(normals);
        launch_normals_forward<float>(a, ctx->stream);
    }
    ctx->timer.end(ctx->stream);
    CUDA_TRY(cudaGetLastError());
    return MSPLAT_OK;
}

msplat_status msplat_normals_backward(msplat_context* ctx, int dtype, const void* dN, const void* depth, const void* T,
                                      const msplat_camera* cam, const msplat_normal_config* ncfg, double seed,
                                      void* dD) {
    CTX_DEVICE_GUARD(ctx);
    if (!ctx || !dN || !depth || !T || !dD)
        return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "normals_backward: gradient shape mismatch");
    msplat_status st = check_ncfg(ncfg);
    if (st != MSPLAT_OK) return st;
    Cam c;
    if ((st = make_cam(cam, c)) != MSPLAT_OK) return st;
    const size_t HW = size_t(c.W) * c.H, R = real_size(dtype);
    CUDA_TRY(ctx->normal_dv.ensure(12 * HW * R));
    ctx->timer.begin(MSPLAT_STAGE_NORMALS_BWD, ctx->stream);
    if (dtype == MSPLAT_F64) {
        auto a = normal_args<double>(c, ncfg, depth, T);
        a.dN = static_cast<const double*>(dN);
        a.dv = ctx->normal_dv.as<double>();
        a.dD = static_cast<double*>(dD);
        a.seed = seed;
        launch_normals_backward<double>(a, ctx->stream);
    } else {
        auto a = normal_args<float>(c, ncfg, depth, T);
        a.dN = static_cast<const float*>(dN);
        a.dv = ctx->normal_dv.as<float>();
        a.dD = static_cast<float*>(dD);
        a.seed = seed;
        launch_normals_backward<float>(a, ctx->stream);
    }
    ctx->timer.end(ctx->stream);
    CUDA_TRY(cudaGetLastError());
    return MSPLAT_OK;
}

static msplat_status backward_checks(const msplat_scene* s, const msplat_camera* cam, const msplat_frame* f,
                                     const msplat_replay* r, const msplat_pixel_grads* pix, const msplat_grads* g) {
    msplat_status st = check_scene(s);
    if (st != MSPLAT_OK) return st;
    if (!r || !r->valid || r->n != s->n || r->deg != s->sh_degree || r->C != s->num_classes || r->dtype != s->dtype)
        return set_error(MSPLAT_ERR_RUNTIME, "rasterize_backward: replay state does not match the scene");
    if (!cam || cam->width != r->W || cam->height != r->H || !f || !f->transmittance)
        return set_error(MSPLAT_ERR_RUNTIME, "rasterize_backward: frame/view size mismatch");
    if (!pix || !pix->dcolor || !pix->ddepth || !pix->dkmap || (s->num_classes > 0 && !pix->dsemantics))
        return set_error(MSPLAT_ERR_RUNTIME, "rasterize_backward: pixel-gradient shape mismatch");
    if (!g || !g->dposition || !g->drotation || !g->dscale || !g->dopacity || !g->dk || !g->dsh ||
        (s->num_classes > 0 && !g->dsemantics))
        return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "rasterize_backward: null gradient buffer");
    return MSPLAT_OK;
}

msplat_status msplat_rasterize_backward(msplat_context* ctx, const msplat_scene* s, const msplat_camera* cam,
                                        const msplat_frame* f, const msplat_replay* r, const msplat_pixel_grads* pix,
                                        msplat_grads* g) {
    CTX_DEVICE_GUARD(ctx);
    if (!ctx) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "null context");
    msplat_status st = backward_checks(s, cam, f, r, pix, g);
    if (st != MSPLAT_OK) return st;
    st = s->dtype == MSPLAT_F64 ? backward_impl<double>(ctx, s, f, r, pix, pix->ddepth, g, 0, 0)
                                : backward_impl<float>(ctx, s, f, r, pix, pix->ddepth, g, 0, 0);
    if (st != MSPLAT_OK) return st;
    return drain_device_error(ctx, r->W);
}

msplat_status msplat_chain_activations(msplat_context* ctx, const msplat_scene* s, msplat_grads* g) {
    CTX_DEVICE_GUARD(ctx);
    if (!ctx || !g) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "chain_activations: null argument");
    msplat_status st = check_scene(s);
    if (st != MSPLAT_OK) return st;
    if (s->dtype == MSPLAT_F64)
        launch_chain<double>(s->n, static_cast<const double*>(s->quats), static_cast<const double*>(s->log_scales),
                             static_cast<const double*>(s->opacity_logits), static_cast<double*>(g->drotation),
                             static_cast<double*>(g->dscale), static_cast<double*>(g->dopacity), ctx->stream);
    else
        launch_chain<float>(s->n, static_cast<const float*>(s->quats), static_cast<const float*>(s->log_scales),
                            static_cast<const float*>(s->opacity_logits), static_cast<float*>(g->drotation),
                            static_cast<float*>(g->dscale), static_cast<float*>(g->dopacity), ctx->stream);
    CUDA_TRY(cudaGetLastError());
    return MSPLAT_OK;
}

msplat_status msplat_fwd_bwd(msplat_context* ctx, const msplat_scene* s, const msplat_camera* cam,
                             const msplat_render_config* cfg, const msplat_normal_config* ncfg, const msplat_frame* f,
                             const msplat_pixel_grads* pix, msplat_grads* g, int chain, int accumulate,
                             msplat_replay* r) {
    CTX_DEVICE_GUARD(ctx);
    if (!ctx || !r || !f || !f->depth || !f->transmittance)
        return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "fwd_bwd: null argument (replay, depth and T required)");
    msplat_status st = check_ncfg(ncfg);
    if (st != MSPLAT_OK) return st;
    // First use of a replay sizes the instance buffers synchronously; later
    // calls stay asynchronous (capturable in a CUDA graph).
    const bool first = r->inst_cap == 0 || !r->valid;
    st = rasterize_entry(ctx, s, cam, cfg, f, r, first);
    if (st != MSPLAT_OK) return st;
    const size_t HW = size_t(r->W) * r->H, R = real_size(s->dtype);
    CUDA_TRY(ctx->ddepth_total.ensure(HW * R));
    CUDA_TRY(cudaMemcpyAsync(ctx->ddepth_total.p, pix->ddepth, HW * R, cudaMemcpyDeviceToDevice, ctx->stream));
    if (f->normals) {
        st = msplat_estimate_normals(ctx, s->dtype, f->depth, f->transmittance, cam, ncfg, f->normals);
        if (st != MSPLAT_OK) return st;
    }
    if (pix->dnormals) {
        st = msplat_normals_backward(ctx, s->dtype, pix->dnormals, f->depth, f->transmittance, cam, ncfg, 1.0,
                                     ctx->ddepth_total.p);
        if (st != MSPLAT_OK) return st;
    }
    st = backward_checks(s, cam, f, r, pix, g);
    if (st != MSPLAT_OK) return st;
    st = s->dtype == MSPLAT_F64
             ? backward_impl<double>(ctx, s, f, r, pix, ctx->ddepth_total.p, g, chain, accumulate)
             : backward_impl<float>(ctx, s, f, r, pix, ctx->ddepth_total.p, g, chain, accumulate);
    return st;
}

static msplat_status adam_range_impl(msplat_context* ctx, int dtype, int64_t n, int C, int deg, int64_t begin,
                                     int64_t count, void* params, const void* grads, void* m, void* v,
                                     int64_t step, const double lr[7], const char* who) {
    if (!ctx || !params || !grads || !m || !v || !lr)
        return set_error(MSPLAT_ERR_INVALID_ARGUMENT, std::string(who) + ": null argument");
    if (step < 1) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, std::string(who) + ": step must be >= 1");
    if (dtype != MSPLAT_F32 && dtype != MSPLAT_F64)
        return set_error(MSPLAT_ERR_INVALID_ARGUMENT, std::string(who) + ": dtype must be MSPLAT_F32 or MSPLAT_F64");
    int64_t off[8];
    msplat_status st = msplat_param_layout(n, C, deg, off);
    if (st != MSPLAT_OK) return st;
    if (count < 0) count = off[7] - begin;
    if (begin < 0 || begin > off[7] || count < 0 || begin + count > off[7])
        return set_error(MSPLAT_ERR_INVALID_ARGUMENT, std::string(who) + ": range outside the packed buffer");
    const double bc1 = 1 - std::pow(0.9, double(step)), bc2 = 1 - std::pow(0.999, double(step));
    ctx->timer.begin(MSPLAT_STAGE_OPTIM, ctx->stream);
    if (dtype == MSPLAT_F64)
        launch_adam<double>(begin, count, off, lr, static_cast<double*>(params), static_cast<const double*>(grads),
                            static_cast<double*>(m), static_cast<double*>(v), bc1, bc2, ctx->stream);
    else
        launch_adam<float>(begin, count, off, lr, static_cast<float*>(params), static_cast<const float*>(grads),
                           static_cast<float*>(m), static_cast<float*>(v), bc1, bc2, ctx->stream);
    ctx->timer.end(ctx->stream);
    CUDA_TRY(cudaGetLastError());
    return MSPLAT_OK;
}

msplat_status msplat_adam_step(msplat_context* ctx, int dtype, int64_t n, int C, int deg, void* params,
                               const void* grads, void* m, void* v, int64_t step, const double lr[7]) {
    CTX_DEVICE_GUARD(ctx);
    return adam_range_impl(ctx, dtype, n, C, deg, 0, -1, params, grads, m, v, step, lr, "adam_step");
}

msplat_status msplat_adam_step_range(msplat_context* ctx, int dtype, int64_t n, int C, int deg, int64_t begin,
                                     int64_t count, void* params, const void* grads, void* m, void* v,
                                     int64_t step, const double lr[7]) {
    CTX_DEVICE_GUARD(ctx);
    return adam_range_impl(ctx, dtype, n, C, deg, begin, count, params, grads, m, v, step, lr, "adam_step_range");
}

msplat_status msplat_accumulate(msplat_context* ctx, int dtype, int64_t count, void* dst, const void* src) {
    CTX_DEVICE_GUARD(ctx);
    if (!ctx || (count > 0 && (!dst || !src))) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "accumulate: null argument");
    if (count < 0) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "accumulate: negative count");
    if (dtype != MSPLAT_F32 && dtype != MSPLAT_F64)
        return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "accumulate: dtype must be MSPLAT_F32 or MSPLAT_F64");
    if (dtype == MSPLAT_F64)
        launch_accumulate<double>(count, static_cast<double*>(dst), static_cast<const double*>(src), ctx->stream);
    else
        launch_accumulate<float>(count, static_cast<float*>(dst), static_cast<const float*>(src), ctx->stream);
    CUDA_TRY(cudaGetLastError());
    return MSPLAT_OK;
}

msplat_status msplat_context_set_timing(msplat_context* ctx, int enable) {
    CTX_DEVICE_GUARD(ctx);
    if (!ctx) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "null context");
    ctx->timer.enabled = enable != 0;
    return MSPLAT_OK;
}

msplat_status msplat_frame_losses(msplat_context* ctx, int dtype, int num_classes, const msplat_camera* camera,
                                  const msplat_normal_config* ncfg, const msplat_frame* frame,
                                  const msplat_ground_truth* gt, const double lambdas[6], msplat_pixel_grads* out,
                                  msplat_loss_report* host_report) {
    CTX_DEVICE_GUARD(ctx);
    if (!ctx || !frame || !gt || !lambdas || !out) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "frame_losses: null argument");
    if (dtype != MSPLAT_F32 && dtype != MSPLAT_F64)
        return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "frame_losses: dtype must be MSPLAT_F32 or MSPLAT_F64");
    Cam c;
    msplat_status st = make_cam(camera, c);
    if (st != MSPLAT_OK) return st;
    if ((st = check_ncfg(ncfg)) != MSPLAT_OK) return st;
    // trainer.cpp:181-224: an enabled modality needs its ground truth
    if ((lambdas[0] > 0 || lambdas[1] > 0) && !gt->rgb)
        return set_error(MSPLAT_ERR_RUNTIME, "rgb loss enabled but the frame has no rgb ground truth (<missing>)");
    if (lambdas[2] > 0 && !gt->normal)
        return set_error(MSPLAT_ERR_RUNTIME, "normal loss enabled but the frame has no normal ground truth (<missing>)");
    if (lambdas[3] > 0 && !gt->depth)
        return set_error(MSPLAT_ERR_RUNTIME, "depth loss enabled but the frame has no depth ground truth (<missing>)");
    if (lambdas[4] > 0 && !gt->labels)
        return set_error(MSPLAT_ERR_RUNTIME,
                         "segmentation loss enabled but the frame has no label ground truth (<missing>)");
    if (lambdas[1] > 0 && (c.W < 11 || c.H < 11))
        return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "ssim_loss: frame smaller than the 11x11 window");
    if (lambdas[4] > 0 && num_classes < 1)
        return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "cross_entropy_seg: no semantic channels");
    if (!frame->color || !frame->depth || !frame->kmap || !frame->transmittance ||
        (lambdas[2] > 0 && !frame->normals) || (num_classes > 0 && !frame->semantics) || !out->dcolor ||
        !out->ddepth || !out->dkmap || (num_classes > 0 && !out->dsemantics))
        return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "frame_losses: missing frame or gradient buffer");
    st = dtype == MSPLAT_F64 ? frame_losses_impl<double>(ctx, num_classes, c, ncfg, frame, gt, lambdas, out)
                             : frame_losses_impl<float>(ctx, num_classes, c, ncfg, frame, gt, lambdas, out);
    if (st != MSPLAT_OK) return st;
    // The normal term reaches the Gaussians through the depth map
    // (trainer.cpp:258-262): dD += normals_backward(seed_normal * dL/dN).
    if (lambdas[2] > 0) {
        st = msplat_normals_backward(ctx, dtype, ctx->loss_dN.p, frame->depth, frame->transmittance, camera, ncfg, 1.0,
                                     const_cast<void*>(out->ddepth));
        if (st != MSPLAT_OK) return st;
    }
    if (host_report) {
        CUDA_TRY(cudaMemcpyAsync(host_report, ctx->loss_report.p, sizeof(msplat_loss_report), cudaMemcpyDeviceToHost,
                                 ctx->stream));
        return drain_device_error(ctx, c.W);
    }
    return MSPLAT_OK;
}

const double* msplat_loss_report_device(msplat_context* ctx) {
    CTX_DEVICE_GUARD(ctx);
    return ctx ? static_cast<const double*>(ctx->loss_report.p) : nullptr;
}

msplat_status msplat_frame_metrics(msplat_context* ctx, int dtype, int width, int height, int num_classes,
                                   const void* color, const void* gt_rgb, const void* depth, const void* gt_depth,
                                   const uint8_t* depth_mask, const void* normals, const void* gt_normal,
                                   const uint8_t* normal_mask, const void* semantics, const uint8_t* gt_labels,
                                   const uint8_t* label_mask, msplat_metric_report* out) {
    CTX_DEVICE_GUARD(ctx);
    if (!ctx || !out) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "frame_metrics: null argument");
    if (width < 1 || height < 1 || num_classes < 0)
        return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "frame_metrics: bad frame size");
    if (dtype != MSPLAT_F32 && dtype != MSPLAT_F64)
        return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "frame_metrics: dtype must be MSPLAT_F32 or MSPLAT_F64");
    const bool do_rgb = color && gt_rgb, do_depth = depth && gt_depth && depth_mask,
               do_normal = normals && gt_normal && normal_mask,
               do_sem = semantics && gt_labels && label_mask && num_classes > 0;
    if (do_rgb && (width < 11 || height < 11))
        return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "ssim_loss: frame smaller than the 11x11 window");
    CUDA_TRY(ctx->metric_acc.ensure(9 * sizeof(double)));
    CUDA_TRY(ctx->metric_hist.ensure(3 * size_t(std::max(num_classes, 1)) * 8));
    double w[11], wsum = 0;
    for (int i = 0; i < 11; ++i) {
        const double d = i - 5.0;
        w[i] = std::exp(-d * d / (2.0 * 1.5 * 1.5));
        wsum += w[i];
    }
    auto fill = [&](auto& a, auto tag) {
        using Real = decltype(tag);
        a.W = width;
        a.H = height;
        a.C = do_sem ? num_classes : 0;
        for (int i = 0; i < 11; ++i) a.ssim_w[i] = w[i] / wsum;
        a.color = do_rgb ? static_cast<const Real*>(color) : nullptr;
        a.gt_rgb = static_cast<const Real*>(gt_rgb);
        a.depth = do_depth ? static_cast<const Real*>(depth) : nullptr;
        a.gt_depth = static_cast<const Real*>(gt_depth);
        a.depth_mask = depth_mask;
        a.normals = do_normal ? static_cast<const Real*>(normals) : nullptr;
        a.gt_normal = static_cast<const Real*>(gt_normal);
        a.normal_mask = normal_mask;
        a.sem = do_sem ? static_cast<const Real*>(semantics) : nullptr;
        a.labels = gt_labels;
        a.label_mask = label_mask;
        a.acc = ctx->metric_acc.as<double>();
        a.hist = ctx->metric_hist.as<unsigned long long>();
        a.err = ctx->d_err;
    };
    if (dtype == MSPLAT_F64) {
        MetricArgs<double> a{};
        fill(a, double{});
        launch_frame_metrics<double>(a, ctx->stream);
    } else {
        MetricArgs<float> a{};
        fill(a, float{});
        launch_frame_metrics<float>(a, ctx->stream);
    }
    CUDA_TRY(cudaGetLastError());
    double acc[9];
    std::vector<unsigned long long> hist(3 * size_t(std::max(num_classes, 1)), 0);
    CUDA_TRY(cudaMemcpyAsync(acc, ctx->metric_acc.p, sizeof acc, cudaMemcpyDeviceToHost, ctx->stream));
    if (do_sem)
        CUDA_TRY(cudaMemcpyAsync(hist.data(), ctx->metric_hist.p, hist.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
    msplat_status st = drain_device_error(ctx, width);
    if (st != MSPLAT_OK) return st;
    *out = msplat_metric_report{};
    const double HW = double(width) * height;
    if (do_rgb) {  // metrics.cpp:68-82, 84
        const double mse = acc[0] / (3 * HW);
        out->psnr = mse <= 1e-10 ? 100.0 : std::min(100.0, 10.0 * std::log10(1.0 / mse));
        out->has_psnr = 1;
        const double inv = 1.0 / (double(width - 10) * double(height - 10) * 3);
        out->ssim = 1.0 - (1.0 - acc[8] * inv);
        out->has_ssim = 1;
    }
    if (do_depth) {  // metrics.cpp:86-119
        if (acc[2] > 0) {
            out->abs_rel = acc[1] / acc[2];
            out->has_abs_rel = 1;
        }
        if (acc[4] > 0) {
            out->rmse = std::sqrt(acc[3] / acc[4]);
            out->has_rmse = 1;
        }
    }
    if (do_normal && acc[6] > 0) {  // metrics.cpp:121-137
        out->cos_simi = acc[5] / acc[6];
        out->has_cos_simi = 1;
    }
    if (do_sem && acc[7] > 0) {  // metrics.cpp:152-187
        double sum = 0;
        int classes = 0;
        for (int c = 0; c < num_classes; ++c) {
            const unsigned long long inter = hist[size_t(c)], pred = hist[size_t(num_classes + c)],
                                     truth = hist[size_t(2 * num_classes + c)];
            const unsigned long long uni = pred + truth - inter;
            if (uni == 0) continue;
            sum += double(inter) / double(uni);
            ++classes;
        }
        if (classes > 0) {
            out->miou = sum / classes;
            out->has_miou = 1;
        }
    }
    return MSPLAT_OK;
}

static msplat_status io_status(const IoResult& r) {
    if (r.code == 0) return MSPLAT_OK;
    if (r.code == 1) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, r.msg.c_str());
    if (r.code == 4) return set_error(MSPLAT_ERR_CUDA, r.msg.c_str());
    return set_error(MSPLAT_ERR_RUNTIME, r.msg.c_str());
}

msplat_status msplat_ply_scene_info(const char* path, int64_t* n, int* num_classes, int* sh_degree) {
    if (!path || !n || !num_classes || !sh_degree) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "ply: null argument");
    return io_status(ply_scene_info(path, n, num_classes, sh_degree));
}

msplat_status msplat_load_scene_ply(msplat_context* ctx, const char* path, int dtype, void* params) {
    CTX_DEVICE_GUARD(ctx);
    if (!ctx || !path || !params) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "load_scene_ply: null argument");
    if (dtype == MSPLAT_F64) return io_status(ply_load_scene<double>(path, static_cast<double*>(params), ctx->stream, ctx->d_err));
    if (dtype == MSPLAT_F32) return io_status(ply_load_scene<float>(path, static_cast<float*>(params), ctx->stream, ctx->d_err));
    return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "load_scene_ply: dtype must be MSPLAT_F32 or MSPLAT_F64");
}

msplat_status msplat_save_scene_ply(msplat_context* ctx, const char* path, int dtype, int64_t n, int num_classes,
                                    int sh_degree, const void* params) {
    CTX_DEVICE_GUARD(ctx);
    if (!ctx || !path || (n > 0 && !params)) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "save_scene_ply: null argument");
    if (sh_degree < 0 || sh_degree > 3) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "Scene: sh_degree must be in [0,3]");
    if (num_classes < 0) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "Scene: num_classes must be >= 0");
    if (dtype == MSPLAT_F64)
        return io_status(ply_save_scene<double>(path, n, num_classes, sh_degree, static_cast<const double*>(params), ctx->stream));
    if (dtype == MSPLAT_F32)
        return io_status(ply_save_scene<float>(path, n, num_classes, sh_degree, static_cast<const float*>(params), ctx->stream));
    return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "save_scene_ply: dtype must be MSPLAT_F32 or MSPLAT_F64");
}

msplat_status msplat_init_scene(msplat_context* ctx, int dtype, int64_t n, const double* points, const double* colors,
                                int num_classes, int sh_degree, double k_reset, void* params) {
    CTX_DEVICE_GUARD(ctx);
    if (!ctx || !params) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "init_scene: null argument");
    if (n <= 0 || !points) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "init_scene: empty point list");
    if (!colors) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "init_scene: point/color count mismatch");
    if (num_classes < 0 || sh_degree < 0 || sh_degree > 3)
        return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "init_scene: bad class count or SH degree");
    if (dtype != MSPLAT_F32 && dtype != MSPLAT_F64)
        return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "init_scene: dtype must be MSPLAT_F32 or MSPLAT_F64");
    const size_t nn = size_t(n);
    CUDA_TRY(ctx->init_pts.ensure(nn * 3 * 8));
    CUDA_TRY(ctx->init_cols.ensure(nn * 3 * 8));
    CUDA_TRY(ctx->init_logs.ensure(nn * 8));
    CUDA_TRY(cudaMemcpyAsync(ctx->init_pts.p, points, nn * 3 * 8, cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(ctx->init_cols.p, colors, nn * 3 * 8, cudaMemcpyHostToDevice, ctx->stream));
    if (dtype == MSPLAT_F64)
        launch_init_scene<double>(n, num_classes, sh_degree, ctx->init_pts.as<double>(), ctx->init_cols.as<double>(),
                                  ctx->init_logs.as<double>(), k_reset, static_cast<double*>(params), ctx->stream);
    else
        launch_init_scene<float>(n, num_classes, sh_degree, ctx->init_pts.as<double>(), ctx->init_cols.as<double>(),
                                 ctx->init_logs.as<double>(), k_reset, static_cast<float*>(params), ctx->stream);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));  // the host point arrays may be released
    return MSPLAT_OK;
}

msplat_status msplat_prune_compact(msplat_context* ctx, int dtype, int64_t n, int num_classes, int sh_degree,
                                   const uint8_t* keep, int64_t kept, const void* const in[3], void* const out[3],
                                   double k_reset) {
    CTX_DEVICE_GUARD(ctx);
    if (!ctx || !keep || !in || !out || !in[0] || !out[0])
        return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "prune: null argument");
    if (kept <= 0) return set_error(MSPLAT_ERR_RUNTIME, "prune: every gaussian would be removed");
    if (kept > n || num_classes < 0 || sh_degree < 0 || sh_degree > 3)
        return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "prune: bad size");
    const size_t nn = size_t(n);
    CUDA_TRY(ctx->cmp_k32.ensure(nn * 4));
    CUDA_TRY(ctx->cmp_idx.ensure(nn * 4));
    CUDA_TRY(ctx->cmp_tiles.ensure((nn + kScanTile - 1) / kScanTile * 4 + 8));
    CUDA_TRY(ctx->cmp_total.ensure(8));
    if (dtype == MSPLAT_F64) {
        const double* const i3[3] = {static_cast<const double*>(in[0]), static_cast<const double*>(in[1]),
                                     static_cast<const double*>(in[2])};
        double* const o3[3] = {static_cast<double*>(out[0]), static_cast<double*>(out[1]), static_cast<double*>(out[2])};
        launch_prune_compact<double>(n, num_classes, sh_degree, keep, kept, i3, o3, k_reset, ctx->cmp_k32.as<uint32_t>(),
                                     ctx->cmp_idx.as<uint32_t>(), ctx->cmp_tiles.as<uint32_t>(),
                                     ctx->cmp_total.as<uint32_t>(), ctx->stream);
    } else {
        const float* const i3[3] = {static_cast<const float*>(in[0]), static_cast<const float*>(in[1]),
                                    static_cast<const float*>(in[2])};
        float* const o3[3] = {static_cast<float*>(out[0]), static_cast<float*>(out[1]), static_cast<float*>(out[2])};
        launch_prune_compact<float>(n, num_classes, sh_degree, keep, kept, i3, o3, k_reset, ctx->cmp_k32.as<uint32_t>(),
                                    ctx->cmp_idx.as<uint32_t>(), ctx->cmp_tiles.as<uint32_t>(),
                                    ctx->cmp_total.as<uint32_t>(), ctx->stream);
    }
    CUDA_TRY(cudaGetLastError());
    return MSPLAT_OK;
}

msplat_status msplat_context_set_deterministic(msplat_context* ctx, int enable) {
    CTX_DEVICE_GUARD(ctx);
    if (!ctx) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "null context");
    ctx->deterministic = enable != 0;
    return MSPLAT_OK;
}

msplat_status msplat_context_timings(msplat_context* ctx, double ms[MSPLAT_STAGE_COUNT],
                                     int64_t calls[MSPLAT_STAGE_COUNT]) {
    CTX_DEVICE_GUARD(ctx);
    if (!ctx || !ms) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "null argument");
    ctx->timer.collect(ms, calls);
    CUDA_TRY(cudaGetLastError());
    return MSPLAT_OK;
}

int64_t msplat_kernel_launches(void) { return int64_t(g_launches.load()); }

msplat_status msplat_prune_mask(msplat_context* ctx, int dtype, int64_t n, const void* k, double threshold,
                                int keep_small, uint8_t* keep, int64_t* kept) {
    CTX_DEVICE_GUARD(ctx);
    if (!ctx || !k || !keep) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "prune: null argument");
    CUDA_TRY(ctx->kept.ensure(8));
    CUDA_TRY(cudaMemsetAsync(ctx->kept.p, 0, 8, ctx->stream));
    if (dtype == MSPLAT_F64)
        launch_prune_mask<double>(n, static_cast<const double*>(k), threshold, keep_small, keep,
                                  ctx->kept.as<unsigned long long>(), ctx->stream);
    else
        launch_prune_mask<float>(n, static_cast<const float*>(k), threshold, keep_small, keep,
                                 ctx->kept.as<unsigned long long>(), ctx->stream);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(ctx->h_u64, ctx->kept.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    const int64_t kk = int64_t(ctx->h_u64[0]);
    if (kept) *kept = kk;
    if (kk == 0 && n > 0) {
        char buf[128];
        snprintf(buf, sizeof buf, "prune: threshold %f would remove every gaussian", threshold);
        return set_error(MSPLAT_ERR_RUNTIME, buf);
    }
    return MSPLAT_OK;
}

msplat_status msplat_replay_counters(msplat_replay* r, msplat_counters* out) {
    REPLAY_DEVICE_GUARD(r);
    if (!r || !out || !r->valid) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "replay: no forward recorded");
    cudaStream_t st = r->ctx->stream;
    const int64_t tiles = int64_t(r->tiles_x) * r->tiles_y;
    std::vector<uint2> ranges(static_cast<size_t>(tiles));
    unsigned long long vis = 0;
    int64_t inst = 0;
    CUDA_TRY(cudaMemcpyAsync(&vis, r->visible_count.p, 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(&inst, r->d_inst_count.p, 8, cudaMemcpyDeviceToHost, st));
    if (tiles) CUDA_TRY(cudaMemcpyAsync(ranges.data(), r->tile_range.p, size_t(tiles) * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    int64_t mx = 0;
    for (const auto& rg : ranges) mx = std::max<int64_t>(mx, int64_t(rg.y) - int64_t(rg.x));
    out->n = r->n;
    out->visible = int64_t(vis);
    out->instances = inst;
    out->tiles = tiles;
    out->max_tile_list = mx;
    return MSPLAT_OK;
}

msplat_status msplat_replay_bins(msplat_replay* r, int64_t* tile_offsets, int32_t* values, int64_t capacity) {
    REPLAY_DEVICE_GUARD(r);
    if (!r || !r->valid) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "replay: no forward recorded");
    cudaStream_t st = r->ctx->stream;
    const int64_t tiles = int64_t(r->tiles_x) * r->tiles_y;
    std::vector<uint2> ranges(static_cast<size_t>(tiles));
    int64_t inst = 0;
    CUDA_TRY(cudaMemcpyAsync(&inst, r->d_inst_count.p, 8, cudaMemcpyDeviceToHost, st));
    if (tiles) CUDA_TRY(cudaMemcpyAsync(ranges.data(), r->tile_range.p, size_t(tiles) * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (tile_offsets) {
        // Ranges are contiguous in tile order: offsets follow from the lengths.
        int64_t off = 0;
        for (int64_t t = 0; t < tiles; ++t) {
            tile_offsets[t] = off;
            off += int64_t(ranges[size_t(t)].y) - int64_t(ranges[size_t(t)].x);
        }
        tile_offsets[tiles] = off;
    }
    if (values && capacity >= inst && inst > 0)
        CUDA_TRY(cudaMemcpy(values, r->sorted_gauss, size_t(inst) * 4, cudaMemcpyDeviceToHost));
    return MSPLAT_OK;
}

msplat_status msplat_replay_splats(msplat_replay* r, uint8_t* visible, double* center, double* conic,
                                   double* sort_depth, double* radius, double* rgb, uint8_t* clamped) {
    REPLAY_DEVICE_GUARD(r);
    if (!r || !r->valid) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "replay: no forward recorded");
    if (!(r->capture & 1) && (center || conic || sort_depth || radius || rgb))
        return set_error(MSPLAT_ERR_LOGIC, "replay: splat capture was not enabled (msplat_replay_set_capture)");
    CUDA_TRY(cudaStreamSynchronize(r->ctx->stream));
    const size_t n = size_t(r->n);
    if (!n) return MSPLAT_OK;
    if (visible) CUDA_TRY(cudaMemcpy(visible, r->visible.p, n, cudaMemcpyDeviceToHost));
    if (center) CUDA_TRY(cudaMemcpy(center, r->cap_center.p, n * 16, cudaMemcpyDeviceToHost));
    if (conic) CUDA_TRY(cudaMemcpy(conic, r->cap_conic.p, n * 24, cudaMemcpyDeviceToHost));
    if (sort_depth) CUDA_TRY(cudaMemcpy(sort_depth, r->cap_depth.p, n * 8, cudaMemcpyDeviceToHost));
    if (radius) CUDA_TRY(cudaMemcpy(radius, r->cap_radius.p, n * 8, cudaMemcpyDeviceToHost));
    if (rgb) CUDA_TRY(cudaMemcpy(rgb, r->cap_rgb.p, n * 24, cudaMemcpyDeviceToHost));
    if (clamped) {
        std::vector<uint8_t> bits(n);
        CUDA_TRY(cudaMemcpy(bits.data(), r->clamped.p, n, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < n; ++i)
            for (int c = 0; c < 3; ++c) clamped[3 * i + c] = (bits[i] >> c) & 1;
    }
    return MSPLAT_OK;
}

msplat_status msplat_replay_terminus(msplat_replay* r, int32_t* terminus) {
    REPLAY_DEVICE_GUARD(r);
    if (!r || !r->valid || !terminus) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "replay: no forward recorded");
    CUDA_TRY(cudaStreamSynchronize(r->ctx->stream));
    CUDA_TRY(cudaMemcpy(terminus, r->terminus.p, size_t(r->W) * r->H * 4, cudaMemcpyDeviceToHost));
    return MSPLAT_OK;
}

msplat_status msplat_replay_weight_sums(msplat_replay* r, double* ws) {
    REPLAY_DEVICE_GUARD(r);
    if (!r || !r->valid || !ws) return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "replay: no forward recorded");
    if (!(r->capture & 2)) return set_error(MSPLAT_ERR_LOGIC, "replay: weight-sum capture was not enabled");
    CUDA_TRY(cudaStreamSynchronize(r->ctx->stream));
    const size_t n = size_t(r->n);
    if (!n) return MSPLAT_OK;
    if (r->dtype == MSPLAT_F64) {
        CUDA_TRY(cudaMemcpy(ws, r->weight_sums.p, n * 8, cudaMemcpyDeviceToHost));
    } else {
        std::vector<float> tmp(n);
        CUDA_TRY(cudaMemcpy(tmp.data(), r->weight_sums.p, n * 4, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < n; ++i) ws[i] = tmp[i];
    }
    return MSPLAT_OK;
}

msplat_status msplat_bin_and_sort_host(msplat_context* ctx, int64_t n, const uint8_t* visible, const double* center,
                                       const double* radius, const double* sort_depth, int width, int height,
                                       int64_t* tile_offsets, int32_t* values, int64_t capacity, int64_t* count) {
    CTX_DEVICE_GUARD(ctx);
    if (!ctx || (n > 0 && (!visible || !center || !radius || !sort_depth)) || width < 1 || height < 1)
        return set_error(MSPLAT_ERR_INVALID_ARGUMENT, "bin_and_sort: bad argument");
    msplat_replay r;
    r.ctx = ctx;
    msplat_status st = size_replay(&r, MSPLAT_F64, n, 0, 0, width, height);
    if (st != MSPLAT_OK) return st;
    DevBuf dv, dc, dr, dd;
    const size_t nn = size_t(std::max<int64_t>(n, 1));
    CUDA_TRY(dv.ensure(nn));
    CUDA_TRY(dc.ensure(nn * 16));
    CUDA_TRY(dr.ensure(nn * 8));
    CUDA_TRY(dd.ensure(nn * 8));
    if (n > 0) {
        CUDA_TRY(cudaMemcpy(dv.p, visible, size_t(n), cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(dc.p, center, size_t(n) * 16, cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(dr.p, radius, size_t(n) * 8, cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(dd.p, sort_depth, size_t(n) * 8, cudaMemcpyHostToDevice));
    }
    launch_rects_from_splats(n, dv.as<uint8_t>(), dc.as<double>(), dr.as<double>(), dd.as<double>(), width, height,
                             r.depth_key.as<uint64_t>(), r.order.as<uint32_t>(), r.tile_count.as<uint32_t>(),
                             r.tile_rect.as<uint2>(), ctx->stream);
    r.binned_explicit = true;
    st = binning_with_capacity(&r, true);
    if (st == MSPLAT_OK) st = drain_device_error(ctx, width);
    if (st == MSPLAT_OK) {
        r.valid = true;
        int64_t inst = 0;
        cudaMemcpy(&inst, r.d_inst_count.p, 8, cudaMemcpyDeviceToHost);
        if (count) *count = inst;
        st = msplat_replay_bins(&r, tile_offsets, values, capacity);
    }
    cudaStreamSynchronize(ctx->stream);
    r.release_all();
    for (DevBuf* b : {&dv, &dc, &dr, &dd}) b->release();
    return st;
}

}  // extern "C"
