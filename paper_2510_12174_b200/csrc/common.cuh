// Shared device definitions for the sm_100a msplat kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace msplat_cuda {

constexpr int kTile = 16;                     // TileBins::kTileSize (msplat/rasterizer.hpp:34)
constexpr int kTilePixels = kTile * kTile;    // one CTA per tile, one thread per pixel
constexpr double kNearPlane = 0.01;           // msplat/geometry.hpp:63
constexpr double kCovFloor = 0.3;             // msplat/geometry.hpp:64
constexpr double kMinAlpha = 1.0 / 255.0;     // msplat/geometry.hpp:65
constexpr double kMaxAlpha = 0.99;            // msplat/geometry.hpp:66
constexpr double kDegenerateScale = 1e-8;     // msplat/geometry.hpp:30

// Device error word: first fault wins (atomicCAS on code).  Codes mirror the
// reference exception sites.
enum ErrCode : int {
    kErrNone = 0,
    kErrNonFiniteBlend = 1,    // rasterizer.cpp:148-151  (a = pixel, b = primitive)
    kErrNonFiniteOutput = 2,   // rasterizer.cpp:179-183  (a = pixel)
    kErrSceneModified = 3,     // rasterizer_backward.cpp:40-44 (b = primitive)
    kErrNonFiniteGrad = 4,     // scene.cpp:97-106 (b = primitive)
    kErrZeroQuat = 5,          // scene.cpp:49-51 (b = primitive)
    kErrNonFiniteParam = 6,    // scene.cpp:36-38 (b = primitive)
    kErrInstanceOverflow = 7,  // internal: tile-instance buffer too small (a = needed)
    kErrLabelRange = 8,        // losses.cpp:245-249 (a = pixel, b = label)
    kErrMiouLabel = 9,         // metrics.cpp:165-166 (a = pixel, b = label)
    kErrPairOverflow = 10,     // internal: pair-record buffer too small (a = needed, b = capacity)
};

struct DeviceError {
    int code;
    int pad;
    long long a;
    long long b;
    unsigned long long min_b;  // ~(lowest primitive) of an ordered error (raise_error_ordered), 0 = unset
};

__device__ __forceinline__ void raise_error(DeviceError* e, int code, long long a, long long b) {
    if (atomicCAS(&e->code, 0, code) == 0) {
        e->a = a;
        e->b = b;
    }
}

// Errors the reference raises from a sequential scan over primitives
// (Scene::validate scene.cpp:22-40, activate :43-51, check_finite :97-106,
// rasterize_backward's modification check rasterizer_backward.cpp:40-44)
// report the LOWEST offending primitive, whichever thread faults first.
__device__ __forceinline__ void raise_error_ordered(DeviceError* e, int code, long long b) {
    const int old = atomicCAS(&e->code, 0, code);
    if (old != 0 && old != code) return;
    atomicMax(&e->min_b, ~static_cast<unsigned long long>(b));
}

// Camera with the derived world->cam pose, both in double (CameraView).
struct Cam {
    double fx, fy, cx, cy;
    int W, H;
    double Rc2w[9], tc2w[3], Rw2c[9], tw2c[3];
};

// Render constants passed by value to the blend kernels.
struct RenderParams {
    double sigma_scale;
    double bg[3];
    double early_stop_T;
    int early_termination;
};

template <typename Real>
struct Vec3T {
    Real x, y, z;
};

// Per-visible-Gaussian records written by K1 and gathered per tile by K6/K9.
// Alpha-test record (everything a visited pair needs), 12 Reals.
template <typename Real>
struct __align__(16) AlphaRec {  // 64 B (FP32): four 16-byte stores / loads
    Real cx, cy;      // splat centre (pixels)
    Real ca, cb, cc;  // conic (xx, xy, yy)
    Real opacity;     // activated alpha (logistic of the logit)
    Real log_thr;     // log(1/(255*opacity)): power >= log_thr  <=>  alpha >= 1/255
    Real pad;
    // Conservative pixel-space box of the alpha >= 1/255 support (the ellipse
    // power >= log_thr - 1e-3 grown by 0.1% + 1e-3 px).  Used only to skip
    // pairs that would fail the alpha test anyway: results are unchanged.
    Real bx0, bx1, by0, by1;
    // View-dependent colour and gradient factor: the forward reads them with
    // the record it already stages (no per-event gather from BlendRec).
    Real rgb[3], k;
};

// Blend record (everything a blended pair needs beyond the alpha test).
// Rt is R^T of the activated rotation, row-major; inv_axes = 1/(sigma*s).
template <typename Real>
struct __align__(16) BlendRec {  // 128 B (FP32): eight 16-byte stores
    Real Rt[9];
    Real axes[3];     // sigma * s (double path divides like the reference)
    Real inv_axes[3]; // 1 / (sigma * s)
    Real vs[3];       // v_s = R^T (o - mu) / axes   (per view constant)
    Real csq;         // |v_s|^2 - 1
    Real zc;          // sort depth (camera-z of the centre): no-hit fallback
    Real rgb[3];      // view-dependent colour
    Real k;           // gradient factor
    Real hit_ok;      // 0 when an axis is degenerate (< 1e-8): never intersects
    Real q[4];        // unit quaternion (w,x,y,z) of the activated rotation
    Real vl[3];       // v_l = R^T (o - mu), unscaled local camera offset (per view)
};

// FP32 forward depth of a blended pair (K6's depth flush), per Gaussian and
// view: intersect (core/src/geometry.cpp:37-68) rewritten as quadratic forms
// in the pixel offset (dx, dy) from the projected centre (the AlphaRec's
// cx, cy).  With the unnormalised ray d~ = R_c2w (p~ = ((px-cx)/fx,
// (py-cy)/fy, 1)), m = M d~ (M = diag(1/axes) R^T) and v_s:
//   a~ = |m|^2            = A0 + A1 dx + A2 dy + A3 dx^2 + A4 dx dy + A5 dy^2
//   h  = v_s . m          = H0 + H1 dx + H2 dy
//   disc/4 = |m|^2 - |v_s x m|^2 (the Lagrange form of h^2 - a~ c)
//                         = E0 + E1 dx + E2 dy + E3 dx^2 + E4 dx dy + E5 dy^2
// hit <=> disc >= 0 and t = -h / a~ > 0, and the midpoint depth is
// zoff - h / a~ (d~ has camera z = 1).  The coefficients are computed in
// FP64 by K1 about the centre, so the FP32 evaluation is well conditioned;
// decisions within 1e-5 of the terms' magnitude are re-taken in FP64 exactly
// as the reference computes them (intersect_fp64).  A degenerate splat
// (axis < 1e-8) has E = (-1, 0, ...): never a hit.
// The backward (phase B) also needs the small offset of the midpoint from the
// centre: Delta = t - z_c = -(h + z_c a~) / a~ with K = H + z_c A (FP64), and
// (ex, ey) = camera-space (x, y) of the mean minus z_c p0 (p0 = the centre's
// normalised image point), so that P - mu in camera space is
//   (Delta p0x + t dx / fx - ex, Delta p0y + t dy / fy - ey, Delta)
// without cancellation.  The forward reads the first 64 bytes only.
struct __align__(16) DepthRec {  // 96 B
    float E[6];
    float H[3];
    float zc;  // camera-z of the centre: the no-hit depth
    float A[6];
    float K[6];
    float ex, ey;
};

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

}  // namespace msplat_cuda
