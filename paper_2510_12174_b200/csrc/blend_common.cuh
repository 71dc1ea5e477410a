// Per-pixel math shared by the forward (K6) and backward (K9) blends.  Both
// kernels must take identical alpha decisions for a (pixel, Gaussian) pair, so
// the test lives here once.
#pragma once

#include "common.cuh"

namespace msplat_cuda {

template <typename Real>
__device__ __forceinline__ Real fast_exp(Real x);
template <>
__device__ __forceinline__ float fast_exp<float>(float x) { return __expf(x); }
template <>
__device__ __forceinline__ double fast_exp<double>(double x) { return exp(x); }

template <typename Real>
struct PixelRay {
    Real px, py;     // pixel centre (x + 0.5, y + 0.5)
    Real o[3];       // ray origin (camera centre, world)
    Real d[3];       // unit direction (world)
    Real dz;         // R_w2c.row(2) . d  = d(depth)/d(t)
    Real zoff;       // R_w2c.row(2) . o + t_w2c.z  (~0; exact FP64 constant)
};

// compute_ray (core/src/geometry.cpp:31-35) at (x + 0.5, y + 0.5).
template <typename Real>
__device__ __forceinline__ PixelRay<Real> make_ray(const Cam& c, int x, int y) {
    PixelRay<Real> r;
    r.px = Real(x) + Real(0.5);
    r.py = Real(y) + Real(0.5);
    const Real pd[3] = {(r.px - Real(c.cx)) / Real(c.fx), (r.py - Real(c.cy)) / Real(c.fy), Real(1)};
    Real v[3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
        v[i] = Real(c.Rc2w[i * 3 + 0]) * pd[0] + Real(c.Rc2w[i * 3 + 1]) * pd[1] +
               Real(c.Rc2w[i * 3 + 2]) * pd[2];
    const Real nn = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
    const Real inv = nn > Real(0) ? Real(1) / sqrt(nn) : Real(1);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        r.d[i] = v[i] * inv;
        r.o[i] = Real(c.tc2w[i]);
    }
    r.dz = Real(c.Rw2c[6]) * r.d[0] + Real(c.Rw2c[7]) * r.d[1] + Real(c.Rw2c[8]) * r.d[2];
    const double zo = c.Rw2c[6] * c.tc2w[0] + c.Rw2c[7] * c.tc2w[1] + c.Rw2c[8] * c.tc2w[2] + c.tw2c[2];
    r.zoff = Real(zo);
    return r;
}

template <typename Real>
struct AlphaEval {
    Real alpha, gauss, dx, dy;
    bool clamped;
    bool pass;  // alpha >= 1/255
};

// eval_alpha_full (core/src/geometry.cpp:138-152) + the 1/255 skip test
// (rasterizer.cpp:139, rasterizer_backward.cpp:191).  A pre-test on the
// exponent (power < log(1/(255*opacity)) - 1e-3 implies alpha < 1/255 with a
// margin far above rounding) skips the exp for the ~96% of visited pairs that
// fail, without changing any decision.
template <typename Real>
__device__ __forceinline__ AlphaEval<Real> eval_alpha(const AlphaRec<Real>& g, Real px, Real py) {
    AlphaEval<Real> e;
    e.dx = px - g.cx;
    e.dy = py - g.cy;
    const Real power = Real(-0.5) * (g.ca * e.dx * e.dx + g.cc * e.dy * e.dy) - g.cb * e.dx * e.dy;
    e.pass = false;
    e.clamped = false;
    e.alpha = Real(0);
    e.gauss = Real(0);
    if (power > Real(0) || power < g.log_thr - Real(1e-3)) return e;
    e.gauss = fast_exp<Real>(power);
    const Real raw = g.opacity * e.gauss;
    e.clamped = raw > Real(kMaxAlpha);
    e.alpha = e.clamped ? Real(kMaxAlpha) : raw;
    e.pass = !(e.alpha < Real(kMinAlpha));
    return e;
}

template <typename Real>
struct HitEval {
    bool hit;
    Real t_mid, a, b;
    Real ds[3];
};

// intersect (core/src/geometry.cpp:37-64) with the per-view constant v_s and
// |v_s|^2 - 1 precomputed by K1.
template <typename Real>
__device__ __forceinline__ HitEval<Real> intersect(const BlendRec<Real>& g, const PixelRay<Real>& r) {
    HitEval<Real> h;
    h.hit = false;
    if (g.hit_ok == Real(0)) return h;
    Real dl[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) dl[i] = g.Rt[i * 3 + 0] * r.d[0] + g.Rt[i * 3 + 1] * r.d[1] + g.Rt[i * 3 + 2] * r.d[2];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        if constexpr (sizeof(Real) == 8)
            h.ds[i] = dl[i] / g.axes[i];
        else
            h.ds[i] = dl[i] * g.inv_axes[i];
    }
    h.a = h.ds[0] * h.ds[0] + h.ds[1] * h.ds[1] + h.ds[2] * h.ds[2];
    h.b = Real(2) * (g.vs[0] * h.ds[0] + g.vs[1] * h.ds[1] + g.vs[2] * h.ds[2]);
    const Real disc = h.b * h.b - Real(4) * h.a * g.csq;
    if (disc < Real(0) || h.a <= Real(0)) return h;
    h.t_mid = -h.b / (Real(2) * h.a);
    if (h.t_mid <= Real(0)) return h;
    h.hit = true;
    return h;
}

// midpoint_depth (core/src/geometry.cpp:66-68): camera-z of o + t d.
template <typename Real>
__device__ __forceinline__ Real midpoint_depth(const Cam& c, const PixelRay<Real>& r, Real t) {
    if constexpr (sizeof(Real) == 8) {
        const double p0 = r.o[0] + t * r.d[0], p1 = r.o[1] + t * r.d[1], p2 = r.o[2] + t * r.d[2];
        return c.Rw2c[6] * p0 + c.Rw2c[7] * p1 + c.Rw2c[8] * p2 + c.tw2c[2];
    } else {
        return t * r.dz + r.zoff;  // same value without the o-vs-t_w2c cancellation in fp32
    }
}

// Tile-local pixel coordinates: warps cover 8x4 pixel blocks, 2 across x 4 down.
__device__ __forceinline__ int tile_pixel_x(int warp, int lane) { return (warp & 1) * 8 + (lane & 7); }
__device__ __forceinline__ int tile_pixel_y(int warp, int lane) { return (warp >> 1) * 4 + (lane >> 3); }
__device__ __forceinline__ int tile_pixel_index(int warp, int lane) {
    return tile_pixel_y(warp, lane) * kTile + tile_pixel_x(warp, lane);
}

}  // namespace msplat_cuda
