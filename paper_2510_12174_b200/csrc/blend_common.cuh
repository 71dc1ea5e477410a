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

// FP32 blends keep the 32 rays of a warp's 8x4 pixel block in shared memory
// ({d, dz} per pixel plus the camera's zoff), computed once by make_ray, so a
// pair's ray costs one 16-byte load instead of the camera conversions,
// divisions and normalisation.  Values are make_ray's bit for bit (o is not
// used by the FP32 intersect / midpoint_depth).
__device__ __forceinline__ float4 ray_cache_entry(const PixelRay<float>& r) { return make_float4(r.d[0], r.d[1], r.d[2], r.dz); }
__device__ __forceinline__ PixelRay<float> cached_ray(const float4 c, float zoff, int x, int y) {
    PixelRay<float> r;
    r.px = float(x) + 0.5f;
    r.py = float(y) + 0.5f;
    r.d[0] = c.x;
    r.d[1] = c.y;
    r.d[2] = c.z;
    r.dz = c.w;
    r.o[0] = r.o[1] = r.o[2] = 0.f;
    r.zoff = zoff;
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
    Real ds[3];       // d_s = d_l / axes
    Real dl[3];       // d_l = R^T d (unscaled local direction)
    Real depth_fp64;  // set when the FP64 re-decision ran (< 0 otherwise)
};

// Raw scene parameters, for the FP64 re-decision of near-silhouette pairs.
template <typename Real>
struct RawParams {
    const Real *means, *quats, *log_scales;
    double sigma;
};

// intersect() exactly as the reference evaluates it, in FP64 from the raw
// parameters (activate: scene.cpp:42-60; compute_ray: geometry.cpp:31-35;
// intersect: geometry.cpp:37-64).  Used by the FP32 kernels when the FP32
// discriminant or t_mid is too close to zero to decide reliably, so hit/miss
// decisions match the FP64 oracle.  Not inlined: it runs for a tiny fraction
// of blended pairs (grazing rays).
template <typename Real>
__device__ __forceinline__ bool intersect_fp64_impl(const Cam& c, const RawParams<Real>& rp, uint32_t g, Real px,
                                                    Real py, double* t_out, double* a_out, double* b_out,
                                                    double* ds_out, double* depth_out) {
    const double pd[3] = {(double(px) - c.cx) / c.fx, (double(py) - c.cy) / c.fy, 1.0};
    double d[3];
    for (int i = 0; i < 3; ++i) {
        double t = c.Rc2w[i * 3] * pd[0];
        t += c.Rc2w[i * 3 + 1] * pd[1];
        t += c.Rc2w[i * 3 + 2] * pd[2];
        d[i] = t;
    }
    {
        double z = d[0] * d[0];
        z += d[1] * d[1];
        z += d[2] * d[2];
        const double n = sqrt(z);
        for (int i = 0; i < 3; ++i) d[i] = d[i] / n;
    }
    double q[4], n2 = 0;
    for (int j = 0; j < 4; ++j) q[j] = double(rp.quats[4 * size_t(g) + j]);
    n2 = q[0] * q[0];
    n2 += q[1] * q[1];
    n2 += q[2] * q[2];
    n2 += q[3] * q[3];
    double qn = sqrt(n2);
    for (int j = 0; j < 4; ++j) q[j] = q[j] / qn;
    n2 = q[0] * q[0];
    n2 += q[1] * q[1];
    n2 += q[2] * q[2];
    n2 += q[3] * q[3];
    qn = sqrt(n2);
    const double w = q[0] / qn, x = q[1] / qn, y = q[2] / qn, z = q[3] / qn;
    const double R[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                         2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                         2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
    double axes[3], rel[3], vs[3], ds[3];
    for (int j = 0; j < 3; ++j) {
        axes[j] = rp.sigma * exp(double(rp.log_scales[3 * size_t(g) + j]));
        rel[j] = c.tc2w[j] - double(rp.means[3 * size_t(g) + j]);
    }
    if (fmin(axes[0], fmin(axes[1], axes[2])) < kDegenerateScale) return false;
    for (int j = 0; j < 3; ++j) {
        double tv = R[0 * 3 + j] * rel[0];
        tv += R[1 * 3 + j] * rel[1];
        tv += R[2 * 3 + j] * rel[2];
        double td = R[0 * 3 + j] * d[0];
        td += R[1 * 3 + j] * d[1];
        td += R[2 * 3 + j] * d[2];
        vs[j] = tv / axes[j];
        ds[j] = td / axes[j];
    }
    double a = ds[0] * ds[0];
    a += ds[1] * ds[1];
    a += ds[2] * ds[2];
    double bb = vs[0] * ds[0];
    bb += vs[1] * ds[1];
    bb += vs[2] * ds[2];
    const double b = 2.0 * bb;
    double cc = vs[0] * vs[0];
    cc += vs[1] * vs[1];
    cc += vs[2] * vs[2];
    cc = cc - 1.0;
    const double disc = b * b - 4.0 * a * cc;
    if (disc < 0 || a <= 0) return false;
    const double t = -b / (2.0 * a);
    if (t <= 0) return false;
    *t_out = t;
    *a_out = a;
    *b_out = b;
    for (int j = 0; j < 3; ++j) ds_out[j] = ds[j];
    double p0 = c.tc2w[0] + t * d[0], p1 = c.tc2w[1] + t * d[1], p2 = c.tc2w[2] + t * d[2];
    double dz = c.Rw2c[6] * p0;
    dz += c.Rw2c[7] * p1;
    dz += c.Rw2c[8] * p2;
    *depth_out = dz + c.tw2c[2];
    return true;
}

template <typename Real>
__device__ __noinline__ bool intersect_fp64(const Cam& c, const RawParams<Real>& rp, uint32_t g, Real px,
                                            Real py, double* t_out, double* a_out, double* b_out,
                                            double* ds_out, double* depth_out) {
    return intersect_fp64_impl<Real>(c, rp, g, px, py, t_out, a_out, b_out, ds_out, depth_out);
}

// How the FP32 intersect re-decides a near-boundary pair in FP64.
enum : int {
    kFp64Undecided = 0,  // not at all: hit = false, depth_fp64 = -2 ("undecided"); the caller re-runs the pair
    kFp64Call = 1,       // a call to the out-of-line intersect_fp64
    kFp64Inline = 2,     // inlined (callers with many live registers: no call-site spills)
};

// intersect (core/src/geometry.cpp:37-64) with the per-view constant v_s and
// |v_s|^2 - 1 precomputed by K1.  In FP32, a discriminant or t_mid within a
// relative 1e-4 of zero is re-decided in FP64 (intersect_fp64), as kFp64
// selects.
template <typename Real, int kFp64 = kFp64Call>
__device__ __forceinline__ HitEval<Real> intersect(const BlendRec<Real>& g, const PixelRay<Real>& r,
                                                   const Cam& cam, const RawParams<Real>& rp, uint32_t gid) {
    HitEval<Real> h;
    h.hit = false;
    h.depth_fp64 = Real(-1);
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
    for (int i = 0; i < 3; ++i) h.dl[i] = dl[i];
    h.a = h.ds[0] * h.ds[0] + h.ds[1] * h.ds[1] + h.ds[2] * h.ds[2];
    if constexpr (sizeof(Real) == 8) {
        // The reference's own formulation (geometry.cpp:44-58).
        const Real vd = g.vs[0] * h.ds[0] + g.vs[1] * h.ds[1] + g.vs[2] * h.ds[2];
        h.b = Real(2) * vd;
        const Real disc = h.b * h.b - Real(4) * h.a * g.csq;
        if (disc < Real(0) || h.a <= Real(0)) return h;
        h.t_mid = -h.b / (Real(2) * h.a);
    } else {
        // disc/4 = (v_s.d_s)^2 - |d_s|^2 (|v_s|^2 - 1) = |d_s|^2 - |v_s x d_s|^2 (Lagrange
        // identity).  For flat splats |v_s| ~ 1e3, so b^2 and 4ac agree to ~1e-7
        // and the textbook form has no correct FP32 digit; the cross product is
        // taken in unscaled local space (v_l x d_l) where it is well conditioned:
        //   (v_s x d_s)_i = (v_l x d_l)_i / (axes_j axes_k).
        const Real* ia = g.inv_axes;
        const Real w0 = g.vl[1] * dl[2] - g.vl[2] * dl[1];
        const Real w1 = g.vl[2] * dl[0] - g.vl[0] * dl[2];
        const Real w2 = g.vl[0] * dl[1] - g.vl[1] * dl[0];
        const Real c0 = w0 * ia[1] * ia[2], c1 = w1 * ia[0] * ia[2], c2 = w2 * ia[0] * ia[1];
        const Real disc4 = h.a - (c0 * c0 + c1 * c1 + c2 * c2);
        const Real vd = g.vl[0] * dl[0] * ia[0] * ia[0] + g.vl[1] * dl[1] * ia[1] * ia[1] +
                        g.vl[2] * dl[2] * ia[2] * ia[2];
        // Decisions within FP32 noise of the boundary are re-taken in FP64 exactly
        // as the reference computes them (rare: grazing rays / camera on the shell).
        if (fabsf(disc4) <= Real(1e-4) * h.a || fabsf(vd) <= Real(1e-4) * sqrtf(h.a * (g.csq + Real(1)))) {
            if constexpr (kFp64 == kFp64Undecided) {
                h.depth_fp64 = Real(-2);
                return h;
            }
            double t, a, b, ds[3], dep;
            bool ok;
            if constexpr (kFp64 == kFp64Inline)
                ok = intersect_fp64_impl<Real>(cam, rp, gid, r.px, r.py, &t, &a, &b, ds, &dep);
            else
                ok = intersect_fp64<Real>(cam, rp, gid, r.px, r.py, &t, &a, &b, ds, &dep);
            if (!ok) return h;
            h.hit = true;
            h.t_mid = Real(t);
            h.a = Real(a);
            h.b = Real(b);
            for (int i = 0; i < 3; ++i) h.ds[i] = Real(ds[i]);
            h.depth_fp64 = Real(dep);
            return h;
        }
        h.b = Real(2) * vd;
        if (disc4 < Real(0) || h.a <= Real(0)) return h;
        h.t_mid = -vd / h.a;
    }
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

// quat_rotation_backward (core/src/geometry.cpp:17-29): dL/dR -> dL/d(unit q),
// before the tangent projection of chain_activations.
template <typename Real>
__device__ __forceinline__ void quat_rotation_backward(const Real* q, const Real* G, Real* dq) {
    const Real w = q[0], x = q[1], y = q[2], z = q[3];
#define g(i, j) G[(i)*3 + (j)]
    dq[0] = Real(2) * (g(0, 1) * (-z) + g(0, 2) * y + g(1, 0) * z + g(1, 2) * (-x) + g(2, 0) * (-y) +
                       g(2, 1) * x);
    dq[1] = Real(2) * (g(0, 1) * y + g(0, 2) * z + g(1, 0) * y + g(1, 1) * (-2 * x) + g(1, 2) * (-w) +
                       g(2, 0) * z + g(2, 1) * w + g(2, 2) * (-2 * x));
    dq[2] = Real(2) * (g(0, 0) * (-2 * y) + g(0, 1) * x + g(0, 2) * w + g(1, 0) * x + g(1, 2) * z +
                       g(2, 0) * (-w) + g(2, 1) * z + g(2, 2) * (-2 * y));
    dq[3] = Real(2) * (g(0, 0) * (-2 * z) + g(0, 1) * (-w) + g(0, 2) * x + g(1, 0) * w +
                       g(1, 1) * (-2 * z) + g(1, 2) * y + g(2, 0) * x + g(2, 1) * y);
#undef g
}

// Tile-local pixel coordinates: warps cover 8x4 pixel blocks, 2 across x 4 down.
// Asynchronous staging of F_j = [rgb, k, sem] (the per-Gaussian row the
// backward reads every event) into a shared row with cp.async: issued one event
// ahead into the other half of a double buffer, it costs no registers and the
// L2 latency overlaps the current event.  Channels >= C + 4 of the row are
// never written (callers zero them once).
template <typename Real>
__device__ __forceinline__ void stage_F_async(Real* row, const BlendRec<Real>* brec, const Real* semantics, int C,
                                              uint32_t g, int lane) {
    const int S = C + 4;
    for (int ch = lane; ch < S; ch += 32) {
        const Real* src = ch < 3 ? &brec[g].rgb[ch] : (ch == 3 ? &brec[g].k : semantics + size_t(g) * C + (ch - 4));
        const unsigned dst = unsigned(__cvta_generic_to_shared(row + ch));
        if constexpr (sizeof(Real) == 4)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
        else
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void stage_F_commit_empty() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// Waits until at most the lookahead row is in flight, then makes the completed
// rows warp-visible.
__device__ __forceinline__ void stage_F_wait_prev() {
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncwarp();
}

// ---- warp-level tensor-core helpers (mma.sync m16n8k8 TF32, FP32 accumulate)
// with a hi/lo operand split: a.b ~ a_hi b_hi + a_hi b_lo + a_lo b_hi, i.e.
// FP32-level accuracy for the blend contractions.
// hi = x truncated to TF32 (one AND), lo = x - hi exactly (<= 13 significant
// bits, which the tensor core truncates to TF32): |a b - (a_hi b_hi + a_hi b_lo
// + a_lo b_hi)| <= ~2^-20 |a b|.  (cvt.rna.tf32 lowers to a compare, an add
// and a mask; this split is two instructions.)
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
    hi = __float_as_uint(x) & 0xffffe000u;
    lo = __float_as_uint(x - __uint_as_float(hi));
}

__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// d += A B with the 3-term split (A: 4 fp32 fragment values, B: 2).
__device__ __forceinline__ void mma_3xtf32(float (&d)[4], const float (&a)[4], const float (&b)[2]) {
    uint32_t ah[4], al[4], bh[2], bl[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) split_tf32(a[i], ah[i], al[i]);
#pragma unroll
    for (int i = 0; i < 2; ++i) split_tf32(b[i], bh[i], bl[i]);
    mma_tf32(d, al, bh);
    mma_tf32(d, ah, bl);
    mma_tf32(d, ah, bh);
}

__device__ __forceinline__ int tile_pixel_x(int warp, int lane) { return (warp & 1) * 8 + (lane & 7); }
__device__ __forceinline__ int tile_pixel_y(int warp, int lane) { return (warp >> 1) * 4 + (lane >> 3); }
__device__ __forceinline__ int tile_pixel_index(int warp, int lane) {
    return tile_pixel_y(warp, lane) * kTile + tile_pixel_x(warp, lane);
}

}  // namespace msplat_cuda
