// K1: per-Gaussian preprocess (one thread per Gaussian).
//
// Replaces prepare_view (core/src/rasterizer.cpp:55-74): activate
// (core/src/scene.cpp:42-60), project_gaussian (core/src/geometry.cpp:107-136),
// eval_sh_color (core/src/sh.cpp:75-84), the pixel-rect/tile-range rule of
// bin_and_sort (core/src/rasterizer.cpp:32-39) and the per-view constant part
// of intersect (core/src/geometry.cpp:39-52).
//
// Everything that decides integer binning output (centre, covariance,
// determinant, radius, depth key, tile rect) is computed in FP64 with the
// reference's evaluation order and WITHOUT FMA contraction: this translation
// unit is compiled with --fmad=false, so every a*b+c below rounds twice like
// the reference's -ffp-contract=off double arithmetic.  That is what makes the
// tile lists, their order and the per-tile ranges bit-exact.  Blend records are
// then rounded to the kernel precision (float or double).
#include "common.cuh"
#include "kernels.h"

#include <type_traits>

namespace msplat_cuda {

constexpr int kPreThreads = 256;

namespace {

__device__ __forceinline__ double dot3(const double* a, const double* b) {
    double s = a[0] * b[0];
    s += a[1] * b[1];
    s += a[2] * b[2];
    return s;
}
__device__ __forceinline__ void cross3(const double* a, const double* b, double* o) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}

// x86 cvttsd2si semantics of the reference's int(std::floor(v)): NaN and
// out-of-range values become INT_MIN (rasterizer.cpp:32-35 on this platform).
__device__ __forceinline__ int floor_to_int(double v) {
    const double f = floor(v);
    if (!(f >= -2147483648.0 && f < 2147483648.0)) return int(0x80000000u);
    return int(f);
}

__device__ __forceinline__ void quat_to_rotation(const double* q, double* R) {
    double n2 = q[0] * q[0];
    n2 += q[1] * q[1];
    n2 += q[2] * q[2];
    n2 += q[3] * q[3];
    const double n = sqrt(n2);
    const double w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
    R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z); R[2] = 2 * (x * z + w * y);
    R[3] = 2 * (x * y + w * z); R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
    R[6] = 2 * (x * z - w * y); R[7] = 2 * (y * z + w * x); R[8] = 1 - 2 * (x * x + y * y);
}

template <typename T>
__device__ __forceinline__ void sh_basis(int deg, T x, T y, T z, T* b) {
    const T C0 = T(0.28209479177387814), C1 = T(0.4886025119029199);
    b[0] = C0;
    if (deg >= 1) { b[1] = -C1 * y; b[2] = C1 * z; b[3] = -C1 * x; }
    if (deg >= 2) {
        const T xx = x * x, yy = y * y, zz = z * z;
        b[4] = T(1.0925484305920792) * x * y;
        b[5] = -T(1.0925484305920792) * y * z;
        b[6] = T(0.31539156525252005) * (T(2) * zz - xx - yy);
        b[7] = -T(1.0925484305920792) * x * z;
        b[8] = T(0.5462742152960396) * (xx - yy);
    }
    if (deg >= 3) {
        const T xx = x * x, yy = y * y, zz = z * z;
        b[9] = -T(0.5900435899266435) * y * (T(3) * xx - yy);
        b[10] = T(2.890611442640554) * x * y * z;
        b[11] = -T(0.4570457994644658) * y * (T(4) * zz - xx - yy);
        b[12] = T(0.3731763325901154) * z * (T(2) * zz - 3 * xx - T(3) * yy);
        b[13] = -T(0.4570457994644658) * x * (T(4) * zz - xx - yy);
        b[14] = T(1.445305721320277) * z * (xx - yy);
        b[15] = -T(0.5900435899266435) * x * (xx - T(3) * yy);
    }
}

// Copies count contiguous values to dst (when given) and reports whether any
// of those this thread touched is non-finite: 16-byte vectors, four in flight
// per thread, when src is 16-byte aligned (block offsets are; the tensor base
// normally is), scalars otherwise and for the tail.
template <typename Real>
__device__ __forceinline__ bool stage_and_scan(const Real* __restrict__ src, Real* dst, int count) {
    constexpr int W = 16 / int(sizeof(Real));
    constexpr uint64_t kExp = sizeof(Real) == 4 ? 0x7f800000ull : 0x7ff0000000000000ull;
    using Bits = std::conditional_t<sizeof(Real) == 4, uint32_t, uint64_t>;
    bool bad = false;
    int done = 0;
    if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
        const int nv = count / W;
        const uint4* s = reinterpret_cast<const uint4*>(src);
        uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll 4
        for (int v = threadIdx.x; v < nv; v += kPreThreads) {
            const uint4 x = __ldg(s + v);
            if (dst) d[v] = x;
            if constexpr (sizeof(Real) == 4) {
                bad |= (x.x & 0x7f800000u) == 0x7f800000u || (x.y & 0x7f800000u) == 0x7f800000u ||
                       (x.z & 0x7f800000u) == 0x7f800000u || (x.w & 0x7f800000u) == 0x7f800000u;
            } else {
                bad |= (x.y & 0x7ff00000u) == 0x7ff00000u || (x.w & 0x7ff00000u) == 0x7ff00000u;
            }
        }
        done = nv * W;
    }
    for (int e = done + int(threadIdx.x); e < count; e += kPreThreads) {
        const Real v = src[e];
        if (dst) dst[e] = v;
        Bits b;
        memcpy(&b, &v, sizeof(b));
        bad |= (uint64_t(b) & kExp) == kExp;
    }
    return bad;
}

template <typename Real>
__device__ __forceinline__ bool finite_params(const PreprocessArgs<Real>& a, int64_t i) {
    bool ok = true;
    for (int j = 0; j < 3; ++j)
        ok &= isfinite(a.means[3 * i + j]) && isfinite(a.log_scales[3 * i + j]);
    for (int j = 0; j < 4; ++j) ok &= isfinite(a.quats[4 * i + j]);
    ok &= isfinite(a.opacity_logits[i]) && isfinite(a.k[i]);
    return ok;
}

}  // namespace

template <typename Real>
#ifndef K1_MINB
#define K1_MINB 3  // 3 CTAs per SM (85 registers): measured 0.18 ms vs 0.22 at 2
#endif
__global__ void __launch_bounds__(kPreThreads, K1_MINB) preprocess_kernel(const __grid_constant__ PreprocessArgs<Real> a) {
    // The block's SH rows (3K values per Gaussian, contiguous) are staged in
    // shared memory by one coalesced copy, and the semantic rows are scanned for
    // non-finite values the same way; per-thread strided row reads would thrash
    // L1.  Row pitch 3K is odd for K = 1, 9: conflict-free FP32 row reads.
    extern __shared__ __align__(16) unsigned char pre_smem[];
    Real* const sh_s = reinterpret_cast<Real*>(pre_smem);
    uint8_t* const bad_s = reinterpret_cast<uint8_t*>(sh_s + size_t(kPreThreads) * 3 * a.K);
    const int64_t base = int64_t(blockIdx.x) * kPreThreads;
    const int cnt = int(a.n - base < kPreThreads ? a.n - base : kPreThreads);
    {
        const int rs = 3 * a.K;
        bad_s[threadIdx.x] = 0;
        // Fast path: 16-byte vector copies / scans with a block-wide "any
        // non-finite" vote; the rows are only identified when the vote fires.
        bool bad = stage_and_scan<Real>(a.sh + base * rs, sh_s, cnt * rs);
        if (a.C > 0) bad |= stage_and_scan<Real>(a.semantics + base * a.C, nullptr, cnt * a.C);
        if (__syncthreads_or(bad)) {
            // (element -> row index by a running quotient: no integer division per element)
            const Real* src = a.sh + base * rs;
            for (int e = threadIdx.x, row = threadIdx.x / rs, rem = threadIdx.x % rs; e < cnt * rs;
                 e += kPreThreads, rem += kPreThreads % rs, row += kPreThreads / rs) {
                if (rem >= rs) { rem -= rs; ++row; }
                if (!isfinite(src[e])) bad_s[row] = 1;
            }
            if (a.C > 0) {
                const Real* sem = a.semantics + base * a.C;
                for (int e = threadIdx.x, row = threadIdx.x / a.C, rem = threadIdx.x % a.C; e < cnt * a.C;
                     e += kPreThreads, rem += kPreThreads % a.C, row += kPreThreads / a.C) {
                    if (rem >= a.C) { rem -= a.C; ++row; }
                    if (!isfinite(sem[e])) bad_s[row] = 1;
                }
            }
            __syncthreads();
        }
    }
    const int64_t i = base + threadIdx.x;
    if (i >= a.n) return;
    const Cam& c = a.cam;

    a.depth_key[i] = ~0ull;  // not binned unless proven otherwise
    a.order[i] = uint32_t(i);
    a.tile_count[i] = 0;
    a.visible[i] = 0;

    if (bad_s[threadIdx.x] || !finite_params(a, i)) {  // Scene::validate / activate (scene.cpp:36-38, 43-45)
        raise_error_ordered(a.err, kErrNonFiniteParam, i);
        return;
    }
    // ---- activate (scene.cpp:42-60)
    double q[4] = {double(a.quats[4 * i]), double(a.quats[4 * i + 1]), double(a.quats[4 * i + 2]),
                   double(a.quats[4 * i + 3])};
    double n2 = q[0] * q[0];
    n2 += q[1] * q[1];
    n2 += q[2] * q[2];
    n2 += q[3] * q[3];
    const double qn = sqrt(n2);
    if (qn < 1e-12) {
        raise_error_ordered(a.err, kErrZeroQuat, i);
        return;
    }
    for (int j = 0; j < 4; ++j) q[j] = q[j] / qn;
    double R[9];
    quat_to_rotation(q, R);
    const double mu[3] = {double(a.means[3 * i]), double(a.means[3 * i + 1]), double(a.means[3 * i + 2])};
    const double s[3] = {exp(double(a.log_scales[3 * i])), exp(double(a.log_scales[3 * i + 1])),
                         exp(double(a.log_scales[3 * i + 2]))};
    // opacity / log threshold only feed Real-precision records
    const Real opacity = Real(1) / (Real(1) + exp(-a.opacity_logits[i]));

    // ---- project_gaussian (geometry.cpp:107-136)
    double pc[3];
    for (int r = 0; r < 3; ++r) {
        double t = c.Rw2c[r * 3 + 0] * mu[0];
        t += c.Rw2c[r * 3 + 1] * mu[1];
        t += c.Rw2c[r * 3 + 2] * mu[2];
        pc[r] = t + c.tw2c[r];
    }
    if (pc[2] <= kNearPlane) return;
    const double x = pc[0], y = pc[1], z = pc[2];
    const double cxp = c.fx * x / z + c.cx;
    const double cyp = c.fy * y / z + c.cy;
    const double J[6] = {c.fx / z, 0, -c.fx * x / (z * z), 0, c.fy / z, -c.fy * y / (z * z)};
    double V[9];
    {
        double RD[9];
        for (int r = 0; r < 3; ++r)
            for (int q2 = 0; q2 < 3; ++q2) RD[r * 3 + q2] = R[r * 3 + q2] * (s[q2] * s[q2]);
        for (int r = 0; r < 3; ++r)
            for (int q2 = 0; q2 < 3; ++q2) {
                double t = RD[r * 3 + 0] * R[q2 * 3 + 0];
                t += RD[r * 3 + 1] * R[q2 * 3 + 1];
                t += RD[r * 3 + 2] * R[q2 * 3 + 2];
                V[r * 3 + q2] = t;
            }
    }
    double T[6], TV[6], cov[4];
    for (int r = 0; r < 2; ++r)
        for (int q2 = 0; q2 < 3; ++q2) {
            double t = J[r * 3 + 0] * c.Rw2c[0 * 3 + q2];
            t += J[r * 3 + 1] * c.Rw2c[1 * 3 + q2];
            t += J[r * 3 + 2] * c.Rw2c[2 * 3 + q2];
            T[r * 3 + q2] = t;
        }
    for (int r = 0; r < 2; ++r)
        for (int q2 = 0; q2 < 3; ++q2) {
            double t = T[r * 3 + 0] * V[0 * 3 + q2];
            t += T[r * 3 + 1] * V[1 * 3 + q2];
            t += T[r * 3 + 2] * V[2 * 3 + q2];
            TV[r * 3 + q2] = t;
        }
    for (int r = 0; r < 2; ++r)
        for (int q2 = 0; q2 < 2; ++q2) {
            double t = TV[r * 3 + 0] * T[q2 * 3 + 0];
            t += TV[r * 3 + 1] * T[q2 * 3 + 1];
            t += TV[r * 3 + 2] * T[q2 * 3 + 2];
            cov[r * 2 + q2] = t;
        }
    cov[0] += kCovFloor;
    cov[3] += kCovFloor;
    const double det = cov[0] * cov[3] - cov[2] * cov[1];
    const bool proj_ok = det > 0;
    {  // one atomic per warp for the visible count (a same-address atomic per
       // Gaussian serialises in L2)
        const unsigned act = __activemask();
        const unsigned vis = __ballot_sync(act, proj_ok);
        if (proj_ok && (threadIdx.x & 31) == __ffs(vis) - 1) atomicAdd(a.visible_count, (unsigned long long)__popc(vis));
    }
    if (!proj_ok) return;
    const double ca = cov[3] / det, cb = -cov[1] / det, cc = cov[0] / det;
    const double mid = 0.5 * (cov[0] + cov[3]);
    const double m2 = mid * mid - det;
    const double lambda_max = mid + sqrt(0.1 < m2 ? m2 : 0.1);
    const double radius = 3.0 * sqrt(lambda_max);
    a.visible[i] = 1;

    // ---- pixel rect -> tile rect (rasterizer.cpp:32-39)
    int x0 = floor_to_int(cxp - radius), x1 = floor_to_int(cxp + radius);
    int y0 = floor_to_int(cyp - radius), y1 = floor_to_int(cyp + radius);
    x0 = x0 > 0 ? x0 : 0;
    x1 = x1 < a.W - 1 ? x1 : a.W - 1;
    y0 = y0 > 0 ? y0 : 0;
    y1 = y1 < a.H - 1 ? y1 : a.H - 1;
    if (!(x1 < x0 || y1 < y0)) {
        const int tx0 = x0 / kTile, tx1 = x1 / kTile, ty0 = y0 / kTile, ty1 = y1 / kTile;
        a.tile_rect[i] = make_uint2(uint32_t(tx0) | (uint32_t(tx1) << 16),
                                    uint32_t(ty0) | (uint32_t(ty1) << 16));
        a.tile_count[i] = uint32_t((tx1 - tx0 + 1) * (ty1 - ty0 + 1));
        // Positive doubles order like their IEEE bit patterns (z > 0.01 here).
        a.depth_key[i] = uint64_t(__double_as_longlong(z));
    }

    // ---- view-dependent colour (rasterizer.cpp:66-71, sh.cpp:75-84)
    // In the kernel precision: the colour only feeds Real records (FP64 keeps
    // the reference's double evaluation).
    Real rgb[3];
    uint8_t clamped[3];
    {
        const double tg[3] = {mu[0] - c.tc2w[0], mu[1] - c.tc2w[1], mu[2] - c.tc2w[2]};
        const double nrm = sqrt(dot3(tg, tg));
        double dx = 0, dy = 0, dz = 1;
        if (nrm > 1e-12) { dx = tg[0] / nrm; dy = tg[1] / nrm; dz = tg[2] / nrm; }
        Real b[16];
        sh_basis<Real>(a.deg, Real(dx), Real(dy), Real(dz), b);
        for (int ch = 0; ch < 3; ++ch) {
            const Real* shc = sh_s + (size_t(threadIdx.x) * 3 + ch) * a.K;
            Real t = shc[0] * b[0];
            for (int j = 1; j < a.K; ++j) t += shc[j] * b[j];
            const Real raw = t + Real(0.5);
            clamped[ch] = raw < Real(0);
            rgb[ch] = clamped[ch] ? Real(0) : raw;
        }
    }

    // ---- per-view constant part of intersect (geometry.cpp:39-52)
    const double axes[3] = {a.sigma * s[0], a.sigma * s[1], a.sigma * s[2]};
    double amin = axes[0];
    if (axes[1] < amin) amin = axes[1];
    if (axes[2] < amin) amin = axes[2];
    const double rel[3] = {c.tc2w[0] - mu[0], c.tc2w[1] - mu[1], c.tc2w[2] - mu[2]};
    double vs[3], vl[3];
    for (int j = 0; j < 3; ++j) {
        double t = R[0 * 3 + j] * rel[0];
        t += R[1 * 3 + j] * rel[1];
        t += R[2 * 3 + j] * rel[2];
        vl[j] = t;
        vs[j] = t / axes[j];
    }
    const double csq = dot3(vs, vs) - 1.0;

    AlphaRec<Real> ar;
    ar.cx = Real(cxp);
    ar.cy = Real(cyp);
    ar.ca = Real(ca);
    ar.cb = Real(cb);
    ar.cc = Real(cc);
    ar.opacity = Real(opacity);
    const Real log_thr = log(Real(1) / (Real(255) * opacity));
    ar.log_thr = log_thr;
    ar.pad = Real(1) / opacity;  // phase B's dopacity = dpower / opacity
    {
        // d^T conic d <= r2 with r2 = -2 (log_thr - 1e-3); the tight box of that
        // ellipse has half-widths sqrt(r2 cov_xx), sqrt(r2 cov_yy) (cov = conic^-1).
        const double r2 = -2.0 * (double(log_thr) - 1e-3);
        if (r2 > 0) {
            const double hx = sqrt(r2 * cov[0]) * 1.001 + 1e-3, hy = sqrt(r2 * cov[3]) * 1.001 + 1e-3;
            ar.bx0 = Real(cxp - hx);
            ar.bx1 = Real(cxp + hx);
            ar.by0 = Real(cyp - hy);
            ar.by1 = Real(cyp + hy);
        } else {  // opacity < 1/255: no pixel can pass
            ar.bx0 = ar.by0 = Real(1e30);
            ar.bx1 = ar.by1 = Real(-1e30);
        }
    }
    for (int j = 0; j < 3; ++j) ar.rgb[j] = Real(rgb[j]);
    ar.k = a.k[i];
    a.arec[i] = ar;

    BlendRec<Real> br;
    for (int r = 0; r < 3; ++r)
        for (int q2 = 0; q2 < 3; ++q2) br.Rt[r * 3 + q2] = Real(R[q2 * 3 + r]);
    for (int j = 0; j < 3; ++j) {
        br.axes[j] = Real(axes[j]);
        br.inv_axes[j] = Real(1.0 / axes[j]);
        br.vs[j] = Real(vs[j]);
        br.rgb[j] = Real(rgb[j]);
        br.vl[j] = Real(vl[j]);
    }
    br.csq = Real(csq);
    br.zc = Real(z);
    br.k = a.k[i];
    br.hit_ok = Real(amin < kDegenerateScale ? 0 : 1);
    for (int j = 0; j < 4; ++j) br.q[j] = Real(q[j]);
    if (a.brec) a.brec[i] = br;

    if constexpr (sizeof(Real) == 4) {
        if (a.drec) {  // DepthRec (common.cuh): the forward depth as quadratic forms about the centre
            DepthRec dr;
            dr.zc = float(z);
            if (amin < kDegenerateScale) {
                for (int j = 0; j < 6; ++j) dr.E[j] = dr.A[j] = dr.K[j] = 0.f;
                for (int j = 0; j < 3; ++j) dr.H[j] = 0.f;
                dr.E[0] = -1.f;
                dr.A[0] = 1.f;
                dr.ex = dr.ey = 0.f;
            } else {
                const double u0 = double(float(cxp)), v0 = double(float(cyp));  // the AlphaRec centre
                const double ifx = 1.0 / c.fx, ify = 1.0 / c.fy;
                const double p0[2] = {(u0 - c.cx) * ifx, (v0 - c.cy) * ify};
                double m0[3], mx[3], my[3];
#pragma unroll 1
                for (int j = 0; j < 3; ++j) {
                    double mc[3];  // row j of M R_c2w
                    const double ia = 1.0 / axes[j];
                    for (int k2 = 0; k2 < 3; ++k2) {
                        double t = R[0 * 3 + j] * c.Rc2w[0 * 3 + k2];
                        t += R[1 * 3 + j] * c.Rc2w[1 * 3 + k2];
                        t += R[2 * 3 + j] * c.Rc2w[2 * 3 + k2];
                        mc[k2] = t * ia;
                    }
                    m0[j] = mc[0] * p0[0] + mc[1] * p0[1] + mc[2];
                    mx[j] = mc[0] * ifx;
                    my[j] = mc[1] * ify;
                }
                double w0[3], wx[3], wy[3];
                cross3(vs, m0, w0);
                cross3(vs, mx, wx);
                cross3(vs, my, wy);
                const double A[6] = {dot3(m0, m0), 2.0 * dot3(m0, mx), 2.0 * dot3(m0, my),
                                     dot3(mx, mx), 2.0 * dot3(mx, my), dot3(my, my)};
                const double W2[6] = {dot3(w0, w0), 2.0 * dot3(w0, wx), 2.0 * dot3(w0, wy),
                                      dot3(wx, wx), 2.0 * dot3(wx, wy), dot3(wy, wy)};
                for (int j = 0; j < 6; ++j) {
                    dr.A[j] = float(A[j]);
                    dr.E[j] = float(A[j] - W2[j]);
                }
                const double H[3] = {dot3(vs, m0), dot3(vs, mx), dot3(vs, my)};
                for (int j = 0; j < 3; ++j) dr.H[j] = float(H[j]);
                for (int j = 0; j < 6; ++j) dr.K[j] = float((j < 3 ? H[j] : 0.0) + z * A[j]);
                dr.ex = float(x - z * p0[0]);
                dr.ey = float(y - z * p0[1]);
            }
            a.drec[i] = dr;
        }
    }

    a.clamped_bits[i] = uint8_t(clamped[0] | (clamped[1] << 1) | (clamped[2] << 2));
    if (a.cap_center) {  // replay capture for parity checks (msplat_replay_splats)
        a.cap_center[2 * i] = cxp;
        a.cap_center[2 * i + 1] = cyp;
        a.cap_conic[3 * i] = ca;
        a.cap_conic[3 * i + 1] = cb;
        a.cap_conic[3 * i + 2] = cc;
        a.cap_depth[i] = z;
        a.cap_radius[i] = radius;
        for (int j = 0; j < 3; ++j) a.cap_rgb[3 * i + j] = rgb[j];
    }
}

template <typename Real>
void launch_preprocess(const PreprocessArgs<Real>& a, cudaStream_t s) {
    if (a.n == 0) return;
    const int64_t blocks = (a.n + kPreThreads - 1) / kPreThreads;
    const size_t smem = sizeof(Real) * size_t(kPreThreads) * 3 * a.K + kPreThreads;
    static std::atomic<unsigned long long> attr{0};  // per instantiation, per device
    opt_in_smem(reinterpret_cast<const void*>(preprocess_kernel<Real>), attr, 200 * 1024);
    preprocess_kernel<Real><<<unsigned(blocks), kPreThreads, smem, s>>>(a);
    count_launches(1);
}

__global__ void rects_from_splats_kernel(int64_t n, const uint8_t* __restrict__ visible,
                                         const double* __restrict__ center,
                                         const double* __restrict__ radius,
                                         const double* __restrict__ depth, int W, int H,
                                         uint64_t* depth_key, uint32_t* order, uint32_t* tile_count,
                                         uint2* tile_rect) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    order[i] = uint32_t(i);
    depth_key[i] = ~0ull;
    tile_count[i] = 0;
    if (!visible[i]) return;
    const double cx = center[2 * i], cy = center[2 * i + 1], r = radius[i];
    int x0 = floor_to_int(cx - r), x1 = floor_to_int(cx + r);
    int y0 = floor_to_int(cy - r), y1 = floor_to_int(cy + r);
    x0 = x0 > 0 ? x0 : 0;
    x1 = x1 < W - 1 ? x1 : W - 1;
    y0 = y0 > 0 ? y0 : 0;
    y1 = y1 < H - 1 ? y1 : H - 1;
    if (x1 < x0 || y1 < y0) return;
    const int tx0 = x0 / kTile, tx1 = x1 / kTile, ty0 = y0 / kTile, ty1 = y1 / kTile;
    tile_rect[i] = make_uint2(uint32_t(tx0) | (uint32_t(tx1) << 16), uint32_t(ty0) | (uint32_t(ty1) << 16));
    tile_count[i] = uint32_t((tx1 - tx0 + 1) * (ty1 - ty0 + 1));
    // Arbitrary doubles: map to an order-preserving unsigned key (negative
    // values flip all bits, positive set the sign bit) -- the explicit-splat
    // entry point is not restricted to z > 0.  -0.0 + 0.0 = +0.0: the two
    // zeros compare equal in the reference's comparator (index tie-break).
    const uint64_t b = uint64_t(__double_as_longlong(depth[i] + 0.0));
    depth_key[i] = (b >> 63) ? ~b : (b | (1ull << 63));
}

void launch_rects_from_splats(int64_t n, const uint8_t* visible, const double* center,
                              const double* radius, const double* depth, int W, int H,
                              uint64_t* depth_key, uint32_t* order, uint32_t* tile_count,
                              uint2* tile_rect, cudaStream_t s) {
    if (n == 0) return;
    rects_from_splats_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(
        n, visible, center, radius, depth, W, H, depth_key, order, tile_count, tile_rect);
    count_launches(1);
}

template void launch_preprocess<float>(const PreprocessArgs<float>&, cudaStream_t);
template void launch_preprocess<double>(const PreprocessArgs<double>&, cudaStream_t);

}  // namespace msplat_cuda
