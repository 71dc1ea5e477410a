// K10: per-Gaussian projection / SH adjoint (projection_backward,
// core/src/rasterizer_backward.cpp:57-123; eval_sh_color_backward, sh.cpp:86-99)
// with chain_activations (scene.cpp:108-129) and check_finite
// (scene.cpp:97-106) fused; the standalone chain kernel; check_replay's scene
// comparison (rasterizer_backward.cpp:40-44).  K9 lives in backward_blend.cu.
#include "blend_common.cuh"
#include "kernels.h"

namespace msplat_cuda {

// ------------------------------------------------------------------ K10
// SH colour adjoint (sh.cpp:45-73, 86-99) for a compile-time degree: dsh +=
// g (x) basis, and the view-direction gradient through the basis Jacobian.
template <typename Real, int DEG>
__device__ __forceinline__ void sh_adjoint(const Real* sh, Real* g_sh, Real dx, Real dy, Real dz, const Real* g3,
                                           Real* ddir) {
    constexpr int K = (DEG + 1) * (DEG + 1);
    Real b[K], Jb[K][3];
    const Real C0 = Real(0.28209479177387814), C1 = Real(0.4886025119029199);
    const Real k0 = Real(1.0925484305920792), k1 = Real(-1.0925484305920792), k2 = Real(0.31539156525252005),
               k3 = Real(-1.0925484305920792), k4 = Real(0.5462742152960396);
    const Real m0 = Real(-0.5900435899266435), m1 = Real(2.890611442640554), m2 = Real(-0.4570457994644658),
               m3 = Real(0.3731763325901154), m4 = Real(-0.4570457994644658), m5 = Real(1.445305721320277),
               m6 = Real(-0.5900435899266435);
#pragma unroll
    for (int j = 0; j < K; ++j) Jb[j][0] = Jb[j][1] = Jb[j][2] = Real(0);
    const Real xx = dx * dx, yy = dy * dy, zz = dz * dz;
    b[0] = C0;
    if constexpr (DEG >= 1) {
        b[1] = -C1 * dy; b[2] = C1 * dz; b[3] = -C1 * dx;
        Jb[1][1] = -C1; Jb[2][2] = C1; Jb[3][0] = -C1;
    }
    if constexpr (DEG >= 2) {
        b[4] = k0 * dx * dy; b[5] = k1 * dy * dz; b[6] = k2 * (2 * zz - xx - yy);
        b[7] = k3 * dx * dz; b[8] = k4 * (xx - yy);
        Jb[4][0] = k0 * dy; Jb[4][1] = k0 * dx;
        Jb[5][1] = k1 * dz; Jb[5][2] = k1 * dy;
        Jb[6][0] = -2 * k2 * dx; Jb[6][1] = -2 * k2 * dy; Jb[6][2] = 4 * k2 * dz;
        Jb[7][0] = k3 * dz; Jb[7][2] = k3 * dx;
        Jb[8][0] = 2 * k4 * dx; Jb[8][1] = -2 * k4 * dy;
    }
    if constexpr (DEG >= 3) {
        b[9] = m0 * dy * (3 * xx - yy); b[10] = m1 * dx * dy * dz; b[11] = m2 * dy * (4 * zz - xx - yy);
        b[12] = m3 * dz * (2 * zz - 3 * xx - 3 * yy); b[13] = m4 * dx * (4 * zz - xx - yy);
        b[14] = m5 * dz * (xx - yy); b[15] = m6 * dx * (xx - 3 * yy);
        Jb[9][0] = m0 * 6 * dx * dy; Jb[9][1] = m0 * (3 * xx - 3 * yy);
        Jb[10][0] = m1 * dy * dz; Jb[10][1] = m1 * dx * dz; Jb[10][2] = m1 * dx * dy;
        Jb[11][0] = -2 * m2 * dx * dy; Jb[11][1] = m2 * (4 * zz - xx - 3 * yy); Jb[11][2] = 8 * m2 * dy * dz;
        Jb[12][0] = -6 * m3 * dx * dz; Jb[12][1] = -6 * m3 * dy * dz; Jb[12][2] = m3 * (6 * zz - 3 * xx - 3 * yy);
        Jb[13][0] = m4 * (4 * zz - 3 * xx - yy); Jb[13][1] = -2 * m4 * dx * dy; Jb[13][2] = 8 * m4 * dx * dz;
        Jb[14][0] = 2 * m5 * dx * dz; Jb[14][1] = -2 * m5 * dy * dz; Jb[14][2] = m5 * (xx - yy);
        Jb[15][0] = m6 * (3 * xx - 3 * yy); Jb[15][1] = -6 * m6 * dx * dy;
    }
#pragma unroll
    for (int j = 0; j < K; ++j) {
        const Real shg = sh[0 * K + j] * g3[0] + sh[1 * K + j] * g3[1] + sh[2 * K + j] * g3[2];
        for (int k = 0; k < 3; ++k) ddir[k] += Jb[j][k] * shg;
        for (int ch = 0; ch < 3; ++ch) g_sh[ch * K + j] += g3[ch] * b[j];
    }
}

// Per-Gaussian part of K10; sh / g_sh point at the Gaussian's staged rows.
// Returns whether the Gaussian's small gradients (position, rotation, scale,
// opacity, k) are finite.
template <typename Real>
__device__ __forceinline__ bool projection_backward_one(const ProjBackwardArgs<Real>& a, int64_t i, const Real* sh,
                                                        Real* g_sh) {
    const Cam& c = a.cam;
    // Activation (scene.cpp:42-60) in the kernel precision.
    Real q[4];
    Real n2 = 0;
    for (int j = 0; j < 4; ++j) {
        q[j] = a.quats[4 * i + j];
        n2 += q[j] * q[j];
    }
    const Real qn = sqrt(n2);
    Real u[4];
    for (int j = 0; j < 4; ++j) u[j] = q[j] / qn;
    const Real s[3] = {exp(a.log_scales[3 * i]), exp(a.log_scales[3 * i + 1]), exp(a.log_scales[3 * i + 2])};
    Real gp[3] = {a.g_pos[3 * i], a.g_pos[3 * i + 1], a.g_pos[3 * i + 2]};
    Real gr[4] = {a.g_rot[4 * i], a.g_rot[4 * i + 1], a.g_rot[4 * i + 2], a.g_rot[4 * i + 3]};
    Real gs[3] = {a.g_scale[3 * i], a.g_scale[3 * i + 1], a.g_scale[3 * i + 2]};
    Real go = a.g_opac[i];
    // K9's per-pair sums (acc16 row): opacity, position, rotation, scale
    const Real* A16 = a.acc16 + size_t(i) * 16;
    // FP32 phase B (depth_moments): A16[0..2] are the moments sum dpower,
    // sum dpower dx, sum dpower dy; dopacity = [0] / opacity and dmean2d =
    // conic . ([1], [2]) below
    if (!a.depth_moments) go += A16[0];
    if (a.depth_moments) {
        // The FP32 phase B's depth moments (backward_blend.cu depth_moments):
        // dposition = Sigma^-1 R_c2w u + miss * z_cam, dL/dR = S R D,
        // dscale_k = -sigma (R^T S R)_kk / a_k^3 with S = R_c2w S_c R_c2w^T
        // (rotations and diagonal scalings only: well conditioned in FP32).
        float R[9], ia2[3], dR[9];
        {
            const float w = float(u[0]), x = float(u[1]), y = float(u[2]), z = float(u[3]);
            R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z); R[2] = 2 * (x * z + w * y);
            R[3] = 2 * (x * y + w * z); R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
            R[6] = 2 * (x * z - w * y); R[7] = 2 * (y * z + w * x); R[8] = 1 - 2 * (x * x + y * y);
        }
        float sig_a3[3];
        for (int k = 0; k < 3; ++k) {
            const float ak = float(a.sigma) * float(s[k]);
            ia2[k] = 1.f / (ak * ak);
            sig_a3[k] = float(a.sigma) * ia2[k] / ak;
        }
        const float Sc[9] = {float(A16[9]), float(A16[12]), float(A16[13]), float(A16[12]), float(A16[10]),
                             float(A16[14]), float(A16[13]), float(A16[14]), float(A16[11])};
        float Mc[9];  // camera -> world
        for (int k = 0; k < 9; ++k) Mc[k] = float(c.Rc2w[k]);
        float uw[3], RtM[9], B[9];
        for (int r = 0; r < 3; ++r)
            uw[r] = Mc[r * 3] * float(A16[6]) + Mc[r * 3 + 1] * float(A16[7]) + Mc[r * 3 + 2] * float(A16[8]);
        // R^T S R = (R^T Mc) S_c (R^T Mc)^T; S R = Mc S_c (R^T Mc)^T
        for (int r = 0; r < 3; ++r)
            for (int k = 0; k < 3; ++k) RtM[r * 3 + k] = R[r] * Mc[k] + R[3 + r] * Mc[3 + k] + R[6 + r] * Mc[6 + k];
        for (int r = 0; r < 3; ++r)  // B = S_c (R^T Mc)^T
            for (int k = 0; k < 3; ++k)
                B[r * 3 + k] = Sc[r * 3] * RtM[k * 3] + Sc[r * 3 + 1] * RtM[k * 3 + 1] + Sc[r * 3 + 2] * RtM[k * 3 + 2];
        const float miss = float(A16[15]);
        float Rtu[3];
        for (int k = 0; k < 3; ++k) Rtu[k] = (R[k] * uw[0] + R[3 + k] * uw[1] + R[6 + k] * uw[2]) * ia2[k];
        for (int r = 0; r < 3; ++r)
            gp[r] += Real(R[r * 3] * Rtu[0] + R[r * 3 + 1] * Rtu[1] + R[r * 3 + 2] * Rtu[2] + miss * float(c.Rw2c[6 + r]));
        for (int r = 0; r < 3; ++r)
            for (int k = 0; k < 3; ++k)
                dR[r * 3 + k] = (Mc[r * 3] * B[k] + Mc[r * 3 + 1] * B[3 + k] + Mc[r * 3 + 2] * B[6 + k]) * ia2[k];
        for (int k = 0; k < 3; ++k) {
            const float d = RtM[k * 3] * B[k] + RtM[k * 3 + 1] * B[3 + k] + RtM[k * 3 + 2] * B[6 + k];
            gs[k] += Real(-d * sig_a3[k]);
        }
        float uf[4] = {float(u[0]), float(u[1]), float(u[2]), float(u[3])}, dq[4];
        quat_rotation_backward<float>(uf, dR, dq);
        for (int j = 0; j < 4; ++j) gr[j] += Real(dq[j]);
    } else {
        for (int k = 0; k < 3; ++k) gp[k] += A16[6 + k];
        for (int k = 0; k < 4; ++k) gr[k] += A16[9 + k];
        for (int k = 0; k < 3; ++k) gs[k] += A16[13 + k];
    }

    if (a.visible[i]) {
        Real R[9];
        {
            const Real w = u[0], x = u[1], y = u[2], z = u[3];
            R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z); R[2] = 2 * (x * z + w * y);
            R[3] = 2 * (x * y + w * z); R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
            R[6] = 2 * (x * z - w * y); R[7] = 2 * (y * z + w * x); R[8] = 1 - 2 * (x * x + y * y);
        }
        const Real mu[3] = {a.means[3 * i], a.means[3 * i + 1], a.means[3 * i + 2]};
        // conic of this splat, recomputed (projection_backward uses splat.conic)
        Real pc[3];
        for (int r = 0; r < 3; ++r)
            pc[r] = Real(c.Rw2c[r * 3]) * mu[0] + Real(c.Rw2c[r * 3 + 1]) * mu[1] + Real(c.Rw2c[r * 3 + 2]) * mu[2] +
                    Real(c.tw2c[r]);
        const Real x = pc[0], y = pc[1], z = pc[2];
        const Real fx = Real(c.fx), fy = Real(c.fy);
        const Real J[6] = {fx / z, 0, -fx * x / (z * z), 0, fy / z, -fy * y / (z * z)};
        Real T[6];
        for (int r = 0; r < 2; ++r)
            for (int k = 0; k < 3; ++k)
                T[r * 3 + k] = J[r * 3] * Real(c.Rw2c[k]) + J[r * 3 + 1] * Real(c.Rw2c[3 + k]) +
                               J[r * 3 + 2] * Real(c.Rw2c[6 + k]);
        Real V[9];
        for (int r = 0; r < 3; ++r)
            for (int k = 0; k < 3; ++k)
                V[r * 3 + k] = R[r * 3] * (s[0] * s[0]) * R[k * 3] + R[r * 3 + 1] * (s[1] * s[1]) * R[k * 3 + 1] +
                               R[r * 3 + 2] * (s[2] * s[2]) * R[k * 3 + 2];
        Real TV[6], cov[4];
        for (int r = 0; r < 2; ++r)
            for (int k = 0; k < 3; ++k)
                TV[r * 3 + k] = T[r * 3] * V[k] + T[r * 3 + 1] * V[3 + k] + T[r * 3 + 2] * V[6 + k];
        for (int r = 0; r < 2; ++r)
            for (int k = 0; k < 2; ++k)
                cov[r * 2 + k] = TV[r * 3] * T[k * 3] + TV[r * 3 + 1] * T[k * 3 + 1] + TV[r * 3 + 2] * T[k * 3 + 2];
        cov[0] += Real(kCovFloor);
        cov[3] += Real(kCovFloor);
        const Real det = cov[0] * cov[3] - cov[2] * cov[1];
        const Real con[4] = {cov[3] / det, -cov[1] / det, -cov[1] / det, cov[0] / det};
        // dcov2d = -conic Gc conic (rasterizer_backward.cpp:66-69)
        const Real Gc[4] = {A16[3], A16[4], A16[4], A16[5]};
        Real t1[4], dcov[4];
        for (int r = 0; r < 2; ++r)
            for (int k = 0; k < 2; ++k) t1[r * 2 + k] = -(con[r * 2] * Gc[k] + con[r * 2 + 1] * Gc[2 + k]);
        for (int r = 0; r < 2; ++r)
            for (int k = 0; k < 2; ++k) dcov[r * 2 + k] = t1[r * 2] * con[k] + t1[r * 2 + 1] * con[2 + k];
        // dV = T^T dcov T ; dT = 2 dcov T V ; dJ = dT R_w2c^T   (:81-83)
        Real TtD[6], dV[9], D2T[6], dT[6], dJ[6];
        for (int r = 0; r < 3; ++r)
            for (int k = 0; k < 2; ++k) TtD[r * 2 + k] = T[r] * dcov[k] + T[3 + r] * dcov[2 + k];
        for (int r = 0; r < 3; ++r)
            for (int k = 0; k < 3; ++k) dV[r * 3 + k] = TtD[r * 2] * T[k] + TtD[r * 2 + 1] * T[3 + k];
        for (int r = 0; r < 2; ++r)
            for (int k = 0; k < 3; ++k)
                D2T[r * 3 + k] = Real(2) * (dcov[r * 2] * T[k] + dcov[r * 2 + 1] * T[3 + k]);
        for (int r = 0; r < 2; ++r)
            for (int k = 0; k < 3; ++k)
                dT[r * 3 + k] = D2T[r * 3] * V[k] + D2T[r * 3 + 1] * V[3 + k] + D2T[r * 3 + 2] * V[6 + k];
        for (int r = 0; r < 2; ++r)
            for (int k = 0; k < 3; ++k)
                dJ[r * 3 + k] = dT[r * 3] * Real(c.Rw2c[k * 3]) + dT[r * 3 + 1] * Real(c.Rw2c[k * 3 + 1]) +
                                dT[r * 3 + 2] * Real(c.Rw2c[k * 3 + 2]);
        const Real z2 = z * z, z3 = z2 * z;
        Real dp[3];
        dp[0] = dJ[2] * (-fx / z2);
        dp[1] = dJ[5] * (-fy / z2);
        dp[2] = dJ[0] * (-fx / z2) + dJ[4] * (-fy / z2) + dJ[2] * (2 * fx * x / z3) + dJ[5] * (2 * fy * y / z3);
        Real dm0 = A16[1], dm1 = A16[2];
        if (a.depth_moments) {
            dm0 = con[0] * A16[1] + con[1] * A16[2];
            dm1 = con[1] * A16[1] + con[3] * A16[2];
            go += A16[0] * (Real(1) + exp(-a.opacity_logits[i]));  // / opacity
        }
        dp[0] += dm0 * fx / z;
        dp[1] += dm1 * fy / z;
        dp[2] += -dm0 * fx * x / z2 - dm1 * fy * y / z2;
        for (int r = 0; r < 3; ++r)
            gp[r] += Real(c.Rc2w[r * 3]) * dp[0] + Real(c.Rc2w[r * 3 + 1]) * dp[1] + Real(c.Rc2w[r * 3 + 2]) * dp[2];
        // V = M M^T, M = R diag(s): dM = 2 dV M, dR = dM diag(s), ds += diag(R^T dM)   (:100-106)
        Real dM[9], dR[9];
        for (int r = 0; r < 3; ++r)
            for (int k = 0; k < 3; ++k)
                dM[r * 3 + k] = Real(2) * (dV[r * 3] * R[k] + dV[r * 3 + 1] * R[3 + k] + dV[r * 3 + 2] * R[6 + k]) * s[k];
        for (int r = 0; r < 3; ++r)
            for (int k = 0; k < 3; ++k) dR[r * 3 + k] = dM[r * 3 + k] * s[k];
        Real dq[4];
        quat_rotation_backward<Real>(u, dR, dq);
        for (int j = 0; j < 4; ++j) gr[j] += dq[j];
        for (int k = 0; k < 3; ++k) gs[k] += R[k] * dM[k] + R[3 + k] * dM[3 + k] + R[6 + k] * dM[6 + k];
        // SH + view-direction chain (:108-120, sh.cpp:86-99)
        Real g3[3] = {a.acc_dcolor[3 * i], a.acc_dcolor[3 * i + 1], a.acc_dcolor[3 * i + 2]};
        if (g3[0] * g3[0] + g3[1] * g3[1] + g3[2] * g3[2] != Real(0)) {
            const Real tg[3] = {mu[0] - Real(c.tc2w[0]), mu[1] - Real(c.tc2w[1]), mu[2] - Real(c.tc2w[2])};
            const Real nrm = sqrt(tg[0] * tg[0] + tg[1] * tg[1] + tg[2] * tg[2]);
            if (nrm > Real(1e-12)) {
                const Real dx = tg[0] / nrm, dy = tg[1] / nrm, dz = tg[2] / nrm;
                const uint8_t cl = a.clamped_bits[i];
                for (int ch = 0; ch < 3; ++ch)
                    if (cl & (1 << ch)) g3[ch] = 0;
                Real ddir[3] = {0, 0, 0};
                switch (a.deg) {  // compile-time K: basis and Jacobian stay in registers
                    case 0: sh_adjoint<Real, 0>(sh, g_sh, dx, dy, dz, g3, ddir); break;
                    case 1: sh_adjoint<Real, 1>(sh, g_sh, dx, dy, dz, g3, ddir); break;
                    case 2: sh_adjoint<Real, 2>(sh, g_sh, dx, dy, dz, g3, ddir); break;
                    default: sh_adjoint<Real, 3>(sh, g_sh, dx, dy, dz, g3, ddir); break;
                }
                const Real dirv[3] = {dx, dy, dz};
                const Real dd = dx * ddir[0] + dy * ddir[1] + dz * ddir[2];
                for (int k = 0; k < 3; ++k) gp[k] += (ddir[k] - dirv[k] * dd) / nrm;
            }
        }
    }
    if (a.chain) {  // chain_activations (scene.cpp:108-129)
        const Real qd = u[0] * gr[0] + u[1] * gr[1] + u[2] * gr[2] + u[3] * gr[3];
        for (int j = 0; j < 4; ++j) gr[j] = (gr[j] - u[j] * qd) / qn;
        for (int k = 0; k < 3; ++k) gs[k] *= s[k];
        const Real al = Real(1) / (Real(1) + exp(-a.opacity_logits[i]));
        go *= al * (Real(1) - al);
    }
    bool ok = true;
    for (int k = 0; k < 3; ++k) {
        a.g_pos[3 * i + k] = gp[k];
        a.g_scale[3 * i + k] = gs[k];
        ok &= isfinite(gp[k]) && isfinite(gs[k]);
    }
    for (int j = 0; j < 4; ++j) {
        a.g_rot[4 * i + j] = gr[j];
        ok &= isfinite(gr[j]);
    }
    a.g_opac[i] = go;
    ok &= isfinite(go) && isfinite(a.g_k[i]);
    return ok;
}

// One thread per Gaussian.  The wide rows (SH and its gradient, 3K values;
// the semantic gradient, C values) are moved block-wide: the block's rows are
// one contiguous range, staged through shared memory (SH, SH gradient) or
// scanned in place (semantic gradient finiteness) with coalesced accesses,
// instead of each thread striding through its own 108- / 200-byte row.
constexpr int kK10Threads = 128;

// A CTA's contiguous row range: dst[0, count) = src[0, count) (dst may be null:
// scan only), returning whether this thread saw a non-finite value.  16-byte
// vectors when both ends are 16-byte aligned (the packed layouts normally are),
// scalars otherwise and for the tail.
template <typename Real>
__device__ __forceinline__ bool k10_move_scan(const Real* src, Real* dst, int count, bool scan) {
    constexpr int W = 16 / int(sizeof(Real));
    bool bad = false;
    int done = 0;
    if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
        const int nv = count / W;
        const uint4* s = reinterpret_cast<const uint4*>(src);
        uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll 4
        for (int v = threadIdx.x; v < nv; v += kK10Threads) {
            const uint4 x = s[v];
            if (dst) d[v] = x;
            if (scan) {
                if constexpr (sizeof(Real) == 4)
                    bad |= (x.x & 0x7f800000u) == 0x7f800000u || (x.y & 0x7f800000u) == 0x7f800000u ||
                           (x.z & 0x7f800000u) == 0x7f800000u || (x.w & 0x7f800000u) == 0x7f800000u;
                else
                    bad |= (x.y & 0x7ff00000u) == 0x7ff00000u || (x.w & 0x7ff00000u) == 0x7ff00000u;
            }
        }
        done = nv * W;
    }
    for (int e = done + int(threadIdx.x); e < count; e += kK10Threads) {
        const Real v = src[e];
        if (dst) dst[e] = v;
        if (scan) bad |= !isfinite(v);
    }
    return bad;
}

template <typename Real>
size_t k10_smem_bytes(int K) { return size_t(2) * kK10Threads * 3 * K * sizeof(Real); }

template <typename Real>
#ifndef K10_MINB
#define K10_MINB 7  // 7 CTAs per SM (72 registers): measured 0.193 ms vs 0.203 at 6, 0.23 at 5
#endif
__global__ void __launch_bounds__(kK10Threads, K10_MINB) projection_backward_kernel(const __grid_constant__ ProjBackwardArgs<Real> a) {
    extern __shared__ __align__(16) unsigned char k10_smem[];
    const int RK = 3 * a.K;
    Real* const s_sh = reinterpret_cast<Real*>(k10_smem);
    Real* const s_gsh = s_sh + kK10Threads * RK;
    const int64_t i0 = int64_t(blockIdx.x) * kK10Threads;
    const int nb = int(a.n - i0 < kK10Threads ? a.n - i0 : kK10Threads);
    k10_move_scan<Real>(a.sh + size_t(i0) * RK, s_sh, nb * RK, false);
    k10_move_scan<Real>(a.g_sh + size_t(i0) * RK, s_gsh, nb * RK, false);
    __syncthreads();
    const int64_t i = i0 + threadIdx.x;
    bool ok = true;
    if (i < a.n) ok = projection_backward_one<Real>(a, i, s_sh + threadIdx.x * RK, s_gsh + threadIdx.x * RK);
    if (!ok) raise_error_ordered(a.err, kErrNonFiniteGrad, i);
    __syncthreads();
    // write the SH gradient back; finiteness of the SH and semantic rows (a
    // block-wide vote; the rows are only identified when it fires)
    bool any = k10_move_scan<Real>(s_gsh, a.g_sh + size_t(i0) * RK, nb * RK, true);
    if (a.C > 0) any |= k10_move_scan<Real>(a.g_sem + size_t(i0) * a.C, nullptr, nb * a.C, true);
    if (__syncthreads_or(any)) {
        int bad = -1;
        for (int e = threadIdx.x; e < nb * RK; e += kK10Threads)
            if (!isfinite(s_gsh[e]) && bad < 0) bad = e / RK;
        const Real* __restrict__ gsem = a.g_sem + size_t(i0) * a.C;
        for (int e = threadIdx.x; e < nb * a.C; e += kK10Threads)
            if (!isfinite(gsem[e]) && bad < 0) bad = e / a.C;
        if (bad >= 0) raise_error_ordered(a.err, kErrNonFiniteGrad, i0 + bad);
    }
}


template <typename Real>
__global__ void chain_kernel(int64_t n, const Real* __restrict__ quats, const Real* __restrict__ log_scales,
                             const Real* __restrict__ opac, Real* g_rot, Real* g_scale, Real* g_opac) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Real q[4], n2 = 0;
    for (int j = 0; j < 4; ++j) {
        q[j] = quats[4 * i + j];
        n2 += q[j] * q[j];
    }
    const Real qn = sqrt(n2);
    Real qd = 0;
    for (int j = 0; j < 4; ++j) qd += (q[j] / qn) * g_rot[4 * i + j];
    for (int j = 0; j < 4; ++j) g_rot[4 * i + j] = (g_rot[4 * i + j] - (q[j] / qn) * qd) / qn;
    for (int k = 0; k < 3; ++k) g_scale[3 * i + k] *= exp(log_scales[3 * i + k]);
    const Real al = Real(1) / (Real(1) + exp(-opac[i]));
    g_opac[i] *= al * (Real(1) - al);
}

template <typename Real>
__global__ void check_replay_kernel(int64_t n, const Real* __restrict__ means, const Real* __restrict__ k,
                                    const Real* __restrict__ saved_means, const Real* __restrict__ saved_k,
                                    DeviceError* err) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    bool same = k[i] == saved_k[i];
    for (int j = 0; j < 3; ++j) same &= means[3 * i + j] == saved_means[3 * i + j];
    if (!same) raise_error_ordered(err, kErrSceneModified, i);
}

template <typename Real>
void launch_projection_backward(const ProjBackwardArgs<Real>& a, cudaStream_t s) {
    if (a.n == 0) return;
    const size_t smem = k10_smem_bytes<Real>(a.K);
    static std::atomic<unsigned long long> attr{0};  // per instantiation, per device
    opt_in_smem(reinterpret_cast<const void*>(projection_backward_kernel<Real>), attr);
    projection_backward_kernel<Real><<<unsigned((a.n + kK10Threads - 1) / kK10Threads), kK10Threads, smem, s>>>(a);
    count_launches(1);
}

template <typename Real>
void launch_chain(int64_t n, const Real* quats, const Real* log_scales, const Real* opac, Real* g_rot,
                  Real* g_scale, Real* g_opac, cudaStream_t s) {
    if (n == 0) return;
    chain_kernel<Real><<<unsigned((n + 255) / 256), 256, 0, s>>>(n, quats, log_scales, opac, g_rot, g_scale, g_opac);
    count_launches(1);
}

template <typename Real>
void launch_check_replay(int64_t n, const Real* means, const Real* k, const Real* saved_means,
                         const Real* saved_k, DeviceError* err, cudaStream_t s) {
    if (n == 0) return;
    check_replay_kernel<Real><<<unsigned((n + 255) / 256), 256, 0, s>>>(n, means, k, saved_means, saved_k, err);
    count_launches(1);
}

#define MSPLAT_INST(R)                                                                                  \
    template void launch_projection_backward<R>(const ProjBackwardArgs<R>&, cudaStream_t);             \
    template void launch_chain<R>(int64_t, const R*, const R*, const R*, R*, R*, R*, cudaStream_t);     \
    template void launch_check_replay<R>(int64_t, const R*, const R*, const R*, const R*, DeviceError*, \
                                         cudaStream_t);
MSPLAT_INST(float)
MSPLAT_INST(double)
#undef MSPLAT_INST

}  // namespace msplat_cuda
