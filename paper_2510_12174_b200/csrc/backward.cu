// K9: per-tile reverse blend (rasterize_backward's tile loop,
// core/src/rasterizer_backward.cpp:140-255, with intersection_backward
// core/src/geometry.cpp:70-105 and quat_rotation_backward :17-29).
// K10: per-Gaussian projection / SH adjoint (projection_backward,
// rasterizer_backward.cpp:57-123; eval_sh_color_backward, sh.cpp:86-99) with
// chain_activations (scene.cpp:108-129) and check_finite (scene.cpp:97-106)
// fused.  Plus check_replay's scene comparison (rasterizer_backward.cpp:40-44).
//
// K9 layout: one CTA per tile, one thread per pixel (8x4 pixel block per warp).
// Each pixel replays its list from terminus-1 down to 0 with the forward's
// alpha test, restores T by division, and forms the reference's per-pair
// gradients.  Two reductions replace the reference's per-thread accumulators:
//   * "seed-linear" gradients (dcolor, dk, dsemantics = w * seed of the pixel)
//     are reduced channel-parallel: lane ch sums w_L * seed_L[ch] over the
//     blending lanes L of the warp (seeds staged once per tile in shared
//     memory, pixel-major rows), then one coalesced atomic per channel;
//   * the 16 "geometric" gradients (dopacity, dmean2d, dconic, and the depth
//     chain's dposition/drotation/dscale) are written per lane to a per-warp
//     shared scratch row and summed by lanes 0..15, one atomic each.
// Per (warp, Gaussian) event that is O(active lanes) work instead of a
// 5-level shuffle tree per value.
// The semantic part of dalpha uses the scalar recursion
//   A <- a_last * (sem_last . dO) + (1 - a_last) * A
// which equals sum_ch accum_sem[ch] * dO[ch] of the reference (:224-231).
#include "blend_common.cuh"
#include "kernels.h"

namespace msplat_cuda {

namespace {

constexpr int kBatch = 256;
constexpr int kThreads = 256;
constexpr int kGeo = 16;         // geometric values per pair
constexpr int kRedPitch = kGeo + 1;  // + w, odd pitch

__host__ __device__ inline int seed_pitch(int C) { return (C + 4) | 1; }

template <typename Real>
size_t backward_smem_bytes(int C) {
    return sizeof(AlphaRec<Real>) * kBatch + sizeof(uint32_t) * kBatch +
           sizeof(Real) * size_t(kTilePixels) * seed_pitch(C) +
           sizeof(Real) * 8 * 32 * kRedPitch + 16;
}

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

}  // namespace

template <typename Real>
__global__ void __launch_bounds__(kThreads) backward_kernel(const BackwardArgs<Real> a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    AlphaRec<Real>* s_rec = reinterpret_cast<AlphaRec<Real>*>(smem_raw);
    uint32_t* s_gid = reinterpret_cast<uint32_t*>(s_rec + kBatch);
    Real* s_seed = reinterpret_cast<Real*>(s_gid + kBatch);      // [256][seed_pitch]
    const int C = a.C, sp = seed_pitch(C), S = C + 4;
    Real* s_red = s_seed + size_t(kTilePixels) * sp;              // [8][32][kRedPitch]
    int* s_maxterm = reinterpret_cast<int*>(s_red + 8 * 32 * kRedPitch);

    const int tile = blockIdx.x;
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int x = tx * kTile + tile_pixel_x(warp, lane);
    const int y = ty * kTile + tile_pixel_y(warp, lane);
    const int pl = tile_pixel_index(warp, lane);
    const bool inside = x < a.W && y < a.H;
    const size_t HW = size_t(a.W) * a.H, p = size_t(y) * a.W + x;
    if (threadIdx.x == 0) *s_maxterm = 0;

    // Per-pixel seeds: dC, dK and dO into shared memory; dD in a register.
    Real* my_seed = s_seed + size_t(pl) * sp;
    int term = 0;
    Real T_final = Real(1), dD = Real(0);
    bool any = false;
    if (inside) {
        term = a.terminus[p];
        T_final = a.T_final[p];
        dD = a.ddepth[p];
        for (int ch = 0; ch < 3; ++ch) {
            my_seed[ch] = a.dcolor[ch * HW + p];
            any |= my_seed[ch] != Real(0);
        }
        my_seed[3] = a.dkmap[p];
        any |= my_seed[3] != Real(0) || dD != Real(0);
        for (int ch = 0; ch < C; ++ch) {
            my_seed[4 + ch] = a.dsem[size_t(ch) * HW + p];
            any |= my_seed[4 + ch] != Real(0);
        }
    } else {
        for (int ch = 0; ch < S; ++ch) my_seed[ch] = Real(0);
    }
    // rasterize_backward.cpp:156-171: nothing to do without blends or seeds.
    const bool active_px = inside && term > 0 && any;
    if (!active_px) term = 0;
    __syncthreads();
    if (term > 0) atomicMax(s_maxterm, term);
    __syncthreads();
    const int maxterm = *s_maxterm;
    if (maxterm == 0) return;

    const PixelRay<Real> ray = make_ray<Real>(a.cam, x, y);
    const Real dC0 = my_seed[0], dC1 = my_seed[1], dC2 = my_seed[2], dK = my_seed[3];
    const Real bg_dot = Real(a.rp.bg[0]) * dC0 + Real(a.rp.bg[1]) * dC1 + Real(a.rp.bg[2]) * dC2;
    const Real sigma = Real(a.rp.sigma_scale);
    Real T = T_final;
    Real ac0 = 0, ac1 = 0, ac2 = 0, lc0 = 0, lc1 = 0, lc2 = 0;
    Real acc_k = 0, last_k = 0, acc_sd = 0, last_sd = 0, last_alpha = 0;
    Real* my_red = s_red + size_t(warp * 32 + lane) * kRedPitch;
    const Real* warp_red = s_red + size_t(warp * 32) * kRedPitch;

    const uint2 range = a.tile_range[tile];
    const uint32_t list_end = range.x + uint32_t(maxterm);
    for (int64_t bend = int64_t(list_end); bend > int64_t(range.x); bend -= kBatch) {
        const uint32_t bstart = uint32_t(max(int64_t(range.x), bend - kBatch));
        const int nb = int(uint32_t(bend) - bstart);
        __syncthreads();
        if (int(threadIdx.x) < nb) {
            const uint32_t g = a.inst_gauss[bstart + threadIdx.x];
            s_gid[threadIdx.x] = g;
            s_rec[threadIdx.x] = a.arec[g];
        }
        __syncthreads();
        for (int j = nb - 1; j >= 0; --j) {
            const int pos = int(bstart - range.x) + j;  // index in the tile list
            AlphaEval<Real> ae;
            ae.pass = false;
            if (pos < term) ae = eval_alpha<Real>(s_rec[j], ray.px, ray.py);
            const unsigned mask = __ballot_sync(0xffffffffu, ae.pass);
            if (mask == 0) continue;
            const uint32_t g = s_gid[j];
            if (ae.pass) {
                Real v[kRedPitch];
#pragma unroll
                for (int i = 0; i < kRedPitch; ++i) v[i] = Real(0);
                T = T / (Real(1) - ae.alpha);
                const Real w = ae.alpha * T;
                v[kGeo] = w;
                const BlendRec<Real> br = a.brec[g];
                // Depth chain (rasterizer_backward.cpp:205-218).
                const Real dd = dD * w;
                if (dd != Real(0)) {
                    const HitEval<Real> h = intersect<Real>(br, ray, a.cam, a.raw, g);
                    if (h.hit) {
                        if constexpr (sizeof(Real) == 4) {
                            // Same adjoint, rewritten around the small midpoint offset
                            // p_l = v_l + t d_l (p_s = p_l / axes) so nothing cancels:
                            //   g_vs = -k d_s, g_ds = -k (p_s + t d_s), k = g_t / a
                            //   dscale = 2k (d_s o p_s) / s
                            //   dR = v g_vl^T + d g_dl^T = -k [(R p_l)(d_s/axes)^T + d (p_s/axes)^T]
                            if (!(fabsf(h.a) < 1e-12f)) {
                                const Real kk = dd * ray.dz / h.a;
                                const Real t = h.t_mid;
                                Real ps[3], pl[3], ga[3], gb[3];
#pragma unroll
                                for (int i = 0; i < 3; ++i) {
                                    pl[i] = br.vl[i] + t * h.dl[i];
                                    ps[i] = pl[i] * br.inv_axes[i];
                                    v[13 + i] = Real(2) * kk * h.ds[i] * ps[i] * sigma * br.inv_axes[i];
                                    ga[i] = h.ds[i] * br.inv_axes[i];  // -g_vl / k
                                    gb[i] = ps[i] * br.inv_axes[i];
                                }
                                Real Rp[3];
#pragma unroll
                                for (int i = 0; i < 3; ++i) {
                                    // dposition = -(R g_vl) = k R (d_s/axes); R = Rt^T
                                    v[6 + i] = kk * (br.Rt[0 * 3 + i] * ga[0] + br.Rt[1 * 3 + i] * ga[1] +
                                                     br.Rt[2 * 3 + i] * ga[2]);
                                    Rp[i] = br.Rt[0 * 3 + i] * pl[0] + br.Rt[1 * 3 + i] * pl[1] +
                                            br.Rt[2 * 3 + i] * pl[2];
                                }
                                Real G[9];
#pragma unroll
                                for (int r = 0; r < 3; ++r)
#pragma unroll
                                    for (int c = 0; c < 3; ++c) G[r * 3 + c] = -kk * (Rp[r] * ga[c] + ray.d[r] * gb[c]);
                                quat_rotation_backward<Real>(br.q, G, v + 9);
                            }
                        } else if (!(fabs(double(h.a)) < 1e-12)) {
                            const Real g_t = dd * ray.dz;
                            Real gvs[3], gds[3], gvl[3], gdl[3];
                            const Real inv_a = Real(1) / h.a;
                            const Real ba2 = h.b / (h.a * h.a);
#pragma unroll
                            for (int i = 0; i < 3; ++i) {
                                gvs[i] = g_t * (-h.ds[i] * inv_a);
                                gds[i] = g_t * (ba2 * h.ds[i] - br.vs[i] * inv_a);
                                // ds = -(g_vs o v_s + g_ds o d_s) / s,  s = axes / sigma
                                v[13 + i] = -((gvs[i] * br.vs[i] + gds[i] * h.ds[i]) * sigma * br.inv_axes[i]);
                                gvl[i] = gvs[i] * br.inv_axes[i];
                                gdl[i] = gds[i] * br.inv_axes[i];
                            }
                            // dposition = -(R g_vl); R = Rt^T.
                            Real vv[3];
#pragma unroll
                            for (int i = 0; i < 3; ++i) {
                                v[6 + i] = -(br.Rt[0 * 3 + i] * gvl[0] + br.Rt[1 * 3 + i] * gvl[1] +
                                             br.Rt[2 * 3 + i] * gvl[2]);
                                // v = o - mu = R (v_s o axes)
                                vv[i] = br.Rt[0 * 3 + i] * (br.vs[0] * br.axes[0]) +
                                        br.Rt[1 * 3 + i] * (br.vs[1] * br.axes[1]) +
                                        br.Rt[2 * 3 + i] * (br.vs[2] * br.axes[2]);
                            }
                            Real G[9];
#pragma unroll
                            for (int r = 0; r < 3; ++r)
#pragma unroll
                                for (int c = 0; c < 3; ++c) G[r * 3 + c] = vv[r] * gvl[c] + ray.d[r] * gdl[c];
                            quat_rotation_backward<Real>(br.q, G, v + 9);
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 3; ++i) v[6 + i] = dd * Real(a.cam.Rw2c[6 + i]);
                    }
                }
                // Alpha gradient (rasterizer_backward.cpp:222-244); depth excluded.
                ac0 = last_alpha * lc0 + (Real(1) - last_alpha) * ac0;
                ac1 = last_alpha * lc1 + (Real(1) - last_alpha) * ac1;
                ac2 = last_alpha * lc2 + (Real(1) - last_alpha) * ac2;
                acc_k = last_alpha * last_k + (Real(1) - last_alpha) * acc_k;
                acc_sd = last_alpha * last_sd + (Real(1) - last_alpha) * acc_sd;
                Real sd = Real(0);
                {
                    const Real* semg = a.semantics + size_t(g) * C;
                    const Real* dO = my_seed + 4;
                    for (int ch = 0; ch < C; ++ch) sd += semg[ch] * dO[ch];
                }
                Real dalpha = ((br.rgb[0] - ac0) * dC0 + (br.rgb[1] - ac1) * dC1 + (br.rgb[2] - ac2) * dC2) * T;
                dalpha += (br.k - acc_k) * dK * T;
                dalpha += (sd - acc_sd) * T;
                dalpha -= (T_final / (Real(1) - ae.alpha)) * bg_dot;
                if (!ae.clamped) {
                    v[0] = ae.gauss * dalpha;
                    const Real dpower = ae.alpha * dalpha;
                    const AlphaRec<Real>& ar = s_rec[j];
                    v[1] = dpower * (ar.ca * ae.dx + ar.cb * ae.dy);
                    v[2] = dpower * (ar.cb * ae.dx + ar.cc * ae.dy);
                    v[3] = dpower * (Real(-0.5) * ae.dx * ae.dx);
                    v[4] = dpower * (Real(-0.5) * ae.dx * ae.dy);
                    v[5] = dpower * (Real(-0.5) * ae.dy * ae.dy);
                }
                lc0 = br.rgb[0];
                lc1 = br.rgb[1];
                lc2 = br.rgb[2];
                last_k = br.k;
                last_sd = sd;
                last_alpha = ae.alpha;
#pragma unroll
                for (int i = 0; i < kRedPitch; ++i) my_red[i] = v[i];
            }
            __syncwarp();
            // Geometric reduction: lane i < 16 sums value i over blending lanes.
            if (lane < kGeo) {
                Real s = Real(0);
                unsigned m = mask;
                while (m) {
                    const int L = __ffs(m) - 1;
                    m &= m - 1;
                    s += warp_red[L * kRedPitch + lane];
                }
                if (s != Real(0)) {
                    Real* dst;
                    if (lane == 0) dst = a.g_opac + g;
                    else if (lane < 3) dst = a.acc_dmean + size_t(g) * 2 + (lane - 1);
                    else if (lane < 6) dst = a.acc_dconic + size_t(g) * 3 + (lane - 3);
                    else if (lane < 9) dst = a.g_pos + size_t(g) * 3 + (lane - 6);
                    else if (lane < 13) dst = a.g_rot + size_t(g) * 4 + (lane - 9);
                    else dst = a.g_scale + size_t(g) * 3 + (lane - 13);
                    atomicAdd(dst, s);
                }
            }
            // Seed-linear reduction, channel-parallel.
            for (int ch = lane; ch < S; ch += 32) {
                Real s = Real(0);
                unsigned m = mask;
                while (m) {
                    const int L = __ffs(m) - 1;
                    m &= m - 1;
                    s += warp_red[L * kRedPitch + kGeo] * s_seed[size_t(tile_pixel_index(warp, L)) * sp + ch];
                }
                if (s != Real(0)) {
                    Real* dst = ch < 3 ? a.acc_dcolor + size_t(g) * 3 + ch
                                       : (ch == 3 ? a.g_k + g : a.g_sem + size_t(g) * C + (ch - 4));
                    atomicAdd(dst, s);
                }
            }
            __syncwarp();
        }
    }
}

// ------------------------------------------------------------------ K10
template <typename Real>
__global__ void __launch_bounds__(256) projection_backward_kernel(const ProjBackwardArgs<Real> a) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= a.n) return;
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
        const Real Gc[4] = {a.acc_dconic[3 * i], a.acc_dconic[3 * i + 1], a.acc_dconic[3 * i + 1],
                            a.acc_dconic[3 * i + 2]};
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
        const Real dm0 = a.acc_dmean[2 * i], dm1 = a.acc_dmean[2 * i + 1];
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
                const int deg = a.deg, K = a.K;
                Real b[16], Jb[16][3];
                const Real C0 = Real(0.28209479177387814), C1 = Real(0.4886025119029199);
                const Real k0 = Real(1.0925484305920792), k1 = Real(-1.0925484305920792), k2 = Real(0.31539156525252005),
                           k3 = Real(-1.0925484305920792), k4 = Real(0.5462742152960396);
                const Real m0 = Real(-0.5900435899266435), m1 = Real(2.890611442640554), m2 = Real(-0.4570457994644658),
                           m3 = Real(0.3731763325901154), m4 = Real(-0.4570457994644658), m5 = Real(1.445305721320277),
                           m6 = Real(-0.5900435899266435);
                for (int j = 0; j < 16; ++j) Jb[j][0] = Jb[j][1] = Jb[j][2] = Real(0);
                const Real xx = dx * dx, yy = dy * dy, zz = dz * dz;
                b[0] = C0;
                if (deg >= 1) {
                    b[1] = -C1 * dy; b[2] = C1 * dz; b[3] = -C1 * dx;
                    Jb[1][1] = -C1; Jb[2][2] = C1; Jb[3][0] = -C1;
                }
                if (deg >= 2) {
                    b[4] = k0 * dx * dy; b[5] = k1 * dy * dz; b[6] = k2 * (2 * zz - xx - yy);
                    b[7] = k3 * dx * dz; b[8] = k4 * (xx - yy);
                    Jb[4][0] = k0 * dy; Jb[4][1] = k0 * dx;
                    Jb[5][1] = k1 * dz; Jb[5][2] = k1 * dy;
                    Jb[6][0] = -2 * k2 * dx; Jb[6][1] = -2 * k2 * dy; Jb[6][2] = 4 * k2 * dz;
                    Jb[7][0] = k3 * dz; Jb[7][2] = k3 * dx;
                    Jb[8][0] = 2 * k4 * dx; Jb[8][1] = -2 * k4 * dy;
                }
                if (deg >= 3) {
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
                Real ddir[3] = {0, 0, 0};
                for (int j = 0; j < K; ++j) {
                    const Real shg = a.sh[(i * 3 + 0) * K + j] * g3[0] + a.sh[(i * 3 + 1) * K + j] * g3[1] +
                                     a.sh[(i * 3 + 2) * K + j] * g3[2];
                    for (int k = 0; k < 3; ++k) ddir[k] += Jb[j][k] * shg;
                    for (int ch = 0; ch < 3; ++ch) a.g_sh[(i * 3 + ch) * K + j] += g3[ch] * b[j];
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
        ok &= isfinite(double(gp[k])) && isfinite(double(gs[k]));
    }
    for (int j = 0; j < 4; ++j) {
        a.g_rot[4 * i + j] = gr[j];
        ok &= isfinite(double(gr[j]));
    }
    a.g_opac[i] = go;
    ok &= isfinite(double(go)) && isfinite(double(a.g_k[i]));
    for (int j = 0; j < 3 * a.K; ++j) ok &= isfinite(double(a.g_sh[i * 3 * a.K + j]));
    for (int j = 0; j < a.C; ++j) ok &= isfinite(double(a.g_sem[i * a.C + j]));
    if (!ok) raise_error(a.err, kErrNonFiniteGrad, 0, i);
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
    if (!same) raise_error(err, kErrSceneModified, 0, i);
}

template <typename Real>
void launch_backward_blend(const BackwardArgs<Real>& a, int ntiles, cudaStream_t s) {
    if (ntiles == 0) return;
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(backward_kernel<Real>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        configured = true;
    }
    backward_kernel<Real><<<ntiles, kThreads, backward_smem_bytes<Real>(a.C), s>>>(a);
    count_launches(1);
}

template <typename Real>
void launch_projection_backward(const ProjBackwardArgs<Real>& a, cudaStream_t s) {
    if (a.n == 0) return;
    projection_backward_kernel<Real><<<unsigned((a.n + 255) / 256), 256, 0, s>>>(a);
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
    template void launch_backward_blend<R>(const BackwardArgs<R>&, int, cudaStream_t);                 \
    template void launch_projection_backward<R>(const ProjBackwardArgs<R>&, cudaStream_t);             \
    template void launch_chain<R>(int64_t, const R*, const R*, const R*, R*, R*, R*, cudaStream_t);     \
    template void launch_check_replay<R>(int64_t, const R*, const R*, const R*, const R*, DeviceError*, \
                                         cudaStream_t);
MSPLAT_INST(float)
MSPLAT_INST(double)
#undef MSPLAT_INST

}  // namespace msplat_cuda
