// K9: per-tile reverse blend -- rasterize_backward's tile loop
// (core/src/rasterizer_backward.cpp:140-255) with intersection_backward
// (core/src/geometry.cpp:70-105) and quat_rotation_backward (:17-29).
//
// One CTA per 16x16 tile, one thread per pixel, warps own 8x4 pixel blocks and
// run INDEPENDENTLY (no block barrier after setup): each warp walks the tile
// list back to front in 32-entry chunks up to its own max terminus, culls each
// chunk with the alpha-support boxes (one ballot), and replays its pixels.
//
// Phase A (per (warp, Gaussian) event, the reference's sequential recursion):
//   alpha test (same code and decisions as K6), T restore by division,
//   w = alpha T and dalpha.  With F_j = [rgb, k, sem] and the pixel seed
//   s_p = [dC, dK, dO], the reference's
//     dalpha = (rgb - acc_c).dC T + (k - acc_k) dK T + sum (sem - acc_s).dO T - bg
//   is (F_j.s_p - A) T - bg with A <- a_last (F_last.s_p) + (1 - a_last) A
//   (rasterizer_backward.cpp:222-232).  F_j is staged once per event and
//   dotted with the pixel's seed row (128-bit shared loads).  The seed-linear
//   gradients (dcolor, dk, dsem = sum_p w s_p) are accumulated channel-parallel
//   over the event's blending lanes, one atomic per channel.  Each blended pair
//   is ENQUEUED with everything phase B needs (self-contained entries, so the
//   queue spans chunks).
// Phase B (flush, 32 pairs per warp vector, every lane busy): dopacity,
//   dmean2d, dconic and the depth chain's dposition / drotation / dscale, then
//   a segmented warp reduction keyed by Gaussian (an event's entries are
//   contiguous) and one atomic per value per Gaussian.
#include "blend_common.cuh"
#include "kernels.h"
#include "radix_sort.cuh"

#ifndef K9_UNROLL
#define K9_UNROLL 8  // full sub-batch: 2.483 ms vs 2.494 at 4, 2.51 at 2
#endif

namespace msplat_cuda {

namespace {

constexpr int kThreads = 256;
constexpr int kQueue = 64;  // per-warp pair queue (flushed at >= 32)

// Seed rows [dC0 dC1 dC2 dK dO...]: the channel count rounded up to the mma K
// step (8) plus 4 -- an odd number of 16-byte units per row, so both per-lane
// row reads and the mma fragment loads (row = lane / 4) are conflict-free.
__host__ __device__ inline int seed_k8(int C) { return ((C + 4 + 7) / 8) * 8; }
__host__ __device__ inline int seed_pitch(int C) { return seed_k8(C) + 4; }

// Blend weight + the pixel's seed-row offset, read together (one 64-bit LDS
// for FP32) by the seed-linear loop.
template <typename Real>
struct __align__(2 * sizeof(Real)) WeightRow {
    Real w;
    uint32_t soff;
};

template <typename Real>
struct PairQueue {
    static constexpr bool kConic = true;  // entries carry the splat centre / conic
    __device__ Real weight(int i) const { return ws[i].w; }
    uint32_t meta[kQueue];  // pixel lane | clamped << 8
    uint32_t gid[kQueue];
    uint32_t inst[kQueue];  // position in the tile-sorted list (deterministic mode)
    WeightRow<Real> ws[kQueue];
    Real da[kQueue], al[kQueue], gs[kQueue];
    Real cx[kQueue], cy[kQueue], ca[kQueue], cb[kQueue], cc[kQueue];
};

template <typename Real>
struct WarpSmem {
    AlphaRec<Real> rec[32];
    uint32_t gid[32];
    uint32_t emask[32];  // blend-event batch: forward lane mask (active lanes only)
    uint32_t pos[32];    //   and list position
    Real dD[32];
    PairQueue<Real> q;
};

template <typename Real>
size_t backward_smem_bytes(int C) {
    const int sp = seed_pitch(C);
    return 8 * (sizeof(WarpSmem<Real>) + sizeof(Real) * size_t(32 + 2) * sp) + 64;
}

template <typename Real>
__device__ __forceinline__ Real dot_rows(const Real* a, const Real* b, int n) {
    Real s = Real(0);
    if constexpr (sizeof(Real) == 4) {
        // four independent FMA chains (latency, not throughput, bound)
        const float4* a4 = reinterpret_cast<const float4*>(a);
        const float4* b4 = reinterpret_cast<const float4*>(b);
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll 4
        for (int i = 0; i < n / 4; ++i) {
            const float4 x = a4[i], y = b4[i];
            s0 = fmaf(x.x, y.x, s0);
            s1 = fmaf(x.y, y.y, s1);
            s2 = fmaf(x.z, y.z, s2);
            s3 = fmaf(x.w, y.w, s3);
        }
        s = (s0 + s1) + (s2 + s3);
    } else {
        for (int i = 0; i < n; ++i) s += a[i] * b[i];
    }
    return s;
}

// Segmented sum toward the first lane of each run of equal keys (runs are
// contiguous).  same[k] = (key of lane + 2^k == my key).
template <typename Real>
__device__ __forceinline__ Real seg_sum(Real v, const bool* same) {
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const Real o = __shfl_down_sync(0xffffffffu, v, 1 << k);
        if (same[k]) v += o;
    }
    return v;
}

// The depth chain of one blended pair (rasterizer_backward.cpp:205-218): the
// ray-ellipsoid midpoint depth's adjoint into dmean (v[6..8]), drotation
// (v[9..12]) and dscale (v[13..15]); dd = dL/ddepth(pixel) * w.
template <typename Real>
__device__ __forceinline__ void depth_chain_adjoint(const BackwardArgs<Real>& a, uint32_t g, const PixelRay<Real>& ray,
                                                    Real dd, Real (&v)[16]) {
    const Real sigma = Real(a.rp.sigma_scale);
    const BlendRec<Real>& br = a.brec[g];
    const HitEval<Real> h = intersect<Real>(br, ray, a.cam, a.raw, g);
    if (h.hit) {
        if constexpr (sizeof(Real) == 4) {
            // Adjoint around the small midpoint offset p_l = v_l + t d_l
            // (p_s = p_l / axes), algebraically the reference's:
            //   g_vs = -k d_s, g_ds = -k (p_s + t d_s), k = g_t / a
            //   dscale = 2k (d_s o p_s) / s
            //   dR = -k [(R p_l)(d_s/axes)^T + d (p_s/axes)^T]
            if (!(fabsf(h.a) < 1e-12f)) {
                const Real kk = dd * ray.dz / h.a;
                const Real t = h.t_mid;
                Real ps[3], pl[3], ga[3], gb[3];
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    pl[i] = br.vl[i] + t * h.dl[i];
                    ps[i] = pl[i] * br.inv_axes[i];
                    v[13 + i] = Real(2) * kk * h.ds[i] * ps[i] * sigma * br.inv_axes[i];
                    ga[i] = h.ds[i] * br.inv_axes[i];
                    gb[i] = ps[i] * br.inv_axes[i];
                }
                Real Rp[3];
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    v[6 + i] = kk * (br.Rt[0 * 3 + i] * ga[0] + br.Rt[1 * 3 + i] * ga[1] + br.Rt[2 * 3 + i] * ga[2]);
                    Rp[i] = br.Rt[0 * 3 + i] * pl[0] + br.Rt[1 * 3 + i] * pl[1] + br.Rt[2 * 3 + i] * pl[2];
                }
                Real G[9];
#pragma unroll
                for (int rr = 0; rr < 3; ++rr)
#pragma unroll
                    for (int cc2 = 0; cc2 < 3; ++cc2)
                        G[rr * 3 + cc2] = -kk * (Rp[rr] * ga[cc2] + ray.d[rr] * gb[cc2]);
                quat_rotation_backward<Real>(br.q, G, v + 9);
            }
        } else if (!(fabs(h.a) < 1e-12)) {
            // The reference's formulation (geometry.cpp:70-105).
            const Real g_t = dd * ray.dz;
            Real gvs[3], gds[3], gvl[3], gdl[3];
            const Real ba2 = h.b / (h.a * h.a);
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                gvs[i] = g_t * (-h.ds[i] / h.a);
                gds[i] = g_t * (ba2 * h.ds[i] - br.vs[i] / h.a);
                v[13 + i] = -((gvs[i] * br.vs[i] + gds[i] * h.ds[i]) * sigma / br.axes[i]);
                gvl[i] = gvs[i] / br.axes[i];
                gdl[i] = gds[i] / br.axes[i];
            }
            Real vv[3];
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                v[6 + i] = -(br.Rt[0 * 3 + i] * gvl[0] + br.Rt[1 * 3 + i] * gvl[1] + br.Rt[2 * 3 + i] * gvl[2]);
                vv[i] = br.Rt[0 * 3 + i] * br.vl[0] + br.Rt[1 * 3 + i] * br.vl[1] + br.Rt[2 * 3 + i] * br.vl[2];
            }
            Real G[9];
#pragma unroll
            for (int rr = 0; rr < 3; ++rr)
#pragma unroll
                for (int cc2 = 0; cc2 < 3; ++cc2) G[rr * 3 + cc2] = vv[rr] * gvl[cc2] + ray.d[rr] * gdl[cc2];
            quat_rotation_backward<Real>(br.q, G, v + 9);
        }
    } else {
#pragma unroll
        for (int i = 0; i < 3; ++i) v[6 + i] = dd * Real(a.cam.Rw2c[6 + i]);
    }
}

// Phase B on the first n queue entries (n <= 32): per-pair geometric
// gradients, segmented by Gaussian, one atomic per value per Gaussian.
template <typename Real, bool DET, typename Queue>
__device__ __forceinline__ void flush_pairs(const BackwardArgs<Real>& a, const Queue& q, const Real* dDw, int n, int bx,
                                            int by) {
    const int lane = threadIdx.x & 31;
    const bool act = lane < n;
    const uint32_t meta = act ? q.meta[lane] : 0u;
    const uint32_t g = act ? q.gid[lane] : 0xffffffffu - lane;  // padding lanes: unique keys
    uint32_t inst = 0u;
    if constexpr (DET) inst = act ? q.inst[lane] : 0u;
    bool same[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const uint32_t o = __shfl_down_sync(0xffffffffu, g, 1 << k);
        same[k] = (lane + (1 << k) < 32) && o == g;
    }
    const uint32_t g_prev = __shfl_up_sync(0xffffffffu, g, 1);
    const bool head = act && (lane == 0 || g_prev != g);
    Real v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = Real(0);
    if (act) {
        const int L = int(meta & 0xffu);
        const bool clamped = (meta >> 8) & 1u;
        const Real w = q.weight(lane), dalpha = q.da[lane], alpha = q.al[lane], gauss = q.gs[lane];
        const int xL = bx + (L & 7), yL = by + (L >> 3);
        Real pcx, pcy, ca, cb, cc;
        if constexpr (Queue::kConic) {
            pcx = q.cx[lane];
            pcy = q.cy[lane];
            ca = q.ca[lane];
            cb = q.cb[lane];
            cc = q.cc[lane];
        } else {  // compact queue: re-read the splat record (L2-resident)
            const AlphaRec<Real> r = a.arec[g];
            pcx = r.cx;
            pcy = r.cy;
            ca = r.ca;
            cb = r.cb;
            cc = r.cc;
        }
        const Real dx = Real(xL) + Real(0.5) - pcx, dy = Real(yL) + Real(0.5) - pcy;
        if (!clamped) {  // rasterizer_backward.cpp:234-244
            v[0] = gauss * dalpha;
            const Real dpower = alpha * dalpha;
            v[1] = dpower * (ca * dx + cb * dy);
            v[2] = dpower * (cb * dx + cc * dy);
            v[3] = dpower * (Real(-0.5) * dx * dx);
            v[4] = dpower * (Real(-0.5) * dx * dy);
            v[5] = dpower * (Real(-0.5) * dy * dy);
        }
        // Depth chain (rasterizer_backward.cpp:205-218).
        const Real dd = dDw[L] * w;
        if (dd != Real(0)) depth_chain_adjoint<Real>(a, g, make_ray<Real>(a.cam, xL, yL), dd, v);
    }
    // Deterministic mode: this (instance, warp) owns a private slot; plain
    // read-modify-write in program order, reduced later in a fixed order.
    Real* const slot = DET ? a.partial + (size_t(inst) * 8 + (threadIdx.x >> 5)) * a.V : nullptr;
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = seg_sum<Real>(v[i], same);
    if (head) {
        if constexpr (DET) {
            if (int64_t(inst) < a.pair_cap)  // else capacity exceeded (zero_det_slots raised it)
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    if (v[i] != Real(0)) slot[i] += v[i];
        } else {
            Real* const row = a.acc16 + size_t(g) * 16;
            if constexpr (sizeof(Real) == 4) {
                // four 16-byte vector reductions into the Gaussian's 64-byte row
#pragma unroll
                for (int i = 0; i < 16; i += 4)
                    if (v[i] != 0.f || v[i + 1] != 0.f || v[i + 2] != 0.f || v[i + 3] != 0.f)
                        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(row + i), "f"(v[i]),
                                     "f"(v[i + 1]), "f"(v[i + 2]), "f"(v[i + 3])
                                     : "memory");
            } else {
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    if (v[i] != Real(0)) atomicAdd(row + i, v[i]);
            }
        }
    }
    __syncwarp();
}

// K9 phase B on n (<= 32) of the 16-byte pair records phase A wrote
// ({gid, pixel lane, dpower = alpha dalpha (0 when alpha was clamped), dd =
// dD w}): dopacity = G dalpha = dpower / opacity, dmean2d / dconic from dpower,
// the depth chain from dd; segmented by Gaussian, one vector reduction per row.
// The depth chain of one blended pair (rasterizer_backward.cpp:205-218,
// geometry.cpp:70-105) as moments: with the unnormalised camera-space ray
// p~ = ((px-cx)/fx, (py-cy)/fy, 1), a~ = |M R_c2w p~|^2, the midpoint P and
// s = dd / a~, the reference's adjoint is
//   dposition = Sigma^-1 R_c2w u,                u = sum s p~
//   dL/dSigma^-1 = -sum s (P - mu) d~^T  ->  S = R_c2w S_c R_c2w^T,
//                S_c = -sum s ((P-mu)_c p~^T + p~ (P-mu)_c^T)
//   drotation = qrb(S R D), dscale_k = -sigma (R^T S R)_kk / a_k^3
// (Sigma^-1 = R D R^T, D = diag(1 / a^2), a = sigma * scale).  Phase B sums
// u (3), S_c (6: xx yy zz xy xz yz) and, for pairs that miss the ellipsoid
// (depth = centre depth), dd (1) per Gaussian; K10 finishes in FP64.  The
// hit decision is the forward's (same DepthRec forms, same FP64 fallback).
__device__ __forceinline__ void depth_moments(const BackwardArgs<float>& a, uint32_t g, int xL, int yL, float dx,
                                              float dy, float u0, float v0, float dd, float (&v)[16]) {
    const float4* const q4 = reinterpret_cast<const float4*>(a.drec + g);
    const float4 e0 = q4[0], e1 = q4[1], e2 = q4[2];  // E0..3 | E4 E5 H0 H1 | H2 zc A0 A1
    const float xx = dx * dx, xy = dx * dy, yy = dy * dy;
    const float t1 = e0.y * dx, t2 = e0.z * dy, t3 = e0.w * xx, t4 = e1.x * xy, t5 = e1.y * yy;
    const float disc = ((e0.x + t1) + (t2 + t3)) + (t4 + t5);
    const float sdisc = ((fabsf(e0.x) + fabsf(t1)) + (fabsf(t2) + fabsf(t3))) + (fabsf(t4) + fabsf(t5));
    const float w1 = e1.w * dx, w2 = e2.x * dy;
    const float h = e1.z + w1 + w2;
    const float sh = fabsf(e1.z) + fabsf(w1) + fabsf(w2);
    bool hit;
    if (fabsf(disc) <= 1e-5f * sdisc || fabsf(h) <= 1e-5f * sh) {  // as the forward: FP64 decision
        double t, aa, bb, ds[3], dep;
        hit = intersect_fp64<float>(a.cam, a.raw, g, float(xL) + 0.5f, float(yL) + 0.5f, &t, &aa, &bb, ds, &dep);
    } else {
        hit = disc >= 0.f && h < 0.f;
    }
    if (!hit) {
        v[15] = dd;
        return;
    }
    const float4 e3 = q4[3], e4 = q4[4], e5 = q4[5];  // A2..5 | K0..3 | K4 K5 ex ey
    const float at = ((e2.z + e2.w * dx) + (e3.x * dy + e3.y * xx)) + (e3.z * xy + e3.w * yy);
    const float kq = ((e4.x + e4.y * dx) + (e4.z * dy + e4.w * xx)) + (e5.x * xy + e5.y * yy);
    const float ra = 1.f / at;
    const float delta = -kq * ra, t = e2.y + delta;  // t - z_c, t
    const float s = dd * ra;
    const float ifx = float(1.0 / a.cam.fx), ify = float(1.0 / a.cam.fy);
    const float p0x = (u0 - float(a.cam.cx)) * ifx, p0y = (v0 - float(a.cam.cy)) * ify;
    const float xp = p0x + dx * ifx, yp = p0y + dy * ify;  // p~
    const float qx = delta * p0x + t * dx * ifx - e5.z, qy = delta * p0y + t * dy * ify - e5.w, qz = delta;
    v[6] = s * xp;
    v[7] = s * yp;
    v[8] = s;
    v[9] = -2.f * s * qx * xp;
    v[10] = -2.f * s * qy * yp;
    v[11] = -2.f * s * qz;
    v[12] = -s * (qx * yp + qy * xp);
    v[13] = -s * (qx + qz * xp);
    v[14] = -s * (qy + qz * yp);
}

__device__ __forceinline__ void flush_records(const BackwardArgs<float>& a, const uint4* rec, int n, int bx, int by) {
    const int lane = threadIdx.x & 31;
    const bool act = lane < n;
    const uint4 r = act ? rec[lane] : make_uint4(0xffffffffu - lane, 0u, 0u, 0u);  // padding: unique keys
    const uint32_t g = r.x;
    // Runs of equal ids are contiguous (an event's pairs): lane's run ends at
    // the next run start, and the segmented sum needs only ceil(log2(longest
    // run)) shuffle steps.
    const uint32_t g_prev = __shfl_up_sync(0xffffffffu, g, 1);
    const bool brk = lane == 0 || g_prev != g;
    const unsigned starts = __ballot_sync(0xffffffffu, brk);
    const bool head = act && brk;
    const unsigned later = lane == 31 ? 0u : (starts >> (lane + 1)) << (lane + 1);
    const int run_end = later ? __ffs(later) - 1 : 32;
    const unsigned longest = __reduce_max_sync(0xffffffffu, brk ? unsigned(run_end - lane) : 0u);
    float v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = 0.f;
    if (act) {
        const int L = int(r.y);
        const int xL = bx + (L & 7), yL = by + (L >> 3);
        const float dpower = __uint_as_float(r.z), dd = __uint_as_float(r.w);
        if (dpower != 0.f || dd != 0.f) {
            const AlphaRec<float>& ar = a.arec[g];
            const float2 c0 = *reinterpret_cast<const float2*>(&ar.cx);  // cx, cy
            const float dx = float(xL) + 0.5f - c0.x, dy = float(yL) + 0.5f - c0.y;
            if (dpower != 0.f) {  // rasterizer_backward.cpp:234-244, as moments (K10: / opacity, conic .)
                v[0] = dpower;
                v[1] = dpower * dx;
                v[2] = dpower * dy;
                v[3] = dpower * (-0.5f * dx * dx);
                v[4] = dpower * (-0.5f * dx * dy);
                v[5] = dpower * (-0.5f * dy * dy);
            }
            if (dd != 0.f) depth_moments(a, g, xL, yL, dx, dy, c0.x, c0.y, dd, v);
        }
    }
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        if ((1u << k) >= longest) break;
        const bool in_run = lane + (1 << k) < run_end;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const float o = __shfl_down_sync(0xffffffffu, v[i], 1 << k);
            if (in_run) v[i] += o;
        }
    }
    if (head) {
        float* const row = a.acc16 + size_t(g) * 16;
#pragma unroll
        for (int i = 0; i < 16; i += 4)
            if (v[i] != 0.f || v[i + 1] != 0.f || v[i + 2] != 0.f || v[i + 3] != 0.f)
                asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(row + i), "f"(v[i]), "f"(v[i + 1]),
                             "f"(v[i + 2]), "f"(v[i + 3])
                             : "memory");
    }
}

}  // namespace

template <typename Real, bool DET>
__global__ void __launch_bounds__(kThreads, 2) backward_kernel(const __grid_constant__ BackwardArgs<Real> a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int C = a.C, sp = seed_pitch(C), S = C + 4;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpSmem<Real>* ws = reinterpret_cast<WarpSmem<Real>*>(smem_raw) + warp;
    Real* const warp_seed = reinterpret_cast<Real*>(reinterpret_cast<WarpSmem<Real>*>(smem_raw) + 8) +
                            size_t(warp) * (32 + 2) * sp;
    Real* const my_seed = warp_seed + size_t(lane) * sp;
    Real* const F_rows = warp_seed + size_t(32) * sp;  // staged F_j, double-buffered
    PairQueue<Real>& Q = ws->q;

    const int tile = blockIdx.x;
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const int bx = tx * kTile + (warp & 1) * 8, by = ty * kTile + (warp >> 1) * 4;
    const int x = bx + (lane & 7), y = by + (lane >> 3);
    const bool inside = x < a.W && y < a.H;
    const size_t HW = size_t(a.W) * a.H, p = size_t(y) * a.W + x;

    // Per-pixel seeds -> this warp's shared rows; dD for the flush.
    int term = 0;
    Real T_final = Real(1), dD = Real(0);
    bool any = false;
    for (int ch = 0; ch < sp; ++ch) my_seed[ch] = Real(0);
    for (int i = lane; i < 2 * sp; i += 32) F_rows[i] = Real(0);
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
    }
    // rasterize_backward.cpp:156-171: nothing to do without blends or seeds.
    if (!(inside && term > 0 && any)) term = 0;
    ws->dD[lane] = dD;
    int wmax = term;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wmax = max(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
    if (wmax == 0) return;
    __syncwarp();

    const Real pxf = Real(x) + Real(0.5), pyf = Real(y) + Real(0.5);
    const Real bg_dot = Real(a.rp.bg[0]) * my_seed[0] + Real(a.rp.bg[1]) * my_seed[1] + Real(a.rp.bg[2]) * my_seed[2];
    Real T = T_final, accA = 0, lastFS = 0, last_alpha = 0;
    const uint2 range = a.tile_range[tile];
    const uint32_t list0 = range.x;
    // Clamped channel indices keep every shared read inside a seed row (C may be 0).
    const int c0 = lane < sp ? lane : 0, c1 = lane + 32 < sp ? lane + 32 : 0;
    // Destination of the F channel this lane accumulates (F = [rgb, k, sem]):
    // base + gid * stride, hoisted out of the event loop.
    Real* const dst0 = lane < 3 ? a.acc_dcolor + lane : (lane == 3 ? a.g_k : a.g_sem + (lane - 4));
    const int stride0 = lane < 3 ? 3 : (lane == 3 ? 1 : C);
    Real* const dst1 = a.g_sem + (lane + 28);  // channel lane + 32
    int qn = 0, fb = 0;
    // The forward's blend-event log for this warp: exactly the (Gaussian, lane
    // mask) events in which some pixel of the block blended, front to back.
    // Replayed back to front in batches of 32 whose ids and alpha records are
    // fetched in parallel; no culling or alpha test of non-blending pairs.
    const unsigned act_mask = __ballot_sync(0xffffffffu, term > 0);
    const uint32_t nev = a.ev_count[size_t(tile) * 8 + warp];
    const uint4* const evl = a.ev_list + size_t(8) * list0 + size_t(warp) * (range.y - list0);

    for (int cb = int(nev) - 1; cb >= 0; cb -= 32) {
        __syncwarp();  // the previous batch's records are no longer read
        {
            const int e = cb - lane;
            if (e >= 0) {
                const uint4 ev = evl[e];
                const uint32_t g = ev.z;
                ws->rec[lane] = a.arec[g];
                ws->gid[lane] = g;
                ws->emask[lane] = ev.y & act_mask;
                ws->pos[lane] = ev.x;
            }
        }
        __syncwarp();
        const int nb = cb + 1 < 32 ? cb + 1 : 32;
        stage_F_async<Real>(F_rows + fb * sp, a.brec, a.semantics, C, ws->gid[0], lane);
        for (int slot = 0; slot < nb; ++slot) {
            const Real* const warp_F = F_rows + fb * sp;
            fb ^= 1;
            // the next event's row streams in while this one is processed
            if (slot + 1 < nb) stage_F_async<Real>(F_rows + fb * sp, a.brec, a.semantics, C, ws->gid[slot + 1], lane);
            else stage_F_commit_empty();
            const unsigned fmask = ws->emask[slot];
            if (fmask == 0) continue;
            AlphaEval<Real> ae;
            ae.pass = false;
            if ((fmask >> lane) & 1u) ae = eval_alpha<Real>(ws->rec[slot], pxf, pyf);
            const unsigned mask = __ballot_sync(0xffffffffu, ae.pass);
            if (mask == 0) continue;
            stage_F_wait_prev();
            const uint32_t g = ws->gid[slot];
            __syncwarp();
            if (ae.pass) {
                // One reciprocal for the T restore and the background term (FP32);
                // FP64 keeps the reference's divisions.
                const Real inv = sizeof(Real) == 4 ? Real(1) / (Real(1) - ae.alpha) : Real(0);
                T = sizeof(Real) == 4 ? T * inv : T / (Real(1) - ae.alpha);
                const Real w = ae.alpha * T;
                const Real FS = dot_rows<Real>(warp_F, my_seed, sp);
                accA = last_alpha * lastFS + (Real(1) - last_alpha) * accA;
                const Real dalpha = (FS - accA) * T - (sizeof(Real) == 4 ? T_final * inv : T_final / (Real(1) - ae.alpha)) * bg_dot;
                lastFS = FS;
                last_alpha = ae.alpha;
                const int e = qn + __popc(mask & ((1u << lane) - 1u));
                const AlphaRec<Real>& ar = ws->rec[slot];
                Q.meta[e] = uint32_t(lane) | (ae.clamped ? (1u << 8) : 0u);
                Q.gid[e] = g;
                if constexpr (DET) Q.inst[e] = list0 + ws->pos[slot];
                Q.ws[e] = WeightRow<Real>{w, uint32_t(lane * sp)};
                Q.da[e] = dalpha;
                Q.al[e] = ae.alpha;
                Q.gs[e] = ae.gauss;
                Q.cx[e] = ar.cx;
                Q.cy[e] = ar.cy;
                Q.ca[e] = ar.ca;
                Q.cb[e] = ar.cb;
                Q.cc[e] = ar.cc;
            }
            __syncwarp();
            // Seed-linear gradients of this event, channel-parallel.
            {
                const int npairs = __popc(mask);
                Real acc0 = Real(0), acc1 = Real(0);
#pragma unroll 2
                for (int e = qn; e < qn + npairs; ++e) {
                    const WeightRow<Real> wr = Q.ws[e];
                    acc0 += wr.w * warp_seed[wr.soff + c0];
                    acc1 += wr.w * warp_seed[wr.soff + c1];
                }
                if constexpr (DET) {  // fields 16 + ch: dcolor, dk, dsem
                    // (beyond the slot capacity: zero_det_slots raised it; nothing is written)
                    const bool in_cap = int64_t(list0 + ws->pos[slot]) < a.pair_cap;
                    Real* const ps = a.partial + (size_t(list0 + ws->pos[slot]) * 8 + warp) * a.V + 16;
                    if (in_cap && lane < S && acc0 != Real(0)) ps[lane] += acc0;
                    if (in_cap && lane + 32 < S && acc1 != Real(0)) ps[lane + 32] += acc1;
                    for (int ch = lane + 64; in_cap && ch < S; ch += 32) {
                        Real s = Real(0);
                        for (int e = qn; e < qn + npairs; ++e) s += Q.ws[e].w * warp_seed[Q.ws[e].soff + ch];
                        if (s != Real(0)) ps[ch] += s;
                    }
                } else if (lane < S && acc0 != Real(0)) {
                    atomicAdd(dst0 + size_t(g) * stride0, acc0);
                }
                if (!DET && lane + 32 < S && acc1 != Real(0)) atomicAdd(dst1 + size_t(g) * C, acc1);
                for (int ch = lane + 64; !DET && ch < S; ch += 32) {  // C > 60
                    Real s = Real(0);
                    for (int e = qn; e < qn + npairs; ++e) s += Q.ws[e].w * warp_seed[Q.ws[e].soff + ch];
                    if (s != Real(0)) atomicAdd(a.g_sem + size_t(g) * C + (ch - 4), s);
                }
                qn += npairs;
            }
            if (qn >= 32) {
                flush_pairs<Real, DET>(a, Q, ws->dD, 32, bx, by);
                const int rest = qn - 32;
                if (lane < rest) {  // reads >= 32, writes < 32: no overlap
                    const int s2 = 32 + lane;
                    Q.meta[lane] = Q.meta[s2];
                    Q.gid[lane] = Q.gid[s2];
                    if constexpr (DET) Q.inst[lane] = Q.inst[s2];
                    Q.ws[lane] = Q.ws[s2];
                    Q.da[lane] = Q.da[s2];
                    Q.al[lane] = Q.al[s2];
                    Q.gs[lane] = Q.gs[s2];
                    Q.cx[lane] = Q.cx[s2];
                    Q.cy[lane] = Q.cy[s2];
                    Q.ca[lane] = Q.ca[s2];
                    Q.cb[lane] = Q.cb[s2];
                    Q.cc[lane] = Q.cc[s2];
                }
                qn = rest;
                __syncwarp();
            }
        }
    }
    if (qn > 0) flush_pairs<Real, DET>(a, Q, ws->dD, qn, bx, by);
}

// ---------------------------------------------------------------------------
// K9 (FP32) on the tensor cores.  The two C-length contractions of the reverse
// blend are GEMMs once a warp's blend events are taken kSub at a time from the
// forward's event log:
//   GEMM1  FS[px][e]  = sum_ch S[px][ch] F_e[ch]        (F_j . s_p for dalpha)
//   GEMM2  dF[ch][e]  = sum_px S[px][ch] w_e[px]         (dcolor, dk, dsem)
// with S the warp's 32 seed rows [dC, dK, dO] and F_e = [rgb, k, sem] of event
// e.  Both run as mma.sync.m16n8k8 TF32 with a hi/lo split of every operand
// (a_hi b_hi + a_hi b_lo + a_lo b_hi: FP32-level accuracy), the events on the
// N = 8 side.  Between them the per-pixel recursion (T restore, w = alpha T,
// dalpha with the suffix accumulator) runs sequentially per event exactly as
// in backward_kernel, reading FS from shared memory and enqueueing pairs for
// the same phase-B flush.
namespace {

constexpr int kK9Unroll = K9_UNROLL;
#ifndef K9B_MINB
#define K9B_MINB 6  // phase-B CTAs per SM (moments: 0.730 ms vs 0.747 at 5, 0.763 at 7)
#endif
#ifndef K9_RED2_MT0
#define K9_RED2_MT0 1  // also the semantic pairs of channel tile 0 (colour / k stay scalar): 2.486 ms vs 2.494
#endif
#ifndef K9_RED2
#define K9_RED2 1  // semantic GEMM2 outputs as 8-byte vector reductions (pairs from the g4^1 lane): 2.495 ms vs 2.509
#endif
#ifndef K9_PIPE
#define K9_PIPE 1  // chunk ids one chunk ahead, F rows prefetched to L2 and records to L1 at chunk start: 2.55 ms vs 2.58
#endif
constexpr int kSub = 8;         // events per sub-batch (mma N)
constexpr int kTilePitch = 36;  // FS / W tiles [kSub][36]: conflict-free fragment stores and row reads


struct WarpSmemTC {
    AlphaRec<float> rec[kSub];
    uint32_t gid[32];
    uint32_t emask[32];
    uint32_t foff[kSub];  // float offset of each staged semantic row inside its 16-byte chunks
    float Tf[32], bgd[32];  // per-pixel T_final and background . dC
    float dDs[32];          // per-pixel dL/ddepth
};


__host__ __device__ inline int tc_stage_floats(int C) {
    const int sp = seed_pitch(C);
    return kSub * sp > kSub * kTilePitch ? kSub * sp : kSub * kTilePitch;
}
__host__ __device__ inline int tc_warp_floats(int C) {
    return 32 * seed_pitch(C) + tc_stage_floats(C) + kSub * kTilePitch;
}
// Phase A in 4-warp CTAs at 4 / SM (the same 16 warps / SM as 8-warp CTAs at
// 2, but CTAs retire at a finer grain at the end of the longest-first order):
// 2.246 ms vs 2.257; 6-warp CTAs at 3 / SM (96 registers): 2.30.
#ifndef K9A_WARPS
#define K9A_WARPS 4  // warps per phase-A CTA (segments are independent: any CTA size works)
#endif
#ifndef K9A_MINB
#define K9A_MINB (16 / K9A_WARPS)
#endif
constexpr int kTcWarps = K9A_WARPS;
size_t backward_tc_smem_bytes(int C) {
    return kTcWarps * (sizeof(WarpSmemTC) + sizeof(float) * size_t(tc_warp_floats(C))) + 64;
}

}  // namespace

// Stages F rows [rgb, k | sem] of n (<= kSub) events into rows of pitch sp:
// one 16-byte copy of (rgb, k) per row from the AlphaRec (offset 48, the line
// the sub-batch's records come from) and the semantic row as the whole
// 16-byte chunks covering it (any 4-byte alignment; a chunk never straddles a
// page), four lanes per event, landing at row + 4 with the row's own data at
// row + 4 + foff[e].  The chunks never pass row + sp (4 ceil((C+3)/4) <= K8).
__device__ __forceinline__ void stage_rows_tc(float* Fb, int sp, const AlphaRec<float>* arec, const float* semantics,
                                              int C, uint32_t* foff, const uint32_t* gid, int n, int lane) {
    if (lane < n) {
        const unsigned dst = unsigned(__cvta_generic_to_shared(Fb + lane * sp));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(&arec[gid[lane]].rgb[0]) : "memory");
    }
    const int e = lane >> 2, part = lane & 3;
    if (e < n && C > 0) {
        const uintptr_t r0 = reinterpret_cast<uintptr_t>(semantics + size_t(gid[e]) * C);
        const uintptr_t c0 = r0 & ~uintptr_t(15);
        const int nch = int(((r0 + uintptr_t(4 * C) + 15) & ~uintptr_t(15)) - c0) >> 4;
        if (part == 0) foff[e] = uint32_t(r0 - c0) >> 2;
        const char* src = reinterpret_cast<const char*>(c0) + 16 * part;
        unsigned dst = unsigned(__cvta_generic_to_shared(Fb + e * sp + 4 + 4 * part));
        for (int q = part; q < nch; q += 4, src += 64, dst += 64)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

// kRows: the forward ran split (forward_split.cu) and left one row of 32 blend
// weights per event (negated where alpha was clamped at 0.99).  The recursion then needs no
// alpha records and no alpha test: w comes from the row, the transmittance is
// restored by addition (T_j = T_{j+1} + w_j, exact in real arithmetic since
// T_{j+1} = T_j (1 - alpha_j) and w_j = alpha_j T_j), alpha_j = w_j / T_j, and
// with B_j = sum_{k>j} w_k FS_k (the pixel's suffix sum) the reference's
//   dalpha = (FS_j - acc) T_j - T_final bg / (1 - alpha_j)
// is T_j (FS_j - (B_j + T_final bg) / T_{j+1}) (rasterizer_backward.cpp:222-232).
// GEMM2 reads the same rows.
template <bool kRows>
__global__ void __launch_bounds__(32 * kTcWarps, K9A_MINB) backward_kernel_tc(const __grid_constant__ BackwardArgs<float> a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int C = a.C, sp = seed_pitch(C), S = C + 4, K8 = seed_k8(C);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g4 = lane >> 2, t4 = lane & 3;  // mma fragment coordinates
    WarpSmemTC* ws = reinterpret_cast<WarpSmemTC*>(smem_raw) + warp;
    float* const warp_seed =
        reinterpret_cast<float*>(reinterpret_cast<WarpSmemTC*>(smem_raw) + kTcWarps) + size_t(warp) * tc_warp_floats(C);
    float* const my_seed = warp_seed + size_t(lane) * sp;
    float* const Fb = warp_seed + size_t(32) * sp;  // [kSub][sp] F rows; then FS [kSub][36] in place
    float* const FSs = Fb;
    float* const Wb = Fb + tc_stage_floats(C);      // [kSub][36] blend weights

    // this warp's (tile, 8x4 block) segment: longest-first order, or in tile order
    const int item = int(blockIdx.x) * kTcWarps + warp;
    if (item >= a.nseg) return;
    const int seg_i = a.work_order ? int(a.work_order[item]) : item;
    const int tile = seg_i >> 3, wl = seg_i & 7;
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const int bx = tx * kTile + (wl & 1) * 8, by = ty * kTile + (wl >> 1) * 4;
    const int x = bx + (lane & 7), y = by + (lane >> 3);
    const bool inside = x < a.W && y < a.H;
    const size_t HW = size_t(a.W) * a.H, p = size_t(y) * a.W + x;

    int term = 0;
    float T_final = 1.f, dD = 0.f;
    bool any = false;
    for (int ch = 0; ch < sp; ++ch) my_seed[ch] = 0.f;
    for (int i = lane; i < tc_stage_floats(C) + kSub * kTilePitch; i += 32) Fb[i] = 0.f;
    if (lane < kSub) ws->foff[lane] = 0u;
    // Non-finite seeds (an error path): check_finite (scene.cpp:97-106) then
    // names the lowest primitive blending at such a pixel.  They are zeroed
    // for the tensor-core products (0 * inf in another event's column would
    // spread NaN to primitives that never touch the pixel) and every primitive
    // the forward blended at such a pixel is reported (a pass over the event
    // log, off the hot loop), so the named primitive is the reference's.
    bool bad = false;
    if (inside) {
        term = a.terminus[p];
        T_final = a.T_final[p];
        dD = a.ddepth[p];
        const float s0 = a.dcolor[p], s1 = a.dcolor[HW + p], s2 = a.dcolor[2 * HW + p], s3 = a.dkmap[p];
        my_seed[0] = s0;
        my_seed[1] = s1;
        my_seed[2] = s2;
        my_seed[3] = s3;
        any = s0 != 0.f || s1 != 0.f || s2 != 0.f || s3 != 0.f || dD != 0.f;
        bad = !isfinite(s0) || !isfinite(s1) || !isfinite(s2) || !isfinite(s3) || !isfinite(dD);
        // the semantic seed planes straight into the pixel's shared row, all in
        // flight at once (cp.async: no register staging)
        for (int ch = 0; ch < C; ++ch)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(unsigned(__cvta_generic_to_shared(
                             my_seed + 4 + ch))),
                         "l"(a.dsem + size_t(ch) * HW + p)
                         : "memory");
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
        for (int ch = 0; ch < C; ++ch) {
            const float v = my_seed[4 + ch];
            any |= v != 0.f;
            bad |= !isfinite(v);
        }
    }
    // rasterize_backward.cpp:156-171: nothing to do without blends or seeds.
    if (!(inside && term > 0 && any)) term = 0;
    if (bad) {
        for (int ch = 0; ch < sp; ++ch) my_seed[ch] = 0.f;
        dD = 0.f;
    }
    const unsigned bad_mask = __ballot_sync(0xffffffffu, bad && term > 0);
    const size_t seg = size_t(seg_i);  // this warp's pair-record segment
    const unsigned act_mask = __ballot_sync(0xffffffffu, term > 0);
    if (act_mask == 0) {
        if (lane == 0) a.pair_n[seg] = 0;
        return;
    }
    __syncwarp();

    // Read-only per-pixel values live in shared memory and the pixel centre is
    // recomputed where used: the event loop keeps only the recursion state
    // (T, accA, lastFS, last_alpha) in registers, so nothing spills to local
    // memory (whose reloads miss the small L1 left by the carve-out).
    ws->Tf[lane] = T_final;
    ws->dDs[lane] = dD;
    ws->bgd[lane] = float(a.rp.bg[0]) * my_seed[0] + float(a.rp.bg[1]) * my_seed[1] + float(a.rp.bg[2]) * my_seed[2];
    float T = T_final, accA = 0.f, lastFS = 0.f, last_alpha = 0.f;
    const float Tfb = T_final * ws->bgd[lane];  // kRows: T_final (bg . dC)
    const uint2 range = a.tile_range[tile];
    const uint32_t list0 = range.x;
    const uint32_t nev = a.ev_count[seg];
    const size_t ev0 = size_t(8) * list0 + size_t(wl) * (range.y - list0);  // this segment's event-log region
    const uint4* const evl = a.ev_list + ev0;
    const float* const wrows = kRows ? a.ev_w + ev0 * 32 : nullptr;
    const int mtiles2 = (S + 15) / 16;  // GEMM2 channel tiles
    if (bad_mask) {  // error path only (warp-uniform)
        for (int e = lane; e < int(nev); e += 32) {
            const uint4 ev = evl[e];
            if (ev.y & bad_mask) raise_error_ordered(a.err, kErrNonFiniteGrad, ev.z);
        }
    }
    int qn = 0;
    const int64_t pbase = a.pair_off[seg];
    const int64_t pcap = a.pair_cap - pbase;  // records this segment may hold

#if K9_PIPE
    // The next 32-event chunk's (id, mask) are loaded one chunk ahead; at a
    // chunk's start its F rows are prefetched into L2 and its alpha records
    // into L1, so only the first sub-batch waits on memory.
    uint32_t nx_gid = 0u, nx_mask = 0u;
    if (int(nev) - 1 - lane >= 0) {
        const uint4 ev = evl[int(nev) - 1 - lane];
        nx_gid = ev.z;
        nx_mask = ev.y & act_mask;
    }
#endif
    for (int cb = int(nev) - 1; cb >= 0; cb -= 32) {
        __syncwarp();
#if K9_PIPE
        if (cb - lane >= 0) {
            const uint32_t g = nx_gid;
            ws->gid[lane] = g;
            ws->emask[lane] = nx_mask;
            const char* row = reinterpret_cast<const char*>(a.semantics + size_t(g) * C);
            asm volatile("prefetch.global.L2 [%0];" ::"l"(row));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(row + 4 * C - 4));
            if (C > 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(row + 128));
            if (!kRows) asm volatile("prefetch.global.L1 [%0];" ::"l"(reinterpret_cast<const char*>(a.arec + g)));
        }
        if (cb - 32 - lane >= 0) {
            const uint4 ev = evl[cb - 32 - lane];
            nx_gid = ev.z;
            nx_mask = ev.y & act_mask;
        }
#else
        {
            const int e = cb - lane;
            if (e >= 0) {
                const uint4 ev = evl[e];
                ws->gid[lane] = ev.z;
                ws->emask[lane] = ev.y & act_mask;
            }
        }
#endif
        __syncwarp();
        const int nb = cb + 1 < 32 ? cb + 1 : 32;
        for (int s0 = 0; s0 < nb; s0 += kSub) {
            const int ns = nb - s0 < kSub ? nb - s0 : kSub;
            // (a) F rows (cp.async) and alpha records of the sub-batch (kRows:
            // the events' weight rows instead; slot s0 + e is event cb - s0 - e).
            if constexpr (kRows) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {  // 8 rows x 8 16-byte pieces
                    const int i = lane + 32 * h, e = i >> 3, q = i & 7;
                    float* const dst = Wb + e * kTilePitch + 4 * q;
                    if (e < ns) {
                        const unsigned d = unsigned(__cvta_generic_to_shared(dst));
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d),
                                     "l"(wrows + size_t(cb - s0 - e) * 32 + 4 * q)
                                     : "memory");
                    } else {
                        *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                }
            }
            stage_rows_tc(Fb, sp, a.arec, a.semantics, C, ws->foff, ws->gid + s0, ns, lane);
            if (!kRows && lane < ns) ws->rec[lane] = a.arec[ws->gid[s0 + lane]];
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncwarp();
            // (b) GEMM1: FS[px][e], px on M (two 16-row tiles), events on N.
            float d1[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
            const int fo = int(ws->foff[g4]);  // event g4's semantic channels start at column 4 + fo
            for (int k0 = 0; k0 < K8; k0 += 8) {
                const float bf[2] = {Fb[g4 * sp + k0 + t4 + (k0 ? fo : 0)], Fb[g4 * sp + k0 + t4 + 4 + fo]};
#pragma unroll
                for (int mt = 0; mt < 2; ++mt) {
                    const float* A0 = warp_seed + (mt * 16 + g4) * sp + k0 + t4;
                    const float af[4] = {A0[0], A0[8 * sp], A0[4], A0[8 * sp + 4]};
                    mma_3xtf32(d1[mt], af, bf);
                }
            }
            __syncwarp();  // every lane is done with Fb: FS overwrites it
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    FSs[(2 * t4 + (i & 1)) * kTilePitch + mt * 16 + 8 * (i >> 1) + g4] = d1[mt][i];
            __syncwarp();
            // (c) the reference's sequential recursion, event by event.
#pragma unroll kK9Unroll
            for (int e = 0; e < ns; ++e) {
                const unsigned fmask = ws->emask[s0 + e];
                if constexpr (kRows) {  // the forward's weights and decisions
                    if ((fmask >> lane) & 1u) {
                        const float ws_ = Wb[e * kTilePitch + lane];
                        const bool clamped = ws_ < 0.f;
                        const float w = fabsf(ws_);
                        Wb[e * kTilePitch + lane] = w;  // GEMM2 reads plain weights
                        const float Tj = T + w;
                        const float FS = FSs[e * kTilePitch + lane];
                        const float rT = T > 0.f ? __fdividef(1.f, T) : 0.f;  // 1 / T_{j+1}
                        const float dalpha = Tj * (FS - (accA + Tfb) * rT);   // accA = B_j here
                        accA = fmaf(w, FS, accA);
                        const float dpower = clamped ? 0.f : __fdividef(w, Tj) * dalpha;  // alpha dalpha
                        const int64_t qe = qn + __popc(fmask & ((1u << lane) - 1u));
                        if (qe < pcap) {
                            a.pr[pbase + qe] = make_uint4(ws->gid[s0 + e], uint32_t(lane), __float_as_uint(dpower),
                                                          __float_as_uint(ws->dDs[lane] * w));
                        } else {
                            raise_error(a.err, kErrPairOverflow, pbase + qe, a.pair_cap);
                        }
                        T = Tj;
                    }
                    qn += __popc(fmask);
                    continue;
                }
                AlphaEval<float> ae;
                ae.pass = false;
                if ((fmask >> lane) & 1u)
                    ae = eval_alpha<float>(ws->rec[e], float(bx + (lane & 7)) + 0.5f, float(by + (lane >> 3)) + 0.5f);
                const unsigned mask = __ballot_sync(0xffffffffu, ae.pass);
                float wv = 0.f;
                if (ae.pass) {
                    const float inv = 1.f / (1.f - ae.alpha);
                    T = T * inv;
                    const float w = ae.alpha * T;
                    const float FS = FSs[e * kTilePitch + lane];
                    accA = last_alpha * lastFS + (1.f - last_alpha) * accA;
                    const float dalpha = (FS - accA) * T - ws->Tf[lane] * inv * ws->bgd[lane];
                    lastFS = FS;
                    last_alpha = ae.alpha;
                    // the pair record for phase B (backward_pairs_kernel)
                    const int64_t qe = qn + __popc(mask & ((1u << lane) - 1u));
                    if (qe < pcap) {
                        const float dpower = ae.clamped ? 0.f : ae.alpha * dalpha;
                        a.pr[pbase + qe] = make_uint4(ws->gid[s0 + e], uint32_t(lane), __float_as_uint(dpower),
                                                      __float_as_uint(ws->dDs[lane] * w));
                    } else {
                        raise_error(a.err, kErrPairOverflow, pbase + qe, a.pair_cap);
                    }
                    wv = w;
                }
                Wb[e * kTilePitch + lane] = wv;
                qn += __popc(mask);
                __syncwarp();
            }
            if (!kRows)
                for (int e = ns; e < kSub; ++e) Wb[e * kTilePitch + lane] = 0.f;
            __syncwarp();
            // (d) GEMM2: dF[ch][e] = sum_px S[px][ch] w_e[px], channels on M.
            // this lane's two events (columns 2 t4, 2 t4 + 1): semantic channel ch
            // lands at sem_base + ch; channels 0..3 (colour, k) are special.
            const uint32_t ge0 = ws->gid[s0 + (2 * t4 < ns ? 2 * t4 : 0)];
            const uint32_t ge1 = ws->gid[s0 + (2 * t4 + 1 < ns ? 2 * t4 + 1 : 0)];
            float* const sem0 = a.g_sem + size_t(ge0) * C - 4;
            float* const sem1 = a.g_sem + size_t(ge1) * C - 4;
            for (int mt = 0; mt < mtiles2; ++mt) {
                float d2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int k0 = 0; k0 < 32; k0 += 8) {
                    const float bf[2] = {Wb[g4 * kTilePitch + k0 + t4], Wb[g4 * kTilePitch + k0 + t4 + 4]};
                    const float* A0 = warp_seed + (k0 + t4) * sp + mt * 16 + g4;
                    const float af[4] = {A0[0], A0[8], A0[4 * sp], A0[4 * sp + 8]};
                    mma_3xtf32(d2, af, bf);
                }
#if K9_RED2
                if ((mt > 0 || K9_RED2_MT0) && a.sem_vec) {
                    // Semantic channels only: pair up channels (c, c + 1) of one event
                    // with the neighbour lane (g4 ^ 1) and issue 8-byte vector reductions.
                    const bool odd = g4 & 1;
                    const int e = 2 * t4 + (odd ? 1 : 0);
                    float* const semE = odd ? sem1 : sem0;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const float mine0 = d2[2 * h], mine1 = d2[2 * h + 1];
                        const float recv = __shfl_xor_sync(0xffffffffu, odd ? mine0 : mine1, 4);
                        const int c = mt * 16 + (g4 & ~1) + 8 * h;  // even channel of the pair
                        const float lo = odd ? recv : mine0, hi = odd ? mine1 : recv;
                        if (c >= 4) {
                            if (c < S && e < ns && (lo != 0.f || hi != 0.f))
                                asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(semE + c), "f"(lo),
                                             "f"(hi)
                                             : "memory");
                        } else {  // colour / k channels (tile 0 only): this lane's own two values
                            const int ch = mt * 16 + g4 + 8 * h;
#pragma unroll
                            for (int q = 0; q < 2; ++q) {
                                const float v = d2[2 * h + q];
                                const uint32_t gg = q ? ge1 : ge0;
                                if (2 * t4 + q < ns && v != 0.f)
                                    atomicAdd(ch < 3 ? a.acc_dcolor + size_t(gg) * 3 + ch : a.g_k + gg, v);
                            }
                        }
                    }
                    continue;
                }
#endif
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int ch = mt * 16 + g4 + 8 * (i >> 1), e = 2 * t4 + (i & 1);
                    if (ch < S && e < ns && d2[i] != 0.f) {
                        const uint32_t gg = (i & 1) ? ge1 : ge0;
                        float* dst = ch >= 4 ? ((i & 1) ? sem1 : sem0) + ch
                                             : (ch < 3 ? a.acc_dcolor + size_t(gg) * 3 + ch : a.g_k + gg);
                        atomicAdd(dst, d2[i]);
                    }
                }
            }
        }
    }
    if (lane == 0) a.pair_n[seg] = uint32_t(qn < pcap ? qn : pcap);
}

// K9 phase B (FP32): one warp per (tile, warp) pair-record segment, the
// geometric terms of every blended pair 32 at a time (flush_records:
// dopacity / dmean2d / dconic and the depth chain as moments, depth_moments),
// reduced per Gaussian inside the warp into the acc16 rows.  Split from phase A
// so that neither carries the other's registers; 5 blocks/SM (48 registers,
// spills hit the large L1 this kernel leaves) hides its gather latency best.
__global__ void __launch_bounds__(256, K9B_MINB) backward_pairs_kernel(const __grid_constant__ BackwardArgs<float> a, int nseg) {
    const int item = int((int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
    if (item >= nseg) return;
    const int seg = a.work_order ? int(a.work_order[item]) : item;
    const uint32_t n = a.pair_n[seg];
    if (n == 0) return;
    const int tile = seg >> 3, w = seg & 7;
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const int bx = tx * kTile + (w & 1) * 8, by = ty * kTile + (w >> 1) * 4;
    const uint4* const rec = a.pr + a.pair_off[seg];
    for (uint32_t k0 = 0; k0 < n; k0 += 32) flush_records(a, rec + k0, int(n - k0 < 32 ? n - k0 : 32), bx, by);
}

// ---------------------------------------------------------------------------
// Longest-first segment order for the backward.  Tile order leaves the last
// wave running a handful of long tiles on an otherwise idle GPU, and a CTA
// holds its shared memory until its slowest warp finishes.  Warp w of CTA b
// instead takes segment order[8 b + w]: CTAs are dispatched in index order, so
// the heaviest segments start first (LPT scheduling) and the eight warps of a
// CTA carry similar work.  The cost is exact here (the forward's per-warp
// event counts).  The forward keeps tile order: its cost proxy (list length)
// is loose, and neighbouring tiles share Gaussian records in L2 (measured:
// ordering made K6 slower, K9 5% faster).
namespace {

constexpr int kOrderThreads = 1024;
constexpr int kOrderBuckets = 1024;

// Bucket of a segment: its event count, heaviest first (counts of 1023 and
// more share bucket 0; a 4K frame's segments stay well below that).
__device__ __forceinline__ uint32_t order_bucket(uint32_t c) {
    return uint32_t(kOrderBuckets - 1) - min(c, uint32_t(kOrderBuckets - 1));
}

// Pass 1: bucket sizes (warp-aggregated global atomics).
__global__ void __launch_bounds__(kOrderThreads) order_hist_kernel(const uint32_t* __restrict__ cost, int nseg,
                                                                   uint32_t* __restrict__ hist) {
    const int i = blockIdx.x * kOrderThreads + threadIdx.x, lane = threadIdx.x & 31;
    const uint32_t b = i < nseg ? order_bucket(cost[i]) : 0xffffffffu;
    const unsigned peers = __match_any_sync(0xffffffffu, b);
    if (b != 0xffffffffu && lane == __ffs(peers) - 1) atomicAdd(&hist[b], __popc(peers));
}

// Pass 2: every CTA scans the 1024 bucket sizes itself (no third launch) and
// scatters its segments to base[b] + a slot from the bucket's global cursor.
__global__ void __launch_bounds__(kOrderThreads) order_scatter_kernel(const uint32_t* __restrict__ cost, int nseg,
                                                                      const uint32_t* __restrict__ hist,
                                                                      uint32_t* __restrict__ cursor,
                                                                      uint32_t* __restrict__ order) {
    __shared__ uint32_t base[kOrderBuckets];
    __shared__ uint32_t wsum[32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int i = blockIdx.x * kOrderThreads + tid;
    const uint32_t b = i < nseg ? order_bucket(cost[i]) : 0xffffffffu;  // issued before the scan
    const uint32_t h = hist[tid];
    uint32_t x = h;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    if (wid == 0) {
        uint32_t v = wsum[lane];
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        wsum[lane] = v;
    }
    __syncthreads();
    base[tid] = x - h + (wid > 0 ? wsum[wid - 1] : 0u);
    __syncthreads();
    const unsigned peers = __match_any_sync(0xffffffffu, b);
    const int leader = __ffs(peers) - 1;
    uint32_t pos = 0;
    if (b != 0xffffffffu && lane == leader) pos = base[b] + atomicAdd(&cursor[b], __popc(peers));
    pos = __shfl_sync(0xffffffffu, pos, leader) + __popc(peers & ((1u << lane) - 1u));
    if (b != 0xffffffffu) order[pos] = uint32_t(i);
}

}  // namespace

void launch_work_order(const uint32_t* seg_cost, int nseg, uint32_t* order, uint32_t* scratch, cudaStream_t s) {
    if (nseg == 0) return;
    cudaMemsetAsync(scratch, 0, 2 * kOrderBuckets * sizeof(uint32_t), s);
    const int blocks = (nseg + kOrderThreads - 1) / kOrderThreads;
    order_hist_kernel<<<blocks, kOrderThreads, 0, s>>>(seg_cost, nseg, scratch);
    order_scatter_kernel<<<blocks, kOrderThreads, 0, s>>>(seg_cost, nseg, scratch, scratch + kOrderBuckets, order);
    count_launches(2);
}


template <typename Real>
void launch_backward_blend(const BackwardArgs<Real>& a, int ntiles, cudaStream_t s) {
    if (ntiles == 0) return;
    static std::atomic<unsigned long long> attr0{0}, attr1{0};  // per instantiation, per device
    opt_in_smem(reinterpret_cast<const void*>(backward_kernel<Real, false>), attr0);
    opt_in_smem(reinterpret_cast<const void*>(backward_kernel<Real, true>), attr1);
    if (a.partial) {
        backward_kernel<Real, true><<<ntiles, kThreads, backward_smem_bytes<Real>(a.C), s>>>(a);
    } else if constexpr (sizeof(Real) == 4) {
        static std::atomic<unsigned long long> attr_tc{0}, attr_rows{0};
        BackwardArgs<float> b = reinterpret_cast<const BackwardArgs<float>&>(a);
        b.nseg = ntiles * 8;
        const unsigned ctas = unsigned((ntiles * 8 + kTcWarps - 1) / kTcWarps);
        if (a.ev_w) {
            opt_in_smem(reinterpret_cast<const void*>(backward_kernel_tc<true>), attr_rows);
            backward_kernel_tc<true><<<ctas, 32 * kTcWarps, backward_tc_smem_bytes(a.C), s>>>(b);
        } else {
            opt_in_smem(reinterpret_cast<const void*>(backward_kernel_tc<false>), attr_tc);
            backward_kernel_tc<false><<<ctas, 32 * kTcWarps, backward_tc_smem_bytes(a.C), s>>>(b);
        }
        backward_pairs_kernel<<<unsigned((ntiles * 8 + 7) / 8), 256, 0, s>>>(a, ntiles * 8);
        count_launches(1);
    } else {
        backward_kernel<Real, false><<<ntiles, kThreads, backward_smem_bytes<Real>(a.C), s>>>(a);
    }
    count_launches(1);
}

namespace {

__global__ void det_keys_kernel(const int64_t* __restrict__ d_count, const uint32_t* __restrict__ sorted_gauss,
                                uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= *d_count) return;
    keys[i] = sorted_gauss[i];
    vals[i] = uint32_t(i);
}

__global__ void det_ranges_kernel(const int64_t* __restrict__ d_count, const uint32_t* __restrict__ gid_sorted,
                                  uint2* __restrict__ range) {
    const int64_t count = *d_count;
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const uint32_t g = gid_sorted[i];
    if (i == 0 || gid_sorted[i - 1] != g) range[g].x = uint32_t(i);
    if (i == count - 1 || gid_sorted[i + 1] != g) range[g].y = uint32_t(i + 1);
}

// One warp per Gaussian, lanes over the V fields; sequential in (instance, warp).
template <typename Real>
__global__ void det_reduce_kernel(const __grid_constant__ BackwardArgs<Real> a, const uint2* __restrict__ range,
                                  const uint32_t* __restrict__ inst_of) {
    const int64_t g = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (g >= a.n) return;
    const uint2 r = range[g];
    if (r.y <= r.x) return;
    const int C = a.C;
    for (int f = lane; f < a.V; f += 32) {
        Real s = Real(0);
        for (uint32_t k = r.x; k < r.y; ++k) {
            const Real* slot = a.partial + size_t(inst_of[k]) * 8 * a.V + f;
#pragma unroll
            for (int w = 0; w < 8; ++w) s += slot[size_t(w) * a.V];
        }
        if (s == Real(0)) continue;
        Real* dst;
        if (f < 16) dst = a.acc16 + g * 16 + f;
        else if (f < 19) dst = a.acc_dcolor + g * 3 + (f - 16);
        else if (f == 19) dst = a.g_k + g;
        else dst = a.g_sem + g * C + (f - 20);
        *dst += s;  // single writer per (Gaussian, field)
    }
}

template <typename Real>
__global__ void zero_det_slots_kernel(Real* __restrict__ partial, const int64_t* __restrict__ d_count, int64_t cap,
                                      int per_item, DeviceError* err) {
    const int64_t count = *d_count;
    if (count > cap) {
        if (blockIdx.x == 0 && threadIdx.x == 0) raise_error(err, kErrPairOverflow, count, cap);
        return;
    }
    const int64_t total = count * per_item;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x)
        partial[i] = Real(0);
}

int bits_for_ids(int64_t v) {
    int b = 1;
    while ((int64_t(1) << b) < v) ++b;
    return b;
}

}  // namespace

template <typename Real>
void launch_deterministic_reduce(const BackwardArgs<Real>& a, const DetScratch& d, const int64_t* d_count,
                                 int64_t count, cudaStream_t s) {
    if (count == 0 || a.n == 0) return;
    const unsigned blocks = unsigned((count + 255) / 256);
    det_keys_kernel<<<blocks, 256, 0, s>>>(d_count, a.inst_gauss, d.keys, d.vals);
    SortScratch sc{d.hist, d.hist_scanned, d.scan_tiles};
    const bool in_b = radix_sort_pairs<uint32_t, 8>(d.keys, d.vals, d.keys_alt, d.vals_alt, d_count, count,
                                                    bits_for_ids(a.n), sc, s);
    const uint32_t* gid_sorted = in_b ? d.keys_alt : d.keys;
    const uint32_t* inst_of = in_b ? d.vals_alt : d.vals;
    cudaMemsetAsync(d.gid_range, 0, sizeof(uint2) * size_t(a.n), s);
    det_ranges_kernel<<<blocks, 256, 0, s>>>(d_count, gid_sorted, d.gid_range);
    det_reduce_kernel<Real><<<unsigned((a.n * 32 + 255) / 256), 256, 0, s>>>(a, d.gid_range, inst_of);
    count_launches(3);
}

template <typename Real>
void launch_zero_det_slots(Real* partial, const int64_t* d_count, int64_t cap, int per_item, DeviceError* err,
                           cudaStream_t s) {
    zero_det_slots_kernel<Real><<<unsigned(device_sm_count() * 8), 256, 0, s>>>(partial, d_count, cap, per_item, err);
    count_launches(1);
}
template void launch_zero_det_slots<float>(float*, const int64_t*, int64_t, int, DeviceError*, cudaStream_t);
template void launch_zero_det_slots<double>(double*, const int64_t*, int64_t, int, DeviceError*, cudaStream_t);

template void launch_deterministic_reduce<float>(const BackwardArgs<float>&, const DetScratch&, const int64_t*,
                                                 int64_t, cudaStream_t);
template void launch_deterministic_reduce<double>(const BackwardArgs<double>&, const DetScratch&, const int64_t*,
                                                  int64_t, cudaStream_t);

template void launch_backward_blend<float>(const BackwardArgs<float>&, int, cudaStream_t);
template void launch_backward_blend<double>(const BackwardArgs<double>&, int, cudaStream_t);

}  // namespace msplat_cuda
