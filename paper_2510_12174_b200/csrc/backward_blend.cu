// K9: per-tile reverse blend -- rasterize_backward's tile loop
// (core/src/rasterizer_backward.cpp:140-255) with intersection_backward
// (core/src/geometry.cpp:70-105) and quat_rotation_backward (:17-29).
//
// One CTA per 16x16 tile, one thread per pixel, warps own 8x4 pixel blocks.
// Each pixel replays its list from terminus-1 down to 0 with the forward's
// alpha test (same code, same decisions), restores T by division, and forms
// the reference's per-pair gradients.  As in K6, each warp culls every batch
// with the alpha-support boxes and walks only surviving entries (now back to
// front).
//
// dalpha without per-channel accumulators.  With the per-pair feature vector
// F_j = [rgb, k, sem] and the pixel seed s_p = [dC, dK, dO], the reference's
//   dalpha = (rgb - acc_c).dC T + (k - acc_k) dK T + sum_ch (sem - acc_s).dO T - bg term
// equals (F_j.s_p - A) T - bg term, where A = acc_c.dC + acc_k dK + acc_s.dO
// obeys the same linear recursion A <- a_last (F_last.s_p) + (1 - a_last) A
// (rasterizer_backward.cpp:222-231).  F_j is staged once per (warp, Gaussian)
// event in shared memory and dotted with the pixel's seed row (128-bit LDS).
//
// Reductions, fused into one loop over the blending lanes L of an event:
//   * seed-linear gradients (dcolor, dk, dsem = w_L * s_L): channel-parallel,
//     lane ch accumulates w_L * s_L[ch] and w_L * s_L[ch+32];
//   * 16 geometric gradients (dopacity, dmean2d, dconic, depth-chain
//     dposition / drotation / dscale): each blending lane wrote them to its
//     shared scratch row; lane i < 16 sums column i;
// then one atomic per non-zero value.  O(active lanes) per event, no shuffle
// trees.
#include "blend_common.cuh"
#include "kernels.h"

namespace msplat_cuda {

namespace {

constexpr int kBatch = 256;
constexpr int kThreads = 256;
constexpr int kMaskWords = kBatch / 32;
constexpr int kGeo = 16;             // geometric values per pair
constexpr int kRedPitch = kGeo + 1;  // + w; odd pitch

// Seed rows [dC0 dC1 dC2 dK dO...]: multiple of 4 (128-bit loads) with an odd
// number of 16-byte units per row (conflict-free when every lane reads its own row).
__host__ __device__ inline int seed_pitch(int C) {
    int p = ((C + 4 + 3) / 4) * 4;
    if (((p / 4) & 1) == 0) p += 4;
    return p;
}

template <typename Real>
size_t backward_smem_bytes(int C) {
    const int sp = seed_pitch(C);
    return sizeof(AlphaRec<Real>) * kBatch + sizeof(uint32_t) * kBatch + sizeof(Real) * size_t(kTilePixels) * sp +
           sizeof(Real) * 8 * 32 * kRedPitch + sizeof(Real) * 8 * sp + 16;
}

template <typename Real>
__device__ __forceinline__ Real dot_rows(const Real* a, const Real* b, int n) {
    Real s = Real(0);
    if constexpr (sizeof(Real) == 4) {
        const float4* a4 = reinterpret_cast<const float4*>(a);
        const float4* b4 = reinterpret_cast<const float4*>(b);
        for (int i = 0; i < n / 4; ++i) {
            const float4 x = a4[i], y = b4[i];
            s += x.x * y.x + x.y * y.y + x.z * y.z + x.w * y.w;
        }
    } else {
        for (int i = 0; i < n; ++i) s += a[i] * b[i];
    }
    return s;
}

}  // namespace

template <typename Real>
__global__ void __launch_bounds__(kThreads, 2) backward_kernel(const BackwardArgs<Real> a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int C = a.C, sp = seed_pitch(C), S = C + 4;
    AlphaRec<Real>* s_rec = reinterpret_cast<AlphaRec<Real>*>(smem_raw);
    Real* s_seed = reinterpret_cast<Real*>(s_rec + kBatch);          // [256][sp], row = warp*32 + lane
    Real* s_red = s_seed + size_t(kTilePixels) * sp;                  // [8][32][kRedPitch]
    Real* s_F = s_red + 8 * 32 * kRedPitch;                           // [8][sp] staged F_j per warp
    uint32_t* s_gid = reinterpret_cast<uint32_t*>(s_F + 8 * sp);
    int* s_maxterm = reinterpret_cast<int*>(s_gid + kBatch);

    const int tile = blockIdx.x;
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int x = tx * kTile + tile_pixel_x(warp, lane);
    const int y = ty * kTile + tile_pixel_y(warp, lane);
    const bool inside = x < a.W && y < a.H;
    const size_t HW = size_t(a.W) * a.H, p = size_t(y) * a.W + x;
    if (threadIdx.x == 0) *s_maxterm = 0;

    Real* const warp_seed = s_seed + size_t(warp * 32) * sp;
    Real* const my_seed = warp_seed + size_t(lane) * sp;
    Real* const warp_red = s_red + size_t(warp * 32) * kRedPitch;
    Real* const my_red = warp_red + lane * kRedPitch;
    Real* const warp_F = s_F + warp * sp;
    for (int i = lane; i < sp; i += 32) warp_F[i] = Real(0);

    // Per-pixel seeds into shared memory (dD, T_final, terminus in registers).
    int term = 0;
    Real T_final = Real(1), dD = Real(0);
    bool any = false;
    for (int ch = 0; ch < sp; ++ch) my_seed[ch] = Real(0);
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
    __syncthreads();
    if (term > 0) atomicMax(s_maxterm, term);
    __syncthreads();
    const int maxterm = *s_maxterm;
    if (maxterm == 0) return;

    const PixelRay<Real> ray = make_ray<Real>(a.cam, x, y);
    const Real bg_dot = Real(a.rp.bg[0]) * my_seed[0] + Real(a.rp.bg[1]) * my_seed[1] + Real(a.rp.bg[2]) * my_seed[2];
    const Real sigma = Real(a.rp.sigma_scale);
    Real T = T_final;
    Real accA = 0, lastFS = 0, last_alpha = 0;

    const Real rx0 = Real(tx * kTile + (warp & 1) * 8) + Real(0.5), rx1 = rx0 + Real(7);
    const Real ry0 = Real(ty * kTile + (warp >> 1) * 4) + Real(0.5), ry1 = ry0 + Real(3);

    const uint2 range = a.tile_range[tile];
    const uint32_t list_end = range.x + uint32_t(maxterm);
    for (int64_t bend = int64_t(list_end); bend > int64_t(range.x); bend -= kBatch) {
        const uint32_t bstart = uint32_t(max(int64_t(range.x), bend - kBatch));
        const int nb = int(uint32_t(bend) - bstart);
        const int pos0 = int(bstart - range.x);
        __syncthreads();
        if (int(threadIdx.x) < nb) {
            const uint32_t g = a.inst_gauss[bstart + threadIdx.x];
            s_gid[threadIdx.x] = g;
            s_rec[threadIdx.x] = a.arec[g];
        }
        __syncthreads();
        if (!__any_sync(0xffffffffu, term > pos0)) continue;
        uint32_t wm[kMaskWords];
#pragma unroll
        for (int r = 0; r < kMaskWords; ++r) {
            const int i = r * 32 + lane;
            bool hit = false;
            if (i < nb) {
                const AlphaRec<Real>& g = s_rec[i];
                hit = !(g.bx1 < rx0 || g.bx0 > rx1 || g.by1 < ry0 || g.by0 > ry1);
            }
            wm[r] = __ballot_sync(0xffffffffu, hit);
        }
#pragma unroll
        for (int r = kMaskWords - 1; r >= 0; --r) {
            unsigned bits = wm[r];
            while (bits) {
                const int bit = 31 - __clz(bits);
                bits &= ~(1u << bit);
                const int j = r * 32 + bit;
                AlphaEval<Real> ae;
                ae.pass = false;
                if (pos0 + j < term) ae = eval_alpha<Real>(s_rec[j], ray.px, ray.py);
                const unsigned mask = __ballot_sync(0xffffffffu, ae.pass);
                if (mask == 0) continue;
                const uint32_t g = s_gid[j];
                const BlendRec<Real>& br = a.brec[g];
                // Stage F_j = [rgb, k, sem] for the dot products.
                if (lane < 3) warp_F[lane] = br.rgb[lane];
                else if (lane == 3) warp_F[3] = br.k;
                {
                    const Real* semg = a.semantics + size_t(g) * C;
                    for (int ch = lane; ch < C; ch += 32) warp_F[4 + ch] = semg[ch];
                }
                __syncwarp();
                if (ae.pass) {
                    Real v[kRedPitch];
#pragma unroll
                    for (int i = 0; i < kRedPitch; ++i) v[i] = Real(0);
                    T = T / (Real(1) - ae.alpha);
                    const Real w = ae.alpha * T;
                    v[kGeo] = w;
                    // Depth chain (rasterizer_backward.cpp:205-218).
                    const Real dd = dD * w;
                    if (dd != Real(0)) {
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
                                        v[6 + i] = kk * (br.Rt[0 * 3 + i] * ga[0] + br.Rt[1 * 3 + i] * ga[1] +
                                                         br.Rt[2 * 3 + i] * ga[2]);
                                        Rp[i] = br.Rt[0 * 3 + i] * pl[0] + br.Rt[1 * 3 + i] * pl[1] +
                                                br.Rt[2 * 3 + i] * pl[2];
                                    }
                                    Real G[9];
#pragma unroll
                                    for (int rr = 0; rr < 3; ++rr)
#pragma unroll
                                        for (int cc = 0; cc < 3; ++cc)
                                            G[rr * 3 + cc] = -kk * (Rp[rr] * ga[cc] + ray.d[rr] * gb[cc]);
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
                                    v[6 + i] = -(br.Rt[0 * 3 + i] * gvl[0] + br.Rt[1 * 3 + i] * gvl[1] +
                                                 br.Rt[2 * 3 + i] * gvl[2]);
                                    vv[i] = br.Rt[0 * 3 + i] * br.vl[0] + br.Rt[1 * 3 + i] * br.vl[1] +
                                            br.Rt[2 * 3 + i] * br.vl[2];
                                }
                                Real G[9];
#pragma unroll
                                for (int rr = 0; rr < 3; ++rr)
#pragma unroll
                                    for (int cc = 0; cc < 3; ++cc)
                                        G[rr * 3 + cc] = vv[rr] * gvl[cc] + ray.d[rr] * gdl[cc];
                                quat_rotation_backward<Real>(br.q, G, v + 9);
                            }
                        } else {
#pragma unroll
                            for (int i = 0; i < 3; ++i) v[6 + i] = dd * Real(a.cam.Rw2c[6 + i]);
                        }
                    }
                    // Alpha gradient (rasterizer_backward.cpp:222-244); depth excluded.
                    const Real FS = dot_rows<Real>(warp_F, my_seed, sp);
                    accA = last_alpha * lastFS + (Real(1) - last_alpha) * accA;
                    const Real dalpha = (FS - accA) * T - (T_final / (Real(1) - ae.alpha)) * bg_dot;
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
                    lastFS = FS;
                    last_alpha = ae.alpha;
#pragma unroll
                    for (int i = 0; i < kRedPitch; ++i) my_red[i] = v[i];
                }
                __syncwarp();
                // Fused reductions over the blending lanes.
                Real acc0 = Real(0), acc1 = Real(0), geo = Real(0);
                const int gl = lane & (kGeo - 1);
                const int c1 = lane + 32 < sp ? lane + 32 : lane;  // clamp: acc1 unused then
                unsigned m = mask;
                while (m) {
                    const int L = __ffs(m) - 1;
                    m &= m - 1;
                    const Real* redL = warp_red + L * kRedPitch;
                    const Real* seedL = warp_seed + L * sp;
                    const Real wL = redL[kGeo];
                    acc0 += wL * seedL[lane];
                    acc1 += wL * seedL[c1];
                    geo += redL[gl];
                }
                if (lane < kGeo && geo != Real(0)) {
                    Real* dst;
                    if (lane == 0) dst = a.g_opac + g;
                    else if (lane < 3) dst = a.acc_dmean + size_t(g) * 2 + (lane - 1);
                    else if (lane < 6) dst = a.acc_dconic + size_t(g) * 3 + (lane - 3);
                    else if (lane < 9) dst = a.g_pos + size_t(g) * 3 + (lane - 6);
                    else if (lane < 13) dst = a.g_rot + size_t(g) * 4 + (lane - 9);
                    else dst = a.g_scale + size_t(g) * 3 + (lane - 13);
                    atomicAdd(dst, geo);
                }
                if (lane < S && acc0 != Real(0)) {
                    Real* dst = lane < 3 ? a.acc_dcolor + size_t(g) * 3 + lane
                                         : (lane == 3 ? a.g_k + g : a.g_sem + size_t(g) * C + (lane - 4));
                    atomicAdd(dst, acc0);
                }
                if (lane + 32 < S && acc1 != Real(0)) atomicAdd(a.g_sem + size_t(g) * C + (lane + 28), acc1);
                for (int ch = lane + 64; ch < S; ch += 32) {  // C > 60
                    Real s = Real(0);
                    unsigned m2 = mask;
                    while (m2) {
                        const int L = __ffs(m2) - 1;
                        m2 &= m2 - 1;
                        s += warp_red[L * kRedPitch + kGeo] * warp_seed[L * sp + ch];
                    }
                    if (s != Real(0)) atomicAdd(a.g_sem + size_t(g) * C + (ch - 4), s);
                }
                __syncwarp();
            }
        }
    }
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

template void launch_backward_blend<float>(const BackwardArgs<float>&, int, cudaStream_t);
template void launch_backward_blend<double>(const BackwardArgs<double>&, int, cudaStream_t);

}  // namespace msplat_cuda
