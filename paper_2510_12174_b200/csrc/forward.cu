// K6: per-tile forward multimodal blend.  Replaces the tile loop of rasterize
// (core/src/rasterizer.cpp:112-187).
//
// One CTA per 16x16 tile, one thread per pixel; warps own 8x4 pixel blocks and
// run INDEPENDENTLY (no block barrier): each warp streams the tile list front
// to back in 32-entry chunks, culls each chunk against its block with the
// conservative alpha-support boxes (one ballot), and walks the surviving
// entries exactly as the reference walks the list: alpha test, skip below
// 1/255, blend, T *= 1-alpha, break after blending once T < early_stop_T.  A
// culled entry would have failed the alpha test, so results are the
// reference's.
//
// Phase A (per (warp, Gaussian) event, sequential per pixel): alpha, w = alpha T,
//   colour / k accumulation, T update, contributor count and terminus; the
//   semantic logits accumulate channel-parallel into shared rows
//   s_O[lane][C] (lane ch adds w_L * sem_j[ch] for each blending lane L, in
//   list order per pixel).  Each blended pair is enqueued (pixel, Gaussian, w).
// Phase B (flush, 32 pairs per warp vector): the ray-ellipsoid midpoint depth
//   (fallback: centre depth) of every queued pair with all lanes busy, and
//   w * depth added to the owning pixel's depth sum.
#include "blend_common.cuh"
#include "kernels.h"

namespace msplat_cuda {

namespace {

constexpr int kThreads = 256;
constexpr int kQueue = 64;

__host__ __device__ inline int sem_pitch(int C) { return C | 1; }  // odd pitch: conflict-free rows

template <typename Real>
struct FwdWarpSmem {
    AlphaRec<Real> rec[32];
    uint32_t gid[32];
    uint32_t q_lane[kQueue];
    uint32_t q_gid[kQueue];
    Real q_w[kQueue];
    Real q_wd[kQueue];
};

template <typename Real>
size_t forward_smem_bytes(int C) {
    return 8 * (sizeof(FwdWarpSmem<Real>) + sizeof(Real) * 32 * size_t(C > 0 ? sem_pitch(C) : 0)) + 64;
}

// Phase B on the first n queue entries (n <= 32).  `own` has bit e set when
// queue entry e belongs to this lane's pixel.
template <typename Real>
__device__ __forceinline__ void flush_depth(const ForwardArgs<Real>& a, FwdWarpSmem<Real>* ws, int n, int bx, int by,
                                         Real& dep, unsigned own) {
    const int lane = threadIdx.x & 31;
    if (lane < n) {
        const int L = int(ws->q_lane[lane]);
        const uint32_t g = ws->q_gid[lane];
        const BlendRec<Real>& br = a.brec[g];
        const int xL = bx + (L & 7), yL = by + (L >> 3);
        const PixelRay<Real> ray = make_ray<Real>(a.cam, xL, yL);
        const HitEval<Real> h = intersect<Real>(br, ray, a.cam, a.raw, g);
        const Real d = !h.hit ? br.zc
                              : (h.depth_fp64 >= Real(0) ? h.depth_fp64 : midpoint_depth<Real>(a.cam, ray, h.t_mid));
        if (!isfinite(d)) raise_error(a.err, kErrNonFiniteBlend, (long long)yL * a.W + xL, g);
        ws->q_wd[lane] = ws->q_w[lane] * d;
    }
    __syncwarp();
    while (own) {  // this pixel's entries, in queue (= list) order
        const int e = __ffs(own) - 1;
        own &= own - 1;
        dep += ws->q_wd[e];
    }
    __syncwarp();
}

}  // namespace

template <typename Real>
__global__ void __launch_bounds__(kThreads, 2) forward_kernel(const __grid_constant__ ForwardArgs<Real> a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int C = a.C, pitch = sem_pitch(C);
    FwdWarpSmem<Real>* ws = reinterpret_cast<FwdWarpSmem<Real>*>(smem_raw) + warp;
    Real* const warp_O = reinterpret_cast<Real*>(reinterpret_cast<FwdWarpSmem<Real>*>(smem_raw) + 8) +
                         size_t(warp) * 32 * pitch;
    Real* const my_O = warp_O + size_t(lane) * pitch;
    for (int ch = 0; ch < C; ++ch) my_O[ch] = Real(0);

    const int tile = blockIdx.x;
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const int bx = tx * kTile + (warp & 1) * 8, by = ty * kTile + (warp >> 1) * 4;
    const int x = bx + (lane & 7), y = by + (lane >> 3);
    const bool inside = x < a.W && y < a.H;
    const Real pxf = Real(x) + Real(0.5), pyf = Real(y) + Real(0.5);
    const Real rx0 = Real(bx) + Real(0.5), rx1 = rx0 + Real(7);
    const Real ry0 = Real(by) + Real(0.5), ry1 = ry0 + Real(3);
    const uint2 range = a.tile_range[tile];
    const int len = int(range.y - range.x);

    Real T = Real(1), col0 = 0, col1 = 0, col2 = 0, dep = 0, kk = 0;
    int count = 0, last = 0;
    bool done = !inside;
    const Real early = Real(a.rp.early_stop_T);
    const bool c0 = lane < C, c1 = lane + 32 < C;
    int qn = 0;
    unsigned long long own = 0;  // queue entries owned by this pixel
    uint2* const evl = a.ev_list ? a.ev_list + size_t(8) * range.x + size_t(warp) * len : nullptr;
    uint32_t n_ev = 0, n_pairs = 0;

    for (int c = 0; c * 32 < len; ++c) {
        if (__all_sync(0xffffffffu, done)) break;
        const int pos = c * 32 + lane;
        bool hit = false;
        if (pos < len) {
            const uint32_t g = a.inst_gauss[range.x + pos];
            const AlphaRec<Real> r = a.arec[g];
            ws->rec[lane] = r;
            ws->gid[lane] = g;
            hit = !(r.bx1 < rx0 || r.bx0 > rx1 || r.by1 < ry0 || r.by0 > ry1);
            if (hit) asm volatile("prefetch.global.L1 [%0];" ::"l"(reinterpret_cast<const char*>(a.brec + g)));
        }
        unsigned bits = __ballot_sync(0xffffffffu, hit);
        __syncwarp();
        while (bits) {
            const int slot = __ffs(bits) - 1;
            bits &= bits - 1;
            AlphaEval<Real> ae;
            ae.pass = false;
            if (!done) ae = eval_alpha<Real>(ws->rec[slot], pxf, pyf);
            const unsigned mask = __ballot_sync(0xffffffffu, ae.pass);
            if (mask == 0) continue;
            if (evl) {  // the backward replays exactly these events
                if (lane == 0) evl[n_ev] = make_uint2(uint32_t(c * 32 + slot), mask);
                ++n_ev;
                n_pairs += __popc(mask);
            }
            const uint32_t g = ws->gid[slot];
            if (ae.pass) {
                if (!isfinite(ae.alpha)) {
                    raise_error(a.err, kErrNonFiniteBlend, (long long)y * a.W + x, g);
                    done = true;
                }
                const AlphaRec<Real>& br = ws->rec[slot];
                const Real w = ae.alpha * T;
                col0 += w * br.rgb[0];
                col1 += w * br.rgb[1];
                col2 += w * br.rgb[2];
                kk += w * br.k;
                if (a.weight_sums) atomicAdd(a.weight_sums + g, w);
                const int e = qn + __popc(mask & ((1u << lane) - 1u));
                own |= 1ull << e;
                ws->q_lane[e] = uint32_t(lane);
                ws->q_gid[e] = g;
                ws->q_w[e] = w;
                T *= (Real(1) - ae.alpha);
                ++count;
                last = c * 32 + slot + 1;
                if (a.rp.early_termination && T < early) done = true;
            }
            __syncwarp();
            const int npairs = __popc(mask);
            if (C > 0) {  // semantic logits, channel-parallel, list order per pixel
                const Real* semg = a.semantics + size_t(g) * C;
                const Real sv0 = c0 ? semg[lane] : Real(0);
                const Real sv1 = c1 ? semg[lane + 32] : Real(0);
                // The event's rows are distinct pixels: batch the loads before the
                // stores so the shared-memory round trips overlap.
                const int cc0 = c0 ? lane : 0, cc1 = c1 ? lane + 32 : 0;
                int e = qn;
                for (; e + 4 <= qn + npairs; e += 4) {
                    Real* r0 = warp_O + int(ws->q_lane[e]) * pitch;
                    Real* r1 = warp_O + int(ws->q_lane[e + 1]) * pitch;
                    Real* r2 = warp_O + int(ws->q_lane[e + 2]) * pitch;
                    Real* r3 = warp_O + int(ws->q_lane[e + 3]) * pitch;
                    const Real w0 = ws->q_w[e], w1 = ws->q_w[e + 1], w2 = ws->q_w[e + 2], w3 = ws->q_w[e + 3];
                    const Real a0 = r0[cc0], a1 = r1[cc0], a2 = r2[cc0], a3 = r3[cc0];
                    const Real b0 = r0[cc1], b1 = r1[cc1], b2 = r2[cc1], b3 = r3[cc1];
                    if (c0) {
                        r0[lane] = a0 + w0 * sv0;
                        r1[lane] = a1 + w1 * sv0;
                        r2[lane] = a2 + w2 * sv0;
                        r3[lane] = a3 + w3 * sv0;
                    }
                    if (c1) {
                        r0[lane + 32] = b0 + w0 * sv1;
                        r1[lane + 32] = b1 + w1 * sv1;
                        r2[lane + 32] = b2 + w2 * sv1;
                        r3[lane + 32] = b3 + w3 * sv1;
                    }
                }
                for (; e < qn + npairs; ++e) {
                    const Real wL = ws->q_w[e];
                    Real* row = warp_O + int(ws->q_lane[e]) * pitch;
                    if (c0) row[lane] += wL * sv0;
                    if (c1) row[lane + 32] += wL * sv1;
                }
                for (int ch = lane + 64; ch < C; ch += 32) {  // C > 64
                    const Real sv = semg[ch];
                    for (int e = qn; e < qn + npairs; ++e) warp_O[int(ws->q_lane[e]) * pitch + ch] += ws->q_w[e] * sv;
                }
                __syncwarp();
            }
            qn += npairs;
            if (qn >= 32) {
                flush_depth<Real>(a, ws, 32, bx, by, dep, unsigned(own));
                own >>= 32;
                const int rest = qn - 32;
                if (lane < rest) {  // reads >= 32, writes < 32
                    ws->q_lane[lane] = ws->q_lane[32 + lane];
                    ws->q_gid[lane] = ws->q_gid[32 + lane];
                    ws->q_w[lane] = ws->q_w[32 + lane];
                }
                qn = rest;
                __syncwarp();
            }
        }
    }
    if (qn > 0) flush_depth<Real>(a, ws, qn, bx, by, dep, unsigned(own));
    if (a.ev_count && lane == 0) {
        a.ev_count[size_t(tile) * 8 + warp] = n_ev;
        a.ev_npairs[size_t(tile) * 8 + warp] = n_pairs;
    }
    if (!inside) return;
    col0 += T * Real(a.rp.bg[0]);
    col1 += T * Real(a.rp.bg[1]);
    col2 += T * Real(a.rp.bg[2]);
    const size_t HW = size_t(a.W) * a.H, p = size_t(y) * a.W + x;
    if (a.color) {
        a.color[p] = col0;
        a.color[HW + p] = col1;
        a.color[2 * HW + p] = col2;
    }
    if (a.depth) a.depth[p] = dep;
    if (a.kmap) a.kmap[p] = kk;
    a.T[p] = T;
    if (a.contributors) a.contributors[p] = count;
    if (a.terminus) a.terminus[p] = last;
    if (a.sem_out)
        for (int ch = 0; ch < C; ++ch) a.sem_out[size_t(ch) * HW + p] = my_O[ch];
    if (!isfinite(col0) || !isfinite(col1) || !isfinite(col2) || !isfinite(dep) || !isfinite(T))
        raise_error(a.err, kErrNonFiniteOutput, (long long)p, -1);
}

template <typename Real>
void launch_forward(const ForwardArgs<Real>& a, int ntiles, cudaStream_t s) {
    if (ntiles == 0) return;
    const size_t smem = forward_smem_bytes<Real>(a.C);
    static bool configured = false;  // per instantiation
    if (!configured) {
        cudaFuncSetAttribute(forward_kernel<Real>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        configured = true;
    }
    forward_kernel<Real><<<ntiles, kThreads, smem, s>>>(a);
    count_launches(1);
}

template void launch_forward<float>(const ForwardArgs<float>&, int, cudaStream_t);
template void launch_forward<double>(const ForwardArgs<double>&, int, cudaStream_t);

}  // namespace msplat_cuda
