// K6: per-tile forward multimodal blend.  Replaces the tile loop of rasterize
// (core/src/rasterizer.cpp:112-187).
//
// One CTA per 16x16 tile, one thread per pixel; warps own 8x4 pixel blocks.
// The tile's Gaussian list is streamed through shared memory in batches of
// kBatch 48-byte alpha records (coalesced loads, one record per thread).
// Each warp then culls the batch against its 8x4 block with the records'
// conservative alpha-support boxes (8 ballots -> a 256-bit mask) and walks only
// the surviving entries, front to back, exactly as the reference walks the
// list: alpha test, skip below 1/255, ray-ellipsoid midpoint depth (fallback:
// centre depth), blend colour/depth/k, T *= 1-alpha, break after blending once
// T < early_stop_T.  A skipped entry would have failed the alpha test, so the
// result is the reference's.
//
// Semantics (C logits per pixel) accumulate in shared memory rows
// s_O[warp*32+lane][C] (warp-local order).  When a warp blends Gaussian j at
// one or more pixels (ballot), its lanes switch to a channel-parallel update:
// lane ch holds sem_j[ch] and sem_j[ch+32] (one coalesced load each) and adds
// w_L * sem_j[ch] into the row of every blending lane L.  Per pixel the
// additions still happen in list order, like the reference's sem_accum.
#include "blend_common.cuh"
#include "kernels.h"

namespace msplat_cuda {

namespace {

constexpr int kBatch = 256;
constexpr int kThreads = 256;
constexpr int kMaskWords = kBatch / 32;

__host__ __device__ inline int sem_pitch(int C) { return C | 1; }  // odd pitch: conflict-free rows

template <typename Real>
size_t forward_smem_bytes(int C) {
    return sizeof(AlphaRec<Real>) * kBatch + sizeof(uint32_t) * kBatch + sizeof(Real) * 8 * 32 +
           sizeof(Real) * kTilePixels * size_t(C > 0 ? sem_pitch(C) : 0);
}

}  // namespace

template <typename Real>
__global__ void __launch_bounds__(kThreads, 2) forward_kernel(const ForwardArgs<Real> a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    AlphaRec<Real>* s_rec = reinterpret_cast<AlphaRec<Real>*>(smem_raw);
    uint32_t* s_gid = reinterpret_cast<uint32_t*>(s_rec + kBatch);
    Real* s_w = reinterpret_cast<Real*>(s_gid + kBatch);  // [8][32]
    Real* s_O = s_w + 8 * 32;                              // [256][pitch], row = warp*32 + lane

    const int tile = blockIdx.x;
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int x = tx * kTile + tile_pixel_x(warp, lane);
    const int y = ty * kTile + tile_pixel_y(warp, lane);
    const bool inside = x < a.W && y < a.H;
    const int C = a.C, pitch = sem_pitch(C);
    Real* const warp_O = s_O + size_t(warp * 32) * pitch;
    Real* const my_O = warp_O + size_t(lane) * pitch;
    Real* const warp_w = s_w + warp * 32;
    for (int ch = 0; ch < C; ++ch) my_O[ch] = Real(0);

    // The warp's pixel-centre rectangle, for culling.
    const Real rx0 = Real(tx * kTile + (warp & 1) * 8) + Real(0.5), rx1 = rx0 + Real(7);
    const Real ry0 = Real(ty * kTile + (warp >> 1) * 4) + Real(0.5), ry1 = ry0 + Real(3);

    const PixelRay<Real> ray = make_ray<Real>(a.cam, x, y);
    const uint2 range = a.tile_range[tile];

    Real T = Real(1), col0 = 0, col1 = 0, col2 = 0, dep = 0, kk = 0;
    int count = 0, last = 0;
    bool done = !inside;
    const Real early = Real(a.rp.early_stop_T);

    for (uint32_t b0 = range.x; b0 < range.y; b0 += kBatch) {
        const int nb = int(min(uint32_t(kBatch), range.y - b0));
        __syncthreads();
        if (int(threadIdx.x) < nb) {
            const uint32_t g = a.inst_gauss[b0 + threadIdx.x];
            s_gid[threadIdx.x] = g;
            s_rec[threadIdx.x] = a.arec[g];
        }
        __syncthreads();
        if (!__all_sync(0xffffffffu, done)) {
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
            for (int r = 0; r < kMaskWords; ++r) {
                unsigned bits = wm[r];
                while (bits) {
                    const int j = r * 32 + __ffs(bits) - 1;
                    bits &= bits - 1;
                    AlphaEval<Real> ae;
                    ae.pass = false;
                    if (!done) ae = eval_alpha<Real>(s_rec[j], ray.px, ray.py);
                    const unsigned mask = __ballot_sync(0xffffffffu, ae.pass);
                    if (mask == 0) continue;
                    const uint32_t g = s_gid[j];
                    if (ae.pass) {
                        const BlendRec<Real>& br = a.brec[g];
                        const HitEval<Real> h = intersect<Real>(br, ray, a.cam, a.raw, g);
                        const Real d = !h.hit ? br.zc
                                              : (h.depth_fp64 >= Real(0) ? h.depth_fp64
                                                                         : midpoint_depth<Real>(a.cam, ray, h.t_mid));
                        if (!isfinite(ae.alpha) || !isfinite(d)) {
                            raise_error(a.err, kErrNonFiniteBlend, (long long)y * a.W + x, g);
                            done = true;
                        }
                        const Real w = ae.alpha * T;
                        col0 += w * br.rgb[0];
                        col1 += w * br.rgb[1];
                        col2 += w * br.rgb[2];
                        dep += w * d;
                        kk += w * br.k;
                        if (a.weight_sums) atomicAdd(a.weight_sums + g, w);
                        warp_w[lane] = w;
                        T *= (Real(1) - ae.alpha);
                        ++count;
                        last = int(b0 - range.x) + j + 1;
                        if (a.rp.early_termination && T < early) done = true;
                    }
                    if (C > 0) {
                        __syncwarp();
                        const Real* semg = a.semantics + size_t(g) * C;
                        const bool c0 = lane < C, c1 = lane + 32 < C;
                        const Real sv0 = c0 ? semg[lane] : Real(0);
                        const Real sv1 = c1 ? semg[lane + 32] : Real(0);
                        unsigned m = mask;
                        while (m) {
                            const int L = __ffs(m) - 1;
                            m &= m - 1;
                            const Real wL = warp_w[L];
                            Real* row = warp_O + L * pitch;
                            if (c0) row[lane] += wL * sv0;
                            if (c1) row[lane + 32] += wL * sv1;
                        }
                        for (int ch = lane + 64; ch < C; ch += 32) {  // C > 64
                            const Real sv = semg[ch];
                            unsigned m2 = mask;
                            while (m2) {
                                const int L = __ffs(m2) - 1;
                                m2 &= m2 - 1;
                                warp_O[L * pitch + ch] += warp_w[L] * sv;
                            }
                        }
                        __syncwarp();
                    }
                }
            }
        }
        if (__syncthreads_and(done)) break;
    }
    __syncwarp();
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
