// K6: per-tile forward multimodal blend.  Replaces the tile loop of rasterize
// (core/src/rasterizer.cpp:112-187).
//
// One CTA per 16x16 tile, one thread per pixel; warps own 8x4 pixel blocks.
// The tile's Gaussian list is streamed through shared memory in batches of
// kBatch 32-byte alpha records (coalesced 128-bit loads, one record per
// thread).  Every thread walks the batch front to back exactly as the
// reference walks the list: alpha test, skip below 1/255, ray-ellipsoid
// midpoint depth (fallback: centre depth), blend colour/depth/k, T *= 1-alpha,
// break after blending once T < early_stop_T.
//
// Semantics (C logits per pixel) are accumulated in shared memory rows
// s_O[pixel][C] rather than registers, so any C works.  When a warp has
// blended Gaussian j at one or more pixels (ballot), its lanes switch to a
// channel-parallel update: lane ch loads sem_j[ch] once (coalesced) and adds
// w_L * sem_j[ch] into the rows of the blending lanes L.  Per pixel the
// additions still happen in list order, like the reference's sem_accum.
#include "blend_common.cuh"
#include "kernels.h"

namespace msplat_cuda {

namespace {

constexpr int kBatch = 256;
constexpr int kThreads = 256;

__host__ __device__ inline int sem_pitch(int C) { return C | 1; }  // odd pitch: conflict-free rows

template <typename Real>
size_t forward_smem_bytes(int C) {
    return sizeof(AlphaRec<Real>) * kBatch + sizeof(uint32_t) * kBatch + sizeof(Real) * 8 * 32 +
           sizeof(Real) * kTilePixels * size_t(C > 0 ? sem_pitch(C) : 0);
}

}  // namespace

template <typename Real>
__global__ void __launch_bounds__(kThreads) forward_kernel(const ForwardArgs<Real> a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    AlphaRec<Real>* s_rec = reinterpret_cast<AlphaRec<Real>*>(smem_raw);
    uint32_t* s_gid = reinterpret_cast<uint32_t*>(s_rec + kBatch);
    Real* s_w = reinterpret_cast<Real*>(s_gid + kBatch);  // [8][32]
    Real* s_O = s_w + 8 * 32;                              // [256][pitch]

    const int tile = blockIdx.x;
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int x = tx * kTile + tile_pixel_x(warp, lane);
    const int y = ty * kTile + tile_pixel_y(warp, lane);
    const int pl = tile_pixel_index(warp, lane);
    const bool inside = x < a.W && y < a.H;
    const int C = a.C, pitch = sem_pitch(C);
    Real* my_O = s_O + size_t(pl) * pitch;
    for (int ch = 0; ch < C; ++ch) my_O[ch] = Real(0);

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
        for (int j = 0; j < nb; ++j) {
            AlphaEval<Real> ae;
            ae.pass = false;
            if (!done) ae = eval_alpha<Real>(s_rec[j], ray.px, ray.py);
            const unsigned mask = __ballot_sync(0xffffffffu, ae.pass);
            if (mask == 0) continue;
            const uint32_t g = s_gid[j];
            if (ae.pass) {
                const BlendRec<Real> br = a.brec[g];
                const HitEval<Real> h = intersect<Real>(br, ray, a.cam, a.raw, g);
                const Real d = !h.hit ? br.zc
                                      : (h.depth_fp64 >= Real(0) ? h.depth_fp64
                                                                 : midpoint_depth<Real>(a.cam, ray, h.t_mid));
                if (!isfinite(double(ae.alpha)) || !isfinite(double(d))) {
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
                s_w[warp * 32 + lane] = w;
                T *= (Real(1) - ae.alpha);
                ++count;
                last = int(b0 - range.x) + j + 1;
                if (a.rp.early_termination && T < early) done = true;
            }
            if (C > 0) {
                __syncwarp();
                const Real* semg = a.semantics + size_t(g) * C;
                for (int ch = lane; ch < C; ch += 32) {
                    const Real sv = semg[ch];
                    unsigned m = mask;
                    while (m) {
                        const int L = __ffs(m) - 1;
                        m &= m - 1;
                        Real* row = s_O + size_t(tile_pixel_index(warp, L)) * pitch;
                        row[ch] += s_w[warp * 32 + L] * sv;
                    }
                }
                __syncwarp();
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
    if (!isfinite(double(col0)) || !isfinite(double(col1)) || !isfinite(double(col2)) ||
        !isfinite(double(dep)) || !isfinite(double(T)))
        raise_error(a.err, kErrNonFiniteOutput, (long long)p, -1);
}

template <typename Real>
void launch_forward(const ForwardArgs<Real>& a, int ntiles, cudaStream_t s) {
    if (ntiles == 0) return;
    const size_t smem = forward_smem_bytes<Real>(a.C);
    static bool configured = false;  // per instantiation
    if (!configured) {
        cudaFuncSetAttribute(forward_kernel<Real>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             227 * 1024);
        configured = true;
    }
    forward_kernel<Real><<<ntiles, kThreads, smem, s>>>(a);
    count_launches(1);
}

template void launch_forward<float>(const ForwardArgs<float>&, int, cudaStream_t);
template void launch_forward<double>(const ForwardArgs<double>&, int, cudaStream_t);

}  // namespace msplat_cuda
