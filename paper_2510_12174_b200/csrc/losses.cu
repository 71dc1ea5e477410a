// K12: frame losses and gradient-seed assembly on the device -- the step on
// either side of the backward:
//   evaluate_frame_losses (core/src/trainer.cpp:171-264) over
//   l1_rgb, ssim_loss, depth_l1, normal_cosine, cross_entropy_seg,
//   gradient_factor_loss and combine (core/src/losses.cpp:87-313).
//
// Sequence (all on the context stream, no host round trip, graph-capturable):
//   1. loss_pixel_kernel   per pixel: |x - t| (rgb), masked |D - gt| and N.gt,
//                          softmax cross-entropy, |K - 1|; block-reduced into
//                          double accumulators (sums and masked counts);
//   2. ssim_fwd_kernel     per valid window centre and channel: the five
//                          windowed moments, SSIM and its three moment
//                          adjoints (losses.cpp:120-146); 32 x 8 tiles, the
//                          horizontal 11-tap sums shared through shared memory;
//   3. ssim_bwd_kernel     per pixel: the adjoint of the valid correlation
//                          (losses.cpp:61-83, 148-156), tiled the same way;
//   4. combine_kernel      one thread: the values, magnitude ratios and seed
//                          scales of combine() (losses.cpp:285-313);
//   5. assemble_kernel     per pixel: the seeded pixel gradients
//                          (trainer.cpp:229-256) and the seeded normal-loss
//                          gradient, which the caller pushes through the
//                          normals backward into ddepth (trainer.cpp:258-262).
#include "common.cuh"
#include "kernels.h"

namespace msplat_cuda {

namespace {

constexpr int kThreadsL = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Adds v[0..N) of every thread of the block into acc[0..N) (one atomic each).
template <int N>
__device__ __forceinline__ void block_accumulate(double (&v)[N], double* acc) {
    __shared__ double part[N][kThreadsL / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const double s = warp_sum(v[i]);
        if (lane == 0) part[i][warp] = s;
    }
    __syncthreads();
    if (threadIdx.x < N) {
        double s = 0;
        for (int w = 0; w < kThreadsL / 32; ++w) s += part[threadIdx.x][w];
        if (s != 0) atomicAdd(acc + threadIdx.x, s);
    }
}

template <typename Real>
__device__ __forceinline__ Real sign_of(Real v) {
    return v > Real(0) ? Real(1) : (v < Real(0) ? Real(-1) : Real(0));
}

template <typename Real>
__device__ __forceinline__ bool normal_supervised(const LossArgs<Real>& a, size_t p, size_t HW) {
    // nstate.valid (a unit normal was written) and a non-zero ground truth
    // (trainer.cpp:198-205)
    const bool valid = a.normals[p] != Real(0) || a.normals[HW + p] != Real(0) || a.normals[2 * HW + p] != Real(0);
    const bool gt_ok =
        a.gt_normal[p] != Real(0) || a.gt_normal[HW + p] != Real(0) || a.gt_normal[2 * HW + p] != Real(0);
    return valid && gt_ok;
}

// Softmax cross-entropy of one pixel; writes the probability normaliser.
template <typename Real>
__device__ __forceinline__ Real ce_pixel(const LossArgs<Real>& a, size_t p, size_t HW, int label, Real& maxl, Real& z) {
    const Real* __restrict__ sem = a.sem + p;
    maxl = sem[0];
    for (int c = 1; c < a.C; ++c) maxl = sem[size_t(c) * HW] > maxl ? sem[size_t(c) * HW] : maxl;
    z = Real(0);
    for (int c = 0; c < a.C; ++c) z += exp(sem[size_t(c) * HW] - maxl);
    return log(z) - (sem[size_t(label) * HW] - maxl);
}

// acc: 0 l1 sum, 1 ssim sum, 2 depth sum, 3 depth count, 4 normal dot sum,
//      5 normal count, 6 cross-entropy sum, 7 |K-1| sum
template <typename Real>
__global__ void __launch_bounds__(kThreadsL) loss_pixel_kernel(const __grid_constant__ LossArgs<Real> a) {
    const size_t HW = size_t(a.W) * a.H;
    double v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (size_t p = size_t(blockIdx.x) * blockDim.x + threadIdx.x; p < HW; p += size_t(gridDim.x) * blockDim.x) {
        if (a.en[0])
            for (int c = 0; c < 3; ++c) v[0] += double(fabs(a.color[c * HW + p] - a.gt_rgb[c * HW + p]));
        if (a.en[3] && a.gt_depth[p] > Real(0)) {
            v[2] += double(fabs(a.depth[p] - a.gt_depth[p]));
            v[3] += 1;
        }
        if (a.en[2] && normal_supervised(a, p, HW)) {
            for (int c = 0; c < 3; ++c) v[4] += double(a.normals[c * HW + p] * a.gt_normal[c * HW + p]);
            v[5] += 1;
        }
        if (a.en[4]) {
            const int label = a.labels[p];
            if (label >= a.C) {
                raise_error(a.err, kErrLabelRange, (long long)p, label);
            } else {
                Real maxl, z;
                v[6] += double(ce_pixel(a, p, HW, label, maxl, z));
                if (a.ce_stats) {  // the seed assembly's softmax reuses them
                    a.ce_stats[p] = maxl;
                    a.ce_stats[HW + p] = z;
                }
            }
        }
        if (a.en[5]) v[7] += double(fabs(a.kmap[p] - Real(1)));
    }
    block_accumulate<8>(v, a.acc);
}

// SSIM tiles: a CTA covers kSsimTX x kSsimTY outputs of one channel (blockIdx.y).
// The 11-tap horizontal sums of the tile's rows are computed once into shared
// memory and shared by the 11 vertical taps of each output, with every output
// summed in the reference's order (losses.cpp:39-58: along x, i = 0..10, then
// along y, j = 0..10) -- the same operations as one output at a time.
constexpr int kSsimTX = 32, kSsimTY = 8, kSsimRows = kSsimTY + 10, kSsimCols = kSsimTX + 10;
static_assert(kSsimTX * kSsimTY == kThreadsL, "one output per thread");

__host__ __device__ inline int ssim_tiles_x(int w) { return (w + kSsimTX - 1) / kSsimTX; }
__host__ __device__ inline int ssim_tiles_y(int h) { return (h + kSsimTY - 1) / kSsimTY; }

// Windowed moments of the valid windows (vx, vy) in [0, W - 10) x [0, H - 10)
// (window rows vy..vy+10, columns vx..vx+10).
template <typename Real>
__global__ void __launch_bounds__(kThreadsL) ssim_fwd_kernel(const __grid_constant__ LossArgs<Real> a) {
    __shared__ Real sx[kSsimRows][kSsimCols], sy[kSsimRows][kSsimCols];
    __shared__ Real hs[5][kSsimRows][kSsimTX];
    const int W = a.W, H = a.H, Wv = W - 10, Hv = H - 10;
    const size_t HW = size_t(W) * H, nv = size_t(Wv) * Hv;
    const int c = blockIdx.y;
    const int tiles_x = ssim_tiles_x(Wv);
    const int bx = int(blockIdx.x % unsigned(tiles_x)) * kSsimTX, by = int(blockIdx.x / unsigned(tiles_x)) * kSsimTY;
    const Real* X = a.color + c * HW;
    const Real* Y = a.gt_rgb + c * HW;
    for (int e = threadIdx.x; e < kSsimRows * kSsimCols; e += kThreadsL) {
        const int r = e / kSsimCols, q = e - r * kSsimCols, gy = by + r, gx = bx + q;
        const bool in = gy < H && gx < W;
        sx[r][q] = in ? X[size_t(gy) * W + gx] : Real(0);
        sy[r][q] = in ? Y[size_t(gy) * W + gx] : Real(0);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < kSsimRows * kSsimTX; e += kThreadsL) {
        const int r = e / kSsimTX, q = e - r * kSsimTX;
        Real hx = 0, hy = 0, hx2 = 0, hy2 = 0, hxy = 0;
        for (int i = 0; i < 11; ++i) {
            const Real wi = Real(a.ssim_w[i]);
            const Real x = sx[r][q + i], y = sy[r][q + i];
            hx += wi * x;
            hy += wi * y;
            hx2 += wi * (x * x);
            hy2 += wi * (y * y);
            hxy += wi * (x * y);
        }
        hs[0][r][q] = hx;
        hs[1][r][q] = hy;
        hs[2][r][q] = hx2;
        hs[3][r][q] = hy2;
        hs[4][r][q] = hxy;
    }
    __syncthreads();
    const int tx = threadIdx.x % kSsimTX, ty = threadIdx.x / kSsimTX;
    const int vx = bx + tx, vy = by + ty;
    double ssum = 0;
    if (vx < Wv && vy < Hv) {
        Real mx = 0, my = 0, ex2 = 0, ey2 = 0, exy = 0;
        for (int j = 0; j < 11; ++j) {
            const Real wj = Real(a.ssim_w[j]);
            mx += wj * hs[0][ty + j][tx];
            my += wj * hs[1][ty + j][tx];
            ex2 += wj * hs[2][ty + j][tx];
            ey2 += wj * hs[3][ty + j][tx];
            exy += wj * hs[4][ty + j][tx];
        }
        const Real C1 = Real(0.01 * 0.01), C2 = Real(0.03 * 0.03);
        const Real vxx = ex2 - mx * mx, vyy = ey2 - my * my, sxy = exy - mx * my;
        const Real a1 = Real(2) * mx * my + C1, a2 = Real(2) * sxy + C2;
        const Real b1 = mx * mx + my * my + C1, b2 = vxx + vyy + C2;
        const Real sv = (a1 * a2) / (b1 * b2);
        ssum = double(sv);
        if (a.ssim_maps) {
            const Real dS = -Real(a.ssim_inv_count);
            Real* G = a.ssim_maps + size_t(c) * nv + size_t(vy) * Wv + vx;  // [3 maps][3 ch][nv]
            G[0] = dS * (Real(2) * my * (a2 - a1) / (b1 * b2) - Real(2) * mx * sv * (Real(1) / b1 - Real(1) / b2));
            G[3 * nv] = dS * (-sv / b2);
            G[6 * nv] = dS * (Real(2) * a1 / (b1 * b2));
        }
    }
    double v[1] = {ssum};
    block_accumulate<1>(v, a.acc + 1);
}

// The adjoint of the valid correlation per pixel (p = (px, py)): the maps G at
// windows (px - i, py - j), i, j in 0..10 and inside the valid range, weighted
// by w_i w_j -- zero-padded outside, which adds exact zeros.
template <typename Real>
__global__ void __launch_bounds__(kThreadsL) ssim_bwd_kernel(const __grid_constant__ LossArgs<Real> a) {
    __shared__ Real sg[3][kSsimRows][kSsimCols];
    __shared__ Real hs[3][kSsimRows][kSsimTX];
    const int W = a.W, H = a.H, Wv = W - 10, Hv = H - 10;
    const size_t HW = size_t(W) * H, nv = size_t(Wv) * Hv;
    const int c = blockIdx.y;
    const int tiles_x = ssim_tiles_x(W);
    const int bx = int(blockIdx.x % unsigned(tiles_x)) * kSsimTX, by = int(blockIdx.x / unsigned(tiles_x)) * kSsimTY;
    const Real* G = a.ssim_maps + size_t(c) * nv;
    // sg[m][r][q] = map m at window (bx - 10 + q, by - 10 + r)
    for (int e = threadIdx.x; e < kSsimRows * kSsimCols; e += kThreadsL) {
        const int r = e / kSsimCols, q = e - r * kSsimCols, wy = by - 10 + r, wx = bx - 10 + q;
        const bool in = wy >= 0 && wy < Hv && wx >= 0 && wx < Wv;
        const size_t o = in ? size_t(wy) * Wv + wx : 0;
        sg[0][r][q] = in ? G[o] : Real(0);
        sg[1][r][q] = in ? G[3 * nv + o] : Real(0);
        sg[2][r][q] = in ? G[6 * nv + o] : Real(0);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < kSsimRows * kSsimTX; e += kThreadsL) {
        const int r = e / kSsimTX, q = e - r * kSsimTX;
        Real hm = 0, h2 = 0, hxy = 0;
        for (int i = 0; i < 11; ++i) {  // window column px - i = bx + q - i -> sg column q + 10 - i
            const Real wi = Real(a.ssim_w[i]);
            hm += wi * sg[0][r][q + 10 - i];
            h2 += wi * sg[1][r][q + 10 - i];
            hxy += wi * sg[2][r][q + 10 - i];
        }
        hs[0][r][q] = hm;
        hs[1][r][q] = h2;
        hs[2][r][q] = hxy;
    }
    __syncthreads();
    const int tx = threadIdx.x % kSsimTX, ty = threadIdx.x / kSsimTX;
    const int px = bx + tx, py = by + ty;
    if (px >= W || py >= H) return;
    Real bm = 0, b2 = 0, bxy = 0;
    for (int j = 0; j < 11; ++j) {  // window row py - j -> hs row ty + 10 - j
        const Real wj = Real(a.ssim_w[j]);
        bm += wj * hs[0][ty + 10 - j][tx];
        b2 += wj * hs[1][ty + 10 - j][tx];
        bxy += wj * hs[2][ty + 10 - j][tx];
    }
    const size_t idx = size_t(c) * HW + size_t(py) * W + px;
    const Real x = a.color[idx], y = a.gt_rgb[idx];
    a.ssim_grad[idx] = bm + Real(2) * x * b2 + y * bxy;
}

// combine() (losses.cpp:285-313) on the reduced sums.
template <typename Real>
__global__ void combine_kernel(const __grid_constant__ LossArgs<Real> a) {
    const double HW = double(a.W) * a.H;
    const double* s = a.acc;
    double* r = a.report;
    const double l1 = a.en[0] ? s[0] / (3 * HW) : 0;
    const double ssim = a.en[1] ? 1.0 - s[1] * a.ssim_inv_count : 0;
    const double depth = a.en[3] && s[3] > 0 ? s[2] / s[3] : 0;
    const double normal = a.en[2] && s[5] > 0 ? 1.0 - s[4] / s[5] : 0;
    const double seg = a.en[4] && HW > 0 ? s[6] / HW : 0;
    const double k = a.en[5] && HW > 0 ? s[7] / HW : 0;
    const double mag = fabs(l1);
    auto ratio = [&](double v) { return fabs(v) < 1e-12 ? 0.0 : mag / fabs(v); };
    r[0] = l1;
    r[1] = ssim;
    r[2] = depth;
    r[3] = normal;
    r[4] = seg;
    r[5] = k;
    r[7] = ratio(ssim);
    r[8] = ratio(normal);
    r[9] = ratio(depth);
    r[10] = ratio(seg);
    r[11] = ratio(k);
    r[12] = a.lambdas[0];
    r[13] = a.lambdas[1] * r[7];
    r[14] = a.lambdas[3] * r[9];
    r[15] = a.lambdas[2] * r[8];
    r[16] = a.lambdas[4] * r[10];
    r[17] = a.lambdas[5] * r[11];
    r[6] = a.lambdas[0] * l1 + r[13] * ssim + r[15] * normal + r[14] * depth + r[16] * seg + r[17] * k;
    // counts for the seed assembly
    r[18] = s[3];
    r[19] = s[5];
}

template <typename Real>
__global__ void __launch_bounds__(kThreadsL) assemble_kernel(const __grid_constant__ LossArgs<Real> a) {
    const size_t HW = size_t(a.W) * a.H;
    const double* r = a.report;
    const Real seed_l1 = Real(r[12]), seed_ssim = Real(r[13]), seed_depth = Real(r[14]), seed_normal = Real(r[15]),
               seed_seg = Real(r[16]), seed_k = Real(r[17]);
    const Real inv_rgb = Real(1.0 / (3.0 * double(HW))), inv_hw = Real(1.0 / double(HW));
    const Real inv_depth = r[18] > 0 ? Real(1.0 / r[18]) : Real(0), inv_normal = r[19] > 0 ? Real(1.0 / r[19]) : Real(0);
    for (size_t p = size_t(blockIdx.x) * blockDim.x + threadIdx.x; p < HW; p += size_t(gridDim.x) * blockDim.x) {
        for (int c = 0; c < 3; ++c) {
            const size_t i = c * HW + p;
            Real g = Real(0);
            if (a.en[0]) g += seed_l1 * (sign_of(a.color[i] - a.gt_rgb[i]) * inv_rgb);
            if (a.en[1] && seed_ssim != Real(0)) g += seed_ssim * a.ssim_grad[i];
            a.dcolor[i] = g;
        }
        Real gd = Real(0);
        if (a.en[3] && seed_depth != Real(0) && a.gt_depth[p] > Real(0))
            gd = seed_depth * (sign_of(a.depth[p] - a.gt_depth[p]) * inv_depth);
        a.ddepth[p] = gd;
        if (a.dN) {
            const bool sup = a.en[2] && seed_normal != Real(0) && normal_supervised(a, p, HW);
            for (int c = 0; c < 3; ++c) a.dN[c * HW + p] = sup ? seed_normal * (-a.gt_normal[c * HW + p] * inv_normal) : Real(0);
        }
        if (a.dsem) {
            const int label = a.en[4] ? int(a.labels[p]) : 0;
            if (a.en[4] && seed_seg != Real(0) && label < a.C) {
                Real maxl, z;
                if (a.ce_stats) {
                    maxl = a.ce_stats[p];
                    z = a.ce_stats[HW + p];
                } else {
                    ce_pixel(a, p, HW, label, maxl, z);
                }
                // logits in batches of 8 loads ahead of their stores (the output
                // does not alias the frame's logits)
                const Real* __restrict__ sem = a.sem + p;
                Real* __restrict__ dsem = a.dsem + p;
                int c = 0;
                for (; c + 8 <= a.C; c += 8) {
                    Real l[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) l[k] = sem[size_t(c + k) * HW];
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const Real pc = exp(l[k] - maxl) / z;
                        dsem[size_t(c + k) * HW] = seed_seg * ((pc - (c + k == label ? Real(1) : Real(0))) * inv_hw);
                    }
                }
                for (; c < a.C; ++c) {
                    const Real pc = exp(sem[size_t(c) * HW] - maxl) / z;
                    dsem[size_t(c) * HW] = seed_seg * ((pc - (c == label ? Real(1) : Real(0))) * inv_hw);
                }
            } else {
                for (int c = 0; c < a.C; ++c) a.dsem[size_t(c) * HW + p] = Real(0);
            }
        }
        a.dkmap[p] = a.en[5] && seed_k != Real(0) ? seed_k * (sign_of(a.kmap[p] - Real(1)) * inv_hw) : Real(0);
    }
}

// Evaluation metrics (core/src/metrics.cpp:68-187): one pass of masked sums,
// counts and per-class label histograms.  acc: 0 sq err (rgb), 1 abs_rel sum,
// 2 abs_rel count, 3 depth sq err, 4 depth count, 5 cos sum, 6 cos count,
// 7 label-valid count; hist: [3][C] (intersection, predicted, truth).
template <typename Real>
__global__ void __launch_bounds__(kThreadsL) metric_pixel_kernel(const __grid_constant__ MetricArgs<Real> a) {
    extern __shared__ unsigned int hist_s[];  // [3][C]
    const size_t HW = size_t(a.W) * a.H;
    for (int i = threadIdx.x; i < 3 * a.C; i += blockDim.x) hist_s[i] = 0;
    __syncthreads();
    double v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (size_t p = size_t(blockIdx.x) * blockDim.x + threadIdx.x; p < HW; p += size_t(gridDim.x) * blockDim.x) {
        if (a.color)
            for (int c = 0; c < 3; ++c) {
                const double d = double(a.color[c * HW + p]) - double(a.gt_rgb[c * HW + p]);
                v[0] += d * d;
            }
        if (a.depth && a.depth_mask[p]) {
            const double d = double(a.depth[p]), g = double(a.gt_depth[p]);
            if (g > 1e-3) {
                v[1] += fabs(d - g) / g;
                v[2] += 1;
            }
            v[3] += (d - g) * (d - g);
            v[4] += 1;
        }
        if (a.normals && a.normal_mask[p]) {
            for (int c = 0; c < 3; ++c) v[5] += double(a.normals[c * HW + p]) * double(a.gt_normal[c * HW + p]);
            v[6] += 1;
        }
        if (a.sem && a.label_mask[p]) {
            int best = 0;  // argmax_labels: the first maximum
            Real bv = a.sem[p];
            for (int c = 1; c < a.C; ++c)
                if (a.sem[size_t(c) * HW + p] > bv) {
                    bv = a.sem[size_t(c) * HW + p];
                    best = c;
                }
            const int g = a.labels[p];
            v[7] += 1;
            if (g >= a.C) {
                raise_error(a.err, kErrMiouLabel, (long long)p, g);
            } else {
                atomicAdd(&hist_s[a.C + best], 1u);
                atomicAdd(&hist_s[2 * a.C + g], 1u);
                if (best == g) atomicAdd(&hist_s[best], 1u);
            }
        }
    }
    block_accumulate<8>(v, a.acc);
    __syncthreads();
    for (int i = threadIdx.x; i < 3 * a.C; i += blockDim.x)
        if (hist_s[i]) atomicAdd(reinterpret_cast<unsigned long long*>(a.hist) + i, (unsigned long long)hist_s[i]);
}

unsigned grid_for(size_t n) {
    const size_t b = (n + kThreadsL - 1) / kThreadsL;
    return unsigned(b < size_t(148 * 8) ? (b ? b : 1) : size_t(148 * 8));
}

}  // namespace

template <typename Real>
void launch_frame_losses(const LossArgs<Real>& a, cudaStream_t s) {
    const size_t HW = size_t(a.W) * a.H;
    cudaMemsetAsync(a.acc, 0, 8 * sizeof(double), s);
    loss_pixel_kernel<Real><<<grid_for(HW), kThreadsL, 0, s>>>(a);
    count_launches(1);
    if (a.en[1]) {
        ssim_fwd_kernel<Real><<<dim3(unsigned(ssim_tiles_x(a.W - 10) * ssim_tiles_y(a.H - 10)), 3), kThreadsL, 0, s>>>(a);
        ssim_bwd_kernel<Real><<<dim3(unsigned(ssim_tiles_x(a.W) * ssim_tiles_y(a.H)), 3), kThreadsL, 0, s>>>(a);
        count_launches(2);
    }
    combine_kernel<Real><<<1, 1, 0, s>>>(a);
    assemble_kernel<Real><<<grid_for(HW), kThreadsL, 0, s>>>(a);
    count_launches(2);
}

template <typename Real>
void launch_frame_metrics(const MetricArgs<Real>& a, cudaStream_t s) {
    const size_t HW = size_t(a.W) * a.H;
    cudaMemsetAsync(a.acc, 0, 9 * sizeof(double), s);
    if (a.C > 0) cudaMemsetAsync(a.hist, 0, 3 * size_t(a.C) * sizeof(unsigned long long), s);
    metric_pixel_kernel<Real><<<grid_for(HW), kThreadsL, 3 * size_t(a.C > 0 ? a.C : 1) * sizeof(unsigned int), s>>>(a);
    count_launches(1);
    if (a.color && a.W >= 11 && a.H >= 11) {  // ssim_metric = mean SSIM over valid windows
        LossArgs<Real> l{};
        l.W = a.W;
        l.H = a.H;
        for (int i = 0; i < 11; ++i) l.ssim_w[i] = a.ssim_w[i];
        l.color = a.color;
        l.gt_rgb = a.gt_rgb;
        l.acc = a.acc + 7;  // ssim sum lands in acc[8]
        ssim_fwd_kernel<Real><<<dim3(unsigned(ssim_tiles_x(a.W - 10) * ssim_tiles_y(a.H - 10)), 3), kThreadsL, 0, s>>>(l);
        count_launches(1);
    }
}

template void launch_frame_metrics<float>(const MetricArgs<float>&, cudaStream_t);
template void launch_frame_metrics<double>(const MetricArgs<double>&, cudaStream_t);
template void launch_frame_losses<float>(const LossArgs<float>&, cudaStream_t);
template void launch_frame_losses<double>(const LossArgs<double>&, cudaStream_t);

}  // namespace msplat_cuda
