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
//                          adjoints (losses.cpp:120-146);
//   3. ssim_bwd_kernel     per pixel: the adjoint of the valid correlation
//                          (losses.cpp:61-83, 148-156);
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
    maxl = a.sem[p];
    for (int c = 1; c < a.C; ++c) maxl = a.sem[size_t(c) * HW + p] > maxl ? a.sem[size_t(c) * HW + p] : maxl;
    z = Real(0);
    for (int c = 0; c < a.C; ++c) z += exp(a.sem[size_t(c) * HW + p] - maxl);
    return log(z) - (a.sem[size_t(label) * HW + p] - maxl);
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
            }
        }
        if (a.en[5]) v[7] += double(fabs(a.kmap[p] - Real(1)));
    }
    block_accumulate<8>(v, a.acc);
}

// Windowed moments of one valid window (separable order of losses.cpp:39-58:
// along x first, then along y).
template <typename Real>
__global__ void __launch_bounds__(kThreadsL) ssim_fwd_kernel(const __grid_constant__ LossArgs<Real> a) {
    const int W = a.W, H = a.H, Wv = W - 10, Hv = H - 10;
    const size_t HW = size_t(W) * H, nv = size_t(Wv) * Hv;
    double ssum = 0;
    for (size_t idx = size_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < 3 * nv;
         idx += size_t(gridDim.x) * blockDim.x) {
        const int c = int(idx / nv);
        const size_t r = idx - size_t(c) * nv;
        const int vy = int(r / Wv), vx = int(r - size_t(vy) * Wv);
        const Real* X = a.color + c * HW;
        const Real* Y = a.gt_rgb + c * HW;
        Real mx = 0, my = 0, ex2 = 0, ey2 = 0, exy = 0;
        for (int j = 0; j < 11; ++j) {
            const size_t row = size_t(vy + j) * W + vx;
            Real hx = 0, hy = 0, hx2 = 0, hy2 = 0, hxy = 0;
            for (int i = 0; i < 11; ++i) {
                const Real wi = Real(a.ssim_w[i]);
                const Real x = X[row + i], y = Y[row + i];
                hx += wi * x;
                hy += wi * y;
                hx2 += wi * (x * x);
                hy2 += wi * (y * y);
                hxy += wi * (x * y);
            }
            const Real wj = Real(a.ssim_w[j]);
            mx += wj * hx;
            my += wj * hy;
            ex2 += wj * hx2;
            ey2 += wj * hy2;
            exy += wj * hxy;
        }
        const Real C1 = Real(0.01 * 0.01), C2 = Real(0.03 * 0.03);
        const Real sx = ex2 - mx * mx, sy = ey2 - my * my, sxy = exy - mx * my;
        const Real a1 = Real(2) * mx * my + C1, a2 = Real(2) * sxy + C2;
        const Real b1 = mx * mx + my * my + C1, b2 = sx + sy + C2;
        const Real s = (a1 * a2) / (b1 * b2);
        ssum += double(s);
        if (!a.ssim_maps) continue;  // metric only
        const Real dS = -Real(a.ssim_inv_count);
        Real* G = a.ssim_maps + size_t(c) * nv + r;  // [3 maps][3 ch][nv]
        G[0] = dS * (Real(2) * my * (a2 - a1) / (b1 * b2) - Real(2) * mx * s * (Real(1) / b1 - Real(1) / b2));
        G[3 * nv] = dS * (-s / b2);
        G[6 * nv] = dS * (Real(2) * a1 / (b1 * b2));
    }
    double v[1] = {ssum};
    block_accumulate<1>(v, a.acc + 1);
}

template <typename Real>
__global__ void __launch_bounds__(kThreadsL) ssim_bwd_kernel(const __grid_constant__ LossArgs<Real> a) {
    const int W = a.W, H = a.H, Wv = W - 10, Hv = H - 10;
    const size_t HW = size_t(W) * H, nv = size_t(Wv) * Hv;
    for (size_t idx = size_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < 3 * HW;
         idx += size_t(gridDim.x) * blockDim.x) {
        const int c = int(idx / HW);
        const size_t p = idx - size_t(c) * HW;
        const int py = int(p / W), px = int(p - size_t(py) * W);
        const Real* G = a.ssim_maps + size_t(c) * nv;
        Real bm = 0, b2 = 0, bxy = 0;
        const int j0 = py - (Hv - 1) > 0 ? py - (Hv - 1) : 0, j1 = py < 10 ? py : 10;
        const int i0 = px - (Wv - 1) > 0 ? px - (Wv - 1) : 0, i1 = px < 10 ? px : 10;
        for (int j = j0; j <= j1; ++j) {
            const size_t row = size_t(py - j) * Wv;
            Real hm = 0, h2 = 0, hxy = 0;
            for (int i = i0; i <= i1; ++i) {
                const Real wi = Real(a.ssim_w[i]);
                const size_t o = row + (px - i);
                hm += wi * G[o];
                h2 += wi * G[3 * nv + o];
                hxy += wi * G[6 * nv + o];
            }
            const Real wj = Real(a.ssim_w[j]);
            bm += wj * hm;
            b2 += wj * h2;
            bxy += wj * hxy;
        }
        const Real x = a.color[idx], y = a.gt_rgb[idx];
        a.ssim_grad[idx] = bm + Real(2) * x * b2 + y * bxy;
    }
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
                ce_pixel(a, p, HW, label, maxl, z);
                for (int c = 0; c < a.C; ++c) {
                    const Real pc = exp(a.sem[size_t(c) * HW + p] - maxl) / z;
                    a.dsem[size_t(c) * HW + p] = seed_seg * ((pc - (c == label ? Real(1) : Real(0))) * inv_hw);
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
        const size_t nv = size_t(a.W - 10) * (a.H - 10);
        ssim_fwd_kernel<Real><<<grid_for(3 * nv), kThreadsL, 0, s>>>(a);
        ssim_bwd_kernel<Real><<<grid_for(3 * HW), kThreadsL, 0, s>>>(a);
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
        const size_t nv = size_t(a.W - 10) * (a.H - 10);
        ssim_fwd_kernel<Real><<<grid_for(3 * nv), kThreadsL, 0, s>>>(l);
        count_launches(1);
    }
}

template void launch_frame_metrics<float>(const MetricArgs<float>&, cudaStream_t);
template void launch_frame_metrics<double>(const MetricArgs<double>&, cudaStream_t);
template void launch_frame_losses<float>(const LossArgs<float>&, cudaStream_t);
template void launch_frame_losses<double>(const LossArgs<double>&, cudaStream_t);

}  // namespace msplat_cuda
