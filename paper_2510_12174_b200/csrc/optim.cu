// K11: optimizer step and prune mask on packed parameter buffers.
//   adam_step  (core/src/trainer.cpp:90-133): m, v, bias-corrected update with
//              per-group learning rates; the packed layout (msplat_param_layout)
//              groups each parameter kind into one contiguous segment, so the
//              learning rate is a function of the element's segment.
//   prune mask (core/src/trainer.cpp:135-147): keep = !(|k-1| > T)
//              (or !(|k-1| < T) with prune_keep_small).
#include "common.cuh"
#include "kernels.h"

namespace msplat_cuda {

namespace {

struct AdamSegments {
    long long start[8];
    double lr[7];
};

template <typename Real>
__global__ void adam_kernel(int64_t total, AdamSegments seg, Real* __restrict__ p, const Real* __restrict__ g,
                            Real* __restrict__ m, Real* __restrict__ v, double bc1, double bc2) {
    const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= total) return;
    int s = 0;
#pragma unroll
    for (int k = 1; k < 7; ++k) s += e >= seg.start[k];
    const Real lr = Real(seg.lr[s]);
    const Real gr = g[e];
    const Real mm = Real(0.9) * m[e] + (Real(1) - Real(0.9)) * gr;
    const Real vv = Real(0.999) * v[e] + (Real(1) - Real(0.999)) * gr * gr;
    m[e] = mm;
    v[e] = vv;
    p[e] -= lr * (mm / Real(bc1)) / (sqrt(vv / Real(bc2)) + Real(1e-15));
}

template <typename Real>
__global__ void prune_mask_kernel(int64_t n, const Real* __restrict__ k, double thr, int keep_small,
                                  uint8_t* __restrict__ keep, unsigned long long* kept) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    bool kp = false;
    if (i < n) {
        const double dev = fabs(double(k[i]) - 1.0);
        const bool anomalous = keep_small ? dev < thr : dev > thr;
        kp = !anomalous;
        keep[i] = uint8_t(kp);
    }
    const unsigned b = __ballot_sync(0xffffffffu, kp);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(kept, (unsigned long long)__popc(b));
}

}  // namespace

template <typename Real>
void launch_adam(int64_t total, const int64_t* seg_starts, const double* lr, Real* params, const Real* grads,
                 Real* m, Real* v, double bc1, double bc2, cudaStream_t s) {
    if (total == 0) return;
    AdamSegments seg;
    for (int i = 0; i < 8; ++i) seg.start[i] = seg_starts[i];
    for (int i = 0; i < 7; ++i) seg.lr[i] = lr[i];
    adam_kernel<Real><<<unsigned((total + 255) / 256), 256, 0, s>>>(total, seg, params, grads, m, v, bc1, bc2);
    count_launches(1);
}

template <typename Real>
void launch_prune_mask(int64_t n, const Real* k, double threshold, int keep_small, uint8_t* keep,
                       unsigned long long* kept, cudaStream_t s) {
    if (n == 0) return;
    prune_mask_kernel<Real><<<unsigned((n + 255) / 256), 256, 0, s>>>(n, k, threshold, keep_small, keep, kept);
    count_launches(1);
}

template void launch_adam<float>(int64_t, const int64_t*, const double*, float*, const float*, float*, float*,
                                 double, double, cudaStream_t);
template void launch_adam<double>(int64_t, const int64_t*, const double*, double*, const double*, double*,
                                  double*, double, double, cudaStream_t);
template void launch_prune_mask<float>(int64_t, const float*, double, int, uint8_t*, unsigned long long*,
                                       cudaStream_t);
template void launch_prune_mask<double>(int64_t, const double*, double, int, uint8_t*, unsigned long long*,
                                        cudaStream_t);

}  // namespace msplat_cuda
