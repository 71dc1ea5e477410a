// K11: optimizer step and prune mask on packed parameter buffers.
//   adam_step  (core/src/trainer.cpp:90-133): m, v, bias-corrected update with
//              per-group learning rates; the packed layout (msplat_param_layout)
//              groups each parameter kind into one contiguous segment, so the
//              learning rate is a function of the element's segment.
//   prune mask (core/src/trainer.cpp:135-147): keep = !(|k-1| > T)
//              (or !(|k-1| < T) with prune_keep_small).
#include <algorithm>
#include <cstdint>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace msplat_cuda {

namespace {

struct AdamSegments {
    long long start[8];
    double lr[7];
};

// Every operation is explicitly rounded (no FMA contraction), so the vector
// loop, the scalar tail and any sharded sub-range give the same bits for an
// element (sharded Adam == replicated Adam), and FP64 follows the reference's
// -ffp-contract=off evaluation (trainer.cpp:90-94, 109-131).
template <typename Real>
__device__ __forceinline__ Real adam_one(Real p, Real gr, Real& m, Real& v, Real lr, double bc1, double bc2) {
    if constexpr (sizeof(Real) == 8) {
        m = __dadd_rn(__dmul_rn(0.9, m), __dmul_rn(1.0 - 0.9, gr));
        v = __dadd_rn(__dmul_rn(0.999, v), __dmul_rn(__dmul_rn(1.0 - 0.999, gr), gr));
        const double num = __dmul_rn(lr, __ddiv_rn(m, bc1));
        return __dsub_rn(p, __ddiv_rn(num, __dadd_rn(__dsqrt_rn(__ddiv_rn(v, bc2)), 1e-15)));
    } else {  // FP32: reciprocals of the bias corrections, one IEEE divide
        m = __fadd_rn(__fmul_rn(0.9f, m), __fmul_rn(1.f - 0.9f, gr));
        v = __fadd_rn(__fmul_rn(0.999f, v), __fmul_rn(__fmul_rn(1.f - 0.999f, gr), gr));
        const float num = __fmul_rn(lr, __fmul_rn(m, float(1.0 / bc1)));
        return __fsub_rn(p, __fdiv_rn(num, __fadd_rn(__fsqrt_rn(__fmul_rn(v, float(1.0 / bc2))), 1e-15f)));
    }
}

__device__ __forceinline__ int adam_segment(const AdamSegments& seg, int64_t e) {
    int s = 0;
#pragma unroll
    for (int k = 1; k < 7; ++k) s += e >= seg.start[k];
    return s;
}

// Grid-stride, 16-byte vectors (4 floats / 2 doubles per access): the update
// is a pure stream over p, g, m, v (28 B per FP32 element).
template <typename Real>
__global__ void __launch_bounds__(256) adam_kernel(int64_t total, AdamSegments seg, Real* __restrict__ p,
                                                   const Real* __restrict__ g, Real* __restrict__ m,
                                                   Real* __restrict__ v, double bc1, double bc2, bool aligned) {
    constexpr int VEC = 16 / sizeof(Real);
    using V = typename std::conditional<sizeof(Real) == 4, float4, double2>::type;
    const int64_t nvec = aligned ? total / VEC : 0;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nvec; i += stride) {
        V pv = reinterpret_cast<const V*>(p)[i];
        const V gv = reinterpret_cast<const V*>(g)[i];
        V mv = reinterpret_cast<const V*>(m)[i];
        V vv = reinterpret_cast<const V*>(v)[i];
        Real* pp = reinterpret_cast<Real*>(&pv);
        const Real* gg = reinterpret_cast<const Real*>(&gv);
        Real* mm = reinterpret_cast<Real*>(&mv);
        Real* ww = reinterpret_cast<Real*>(&vv);
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
            const Real lr = Real(seg.lr[adam_segment(seg, i * VEC + j)]);
            pp[j] = adam_one<Real>(pp[j], gg[j], mm[j], ww[j], lr, bc1, bc2);
        }
        reinterpret_cast<V*>(p)[i] = pv;
        reinterpret_cast<V*>(m)[i] = mv;
        reinterpret_cast<V*>(v)[i] = vv;
    }
    for (int64_t e = nvec * VEC + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
        Real mm = m[e], ww = v[e];
        p[e] = adam_one<Real>(p[e], g[e], mm, ww, Real(seg.lr[adam_segment(seg, e)]), bc1, bc2);
        m[e] = mm;
        v[e] = ww;
    }
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
void launch_adam(int64_t base, int64_t total, const int64_t* seg_starts, const double* lr, Real* params,
                 const Real* grads, Real* m, Real* v, double bc1, double bc2, cudaStream_t s) {
    if (total == 0) return;
    AdamSegments seg;  // segment starts relative to the first element handled
    for (int i = 0; i < 8; ++i) seg.start[i] = seg_starts[i] - base;
    for (int i = 0; i < 7; ++i) seg.lr[i] = lr[i];
    const bool aligned = ((reinterpret_cast<uintptr_t>(params) | reinterpret_cast<uintptr_t>(grads) |
                           reinterpret_cast<uintptr_t>(m) | reinterpret_cast<uintptr_t>(v)) & 15u) == 0;
    const int64_t work = aligned ? (total + 15) / 16 * 4 : total;
    const unsigned blocks = unsigned(std::min<int64_t>((work + 255) / 256, 148 * 16));
    adam_kernel<Real><<<blocks, 256, 0, s>>>(total, seg, params, grads, m, v, bc1, bc2, aligned);
    count_launches(1);
}

template <typename Real>
void launch_prune_mask(int64_t n, const Real* k, double threshold, int keep_small, uint8_t* keep,
                       unsigned long long* kept, cudaStream_t s) {
    if (n == 0) return;
    prune_mask_kernel<Real><<<unsigned((n + 255) / 256), 256, 0, s>>>(n, k, threshold, keep_small, keep, kept);
    count_launches(1);
}

template void launch_adam<float>(int64_t, int64_t, const int64_t*, const double*, float*, const float*, float*,
                                 float*, double, double, cudaStream_t);
template void launch_adam<double>(int64_t, int64_t, const int64_t*, const double*, double*, const double*,
                                  double*, double*, double, double, cudaStream_t);
template void launch_prune_mask<float>(int64_t, const float*, double, int, uint8_t*, unsigned long long*,
                                       cudaStream_t);
template void launch_prune_mask<double>(int64_t, const double*, double, int, uint8_t*, unsigned long long*,
                                        cudaStream_t);

// dst += src over a packed buffer (the per-lane gradient sums of a multi-lane
// training step): grid-stride 16-byte vectors, scalar tail.
template <typename Real>
__global__ void __launch_bounds__(256) accumulate_kernel(int64_t total, Real* __restrict__ dst,
                                                         const Real* __restrict__ src, bool aligned) {
    constexpr int VEC = 16 / sizeof(Real);
    using V = typename std::conditional<sizeof(Real) == 4, float4, double2>::type;
    const int64_t nvec = aligned ? total / VEC : 0;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    const int64_t t0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    for (int64_t i = t0; i < nvec; i += stride) {
        V d = reinterpret_cast<const V*>(dst)[i];
        const V a = reinterpret_cast<const V*>(src)[i];
        Real* dd = reinterpret_cast<Real*>(&d);
        const Real* aa = reinterpret_cast<const Real*>(&a);
#pragma unroll
        for (int j = 0; j < VEC; ++j) dd[j] += aa[j];
        reinterpret_cast<V*>(dst)[i] = d;
    }
    for (int64_t e = nvec * VEC + t0; e < total; e += stride) dst[e] += src[e];
}

template <typename Real>
void launch_accumulate(int64_t total, Real* dst, const Real* src, cudaStream_t s) {
    if (total <= 0) return;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const bool aligned = (reinterpret_cast<uintptr_t>(dst) % 16 == 0) && (reinterpret_cast<uintptr_t>(src) % 16 == 0);
    const int64_t need = (total + 256 * 4 - 1) / (256 * 4);
    const unsigned blocks = unsigned(std::max<int64_t>(1, std::min<int64_t>(need, int64_t(sms) * 8)));
    accumulate_kernel<Real><<<blocks, 256, 0, s>>>(total, dst, src, aligned);
    count_launches(1);
}
template void launch_accumulate<float>(int64_t, float*, const float*, cudaStream_t);
template void launch_accumulate<double>(int64_t, double*, const double*, cudaStream_t);

}  // namespace msplat_cuda
