// K13: trainer support on packed parameter buffers (msplat_param_layout):
//   init_scene (core/src/trainer.cpp:42-86): the isotropic scale from the mean
//     distance to the three nearest neighbours, as a tiled brute-force search
//     in exact FP64 (no contraction, ascending-order sum): the reference's
//     O(N^2) loop, bit for bit, with the point tiles staged in shared memory;
//   prune compaction (core/src/trainer.cpp:150-168): the stable compaction of
//     the parameters and both Adam moments by the keep mask, then k := k_reset.
#include "common.cuh"
#include "kernels.h"
#include "radix_sort.cuh"

namespace msplat_cuda {

namespace {

constexpr int kKnnThreads = 256;
constexpr double kShC0 = 0.28209479177387814;  // sh.cpp:9

__global__ void __launch_bounds__(kKnnThreads) knn3_kernel(int64_t n, const double* __restrict__ pts,
                                                           double* __restrict__ log_scale) {
    __shared__ double tile[kKnnThreads * 3];
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool act = i < n;
    double px = 0, py = 0, pz = 0;
    if (act) {
        px = pts[3 * i];
        py = pts[3 * i + 1];
        pz = pts[3 * i + 2];
    }
    double b0 = 1e308, b1 = 1e308, b2 = 1e308;  // three smallest squared distances, ascending
    for (int64_t base = 0; base < n; base += kKnnThreads) {
        __syncthreads();
        for (int k = threadIdx.x; k < kKnnThreads * 3; k += kKnnThreads) {
            const int64_t e = base * 3 + k;
            tile[k] = e < 3 * n ? pts[e] : 0.0;
        }
        __syncthreads();
        const int cnt = int(n - base < kKnnThreads ? n - base : kKnnThreads);
        if (act)
            for (int j = 0; j < cnt; ++j) {
                if (base + j == i) continue;
                // (points[j] - points[i]).squaredNorm(): x, y, z left to right
                const double dx = __dsub_rn(tile[3 * j], px), dy = __dsub_rn(tile[3 * j + 1], py),
                             dz = __dsub_rn(tile[3 * j + 2], pz);
                const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
                if (d2 < b2) {
                    if (d2 < b1) {
                        b2 = b1;
                        if (d2 < b0) {
                            b1 = b0;
                            b0 = d2;
                        } else {
                            b1 = d2;
                        }
                    } else {
                        b2 = d2;
                    }
                }
            }
    }
    if (!act) return;
    double mean_dist = 0.1;
    if (n > 1) {
        const int kn = n - 1 < 3 ? int(n - 1) : 3;
        double acc = __dsqrt_rn(b0);
        if (kn > 1) acc = __dadd_rn(acc, __dsqrt_rn(b1));
        if (kn > 2) acc = __dadd_rn(acc, __dsqrt_rn(b2));
        mean_dist = __ddiv_rn(acc, double(kn));
        mean_dist = mean_dist > 1e-4 ? mean_dist : 1e-4;
    }
    log_scale[i] = log(mean_dist);
}

template <typename Real>
__global__ void init_params_kernel(int64_t n, int C, int K, const double* __restrict__ pts,
                                   const double* __restrict__ cols, const double* __restrict__ log_scale,
                                   double k_reset, Real* __restrict__ params) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Real* means = params;
    Real* quats = means + 3 * n;
    Real* logs = quats + 4 * n;
    Real* opac = logs + 3 * n;
    Real* k = opac + n;
    Real* sh = k + n;
    Real* sem = sh + size_t(3) * K * n;
    for (int j = 0; j < 3; ++j) {
        means[3 * i + j] = Real(pts[3 * i + j]);
        logs[3 * i + j] = Real(log_scale[i]);
    }
    quats[4 * i] = Real(1);
    quats[4 * i + 1] = quats[4 * i + 2] = quats[4 * i + 3] = Real(0);
    opac[i] = Real(log(0.1 / 0.9));
    k[i] = Real(k_reset);
    for (int c = 0; c < 3; ++c)
        for (int j = 0; j < K; ++j)
            sh[(size_t(i) * 3 + c) * K + j] = j == 0 ? Real((cols[3 * i + c] - 0.5) / kShC0) : Real(0);
    for (int c = 0; c < C; ++c) sem[size_t(i) * C + c] = Real(0);
}

__global__ void keep_to_u32_kernel(int64_t n, const uint8_t* __restrict__ keep, uint32_t* __restrict__ k32) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) k32[i] = keep[i] ? 1u : 0u;
}

// One packed segment of `width` values per Gaussian: out[new(i)] = in[i] for kept i.
template <typename Real>
__global__ void compact_segment_kernel(int64_t n, int width, const uint8_t* __restrict__ keep,
                                       const uint32_t* __restrict__ newidx, const Real* __restrict__ in,
                                       Real* __restrict__ out) {
    const int64_t total = n * width;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = e / width;
        if (keep[i]) out[int64_t(newidx[i]) * width + (e - i * width)] = in[e];
    }
}

template <typename Real>
__global__ void fill_kernel(int64_t n, Real* __restrict__ p, double v) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) p[i] = Real(v);
}

unsigned blocks_for(int64_t n, int t = 256) {
    const int64_t b = (n + t - 1) / t;
    return unsigned(b < 1 ? 1 : (b > 148 * 32 ? 148 * 32 : b));
}

}  // namespace

template <typename Real>
void launch_init_scene(int64_t n, int C, int deg, const double* pts_dev, const double* cols_dev, double* log_scale_dev,
                       double k_reset, Real* params, cudaStream_t s) {
    if (n == 0) return;
    const int K = (deg + 1) * (deg + 1);
    knn3_kernel<<<unsigned((n + kKnnThreads - 1) / kKnnThreads), kKnnThreads, 0, s>>>(n, pts_dev, log_scale_dev);
    init_params_kernel<Real><<<unsigned((n + 255) / 256), 256, 0, s>>>(n, C, K, pts_dev, cols_dev, log_scale_dev,
                                                                       k_reset, params);
    count_launches(2);
}

template <typename Real>
void launch_prune_compact(int64_t n, int C, int deg, const uint8_t* keep, int64_t kept, const Real* const in[3],
                          Real* const out[3], double k_reset, uint32_t* k32, uint32_t* newidx, uint32_t* scan_tiles,
                          uint32_t* d_total, cudaStream_t s) {
    if (n == 0) return;
    keep_to_u32_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(n, keep, k32);
    device_exclusive_scan<uint32_t>(k32, newidx, nullptr, n, scan_tiles, d_total, s);
    const int K = (deg + 1) * (deg + 1);
    const int widths[7] = {3, 4, 3, 1, 1, 3 * K, C};
    for (int b = 0; b < 3; ++b) {
        if (!in[b] || !out[b]) continue;
        int64_t off_in = 0, off_out = 0;
        for (int sgi = 0; sgi < 7; ++sgi) {
            if (widths[sgi] > 0)
                compact_segment_kernel<Real><<<blocks_for(n * widths[sgi]), 256, 0, s>>>(
                    n, widths[sgi], keep, newidx, in[b] + off_in, out[b] + off_out);
            off_in += n * widths[sgi];
            off_out += kept * widths[sgi];
        }
    }
    // prune() resets every surviving k (trainer.cpp:166-167); the k segment
    // starts after means, quats, log_scales, opacity.
    fill_kernel<Real><<<unsigned((kept + 255) / 256), 256, 0, s>>>(kept, out[0] + kept * 11, k_reset);
    count_launches(3 + 7 * 3);
}

template void launch_init_scene<float>(int64_t, int, int, const double*, const double*, double*, double, float*,
                                       cudaStream_t);
template void launch_init_scene<double>(int64_t, int, int, const double*, const double*, double*, double, double*,
                                        cudaStream_t);
template void launch_prune_compact<float>(int64_t, int, int, const uint8_t*, int64_t, const float* const[3],
                                          float* const[3], double, uint32_t*, uint32_t*, uint32_t*, uint32_t*,
                                          cudaStream_t);
template void launch_prune_compact<double>(int64_t, int, int, const uint8_t*, int64_t, const double* const[3],
                                           double* const[3], double, uint32_t*, uint32_t*, uint32_t*, uint32_t*,
                                           cudaStream_t);

}  // namespace msplat_cuda
