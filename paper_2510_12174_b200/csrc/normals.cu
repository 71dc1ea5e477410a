// K7/K8: depth-derived normals and their adjoint.
//
// K7 replaces estimate_normals + backproject (core/src/normals.cpp:16-101):
// one thread per pixel recomputes the nine backprojected stencil points it
// needs straight from the depth map (no P_world buffer), applies the
// two-scale cross products, sign alignment, fusion, normalisation and the
// view-facing flip, and writes planar unit normals (zero when invalid).
// The stencil runs in CAMERA space: P_world = R P_cam + t, so edge vectors,
// cross products, norms and the facing test are rotation-covariant/invariant
// and t cancels exactly; only the output normal is rotated to world space
// (and the incoming gradient rotated back).  Same values as the reference in
// exact arithmetic, without FP32 cancellation against t.
//
// K8 replaces normals_backward (core/src/normals.cpp:103-152).  The reference
// scatters each centre's four edge adjoints onto 8 stencil pixels; a scatter
// needs atomics on a GPU, so it is split in two deterministic passes:
//   K8a  per centre pixel: the 12 adjoint components dvx1, dvy1, dvx2, dvy2
//        (state recomputed from depth/T as K7 does), written planar;
//   K8b  per target pixel: gather the (at most 8) centres that reference it,
//        sum +-dv and dot with the target's camera ray, dD += seed * that.
#include "common.cuh"
#include "kernels.h"

namespace msplat_cuda {

namespace {

template <typename Real>
struct NormalCtx {
    const NormalArgs<Real>* a;
    // Camera-space backprojection pixel_dir_cam * d (normals.cpp:10-12, 16-26).
    __device__ void point(int x, int y, Real* P) const {
        const Cam& c = a->cam;
        const Real d = a->depth[size_t(y) * a->W + x];
        P[0] = ((Real(x) + Real(0.5) - Real(c.cx)) / Real(c.fx)) * d;
        P[1] = ((Real(y) + Real(0.5) - Real(c.cy)) / Real(c.fy)) * d;
        P[2] = d;
    }
    __device__ bool covered(int x, int y) const {
        return a->T[size_t(y) * a->W + x] < Real(a->mask_threshold);
    }
};

template <typename Real>
__device__ __forceinline__ void cross(const Real* u, const Real* v, Real* o) {
    o[0] = u[1] * v[2] - u[2] * v[1];
    o[1] = u[2] * v[0] - u[0] * v[2];
    o[2] = u[0] * v[1] - u[1] * v[0];
}

// Shared state of one centre pixel (normals.cpp:59-88).  Returns false when the
// pixel is not a valid centre (border, mask, degenerate stencil).
template <typename Real>
struct Stencil {
    Real vx1[3], vy1[3], vx2[3], vy2[3], nf[3], norm, sign2;
    bool flipped;
};

template <typename Real>
__device__ bool centre_state(const NormalCtx<Real>& nc, int x, int y, Stencil<Real>& st) {
    const NormalArgs<Real>& a = *nc.a;
    const int s1 = a.step1, s2 = a.step2;
    if (x < s2 || y < s2 || x + s2 >= a.W || y + s2 >= a.H) return false;
    if (!(nc.covered(x, y) && nc.covered(x + s1, y) && nc.covered(x - s1, y) && nc.covered(x, y + s1) &&
          nc.covered(x, y - s1) && nc.covered(x + s2, y) && nc.covered(x - s2, y) &&
          nc.covered(x, y + s2) && nc.covered(x, y - s2)))
        return false;
    Real pa[3], pb[3];
    nc.point(x + s1, y, pa); nc.point(x - s1, y, pb);
    for (int i = 0; i < 3; ++i) st.vx1[i] = pa[i] - pb[i];
    nc.point(x, y + s1, pa); nc.point(x, y - s1, pb);
    for (int i = 0; i < 3; ++i) st.vy1[i] = pa[i] - pb[i];
    nc.point(x + s2, y, pa); nc.point(x - s2, y, pb);
    for (int i = 0; i < 3; ++i) st.vx2[i] = pa[i] - pb[i];
    nc.point(x, y + s2, pa); nc.point(x, y - s2, pb);
    for (int i = 0; i < 3; ++i) st.vy2[i] = pa[i] - pb[i];
    Real n1[3], n2[3];
    cross(st.vx1, st.vy1, n1);
    cross(st.vx2, st.vy2, n2);
    st.sign2 = (n1[0] * n2[0] + n1[1] * n2[1] + n1[2] * n2[2]) < Real(0) ? Real(-1) : Real(1);
    const Real lam = Real(a.lambda);
    for (int i = 0; i < 3; ++i) st.nf[i] = lam * n1[i] + (Real(1) - lam) * (n2[i] * st.sign2);
    st.norm = sqrt(st.nf[0] * st.nf[0] + st.nf[1] * st.nf[1] + st.nf[2] * st.nf[2]);
    if (st.norm < Real(1e-12)) return false;
    Real P[3];
    nc.point(x, y, P);
    Real dv[3] = {-P[0], -P[1], -P[2]};  // camera centre minus the point, camera frame
    const Real dn = sqrt(dv[0] * dv[0] + dv[1] * dv[1] + dv[2] * dv[2]);
    Real ndot = Real(0);
    for (int i = 0; i < 3; ++i) ndot += (st.nf[i] / st.norm) * (dn > Real(0) ? dv[i] / dn : dv[i]);
    st.flipped = ndot > Real(0);
    return true;
}

template <typename Real>
__global__ void normals_forward_kernel(const __grid_constant__ NormalArgs<Real> a) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= a.W || y >= a.H) return;
    const NormalCtx<Real> nc{&a};
    Stencil<Real> st;
    Real N[3] = {0, 0, 0};
    if (centre_state(nc, x, y, st)) {
        const Real s = st.flipped ? Real(-1) : Real(1);
        Real Nc[3];
        for (int i = 0; i < 3; ++i) Nc[i] = s * (st.nf[i] / st.norm);
        for (int i = 0; i < 3; ++i)
            N[i] = Real(a.cam.Rc2w[i * 3]) * Nc[0] + Real(a.cam.Rc2w[i * 3 + 1]) * Nc[1] +
                   Real(a.cam.Rc2w[i * 3 + 2]) * Nc[2];
    }
    const size_t HW = size_t(a.W) * a.H, p = size_t(y) * a.W + x;
    for (int i = 0; i < 3; ++i) a.normals[i * HW + p] = N[i];
}

template <typename Real>
__global__ void normals_adjoint_kernel(const __grid_constant__ NormalArgs<Real> a) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= a.W || y >= a.H) return;
    const size_t HW = size_t(a.W) * a.H, p = size_t(y) * a.W + x;
    Real out[12];
    for (int i = 0; i < 12; ++i) out[i] = Real(0);
    const Real gw[3] = {a.dN[p], a.dN[HW + p], a.dN[2 * HW + p]};
    Real g[3];  // camera-frame gradient R^T gw
    for (int i = 0; i < 3; ++i)
        g[i] = Real(a.cam.Rc2w[i]) * gw[0] + Real(a.cam.Rc2w[3 + i]) * gw[1] + Real(a.cam.Rc2w[6 + i]) * gw[2];
    const NormalCtx<Real> nc{&a};
    Stencil<Real> st;
    if ((g[0] != Real(0) || g[1] != Real(0) || g[2] != Real(0)) && centre_state(nc, x, y, st)) {
        if (st.flipped)
            for (int i = 0; i < 3; ++i) g[i] = -g[i];
        Real N[3];
        for (int i = 0; i < 3; ++i) N[i] = st.nf[i] / st.norm;
        const Real Ng = N[0] * g[0] + N[1] * g[1] + N[2] * g[2];
        Real g1[3], g2[3];
        const Real lam = Real(a.lambda);
        for (int i = 0; i < 3; ++i) {
            const Real gf = (g[i] - N[i] * Ng) / st.norm;
            g1[i] = lam * gf;
            g2[i] = (Real(1) - lam) * st.sign2 * gf;
        }
        cross(st.vy1, g1, out + 0);  // dvx1
        cross(g1, st.vx1, out + 3);  // dvy1
        cross(st.vy2, g2, out + 6);  // dvx2
        cross(g2, st.vx2, out + 9);  // dvy2
    }
    for (int i = 0; i < 12; ++i) a.dv[i * HW + p] = out[i];
}

template <typename Real>
__global__ void normals_gather_kernel(const __grid_constant__ NormalArgs<Real> a) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= a.W || y >= a.H) return;
    const size_t HW = size_t(a.W) * a.H;
    const int s1 = a.step1, s2 = a.step2;
    // (centre offset from this pixel, dv component block, sign) for the 8
    // scatter targets of normals.cpp:141-148.
    const int cx[8] = {-s1, s1, 0, 0, -s2, s2, 0, 0};
    const int cy[8] = {0, 0, -s1, s1, 0, 0, -s2, s2};
    const int blk[8] = {0, 0, 3, 3, 6, 6, 9, 9};
    const Real sg[8] = {1, -1, 1, -1, 1, -1, 1, -1};
    Real dP[3] = {0, 0, 0};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int px = x + cx[k], py = y + cy[k];
        if (px < 0 || py < 0 || px >= a.W || py >= a.H) continue;
        const size_t q = size_t(py) * a.W + px;
        for (int i = 0; i < 3; ++i) dP[i] += sg[k] * a.dv[size_t(blk[k] + i) * HW + q];
    }
    // dD += dP_world . (R pd) = dP_cam . pd   (normals.cpp:110-113)
    const Cam& c = a.cam;
    const Real pd0 = (Real(x) + Real(0.5) - Real(c.cx)) / Real(c.fx);
    const Real pd1 = (Real(y) + Real(0.5) - Real(c.cy)) / Real(c.fy);
    const Real dd = dP[0] * pd0 + dP[1] * pd1 + dP[2];
    const size_t p = size_t(y) * a.W + x;
    a.dD[p] += Real(a.seed) * dd;
}

}  // namespace

template <typename Real>
void launch_normals_forward(const NormalArgs<Real>& a, cudaStream_t s) {
    const dim3 blk(32, 8), grd((a.W + 31) / 32, (a.H + 7) / 8);
    normals_forward_kernel<Real><<<grd, blk, 0, s>>>(a);
    count_launches(1);
}

template <typename Real>
void launch_normals_backward(const NormalArgs<Real>& a, cudaStream_t s) {
    const dim3 blk(32, 8), grd((a.W + 31) / 32, (a.H + 7) / 8);
    normals_adjoint_kernel<Real><<<grd, blk, 0, s>>>(a);
    count_launches(1);
    normals_gather_kernel<Real><<<grd, blk, 0, s>>>(a);
    count_launches(1);
}

template void launch_normals_forward<float>(const NormalArgs<float>&, cudaStream_t);
template void launch_normals_forward<double>(const NormalArgs<double>&, cudaStream_t);
template void launch_normals_backward<float>(const NormalArgs<float>&, cudaStream_t);
template void launch_normals_backward<double>(const NormalArgs<double>&, cudaStream_t);

}  // namespace msplat_cuda
