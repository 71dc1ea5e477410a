// msplat C++ drop-in: host-side scalar helpers of the public API.
//
// The render path itself runs on the B200 (device_path.cpp); these are the
// per-element functions callers and the reference tests use directly, plus the
// untiled brute-force renderer.  Each follows the reference function cited
// (paths relative to /root/reference/proj) in double precision.
#include "parallel.hpp"
#include <cmath>
#include <iostream>
#include <stdexcept>
#include <string>

#include "msplat/camera.hpp"
#include "msplat/geometry.hpp"
#include "msplat/normals.hpp"
#include "msplat/oracle.hpp"
#include "msplat/rasterizer.hpp"
#include "msplat/scene.hpp"
#include "msplat/sh.hpp"

namespace msplat {

namespace {

bool finite_primitive(const GaussianPrimitive& g) {
    return g.position.allFinite() && g.rotation.allFinite() && g.log_scale.allFinite() &&
           std::isfinite(g.opacity_logit) && g.sh.allFinite() && g.semantic_logits.allFinite() &&
           std::isfinite(g.gradient_factor);
}

std::string prim(size_t i) { return "primitive " + std::to_string(i); }

}  // namespace

// ----------------------------------------------------------------- scene
// Scene::validate -- core/src/scene.cpp:22-40
void Scene::validate() const {
    if (sh_degree < 0 || sh_degree > 3) throw std::invalid_argument("Scene: sh_degree must be in [0,3]");
    if (num_classes < 0) throw std::invalid_argument("Scene: num_classes must be >= 0");
    const int ch = sh_coeff_count();
    // contiguous chunks in parallel; each chunk stops at its first bad
    // primitive and the lowest chunk's error is re-thrown: the sequential
    // loop's message
    dropin::parallel_for(gaussians.size(), [&](size_t b, size_t e) {
        for (size_t i = b; i < e; ++i) {
            const GaussianPrimitive& g = gaussians[i];
            if (g.sh.cols() != ch) throw std::invalid_argument("Scene: " + prim(i) + " has wrong SH coefficient count");
            if (g.semantic_logits.size() != num_classes)
                throw std::invalid_argument("Scene: " + prim(i) + " has wrong semantic channel count");
            if (!finite_primitive(g)) throw std::invalid_argument("Scene: " + prim(i) + " has non-finite fields");
        }
    });
}

// activate -- core/src/scene.cpp:42-60
ActivatedGaussian activate(const GaussianPrimitive& g, size_t index) {
    if (!finite_primitive(g)) throw std::invalid_argument("activate: " + prim(index) + " has non-finite fields");
    const Scalar n = g.rotation.norm();
    if (n < 1e-12) throw std::invalid_argument("activate: " + prim(index) + " has a zero quaternion");
    ActivatedGaussian out;
    out.position = g.position;
    out.unit_q = g.rotation / n;
    out.R = quat_to_rotation(out.unit_q);
    out.scale = g.log_scale.array().exp();
    out.alpha = 1.0 / (1.0 + std::exp(-g.opacity_logit));
    out.sh = &g.sh;
    out.semantic_logits = &g.semantic_logits;
    out.k = g.gradient_factor;
    return out;
}

std::vector<ActivatedGaussian> activate_scene(const Scene& scene) {
    std::vector<ActivatedGaussian> out;
    out.reserve(scene.size());
    for (size_t i = 0; i < scene.size(); ++i) out.push_back(activate(scene.gaussians[i], i));
    return out;
}

// GradientBuffer -- core/src/scene.cpp:70-106
void GradientBuffer::resize_zero(const Scene& scene) {
    const size_t n = scene.size();
    dposition.assign(n, Vec3::Zero());
    drotation.assign(n, Vec4::Zero());
    dscale.assign(n, Vec3::Zero());
    dopacity.assign(n, 0.0);
    dsh.assign(n, ShMatrix::Zero(3, scene.sh_coeff_count()));
    dsemantics.assign(n, VecX::Zero(scene.num_classes));
    dk.assign(n, 0.0);
    raw_space = false;
}

void GradientBuffer::add(const GradientBuffer& o) {
    if (o.size() != size()) throw std::invalid_argument("GradientBuffer::add: size mismatch");
    for (size_t i = 0; i < size(); ++i) {
        dposition[i] += o.dposition[i];
        drotation[i] += o.drotation[i];
        dscale[i] += o.dscale[i];
        dopacity[i] += o.dopacity[i];
        dsh[i] += o.dsh[i];
        dsemantics[i] += o.dsemantics[i];
        dk[i] += o.dk[i];
    }
}

void GradientBuffer::check_finite(const char* where) const {
    for (size_t i = 0; i < size(); ++i) {
        const bool ok = dposition[i].allFinite() && drotation[i].allFinite() && dscale[i].allFinite() &&
                        std::isfinite(dopacity[i]) && dsh[i].allFinite() && dsemantics[i].allFinite() &&
                        std::isfinite(dk[i]);
        if (!ok) throw std::runtime_error(std::string(where) + ": non-finite gradient for " + prim(i));
    }
}

// ---------------------------------------------------------------- camera
// CameraView::finalize -- core/src/camera.cpp:8-21
void CameraView::finalize() {
    if (width < 1 || height < 1) throw std::invalid_argument("CameraView: width and height must be >= 1");
    if (!(fx > 0) || !(fy > 0)) throw std::invalid_argument("CameraView: focal lengths must be positive");
    if ((Mat3(R_cam_to_world.transpose() * R_cam_to_world) - Mat3::Identity()).cwiseAbs().maxCoeff() > 1e-6)
        throw std::invalid_argument("CameraView: rotation is not orthonormal (tol 1e-6)");
    if (std::abs(R_cam_to_world.determinant() - 1.0) > 1e-6)
        throw std::invalid_argument("CameraView: rotation determinant is not +1 (tol 1e-6)");
    R_world_to_cam = R_cam_to_world.transpose();
    t_world_to_cam = -(R_world_to_cam * t_cam_to_world);
}

CameraView make_camera(Scalar fx, Scalar fy, Scalar cx, Scalar cy, int width, int height, const Mat3& R_c2w,
                       const Vec3& t_c2w) {
    CameraView v;
    v.fx = fx;
    v.fy = fy;
    v.cx = cx;
    v.cy = cy;
    v.width = width;
    v.height = height;
    v.R_cam_to_world = R_c2w;
    v.t_cam_to_world = t_c2w;
    v.finalize();
    return v;
}

// make_lookat_camera -- core/src/camera.cpp:38-59
CameraView make_lookat_camera(Scalar fx, Scalar fy, Scalar cx, Scalar cy, int width, int height, const Vec3& eye,
                              const Vec3& target, const Vec3& up_hint) {
    Vec3 fwd = target - eye;
    const Scalar n = fwd.norm();
    if (n < 1e-12) throw std::invalid_argument("make_lookat_camera: eye and target coincide");
    fwd /= n;
    Vec3 right = fwd.cross(up_hint);
    if (right.norm() < 1e-9) {
        right = fwd.cross(Vec3(1, 0, 0));
        if (right.norm() < 1e-9) right = fwd.cross(Vec3(0, 0, 1));
    }
    right.normalize();
    Mat3 R;
    R.col(0) = right;
    R.col(1) = fwd.cross(right);
    R.col(2) = fwd;
    return make_camera(fx, fy, cx, cy, width, height, R, eye);
}

// -------------------------------------------------------------- geometry
// quat_to_rotation -- core/src/geometry.cpp:7-15
Mat3 quat_to_rotation(const Vec4& q) {
    const Vec4 u = q / q.norm();
    const Scalar w = u[0], x = u[1], y = u[2], z = u[3];
    Mat3 R;
    R << 1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
         2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
         2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y);
    return R;
}

// quat_rotation_backward -- core/src/geometry.cpp:17-29
Vec4 quat_rotation_backward(const Vec4& q, const Mat3& G) {
    const Scalar w = q[0], x = q[1], y = q[2], z = q[3];
    Vec4 d;
    d[0] = 2 * (G(0, 1) * (-z) + G(0, 2) * y + G(1, 0) * z + G(1, 2) * (-x) + G(2, 0) * (-y) + G(2, 1) * x);
    d[1] = 2 * (G(0, 1) * y + G(0, 2) * z + G(1, 0) * y + G(1, 1) * (-2 * x) + G(1, 2) * (-w) + G(2, 0) * z +
                G(2, 1) * w + G(2, 2) * (-2 * x));
    d[2] = 2 * (G(0, 0) * (-2 * y) + G(0, 1) * x + G(0, 2) * w + G(1, 0) * x + G(1, 2) * z + G(2, 0) * (-w) +
                G(2, 1) * z + G(2, 2) * (-2 * y));
    d[3] = 2 * (G(0, 0) * (-2 * z) + G(0, 1) * (-w) + G(0, 2) * x + G(1, 0) * w + G(1, 1) * (-2 * z) + G(1, 2) * y +
                G(2, 0) * x + G(2, 1) * y);
    return d;
}

// compute_ray -- core/src/geometry.cpp:31-35
void compute_ray(const CameraView& view, Scalar u, Scalar v, Vec3& origin, Vec3& dir) {
    origin = view.t_cam_to_world;
    dir = (view.R_cam_to_world * Vec3((u - view.cx) / view.fx, (v - view.cy) / view.fy, 1.0)).normalized();
}

// intersect -- core/src/geometry.cpp:37-64
std::optional<RayEllipsoidHit> intersect(const ActivatedGaussian& g, const Vec3& origin, const Vec3& dir,
                                         Scalar sigma_scale) {
    RayEllipsoidHit h;
    h.axes = sigma_scale * g.scale;
    if (h.axes.minCoeff() < kDegenerateScale) return std::nullopt;
    h.v_l = g.R.transpose() * (origin - g.position);
    h.d_l = g.R.transpose() * dir;
    h.v_s = h.v_l.cwiseQuotient(h.axes);
    h.d_s = h.d_l.cwiseQuotient(h.axes);
    h.a = h.d_s.squaredNorm();
    h.b = 2.0 * h.v_s.dot(h.d_s);
    const Scalar c = h.v_s.squaredNorm() - 1.0;
    const Scalar disc = h.b * h.b - 4.0 * h.a * c;
    if (disc < 0 || h.a <= 0) return std::nullopt;
    const Scalar sq = std::sqrt(disc);
    h.t1 = (-h.b - sq) / (2.0 * h.a);
    h.t2 = (-h.b + sq) / (2.0 * h.a);
    h.t_mid = -h.b / (2.0 * h.a);
    if (h.t_mid <= 0) return std::nullopt;
    return h;
}

Scalar midpoint_depth(const CameraView& view, const Vec3& origin, const Vec3& dir, Scalar t_mid) {
    return view.cam_depth(origin + t_mid * dir);
}

// intersection_backward -- core/src/geometry.cpp:70-105
IntersectionGrads intersection_backward(const RayEllipsoidHit& h, Scalar dL_dd, const CameraView& view,
                                        const Vec3& origin, const Vec3& dir, const ActivatedGaussian& g) {
    IntersectionGrads out;
    if (std::abs(h.a) < 1e-12) {
        out.degenerate = true;
        return out;
    }
    if (dL_dd == 0) return out;
    const Scalar g_t = dL_dd * view.R_world_to_cam.row(2).dot(dir);
    const Vec3 g_vs = g_t * (-h.d_s / h.a);
    const Vec3 g_ds = g_t * ((h.b / (h.a * h.a)) * h.d_s - h.v_s / h.a);
    out.dscale = -(g_vs.cwiseProduct(h.v_s) + g_ds.cwiseProduct(h.d_s)).cwiseQuotient(g.scale);
    const Vec3 g_vl = g_vs.cwiseQuotient(h.axes), g_dl = g_ds.cwiseQuotient(h.axes);
    out.dposition = -(g.R * g_vl);
    const Mat3 dR = (origin - g.position) * g_vl.transpose() + dir * g_dl.transpose();
    out.dq = quat_rotation_backward(g.unit_q, dR);
    return out;
}

// project_gaussian -- core/src/geometry.cpp:107-136 (no frustum clamp)
std::optional<Splat2D> project_gaussian(const ActivatedGaussian& g, const CameraView& view) {
    const Vec3 pc = view.world_to_cam(g.position);
    if (pc.z() <= kNearPlane) return std::nullopt;
    const Scalar x = pc.x(), y = pc.y(), z = pc.z();
    Splat2D s;
    s.center = Vec2(view.fx * x / z + view.cx, view.fy * y / z + view.cy);
    s.sort_depth = z;
    Mat23 J;
    J << view.fx / z, 0, -view.fx * x / (z * z), 0, view.fy / z, -view.fy * y / (z * z);
    const Mat3 V = g.R * g.scale.cwiseProduct(g.scale).asDiagonal() * g.R.transpose();
    const Mat23 T = J * view.R_world_to_cam;
    s.cov = T * V * T.transpose();
    s.cov(0, 0) += kCovarianceFloor;
    s.cov(1, 1) += kCovarianceFloor;
    const Scalar det = s.cov.determinant();
    if (det <= 0) return std::nullopt;
    s.conic << s.cov(1, 1) / det, -s.cov(0, 1) / det, -s.cov(0, 1) / det, s.cov(0, 0) / det;
    const Scalar mid = 0.5 * (s.cov(0, 0) + s.cov(1, 1));
    s.radius = 3.0 * std::sqrt(mid + std::sqrt(std::max(Scalar(0.1), mid * mid - det)));
    return s;
}

// eval_alpha_full -- core/src/geometry.cpp:138-156
AlphaEval eval_alpha_full(const Splat2D& s, Scalar alpha, Scalar px, Scalar py) {
    AlphaEval e;
    e.dx = px - s.center.x();
    e.dy = py - s.center.y();
    const Scalar power = -0.5 * (s.conic(0, 0) * e.dx * e.dx + s.conic(1, 1) * e.dy * e.dy) - s.conic(0, 1) * e.dx * e.dy;
    if (power > 0) return e;
    e.gauss = std::exp(power);
    const Scalar raw = alpha * e.gauss;
    e.clamped = raw > kMaxAlpha;
    e.alpha = e.clamped ? kMaxAlpha : raw;
    return e;
}

Scalar eval_alpha(const Splat2D& s, Scalar alpha, Scalar px, Scalar py) { return eval_alpha_full(s, alpha, px, py).alpha; }

// Declared (but never defined) by the reference API; the rect rule of
// bin_and_sort (core/src/rasterizer.cpp:32-35).
PixelRect splat_pixel_rect(const Splat2D& s, int width, int height) {
    PixelRect r;
    r.x0 = std::max(0, int(std::floor(s.center.x() - s.radius)));
    r.x1 = std::min(width - 1, int(std::floor(s.center.x() + s.radius)));
    r.y0 = std::max(0, int(std::floor(s.center.y() - s.radius)));
    r.y1 = std::min(height - 1, int(std::floor(s.center.y() + s.radius)));
    return r;
}

// ---------------------------------------------------------------- SH
namespace {
constexpr Scalar C0 = 0.28209479177387814, C1 = 0.4886025119029199;
constexpr Scalar C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
                          0.5462742152960396};
constexpr Scalar C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
                          -0.4570457994644658, 1.445305721320277, -0.5900435899266435};
}  // namespace

// sh_basis -- core/src/sh.cpp:15-43
VecX sh_basis(int degree, const Vec3& d) {
    const Scalar x = d.x(), y = d.y(), z = d.z();
    VecX b((degree + 1) * (degree + 1));
    b[0] = C0;
    if (degree >= 1) {
        b[1] = -C1 * y;
        b[2] = C1 * z;
        b[3] = -C1 * x;
    }
    if (degree >= 2) {
        const Scalar xx = x * x, yy = y * y, zz = z * z;
        b[4] = C2[0] * x * y;
        b[5] = C2[1] * y * z;
        b[6] = C2[2] * (2 * zz - xx - yy);
        b[7] = C2[3] * x * z;
        b[8] = C2[4] * (xx - yy);
        if (degree >= 3) {
            b[9] = C3[0] * y * (3 * xx - yy);
            b[10] = C3[1] * x * y * z;
            b[11] = C3[2] * y * (4 * zz - xx - yy);
            b[12] = C3[3] * z * (2 * zz - 3 * xx - 3 * yy);
            b[13] = C3[4] * x * (4 * zz - xx - yy);
            b[14] = C3[5] * z * (xx - yy);
            b[15] = C3[6] * x * (xx - 3 * yy);
        }
    }
    return b;
}

// sh_basis_jacobian -- core/src/sh.cpp:45-73
Eigen::Matrix<Scalar, Eigen::Dynamic, 3> sh_basis_jacobian(int degree, const Vec3& d) {
    const Scalar x = d.x(), y = d.y(), z = d.z();
    Eigen::Matrix<Scalar, Eigen::Dynamic, 3> J((degree + 1) * (degree + 1), 3);
    J.setZero();
    if (degree >= 1) {
        J.row(1) << 0, -C1, 0;
        J.row(2) << 0, 0, C1;
        J.row(3) << -C1, 0, 0;
    }
    if (degree >= 2) {
        const Scalar xx = x * x, yy = y * y, zz = z * z;
        J.row(4) << C2[0] * y, C2[0] * x, 0;
        J.row(5) << 0, C2[1] * z, C2[1] * y;
        J.row(6) << -2 * C2[2] * x, -2 * C2[2] * y, 4 * C2[2] * z;
        J.row(7) << C2[3] * z, 0, C2[3] * x;
        J.row(8) << 2 * C2[4] * x, -2 * C2[4] * y, 0;
        if (degree >= 3) {
            J.row(9) << C3[0] * 6 * x * y, C3[0] * (3 * xx - 3 * yy), 0;
            J.row(10) << C3[1] * y * z, C3[1] * x * z, C3[1] * x * y;
            J.row(11) << -2 * C3[2] * x * y, C3[2] * (4 * zz - xx - 3 * yy), 8 * C3[2] * y * z;
            J.row(12) << -6 * C3[3] * x * z, -6 * C3[3] * y * z, C3[3] * (6 * zz - 3 * xx - 3 * yy);
            J.row(13) << C3[4] * (4 * zz - 3 * xx - yy), -2 * C3[4] * x * y, 8 * C3[4] * x * z;
            J.row(14) << 2 * C3[5] * x * z, -2 * C3[5] * y * z, C3[5] * (xx - yy);
            J.row(15) << C3[6] * (3 * xx - 3 * yy), -6 * C3[6] * x * y, 0;
        }
    }
    return J;
}

ShColor eval_sh_color(const ShMatrix& sh, int degree, const Vec3& dir) {
    const Vec3 raw = sh * sh_basis(degree, dir) + Vec3::Constant(0.5);
    ShColor out;
    for (int c = 0; c < 3; ++c) {
        out.clamped[c] = raw[c] < 0;
        out.rgb[c] = out.clamped[c] ? 0.0 : raw[c];
    }
    return out;
}

ShColorGrads eval_sh_color_backward(const ShMatrix& sh, int degree, const Vec3& dir, const ShColor& color,
                                    const Vec3& dL_drgb) {
    Vec3 g = dL_drgb;
    for (int c = 0; c < 3; ++c)
        if (color.clamped[c]) g[c] = 0;
    ShColorGrads out;
    out.dsh = g * sh_basis(degree, dir).transpose();
    out.ddir = sh_basis_jacobian(degree, dir).transpose() * (sh.transpose() * g);
    return out;
}

Vec3 rgb_to_sh_dc(const Vec3& rgb) { return (rgb - Vec3::Constant(0.5)) / C0; }
Vec3 sh_dc_to_rgb(const Vec3& dc) { return C0 * dc + Vec3::Constant(0.5); }

// -------------------------------------------------------------- normals
// backproject -- core/src/normals.cpp:16-26
std::vector<Vec3> backproject(const GridF& depth, const CameraView& view) {
    if (depth.width() != view.width || depth.height() != view.height || depth.channels() != 1)
        throw std::invalid_argument("backproject: depth map does not match the view");
    std::vector<Vec3> out(size_t(view.width) * view.height);
    for (int y = 0; y < view.height; ++y)
        for (int x = 0; x < view.width; ++x) {
            const Vec3 pd((x + 0.5 - view.cx) / view.fx, (y + 0.5 - view.cy) / view.fy, 1.0);
            out[size_t(y) * view.width + x] = view.cam_to_world(pd * depth.at(x, y));
        }
    return out;
}

// --------------------------------------------------------------- oracle
// brute_force_render -- core/src/oracle.cpp:13-91: every Gaussian at every
// pixel in global (depth, index) order, same blend rule; host double.
MultimodalFrame brute_force_render(const Scene& scene, const CameraView& view, const RenderConfig& cfg) {
    scene.validate();
    const int W = view.width, H = view.height, C = scene.num_classes;
    MultimodalFrame f;
    f.width = W;
    f.height = H;
    f.num_classes = C;
    f.color = GridF(W, H, 3, 0.0);
    f.depth = GridF(W, H, 1, 0.0);
    f.semantics = GridF(W, H, C, 0.0);
    f.kmap = GridF(W, H, 1, 0.0);
    f.transmittance = GridF(W, H, 1, 1.0);
    f.normals = GridF(W, H, 3, 0.0);
    f.contributors = Grid<int>(W, H, 1, 0);
    const auto act = activate_scene(scene);
    std::vector<std::optional<Splat2D>> sp(scene.size());
    std::vector<Vec3> rgb(scene.size(), Vec3::Zero());
    std::vector<int> order;
    for (size_t i = 0; i < scene.size(); ++i) {
        sp[i] = project_gaussian(act[i], view);
        if (!sp[i]) continue;
        order.push_back(int(i));
        const Vec3 to_g = act[i].position - view.t_cam_to_world;
        const Scalar n = to_g.norm();
        rgb[i] = eval_sh_color(*act[i].sh, scene.sh_degree, n > 1e-12 ? Vec3(to_g / n) : Vec3(0, 0, 1)).rgb;
    }
    std::sort(order.begin(), order.end(), [&](int a, int b) {
        const Scalar da = sp[a]->sort_depth, db = sp[b]->sort_depth;
        return da != db ? da < db : a < b;
    });
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            Vec3 o, d;
            compute_ray(view, x + 0.5, y + 0.5, o, d);
            Vec3 col = Vec3::Zero();
            Scalar dep = 0, kk = 0, T = 1.0;
            std::vector<Scalar> sem(C, 0.0);
            int count = 0;
            for (int idx : order) {
                const Scalar a = eval_alpha(*sp[idx], act[idx].alpha, x + 0.5, y + 0.5);
                if (a < kMinAlpha) continue;
                const auto hit = intersect(act[idx], o, d, cfg.sigma_scale);
                const Scalar dd = hit ? midpoint_depth(view, o, d, hit->t_mid) : sp[idx]->sort_depth;
                const Scalar w = a * T;
                col += w * rgb[idx];
                dep += w * dd;
                for (int ch = 0; ch < C; ++ch) sem[ch] += w * (*act[idx].semantic_logits)[ch];
                kk += w * act[idx].k;
                T *= (1.0 - a);
                ++count;
                if (cfg.early_termination && T < cfg.early_stop_transmittance) break;
            }
            col += T * cfg.background;
            for (int ch = 0; ch < 3; ++ch) f.color.at(x, y, ch) = col[ch];
            f.depth.at(x, y) = dep;
            for (int ch = 0; ch < C; ++ch) f.semantics.at(x, y, ch) = sem[ch];
            f.kmap.at(x, y) = kk;
            f.transmittance.at(x, y) = T;
            f.contributors.at(x, y) = count;
        }
    return f;
}

// finite_diff -- core/src/oracle.cpp:93-105
VecX finite_diff(const std::function<Scalar(const VecX&)>& fn, const VecX& theta, Scalar eps) {
    VecX grad(theta.size());
    VecX probe = theta;
    for (int i = 0; i < theta.size(); ++i) {
        probe[i] = theta[i] + eps;
        const Scalar hi = fn(probe);
        probe[i] = theta[i] - eps;
        const Scalar lo = fn(probe);
        probe[i] = theta[i];
        grad[i] = (hi - lo) / (2 * eps);
    }
    return grad;
}

}  // namespace msplat
