/*
 * msplat_oracle.c -- plain-C double-precision restatement of the UniGS
 * multimodal rasterizer hot path.  TEST INFRASTRUCTURE ONLY (see
 * msplat_oracle.h): the CUDA product never links or calls this file.
 *
 * Every function follows the reference line by line and in the same floating
 * point evaluation order (left-to-right sums, no FMA: built with
 * -ffp-contract=off), so that it is bitwise identical to the reference sources
 * compiled against third_party/eigen_subset (oracle/_ref).  Citations are
 * relative to /root/reference/proj.
 *
 * Single-threaded: equivalent to RenderConfig::threads == 1, the reference
 * default (core/include/msplat/rasterizer.hpp:18).
 */
#include "msplat_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>



#define TILE 16
static const double kNearPlane = 0.01;       /* geometry.hpp:306 (line 30 of the header) */
static const double kCovFloor = 0.3;
static const double kMinAlpha = 1.0 / 255.0;
static const double kMaxAlpha = 0.99;
static const double kDegenerateScale = 1e-8; /* geometry.hpp:273 */

static __thread char g_err[512];

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

const char* mo_last_error(void) { return g_err; }
const char* mo_impl_name(void) { return "c-restatement"; }

/* ---------------------------------------------------------------- camera */
typedef struct {
    double fx, fy, cx, cy;
    int W, H;
    double Rc2w[9], tc2w[3], Rw2c[9], tw2c[3];
} cam_t;

/* CameraView::finalize (core/src/camera.cpp:8-21) */
static int make_cam(const mo_camera* c, cam_t* o) {
    o->fx = c->fx; o->fy = c->fy; o->cx = c->cx; o->cy = c->cy;
    o->W = c->width; o->H = c->height;
    memcpy(o->Rc2w, c->R_c2w, sizeof o->Rc2w);
    memcpy(o->tc2w, c->t_c2w, sizeof o->tc2w);
    if (o->W < 1 || o->H < 1)
        return fail(1, "CameraView: width and height must be >= 1");
    if (!(o->fx > 0) || !(o->fy > 0))
        return fail(1, "CameraView: focal lengths must be positive");
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            o->Rw2c[i * 3 + j] = o->Rc2w[j * 3 + i];
    for (int i = 0; i < 3; ++i) {
        double s = o->Rw2c[i * 3 + 0] * o->tc2w[0];
        s += o->Rw2c[i * 3 + 1] * o->tc2w[1];
        s += o->Rw2c[i * 3 + 2] * o->tc2w[2];
        o->tw2c[i] = -s;
    }
    return 0;
}

static inline void mat3_vec(const double* M, const double* v, double* out) {
    for (int i = 0; i < 3; ++i) {
        double s = M[i * 3 + 0] * v[0];
        s += M[i * 3 + 1] * v[1];
        s += M[i * 3 + 2] * v[2];
        out[i] = s;
    }
}
/* M^T v */
static inline void mat3t_vec(const double* M, const double* v, double* out) {
    for (int i = 0; i < 3; ++i) {
        double s = M[0 * 3 + i] * v[0];
        s += M[1 * 3 + i] * v[1];
        s += M[2 * 3 + i] * v[2];
        out[i] = s;
    }
}
static inline double dot3(const double* a, const double* b) {
    double s = a[0] * b[0];
    s += a[1] * b[1];
    s += a[2] * b[2];
    return s;
}
static inline void cross3(const double* a, const double* b, double* o) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}
/* Eigen::normalized(): v / sqrt(|v|^2) when |v|^2 > 0 */
static inline void normalized3(const double* v, double* o) {
    const double z = dot3(v, v);
    if (z > 0) {
        const double n = sqrt(z);
        o[0] = v[0] / n; o[1] = v[1] / n; o[2] = v[2] / n;
    } else {
        o[0] = v[0]; o[1] = v[1]; o[2] = v[2];
    }
}

/* compute_ray (core/src/geometry.cpp:31-35) */
static void compute_ray(const cam_t* c, double u, double v, double* origin, double* dir) {
    origin[0] = c->tc2w[0]; origin[1] = c->tc2w[1]; origin[2] = c->tc2w[2];
    const double pd[3] = {(u - c->cx) / c->fx, (v - c->cy) / c->fy, 1.0};
    double r[3];
    mat3_vec(c->Rc2w, pd, r);
    normalized3(r, dir);
}

/* ----------------------------------------------------------- activation */
typedef struct {
    double pos[3], q[4], R[9], s[3], alpha, k;
    const double *sh, *sem;
} act_t;

static int all_finite(const mo_scene* S, int64_t i) {
    const int K = (S->sh_degree + 1) * (S->sh_degree + 1), C = S->num_classes;
    for (int j = 0; j < 3; ++j)
        if (!isfinite(S->means[i * 3 + j]) || !isfinite(S->log_scales[i * 3 + j])) return 0;
    for (int j = 0; j < 4; ++j)
        if (!isfinite(S->quats[i * 4 + j])) return 0;
    if (!isfinite(S->opacity_logits[i]) || !isfinite(S->k[i])) return 0;
    for (int j = 0; j < 3 * K; ++j)
        if (!isfinite(S->sh[i * 3 * K + j])) return 0;
    for (int j = 0; j < C; ++j)
        if (!isfinite(S->semantics[i * C + j])) return 0;
    return 1;
}

/* quat_to_rotation (core/src/geometry.cpp:7-15) */
static void quat_to_rotation(const double* q, double* R) {
    double n2 = q[0] * q[0];
    n2 += q[1] * q[1];
    n2 += q[2] * q[2];
    n2 += q[3] * q[3];
    const double n = sqrt(n2);
    const double w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
    R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z); R[2] = 2 * (x * z + w * y);
    R[3] = 2 * (x * y + w * z); R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
    R[6] = 2 * (x * z - w * y); R[7] = 2 * (y * z + w * x); R[8] = 1 - 2 * (x * x + y * y);
}

/* activate (core/src/scene.cpp:42-60) */
static int activate(const mo_scene* S, int64_t i, act_t* a) {
    if (!all_finite(S, i))
        return fail(1, "activate: primitive %lld has non-finite fields", (long long)i);
    const double* q = S->quats + i * 4;
    double n2 = q[0] * q[0];
    n2 += q[1] * q[1];
    n2 += q[2] * q[2];
    n2 += q[3] * q[3];
    const double norm = sqrt(n2);
    if (norm < 1e-12)
        return fail(1, "activate: primitive %lld has a zero quaternion", (long long)i);
    for (int j = 0; j < 3; ++j) a->pos[j] = S->means[i * 3 + j];
    for (int j = 0; j < 4; ++j) a->q[j] = q[j] / norm;
    quat_to_rotation(a->q, a->R);
    for (int j = 0; j < 3; ++j) a->s[j] = exp(S->log_scales[i * 3 + j]);
    a->alpha = 1.0 / (1.0 + exp(-S->opacity_logits[i]));
    const int K = (S->sh_degree + 1) * (S->sh_degree + 1);
    a->sh = S->sh + i * 3 * K;
    a->sem = S->semantics + i * S->num_classes;
    a->k = S->k[i];
    return 0;
}

/* Scene::validate (core/src/scene.cpp:22-40); shapes are implied by the flat layout. */
static int validate(const mo_scene* S) {
    if (S->sh_degree < 0 || S->sh_degree > 3)
        return fail(1, "Scene: sh_degree must be in [0,3]");
    if (S->num_classes < 0)
        return fail(1, "Scene: num_classes must be >= 0");
    for (int64_t i = 0; i < S->n; ++i)
        if (!all_finite(S, i))
            return fail(1, "Scene: primitive %lld has non-finite fields", (long long)i);
    return 0;
}

/* ------------------------------------------------------------------ SH */
static const double kC0 = 0.28209479177387814;
static const double kC1 = 0.4886025119029199;
static const double kC2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                              -1.0925484305920792, 0.5462742152960396};
static const double kC3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                              0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                              -0.5900435899266435};

/* sh_basis (core/src/sh.cpp:15-43) */
static void sh_basis(int deg, const double* d, double* b) {
    const double x = d[0], y = d[1], z = d[2];
    b[0] = kC0;
    if (deg >= 1) { b[1] = -kC1 * y; b[2] = kC1 * z; b[3] = -kC1 * x; }
    if (deg >= 2) {
        const double xx = x * x, yy = y * y, zz = z * z;
        b[4] = kC2[0] * x * y;
        b[5] = kC2[1] * y * z;
        b[6] = kC2[2] * (2 * zz - xx - yy);
        b[7] = kC2[3] * x * z;
        b[8] = kC2[4] * (xx - yy);
    }
    if (deg >= 3) {
        const double xx = x * x, yy = y * y, zz = z * z;
        b[9] = kC3[0] * y * (3 * xx - yy);
        b[10] = kC3[1] * x * y * z;
        b[11] = kC3[2] * y * (4 * zz - xx - yy);
        b[12] = kC3[3] * z * (2 * zz - 3 * xx - 3 * yy);
        b[13] = kC3[4] * x * (4 * zz - xx - yy);
        b[14] = kC3[5] * z * (xx - yy);
        b[15] = kC3[6] * x * (xx - 3 * yy);
    }
}

/* sh_basis_jacobian (core/src/sh.cpp:45-73), J[K][3] */
static void sh_jacobian(int deg, const double* d, double* J) {
    const double x = d[0], y = d[1], z = d[2];
    const int K = (deg + 1) * (deg + 1);
    for (int i = 0; i < K * 3; ++i) J[i] = 0;
#define ROW(r, a, b, c) do { J[(r)*3+0] = (a); J[(r)*3+1] = (b); J[(r)*3+2] = (c); } while (0)
    if (deg >= 1) { ROW(1, 0, -kC1, 0); ROW(2, 0, 0, kC1); ROW(3, -kC1, 0, 0); }
    if (deg >= 2) {
        const double xx = x * x, yy = y * y, zz = z * z;
        ROW(4, kC2[0] * y, kC2[0] * x, 0);
        ROW(5, 0, kC2[1] * z, kC2[1] * y);
        ROW(6, -2 * kC2[2] * x, -2 * kC2[2] * y, 4 * kC2[2] * z);
        ROW(7, kC2[3] * z, 0, kC2[3] * x);
        ROW(8, 2 * kC2[4] * x, -2 * kC2[4] * y, 0);
        if (deg >= 3) {
            ROW(9, kC3[0] * 6 * x * y, kC3[0] * (3 * xx - 3 * yy), 0);
            ROW(10, kC3[1] * y * z, kC3[1] * x * z, kC3[1] * x * y);
            ROW(11, -2 * kC3[2] * x * y, kC3[2] * (4 * zz - xx - 3 * yy), 8 * kC3[2] * y * z);
            ROW(12, -6 * kC3[3] * x * z, -6 * kC3[3] * y * z, kC3[3] * (6 * zz - 3 * xx - 3 * yy));
            ROW(13, kC3[4] * (4 * zz - 3 * xx - yy), -2 * kC3[4] * x * y, 8 * kC3[4] * x * z);
            ROW(14, 2 * kC3[5] * x * z, -2 * kC3[5] * y * z, kC3[5] * (xx - yy));
            ROW(15, kC3[6] * (3 * xx - 3 * yy), -6 * kC3[6] * x * y, 0);
        }
    }
#undef ROW
}

/* eval_sh_color (core/src/sh.cpp:75-84) */
static void eval_sh_color(const double* sh, int deg, const double* dir, double* rgb,
                          unsigned char* clamped) {
    double b[16];
    sh_basis(deg, dir, b);
    const int K = (deg + 1) * (deg + 1);
    for (int c = 0; c < 3; ++c) {
        double s = sh[c * K] * b[0];
        for (int j = 1; j < K; ++j) s += sh[c * K + j] * b[j];
        const double raw = s + 0.5;
        clamped[c] = raw < 0;
        rgb[c] = clamped[c] ? 0.0 : raw;
    }
}

/* ------------------------------------------------------------ projection */
typedef struct {
    double center[2], cov[4], conic[4], depth, radius;
} splat_t;

/* (R diag(s*s)) R^T, as the reference evaluates it (geometry.cpp:118) */
static void world_cov(const double* R, const double* s, double* V) {
    double RD[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) RD[i * 3 + j] = R[i * 3 + j] * (s[j] * s[j]);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double acc = RD[i * 3 + 0] * R[j * 3 + 0];
            acc += RD[i * 3 + 1] * R[j * 3 + 1];
            acc += RD[i * 3 + 2] * R[j * 3 + 2];
            V[i * 3 + j] = acc;
        }
}

/* project_gaussian (core/src/geometry.cpp:107-136).  Returns 1 when visible. */
static int project_gaussian(const act_t* g, const cam_t* c, splat_t* sp) {
    double pc[3];
    mat3_vec(c->Rw2c, g->pos, pc);
    pc[0] += c->tw2c[0]; pc[1] += c->tw2c[1]; pc[2] += c->tw2c[2];
    if (pc[2] <= kNearPlane) return 0;
    const double x = pc[0], y = pc[1], z = pc[2];
    sp->center[0] = c->fx * x / z + c->cx;
    sp->center[1] = c->fy * y / z + c->cy;
    sp->depth = z;
    const double J[6] = {c->fx / z, 0, -c->fx * x / (z * z), 0, c->fy / z, -c->fy * y / (z * z)};
    double V[9];
    world_cov(g->R, g->s, V);
    double T[6];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j) {
            double acc = J[i * 3 + 0] * c->Rw2c[0 * 3 + j];
            acc += J[i * 3 + 1] * c->Rw2c[1 * 3 + j];
            acc += J[i * 3 + 2] * c->Rw2c[2 * 3 + j];
            T[i * 3 + j] = acc;
        }
    double TV[6];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j) {
            double acc = T[i * 3 + 0] * V[0 * 3 + j];
            acc += T[i * 3 + 1] * V[1 * 3 + j];
            acc += T[i * 3 + 2] * V[2 * 3 + j];
            TV[i * 3 + j] = acc;
        }
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) {
            double acc = TV[i * 3 + 0] * T[j * 3 + 0];
            acc += TV[i * 3 + 1] * T[j * 3 + 1];
            acc += TV[i * 3 + 2] * T[j * 3 + 2];
            sp->cov[i * 2 + j] = acc;
        }
    sp->cov[0] += kCovFloor;
    sp->cov[3] += kCovFloor;
    const double det = sp->cov[0] * sp->cov[3] - sp->cov[2] * sp->cov[1];
    if (det <= 0) return 0;
    sp->conic[0] = sp->cov[3] / det;
    sp->conic[1] = -sp->cov[1] / det;
    sp->conic[2] = -sp->cov[1] / det;
    sp->conic[3] = sp->cov[0] / det;
    const double mid = 0.5 * (sp->cov[0] + sp->cov[3]);
    const double m2 = mid * mid - det;
    const double lambda_max = mid + sqrt(0.1 < m2 ? m2 : 0.1);
    sp->radius = 3.0 * sqrt(lambda_max);
    return 1;
}

/* eval_alpha_full (core/src/geometry.cpp:138-152) */
typedef struct { double alpha, gauss, dx, dy; int clamped; } alpha_t;
static alpha_t eval_alpha(const splat_t* sp, double opacity, double px, double py) {
    alpha_t o = {0, 0, 0, 0, 0};
    o.dx = px - sp->center[0];
    o.dy = py - sp->center[1];
    const double power = -0.5 * (sp->conic[0] * o.dx * o.dx + sp->conic[3] * o.dy * o.dy) -
                         sp->conic[1] * o.dx * o.dy;
    if (power > 0) return o;
    o.gauss = exp(power);
    const double raw = opacity * o.gauss;
    o.clamped = raw > kMaxAlpha;
    o.alpha = o.clamped ? kMaxAlpha : raw;
    return o;
}

/* intersect (core/src/geometry.cpp:37-64) */
typedef struct { double t_mid, a, b, vs[3], ds[3], axes[3]; } hit_t;
static int intersect(const act_t* g, const double* o, const double* d, double sigma, hit_t* h) {
    for (int j = 0; j < 3; ++j) h->axes[j] = sigma * g->s[j];
    double mn = h->axes[0];
    if (h->axes[1] < mn) mn = h->axes[1];
    if (h->axes[2] < mn) mn = h->axes[2];
    if (mn < kDegenerateScale) return 0;
    const double rel[3] = {o[0] - g->pos[0], o[1] - g->pos[1], o[2] - g->pos[2]};
    double vl[3], dl[3];
    mat3t_vec(g->R, rel, vl);
    mat3t_vec(g->R, d, dl);
    for (int j = 0; j < 3; ++j) { h->vs[j] = vl[j] / h->axes[j]; h->ds[j] = dl[j] / h->axes[j]; }
    h->a = dot3(h->ds, h->ds);
    h->b = 2.0 * dot3(h->vs, h->ds);
    const double c = dot3(h->vs, h->vs) - 1.0;
    const double disc = h->b * h->b - 4.0 * h->a * c;
    if (disc < 0 || h->a <= 0) return 0;
    h->t_mid = -h->b / (2.0 * h->a);
    if (h->t_mid <= 0) return 0;
    return 1;
}

/* midpoint_depth (core/src/geometry.cpp:66-68) */
static double midpoint_depth(const cam_t* c, const double* o, const double* d, double t) {
    const double p[3] = {o[0] + t * d[0], o[1] + t * d[1], o[2] + t * d[2]};
    return dot3(c->Rw2c + 6, p) + c->tw2c[2];
}

/* quat_rotation_backward (core/src/geometry.cpp:17-29), G row-major */
static void quat_rotation_backward(const double* q, const double* G, double* dq) {
    const double w = q[0], x = q[1], y = q[2], z = q[3];
#define g(i, j) G[(i)*3 + (j)]
    dq[0] = 2 * (g(0, 1) * (-z) + g(0, 2) * y + g(1, 0) * z + g(1, 2) * (-x) + g(2, 0) * (-y) +
                 g(2, 1) * x);
    dq[1] = 2 * (g(0, 1) * y + g(0, 2) * z + g(1, 0) * y + g(1, 1) * (-2 * x) + g(1, 2) * (-w) +
                 g(2, 0) * z + g(2, 1) * w + g(2, 2) * (-2 * x));
    dq[2] = 2 * (g(0, 0) * (-2 * y) + g(0, 1) * x + g(0, 2) * w + g(1, 0) * x + g(1, 2) * z +
                 g(2, 0) * (-w) + g(2, 1) * z + g(2, 2) * (-2 * y));
    dq[3] = 2 * (g(0, 0) * (-2 * z) + g(0, 1) * (-w) + g(0, 2) * x + g(1, 0) * w +
                 g(1, 1) * (-2 * z) + g(1, 2) * y + g(2, 0) * x + g(2, 1) * y);
#undef g
}

/* intersection_backward (core/src/geometry.cpp:70-105); adds into out[10]
 * = dposition[3], dq[4], dscale[3]. */
static void intersection_backward(const hit_t* h, double dL_dd, const cam_t* c, const double* o,
                                  const double* d, const act_t* g, double* dpos, double* dq,
                                  double* ds) {
    dpos[0] = dpos[1] = dpos[2] = 0;
    dq[0] = dq[1] = dq[2] = dq[3] = 0;
    ds[0] = ds[1] = ds[2] = 0;
    if (fabs(h->a) < 1e-12) return;
    if (dL_dd == 0) return;
    const double dd_dt = dot3(c->Rw2c + 6, d);
    const double g_t = dL_dd * dd_dt;
    double gvs[3], gds[3], gvl[3], gdl[3];
    for (int j = 0; j < 3; ++j) {
        gvs[j] = g_t * (-h->ds[j] / h->a);
        gds[j] = g_t * ((h->b / (h->a * h->a)) * h->ds[j] - h->vs[j] / h->a);
    }
    for (int j = 0; j < 3; ++j) ds[j] = -((gvs[j] * h->vs[j] + gds[j] * h->ds[j]) / g->s[j]);
    for (int j = 0; j < 3; ++j) { gvl[j] = gvs[j] / h->axes[j]; gdl[j] = gds[j] / h->axes[j]; }
    double Rg[3];
    mat3_vec(g->R, gvl, Rg);
    for (int j = 0; j < 3; ++j) dpos[j] = -Rg[j];
    const double v[3] = {o[0] - g->pos[0], o[1] - g->pos[1], o[2] - g->pos[2]};
    double G[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) G[i * 3 + j] = v[i] * gvl[j] + d[i] * gdl[j];
    quat_rotation_backward(g->q, G, dq);
}

/* ---------------------------------------------------------- view prepare */
typedef struct {
    int64_t n;
    act_t* act;
    splat_t* sp;
    unsigned char* vis;
    double* rgb;
    unsigned char* clamped;
} view_t;

static void free_view(view_t* v) {
    free(v->act); free(v->sp); free(v->vis); free(v->rgb); free(v->clamped);
    memset(v, 0, sizeof *v);
}

/* prepare_view (core/src/rasterizer.cpp:55-74) */
static int prepare_view(const mo_scene* S, const cam_t* c, view_t* v) {
    memset(v, 0, sizeof *v);
    const int64_t n = S->n;
    v->n = n;
    v->act = (act_t*)calloc(n ? n : 1, sizeof(act_t));
    v->sp = (splat_t*)calloc(n ? n : 1, sizeof(splat_t));
    v->vis = (unsigned char*)calloc(n ? n : 1, 1);
    v->rgb = (double*)calloc(n ? 3 * n : 1, sizeof(double));
    v->clamped = (unsigned char*)calloc(n ? 3 * n : 1, 1);
    for (int64_t i = 0; i < n; ++i) {
        int st = activate(S, i, &v->act[i]);
        if (st) { free_view(v); return st; }
        const act_t* a = &v->act[i];
        v->vis[i] = (unsigned char)project_gaussian(a, c, &v->sp[i]);
        if (v->vis[i]) {
            const double tg[3] = {a->pos[0] - c->tc2w[0], a->pos[1] - c->tc2w[1],
                                  a->pos[2] - c->tc2w[2]};
            const double nrm = sqrt(dot3(tg, tg));
            double dir[3] = {0, 0, 1};
            if (nrm > 1e-12) { dir[0] = tg[0] / nrm; dir[1] = tg[1] / nrm; dir[2] = tg[2] / nrm; }
            eval_sh_color(a->sh, S->sh_degree, dir, v->rgb + 3 * i, v->clamped + 3 * i);
        }
    }
    return 0;
}

/* ------------------------------------------------------------- binning */
/* x86 double->int conversion: out-of-range and NaN give INT_MIN, which the
 * reference's int(std::floor(..)) produces on this platform (rasterizer.cpp:32-35). */
static inline int floor_to_int(double v) {
    const double f = floor(v);
    if (!(f >= -2147483648.0 && f < 2147483648.0)) return (int)0x80000000;
    return (int)f;
}

typedef struct { const splat_t* sp; } sort_ctx_t;
static const splat_t* g_sort_sp;
static int cmp_depth(const void* pa, const void* pb) {
    const int a = *(const int*)pa, b = *(const int*)pb;
    const double da = g_sort_sp[a].depth, db = g_sort_sp[b].depth;
    if (da != db) return da < db ? -1 : 1;
    return a < b ? -1 : (a > b);
}

typedef struct {
    int tiles_x, tiles_y;
    int64_t* off; /* [tiles+1] */
    int32_t* val;
    int64_t count;
} bins_t;

/* bin_and_sort (core/src/rasterizer.cpp:14-45) */
static int bin_and_sort(int64_t n, const unsigned char* vis, const splat_t* sp, int W, int H,
                        bins_t* b) {
    b->tiles_x = (W + TILE - 1) / TILE;
    b->tiles_y = (H + TILE - 1) / TILE;
    const int64_t tiles = (int64_t)b->tiles_x * b->tiles_y;
    int* order = (int*)malloc(sizeof(int) * (n ? n : 1));
    int64_t m = 0;
    for (int64_t i = 0; i < n; ++i)
        if (vis[i]) order[m++] = (int)i;
    g_sort_sp = sp;
    qsort(order, m, sizeof(int), cmp_depth); /* total order: no ties survive (idx) */
    int* rect = (int*)malloc(sizeof(int) * 4 * (m ? m : 1));
    int64_t* cnt = (int64_t*)calloc(tiles + 1, sizeof(int64_t));
    for (int64_t r = 0; r < m; ++r) {
        const splat_t* s = &sp[order[r]];
        int x0 = floor_to_int(s->center[0] - s->radius);
        int x1 = floor_to_int(s->center[0] + s->radius);
        int y0 = floor_to_int(s->center[1] - s->radius);
        int y1 = floor_to_int(s->center[1] + s->radius);
        x0 = x0 > 0 ? x0 : 0;
        x1 = x1 < W - 1 ? x1 : W - 1;
        y0 = y0 > 0 ? y0 : 0;
        y1 = y1 < H - 1 ? y1 : H - 1;
        int* R = rect + 4 * r;
        if (x1 < x0 || y1 < y0) { R[0] = 1; R[1] = 0; R[2] = 1; R[3] = 0; continue; }
        R[0] = x0 / TILE; R[1] = x1 / TILE; R[2] = y0 / TILE; R[3] = y1 / TILE;
        for (int ty = R[2]; ty <= R[3]; ++ty)
            for (int tx = R[0]; tx <= R[1]; ++tx) cnt[(int64_t)ty * b->tiles_x + tx + 1]++;
    }
    b->off = (int64_t*)malloc(sizeof(int64_t) * (tiles + 1));
    b->off[0] = 0;
    for (int64_t t = 0; t < tiles; ++t) b->off[t + 1] = b->off[t] + cnt[t + 1];
    b->count = b->off[tiles];
    b->val = (int32_t*)malloc(sizeof(int32_t) * (b->count ? b->count : 1));
    int64_t* fillp = cnt; /* reuse as cursor */
    for (int64_t t = 0; t < tiles; ++t) fillp[t] = b->off[t];
    for (int64_t r = 0; r < m; ++r) {
        const int* R = rect + 4 * r;
        for (int ty = R[2]; ty <= R[3]; ++ty)
            for (int tx = R[0]; tx <= R[1]; ++tx)
                b->val[fillp[(int64_t)ty * b->tiles_x + tx]++] = order[r];
    }
    free(order); free(rect); free(cnt);
    return 0;
}

static void free_bins(bins_t* b) { free(b->off); free(b->val); memset(b, 0, sizeof *b); }

/* --------------------------------------------------------- public: pre */
int mo_preprocess(const mo_scene* S, const mo_camera* camera, uint8_t* visible, double* center,
                  double* cov, double* conic, double* sort_depth, double* radius, double* rgb,
                  uint8_t* clamped) {
    cam_t c;
    int st = make_cam(camera, &c);
    if (st) return st;
    if ((st = validate(S))) return st;
    view_t v;
    if ((st = prepare_view(S, &c, &v))) return st;
    for (int64_t i = 0; i < S->n; ++i) {
        if (visible) visible[i] = v.vis[i];
        if (center) { center[2 * i] = v.sp[i].center[0]; center[2 * i + 1] = v.sp[i].center[1]; }
        if (cov) for (int j = 0; j < 4; ++j) cov[4 * i + j] = v.sp[i].cov[j];
        if (conic) { conic[3 * i] = v.sp[i].conic[0]; conic[3 * i + 1] = v.sp[i].conic[1];
                     conic[3 * i + 2] = v.sp[i].conic[3]; }
        if (sort_depth) sort_depth[i] = v.sp[i].depth;
        if (radius) radius[i] = v.sp[i].radius;
        if (rgb) for (int j = 0; j < 3; ++j) rgb[3 * i + j] = v.rgb[3 * i + j];
        if (clamped) for (int j = 0; j < 3; ++j) clamped[3 * i + j] = v.clamped[3 * i + j];
    }
    free_view(&v);
    return 0;
}

int64_t mo_bin(int64_t n, const uint8_t* visible, const double* center, const double* radius,
               const double* sort_depth, int W, int H, int64_t* tile_offsets, int32_t* values,
               int64_t capacity) {
    splat_t* sp = (splat_t*)calloc(n ? n : 1, sizeof(splat_t));
    for (int64_t i = 0; i < n; ++i) {
        sp[i].center[0] = center[2 * i]; sp[i].center[1] = center[2 * i + 1];
        sp[i].radius = radius[i]; sp[i].depth = sort_depth[i];
    }
    bins_t b;
    bin_and_sort(n, visible, sp, W, H, &b);
    const int64_t tiles = (int64_t)b.tiles_x * b.tiles_y;
    if (tile_offsets) memcpy(tile_offsets, b.off, sizeof(int64_t) * (tiles + 1));
    if (values && capacity >= b.count) memcpy(values, b.val, sizeof(int32_t) * b.count);
    const int64_t count = b.count;
    free_bins(&b);
    free(sp);
    return count;
}

/* ------------------------------------------------------------- forward */
typedef struct {
    double *color, *depth, *sem, *kmap, *T;
    int32_t *contrib, *terminus;
    double* wsum;
} frame_out_t;

/* rasterize (core/src/rasterizer.cpp:87-205), threads == 1 */
static int render(const mo_scene* S, const cam_t* c, const mo_render_cfg* cfg, const view_t* v,
                  const bins_t* b, frame_out_t* f) {
    const int W = c->W, H = c->H, C = S->num_classes;
    double* sem = (double*)malloc(sizeof(double) * (C ? C : 1));
    for (int64_t tile = 0; tile < (int64_t)b->tiles_x * b->tiles_y; ++tile) {
        const int tx = (int)(tile % b->tiles_x), ty = (int)(tile / b->tiles_x);
        const int32_t* list = b->val + b->off[tile];
        const int64_t len = b->off[tile + 1] - b->off[tile];
        const int px0 = tx * TILE, py0 = ty * TILE;
        const int px1 = px0 + TILE < W ? px0 + TILE : W, py1 = py0 + TILE < H ? py0 + TILE : H;
        for (int y = py0; y < py1; ++y)
            for (int x = px0; x < px1; ++x) {
                double o[3], d[3];
                compute_ray(c, x + 0.5, y + 0.5, o, d);
                double col[3] = {0, 0, 0}, dep = 0, kk = 0, T = 1.0;
                for (int ch = 0; ch < C; ++ch) sem[ch] = 0;
                int count = 0, last = 0;
                for (int64_t pos = 0; pos < len; ++pos) {
                    const int idx = list[pos];
                    const splat_t* sp = &v->sp[idx];
                    const act_t* a = &v->act[idx];
                    const double alpha = eval_alpha(sp, a->alpha, x + 0.5, y + 0.5).alpha;
                    if (alpha < kMinAlpha) continue;
                    double dd;
                    hit_t h;
                    if (intersect(a, o, d, cfg->sigma_scale, &h))
                        dd = midpoint_depth(c, o, d, h.t_mid);
                    else
                        dd = sp->depth;
                    if (!isfinite(alpha) || !isfinite(dd)) {
                        free(sem);
                        return fail(2, "rasterize: non-finite blend at pixel (%d,%d), primitive %d",
                                    x, y, idx);
                    }
                    const double w = alpha * T;
                    for (int j = 0; j < 3; ++j) col[j] = col[j] + w * v->rgb[3 * idx + j];
                    dep += w * dd;
                    for (int ch = 0; ch < C; ++ch) sem[ch] += w * a->sem[ch];
                    kk += w * a->k;
                    if (f->wsum) f->wsum[idx] += w;
                    T *= (1.0 - alpha);
                    ++count;
                    last = (int)pos + 1;
                    if (cfg->early_termination && T < cfg->early_stop_transmittance) break;
                }
                for (int j = 0; j < 3; ++j) col[j] = col[j] + T * cfg->background[j];
                const size_t p = (size_t)y * W + x;
                if (f->color) for (int j = 0; j < 3; ++j) f->color[3 * p + j] = col[j];
                if (f->depth) f->depth[p] = dep;
                if (f->sem) for (int ch = 0; ch < C; ++ch) f->sem[p * C + ch] = sem[ch];
                if (f->kmap) f->kmap[p] = kk;
                if (f->T) f->T[p] = T;
                if (f->contrib) f->contrib[p] = count;
                if (f->terminus) f->terminus[p] = last;
                if (!isfinite(col[0]) || !isfinite(col[1]) || !isfinite(col[2]) || !isfinite(dep) ||
                    !isfinite(T)) {
                    free(sem);
                    return fail(2, "rasterize: non-finite output at pixel (%d,%d)", x, y);
                }
            }
    }
    free(sem);
    return 0;
}

int mo_render(const mo_scene* S, const mo_camera* camera, const mo_render_cfg* cfg, double* color,
              double* depth, double* semantics, double* kmap, double* transmittance,
              int32_t* contributors, int32_t* terminus, double* weight_sums) {
    cam_t c;
    int st = make_cam(camera, &c);
    if (st) return st;
    if ((st = validate(S))) return st;
    view_t v;
    if ((st = prepare_view(S, &c, &v))) return st;
    bins_t b;
    bin_and_sort(S->n, v.vis, v.sp, c.W, c.H, &b);
    if (weight_sums) memset(weight_sums, 0, sizeof(double) * S->n);
    frame_out_t f = {color, depth, semantics, kmap, transmittance, contributors, terminus,
                     weight_sums};
    st = render(S, &c, cfg, &v, &b, &f);
    free_bins(&b);
    free_view(&v);
    return st;
}

/* ------------------------------------------------------------- normals */
static void pixel_dir_cam(const cam_t* c, int x, int y, double* pd) {
    pd[0] = (x + 0.5 - c->cx) / c->fx;
    pd[1] = (y + 0.5 - c->cy) / c->fy;
    pd[2] = 1.0;
}

typedef struct {
    double *P, *vx1, *vy1, *vx2, *vy2, *n1, *n2, *sign2, *nf, *fnorm;
    unsigned char *valid, *flipped;
} nstate_t;

static void free_nstate(nstate_t* s) {
    free(s->P); free(s->vx1); free(s->vy1); free(s->vx2); free(s->vy2); free(s->n1);
    free(s->n2); free(s->sign2); free(s->nf); free(s->fnorm); free(s->valid); free(s->flipped);
}

/* backproject + estimate_normals (core/src/normals.cpp:16-101) */
static int estimate_normals(const double* depth, const double* Tm, const cam_t* c,
                            const mo_normal_cfg* nc, double* normals, nstate_t* st) {
    if (nc->step1 >= nc->step2)
        return fail(1, "estimate_normals: step1 must be smaller than step2");
    if (nc->fuse_lambda < 0 || nc->fuse_lambda > 1)
        return fail(1, "estimate_normals: fuse weight must be in [0,1]");
    const int W = c->W, H = c->H;
    const size_t n = (size_t)W * H;
    st->P = (double*)calloc(3 * n, sizeof(double));
    st->vx1 = (double*)calloc(3 * n, sizeof(double));
    st->vy1 = (double*)calloc(3 * n, sizeof(double));
    st->vx2 = (double*)calloc(3 * n, sizeof(double));
    st->vy2 = (double*)calloc(3 * n, sizeof(double));
    st->n1 = (double*)calloc(3 * n, sizeof(double));
    st->n2 = (double*)calloc(3 * n, sizeof(double));
    st->nf = (double*)calloc(3 * n, sizeof(double));
    st->sign2 = (double*)malloc(n * sizeof(double));
    st->fnorm = (double*)calloc(n, sizeof(double));
    st->valid = (unsigned char*)calloc(n, 1);
    st->flipped = (unsigned char*)calloc(n, 1);
    for (size_t i = 0; i < n; ++i) st->sign2[i] = 1.0;
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            double pd[3], pc[3], pw[3];
            pixel_dir_cam(c, x, y, pd);
            const double d = depth[(size_t)y * W + x];
            pc[0] = pd[0] * d; pc[1] = pd[1] * d; pc[2] = pd[2] * d;
            mat3_vec(c->Rc2w, pc, pw);
            double* P = st->P + 3 * ((size_t)y * W + x);
            P[0] = pw[0] + c->tc2w[0]; P[1] = pw[1] + c->tc2w[1]; P[2] = pw[2] + c->tc2w[2];
        }
    if (normals) memset(normals, 0, sizeof(double) * 3 * n);
#define COV(xx, yy) (Tm[(size_t)(yy) * W + (xx)] < nc->mask_threshold)
#define PT(xx, yy) (st->P + 3 * ((size_t)(yy) * W + (xx)))
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            const int s2 = nc->step2, s1 = nc->step1;
            if (x < s2 || y < s2 || x + s2 >= W || y + s2 >= H) continue;
            int ok = COV(x, y);
            ok = ok && COV(x + s1, y) && COV(x - s1, y) && COV(x, y + s1) && COV(x, y - s1);
            ok = ok && COV(x + s2, y) && COV(x - s2, y) && COV(x, y + s2) && COV(x, y - s2);
            if (!ok) continue;
            const size_t p = (size_t)y * W + x;
            double *vx1 = st->vx1 + 3 * p, *vy1 = st->vy1 + 3 * p, *vx2 = st->vx2 + 3 * p,
                   *vy2 = st->vy2 + 3 * p, *n1 = st->n1 + 3 * p, *n2s = st->n2 + 3 * p,
                   *nf = st->nf + 3 * p;
            for (int j = 0; j < 3; ++j) {
                vx1[j] = PT(x + s1, y)[j] - PT(x - s1, y)[j];
                vy1[j] = PT(x, y + s1)[j] - PT(x, y - s1)[j];
                vx2[j] = PT(x + s2, y)[j] - PT(x - s2, y)[j];
                vy2[j] = PT(x, y + s2)[j] - PT(x, y - s2)[j];
            }
            cross3(vx1, vy1, n1);
            double n2[3];
            cross3(vx2, vy2, n2);
            st->sign2[p] = dot3(n1, n2) < 0 ? -1.0 : 1.0;
            for (int j = 0; j < 3; ++j) n2[j] *= st->sign2[p];
            for (int j = 0; j < 3; ++j) n2s[j] = n2[j];
            const double lam = nc->fuse_lambda;
            for (int j = 0; j < 3; ++j) nf[j] = lam * n1[j] + (1.0 - lam) * n2[j];
            const double norm = sqrt(dot3(nf, nf));
            st->fnorm[p] = norm;
            if (norm < 1e-12) continue;
            double N[3] = {nf[0] / norm, nf[1] / norm, nf[2] / norm};
            const double* P = PT(x, y);
            const double tv[3] = {c->tc2w[0] - P[0], c->tc2w[1] - P[1], c->tc2w[2] - P[2]};
            double dv[3];
            normalized3(tv, dv);
            if (dot3(N, dv) > 0) {
                N[0] = -N[0]; N[1] = -N[1]; N[2] = -N[2];
                st->flipped[p] = 1;
            }
            st->valid[p] = 1;
            if (normals) for (int j = 0; j < 3; ++j) normals[3 * p + j] = N[j];
        }
#undef COV
#undef PT
    return 0;
}

int mo_normals(const double* depth, const double* transmittance, const mo_camera* camera,
               const mo_normal_cfg* ncfg, double* normals, uint8_t* valid, uint8_t* flipped) {
    cam_t c;
    int st = make_cam(camera, &c);
    if (st) return st;
    nstate_t s;
    memset(&s, 0, sizeof s);
    st = estimate_normals(depth, transmittance, &c, ncfg, normals, &s);
    if (!st) {
        const size_t n = (size_t)c.W * c.H;
        if (valid) memcpy(valid, s.valid, n);
        if (flipped) memcpy(flipped, s.flipped, n);
    }
    free_nstate(&s);
    return st;
}

/* normals_backward (core/src/normals.cpp:103-152) */
static void normals_backward(const double* dN, const nstate_t* st, const cam_t* c,
                             const mo_normal_cfg* nc, double* dD) {
    const int W = c->W, H = c->H;
    memset(dD, 0, sizeof(double) * (size_t)W * H);
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            const size_t p = (size_t)y * W + x;
            if (!st->valid[p]) continue;
            double g[3] = {dN[3 * p], dN[3 * p + 1], dN[3 * p + 2]};
            if (dot3(g, g) == 0) continue;
            if (st->flipped[p]) { g[0] = -g[0]; g[1] = -g[1]; g[2] = -g[2]; }
            const double fn = st->fnorm[p];
            const double* nf = st->nf + 3 * p;
            const double N[3] = {nf[0] / fn, nf[1] / fn, nf[2] / fn};
            const double Ng = dot3(N, g);
            double gf[3], g1[3], g2[3];
            for (int j = 0; j < 3; ++j) gf[j] = (g[j] - N[j] * Ng) / fn;
            const double lam = nc->fuse_lambda;
            for (int j = 0; j < 3; ++j) {
                g1[j] = lam * gf[j];
                g2[j] = (1.0 - lam) * st->sign2[p] * gf[j];
            }
            double dvx1[3], dvy1[3], dvx2[3], dvy2[3];
            cross3(st->vy1 + 3 * p, g1, dvx1);
            cross3(g1, st->vx1 + 3 * p, dvy1);
            cross3(st->vy2 + 3 * p, g2, dvx2);
            cross3(g2, st->vx2 + 3 * p, dvy2);
            const int s1 = nc->step1, s2 = nc->step2;
            const int tx[8] = {x + s1, x - s1, x, x, x + s2, x - s2, x, x};
            const int ty[8] = {y, y, y + s1, y - s1, y, y, y + s2, y - s2};
            const double* vec[8] = {dvx1, dvx1, dvy1, dvy1, dvx2, dvx2, dvy2, dvy2};
            const double sgn[8] = {1, -1, 1, -1, 1, -1, 1, -1};
            for (int k = 0; k < 8; ++k) {
                double pd[3], r[3];
                pixel_dir_cam(c, tx[k], ty[k], pd);
                mat3_vec(c->Rc2w, pd, r);
                const double dP[3] = {sgn[k] < 0 ? -vec[k][0] : vec[k][0],
                                      sgn[k] < 0 ? -vec[k][1] : vec[k][1],
                                      sgn[k] < 0 ? -vec[k][2] : vec[k][2]};
                dD[(size_t)ty[k] * W + tx[k]] += dot3(dP, r);
            }
        }
}

int mo_normals_backward(const double* dL_dnormals, const double* depth,
                        const double* transmittance, const mo_camera* camera,
                        const mo_normal_cfg* ncfg, double* dD) {
    cam_t c;
    int st = make_cam(camera, &c);
    if (st) return st;
    nstate_t s;
    memset(&s, 0, sizeof s);
    st = estimate_normals(depth, transmittance, &c, ncfg, NULL, &s);
    if (!st) normals_backward(dL_dnormals, &s, &c, ncfg, dD);
    free_nstate(&s);
    return st;
}

/* ------------------------------------------------------------ losses */
/* core/src/losses.cpp restated; evaluate_frame_losses (trainer.cpp:171-264). */
static double sign_of(double v) { return v > 0 ? 1.0 : (v < 0 ? -1.0 : 0.0); }

/* losses.cpp:24-35 */
static void ssim_window(double* w) {
    double sum = 0;
    for (int i = 0; i < 11; ++i) {
        const double d = i - (11 - 1) / 2.0;
        w[i] = exp(-d * d / (2.0 * 1.5 * 1.5));
        sum += w[i];
    }
    for (int i = 0; i < 11; ++i) w[i] /= sum;
}

/* conv_valid (losses.cpp:39-58): along x, then along y; out is (W-10)x(H-10). */
static void conv_valid(const double* in, int W, int H, const double* w, double* tmp, double* out) {
    const int Wv = W - 10, Hv = H - 10;
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < Wv; ++x) {
            double acc = 0;
            for (int i = 0; i < 11; ++i) acc += w[i] * in[(size_t)y * W + x + i];
            tmp[(size_t)y * Wv + x] = acc;
        }
    for (int y = 0; y < Hv; ++y)
        for (int x = 0; x < Wv; ++x) {
            double acc = 0;
            for (int i = 0; i < 11; ++i) acc += w[i] * tmp[(size_t)(y + i) * Wv + x];
            out[(size_t)y * Wv + x] = acc;
        }
}

/* conv_valid_adjoint (losses.cpp:61-83) */
static void conv_valid_adjoint(const double* in, int W, int H, const double* w, double* tmp, double* out) {
    const int Wv = W - 10, Hv = H - 10;
    memset(out, 0, sizeof(double) * (size_t)W * H);
    memset(tmp, 0, sizeof(double) * (size_t)W * Hv);
    for (int y = 0; y < Hv; ++y)
        for (int x = 0; x < Wv; ++x) {
            const double v = in[(size_t)y * Wv + x];
            if (v == 0) continue;
            for (int i = 0; i < 11; ++i) tmp[(size_t)y * W + x + i] += w[i] * v;
        }
    for (int y = 0; y < Hv; ++y)
        for (int x = 0; x < W; ++x) {
            const double v = tmp[(size_t)y * W + x];
            if (v == 0) continue;
            for (int i = 0; i < 11; ++i) out[(size_t)(y + i) * W + x] += w[i] * v;
        }
}

/* ssim_loss (losses.cpp:104-170) on HWC x/y with 3 channels; grad HWC. */
static double ssim_loss(const double* X, const double* Y, int W, int H, double* grad) {
    const int C = 3, Wv = W - 10, Hv = H - 10;
    const size_t n = (size_t)W * H, nv = (size_t)Wv * Hv;
    const double inv_count = 1.0 / ((double)nv * C), C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
    double w[11];
    ssim_window(w);
    double *x = malloc(sizeof(double) * n), *y = malloc(sizeof(double) * n), *xy = malloc(sizeof(double) * n),
           *x2 = malloc(sizeof(double) * n), *y2 = malloc(sizeof(double) * n), *tmp = malloc(sizeof(double) * n),
           *mx = malloc(sizeof(double) * nv), *my = malloc(sizeof(double) * nv), *ex2 = malloc(sizeof(double) * nv),
           *ey2 = malloc(sizeof(double) * nv), *exy = malloc(sizeof(double) * nv), *gm = malloc(sizeof(double) * nv),
           *g2 = malloc(sizeof(double) * nv), *gxy = malloc(sizeof(double) * nv), *back = malloc(sizeof(double) * n);
    memset(grad, 0, sizeof(double) * n * C);
    double ssim_sum = 0;
    for (int ch = 0; ch < C; ++ch) {
        for (size_t i = 0; i < n; ++i) {
            x[i] = X[i * C + ch];
            y[i] = Y[i * C + ch];
            xy[i] = x[i] * y[i];
            x2[i] = x[i] * x[i];
            y2[i] = y[i] * y[i];
        }
        conv_valid(x, W, H, w, tmp, mx);
        conv_valid(y, W, H, w, tmp, my);
        conv_valid(x2, W, H, w, tmp, ex2);
        conv_valid(y2, W, H, w, tmp, ey2);
        conv_valid(xy, W, H, w, tmp, exy);
        for (size_t i = 0; i < nv; ++i) {
            const double a_ = mx[i], b_ = my[i];
            const double sx = ex2[i] - a_ * a_, sy = ey2[i] - b_ * b_, sxy = exy[i] - a_ * b_;
            const double a1 = 2 * a_ * b_ + C1, a2 = 2 * sxy + C2;
            const double b1 = a_ * a_ + b_ * b_ + C1, b2 = sx + sy + C2;
            const double s = (a1 * a2) / (b1 * b2);
            ssim_sum += s;
            const double dS = -inv_count;
            gm[i] = dS * (2 * b_ * (a2 - a1) / (b1 * b2) - 2 * a_ * s * (1 / b1 - 1 / b2));
            g2[i] = dS * (-s / b2);
            gxy[i] = dS * (2 * a1 / (b1 * b2));
        }
        conv_valid_adjoint(gm, W, H, w, tmp, back);
        for (size_t i = 0; i < n; ++i) grad[i * C + ch] += back[i];
        conv_valid_adjoint(g2, W, H, w, tmp, back);
        for (size_t i = 0; i < n; ++i) grad[i * C + ch] += 2 * x[i] * back[i];
        conv_valid_adjoint(gxy, W, H, w, tmp, back);
        for (size_t i = 0; i < n; ++i) grad[i * C + ch] += y[i] * back[i];
    }
    free(x); free(y); free(xy); free(x2); free(y2); free(tmp); free(mx); free(my); free(ex2); free(ey2);
    free(exy); free(gm); free(g2); free(gxy); free(back);
    return 1.0 - ssim_sum * inv_count;
}

int mo_frame_losses(int W, int H, int C, const mo_camera* camera, const mo_normal_cfg* ncfg,
                    const double* color, const double* depth, const double* semantics, const double* kmap,
                    const double* transmittance, const double* gt_rgb, const double* gt_depth,
                    const double* gt_normal, const uint8_t* gt_labels, const double* lambdas, double* report,
                    double* dcolor, double* ddepth, double* dsemantics, double* dkmap, double* normals_out) {
    cam_t c;
    int st = make_cam(camera, &c);
    if (st) return st;
    const size_t n = (size_t)W * H;
    double* normals = calloc(3 * n, sizeof(double));
    nstate_t ns;
    memset(&ns, 0, sizeof ns);
    st = estimate_normals(depth, transmittance, &c, ncfg, normals, &ns);  /* trainer.cpp:296-297 */
    if (normals_out && !st) memcpy(normals_out, normals, sizeof(double) * 3 * n);
    double* gssim = NULL;
    double* gnorm = NULL;
    double v[6] = {0, 0, 0, 0, 0, 0}; /* l1, ssim, normal, depth, seg, k (lambda order) */
    double cnt_depth = 0, cnt_normal = 0;
#define EN(i) (lambdas[i] > 0)
    if (!st && (EN(0) || EN(1)) && !gt_rgb)
        st = fail(2, "rgb loss enabled but the frame has no rgb ground truth (<missing>)");
    if (!st && EN(2) && !gt_normal)
        st = fail(2, "normal loss enabled but the frame has no normal ground truth (<missing>)");
    if (!st && EN(3) && !gt_depth)
        st = fail(2, "depth loss enabled but the frame has no depth ground truth (<missing>)");
    if (!st && EN(4) && !gt_labels)
        st = fail(2, "segmentation loss enabled but the frame has no label ground truth (<missing>)");
    if (!st && EN(1) && (W < 11 || H < 11)) st = fail(1, "ssim_loss: frame smaller than the 11x11 window");
    if (!st && EN(4) && C < 1) st = fail(1, "cross_entropy_seg: no semantic channels");
    if (!st && EN(4))
        for (size_t p = 0; p < n && !st; ++p)
            if (gt_labels[p] >= C)
                st = fail(1, "cross_entropy_seg: label %d out of range at pixel (%d,%d)", (int)gt_labels[p],
                          (int)(p % W), (int)(p / W));
    if (!st) {
        if (EN(0)) { /* l1_rgb (losses.cpp:87-102) */
            double sum = 0;
            for (size_t i = 0; i < 3 * n; ++i) sum += fabs(color[i] - gt_rgb[i]);
            v[0] = sum / (double)(3 * n);
        }
        if (EN(1)) {
            gssim = malloc(sizeof(double) * 3 * n);
            v[1] = ssim_loss(color, gt_rgb, W, H, gssim);
        }
        if (EN(2)) { /* normal_cosine (losses.cpp:198-222) over valid && gt != 0 */
            gnorm = calloc(3 * n, sizeof(double));
            double dot = 0;
            for (size_t p = 0; p < n; ++p) {
                const int ok = ns.valid[p] && (gt_normal[3 * p] != 0 || gt_normal[3 * p + 1] != 0 || gt_normal[3 * p + 2] != 0);
                if (ok) cnt_normal += 1;
            }
            if (cnt_normal > 0) {
                for (size_t p = 0; p < n; ++p) {
                    const int ok = ns.valid[p] && (gt_normal[3 * p] != 0 || gt_normal[3 * p + 1] != 0 || gt_normal[3 * p + 2] != 0);
                    if (!ok) continue;
                    for (int ch = 0; ch < 3; ++ch) {
                        dot += normals[3 * p + ch] * gt_normal[3 * p + ch];
                        gnorm[3 * p + ch] = -gt_normal[3 * p + ch] / cnt_normal;
                    }
                }
                v[2] = 1.0 - dot / cnt_normal;
            }
        }
        if (EN(3)) { /* depth_l1 (losses.cpp:172-196) over gt > 0 */
            double sum = 0;
            for (size_t p = 0; p < n; ++p) if (gt_depth[p] > 0) cnt_depth += 1;
            if (cnt_depth > 0) {
                for (size_t p = 0; p < n; ++p)
                    if (gt_depth[p] > 0) sum += fabs(depth[p] - gt_depth[p]);
                v[3] = sum / cnt_depth;
            }
        }
        if (EN(4)) { /* cross_entropy_seg (losses.cpp:224-267), all pixels */
            double sum = 0;
            for (size_t p = 0; p < n; ++p) {
                const double* l = semantics + p * C;
                double mx = l[0];
                for (int ch = 1; ch < C; ++ch) mx = l[ch] > mx ? l[ch] : mx;
                double z = 0;
                for (int ch = 0; ch < C; ++ch) z += exp(l[ch] - mx);
                sum += log(z) - (l[gt_labels[p]] - mx);
            }
            v[4] = sum / (double)n;
        }
        if (EN(5)) { /* gradient_factor_loss (losses.cpp:269-283) */
            double sum = 0;
            for (size_t p = 0; p < n; ++p) sum += fabs(kmap[p] - 1.0);
            v[5] = sum / (double)n;
        }
        /* combine (losses.cpp:285-313); report in LossReport order */
        const double l1 = v[0], ssim = v[1], normal = v[2], dep = v[3], seg = v[4], kk = v[5];
        const double mag = fabs(l1);
#define RATIO(x) (fabs(x) < 1e-12 ? 0.0 : mag / fabs(x))
        double r[18];
        r[0] = l1; r[1] = ssim; r[2] = dep; r[3] = normal; r[4] = seg; r[5] = kk;
        r[7] = RATIO(ssim); r[8] = RATIO(normal); r[9] = RATIO(dep); r[10] = RATIO(seg); r[11] = RATIO(kk);
#undef RATIO
        r[12] = lambdas[0];
        r[13] = lambdas[1] * r[7];
        r[15] = lambdas[2] * r[8];
        r[14] = lambdas[3] * r[9];
        r[16] = lambdas[4] * r[10];
        r[17] = lambdas[5] * r[11];
        r[6] = lambdas[0] * l1 + r[13] * ssim + r[15] * normal + r[14] * dep + r[16] * seg + r[17] * kk;
        if (report) memcpy(report, r, sizeof r);
        /* seed assembly (trainer.cpp:229-262) */
        memset(dcolor, 0, sizeof(double) * 3 * n);
        memset(ddepth, 0, sizeof(double) * n);
        if (dsemantics && C > 0) memset(dsemantics, 0, sizeof(double) * n * C);
        memset(dkmap, 0, sizeof(double) * n);
        if (EN(0))
            for (size_t i = 0; i < 3 * n; ++i) dcolor[i] += r[12] * (sign_of(color[i] - gt_rgb[i]) / (double)(3 * n));
        if (EN(1) && r[13] != 0)
            for (size_t i = 0; i < 3 * n; ++i) dcolor[i] += r[13] * gssim[i];
        if (EN(3) && r[14] != 0 && cnt_depth > 0)
            for (size_t p = 0; p < n; ++p)
                if (gt_depth[p] > 0) ddepth[p] += r[14] * (sign_of(depth[p] - gt_depth[p]) / cnt_depth);
        if (EN(4) && r[16] != 0)
            for (size_t p = 0; p < n; ++p) {
                const double* l = semantics + p * C;
                double mx = l[0];
                for (int ch = 1; ch < C; ++ch) mx = l[ch] > mx ? l[ch] : mx;
                double z = 0;
                for (int ch = 0; ch < C; ++ch) z += exp(l[ch] - mx);
                for (int ch = 0; ch < C; ++ch)
                    dsemantics[p * C + ch] += r[16] * ((exp(l[ch] - mx) / z - (ch == gt_labels[p] ? 1.0 : 0.0)) / (double)n);
            }
        if (EN(5) && r[17] != 0)
            for (size_t p = 0; p < n; ++p) dkmap[p] += r[17] * (sign_of(kmap[p] - 1.0) / (double)n);
        if (EN(2) && r[15] != 0) {
            double* dD = malloc(sizeof(double) * n);
            normals_backward(gnorm, &ns, &c, ncfg, dD);
            for (size_t p = 0; p < n; ++p) ddepth[p] += r[15] * dD[p];
            free(dD);
        }
    }
#undef EN
    free(gssim);
    free(gnorm);
    free(normals);
    free_nstate(&ns);
    return st;
}

/* metrics.cpp:68-187 */
int mo_metrics(int W, int H, int C, const double* color, const double* gt_rgb, const double* depth,
               const double* gt_depth, const uint8_t* depth_mask, const double* normals, const double* gt_normal,
               const uint8_t* normal_mask, const double* semantics, const uint8_t* gt_labels,
               const uint8_t* label_mask, double* vals, int* has) {
    const size_t n = (size_t)W * H;
    for (int i = 0; i < 6; ++i) { vals[i] = 0; has[i] = 0; }
    if (color && gt_rgb) {
        if (W < 11 || H < 11) return fail(1, "ssim_loss: frame smaller than the 11x11 window");
        double mse = 0;
        for (size_t i = 0; i < 3 * n; ++i) {
            const double d = color[i] - gt_rgb[i];
            mse += d * d;
        }
        mse /= (double)(3 * n);
        vals[0] = mse <= 1e-10 ? 100.0 : fmin(100.0, 10.0 * log10(1.0 / mse));
        has[0] = 1;
        double* g = malloc(sizeof(double) * 3 * n);
        vals[1] = 1.0 - ssim_loss(color, gt_rgb, W, H, g);
        has[1] = 1;
        free(g);
    }
    if (depth && gt_depth && depth_mask) {
        double sa = 0, sr = 0;
        size_t ca = 0, cr = 0;
        for (size_t p = 0; p < n; ++p) {
            if (!depth_mask[p]) continue;
            if (gt_depth[p] > 1e-3) {
                sa += fabs(depth[p] - gt_depth[p]) / gt_depth[p];
                ++ca;
            }
            const double d = depth[p] - gt_depth[p];
            sr += d * d;
            ++cr;
        }
        if (ca) { vals[2] = sa / (double)ca; has[2] = 1; }
        if (cr) { vals[3] = sqrt(sr / (double)cr); has[3] = 1; }
    }
    if (normals && gt_normal && normal_mask) {
        double sum = 0;
        size_t cnt = 0;
        for (size_t p = 0; p < n; ++p) {
            if (!normal_mask[p]) continue;
            for (int ch = 0; ch < 3; ++ch) sum += normals[3 * p + ch] * gt_normal[3 * p + ch];
            ++cnt;
        }
        if (cnt) { vals[4] = sum / (double)cnt; has[4] = 1; }
    }
    if (semantics && gt_labels && label_mask && C > 0) {
        size_t* inter = calloc((size_t)C, sizeof(size_t));
        size_t* pc = calloc((size_t)C, sizeof(size_t));
        size_t* gc = calloc((size_t)C, sizeof(size_t));
        size_t valid = 0;
        int st = 0;
        for (size_t p = 0; p < n && !st; ++p) {
            if (!label_mask[p]) continue;
            ++valid;
            int best = 0;  /* argmax_labels: first maximum */
            for (int ch = 1; ch < C; ++ch)
                if (semantics[p * C + ch] > semantics[p * C + best]) best = ch;
            const int g = gt_labels[p];
            if (best >= C || g >= C) { st = fail(1, "miou: label out of range"); break; }
            ++pc[best];
            ++gc[g];
            if (best == g) ++inter[best];
        }
        if (!st && valid) {
            double sum = 0;
            int classes = 0;
            for (int c = 0; c < C; ++c) {
                const size_t uni = pc[c] + gc[c] - inter[c];
                if (uni == 0) continue;
                sum += (double)inter[c] / (double)uni;
                ++classes;
            }
            if (classes) { vals[5] = sum / classes; has[5] = 1; }
        }
        free(inter); free(pc); free(gc);
        if (st) return st;
    }
    return 0;
}

/* ------------------------------------------------------------ backward */
static void zero_grads(const mo_scene* S, mo_grads* g) {
    const int64_t n = S->n;
    const int K = (S->sh_degree + 1) * (S->sh_degree + 1), C = S->num_classes;
    memset(g->dposition, 0, sizeof(double) * 3 * n);
    memset(g->drotation, 0, sizeof(double) * 4 * n);
    memset(g->dscale, 0, sizeof(double) * 3 * n);
    memset(g->dopacity, 0, sizeof(double) * n);
    memset(g->dsh, 0, sizeof(double) * 3 * K * n);
    if (C) memset(g->dsemantics, 0, sizeof(double) * C * n);
    memset(g->dk, 0, sizeof(double) * n);
}

/* rasterize_backward (core/src/rasterizer_backward.cpp:127-264), threads == 1 */
static int backward(const mo_scene* S, const cam_t* c, const mo_render_cfg* cfg, const view_t* v,
                    const bins_t* b, const double* Tfin, const int32_t* terminus,
                    const double* dcolor, const double* ddepth, const double* dsem,
                    const double* dkmap, mo_grads* out) {
    const int W = c->W, H = c->H, C = S->num_classes;
    const int64_t n = S->n;
    const int K = (S->sh_degree + 1) * (S->sh_degree + 1);
    zero_grads(S, out);
    double* acc_dcolor = (double*)calloc(3 * (n ? n : 1), sizeof(double));
    double* acc_dmean = (double*)calloc(2 * (n ? n : 1), sizeof(double));
    double* acc_dconic = (double*)calloc(3 * (n ? n : 1), sizeof(double));
    double* accum_sem = (double*)calloc(C ? C : 1, sizeof(double));
    double* last_sem = (double*)calloc(C ? C : 1, sizeof(double));
    for (int64_t tile = 0; tile < (int64_t)b->tiles_x * b->tiles_y; ++tile) {
        const int32_t* list = b->val + b->off[tile];
        if (b->off[tile + 1] == b->off[tile]) continue;
        const int tx = (int)(tile % b->tiles_x), ty = (int)(tile / b->tiles_x);
        const int px0 = tx * TILE, py0 = ty * TILE;
        const int px1 = px0 + TILE < W ? px0 + TILE : W, py1 = py0 + TILE < H ? py0 + TILE : H;
        for (int y = py0; y < py1; ++y)
            for (int x = px0; x < px1; ++x) {
                const size_t p = (size_t)y * W + x;
                const int last_pos = terminus[p];
                if (last_pos == 0) continue;
                const double dC[3] = {dcolor[3 * p], dcolor[3 * p + 1], dcolor[3 * p + 2]};
                const double dD = ddepth[p];
                const double* dO = dsem + p * C;
                const double dK = dkmap[p];
                int any = dD != 0 || dK != 0 || dot3(dC, dC) != 0;
                for (int ch = 0; ch < C && !any; ++ch) any = dO[ch] != 0;
                if (!any) continue;
                double o[3], d[3];
                compute_ray(c, x + 0.5, y + 0.5, o, d);
                const double T_final = Tfin[p];
                const double bg_dot = dot3(cfg->background, dC);
                double T = T_final;
                double acol[3] = {0, 0, 0}, lcol[3] = {0, 0, 0};
                for (int ch = 0; ch < C; ++ch) { accum_sem[ch] = 0; last_sem[ch] = 0; }
                double accum_k = 0, last_k = 0, last_alpha = 0;
                for (int pos = last_pos - 1; pos >= 0; --pos) {
                    const int idx = list[pos];
                    const splat_t* sp = &v->sp[idx];
                    const act_t* a = &v->act[idx];
                    const alpha_t ae = eval_alpha(sp, a->alpha, x + 0.5, y + 0.5);
                    if (ae.alpha < kMinAlpha) continue;
                    T /= (1.0 - ae.alpha);
                    const double w = ae.alpha * T;
                    for (int j = 0; j < 3; ++j) acc_dcolor[3 * idx + j] += w * dC[j];
                    for (int ch = 0; ch < C; ++ch) out->dsemantics[(int64_t)idx * C + ch] += w * dO[ch];
                    out->dk[idx] += w * dK;
                    const double ddv = dD * w;
                    if (ddv != 0) {
                        hit_t h;
                        if (intersect(a, o, d, cfg->sigma_scale, &h)) {
                            double gp[3], gq[4], gs[3];
                            intersection_backward(&h, ddv, c, o, d, a, gp, gq, gs);
                            for (int j = 0; j < 3; ++j) out->dposition[3 * idx + j] += gp[j];
                            for (int j = 0; j < 4; ++j) out->drotation[4 * idx + j] += gq[j];
                            for (int j = 0; j < 3; ++j) out->dscale[3 * idx + j] += gs[j];
                        } else {
                            for (int j = 0; j < 3; ++j)
                                out->dposition[3 * idx + j] += ddv * c->Rw2c[6 + j];
                        }
                    }
                    for (int j = 0; j < 3; ++j)
                        acol[j] = last_alpha * lcol[j] + (1.0 - last_alpha) * acol[j];
                    accum_k = last_alpha * last_k + (1.0 - last_alpha) * accum_k;
                    for (int ch = 0; ch < C; ++ch)
                        accum_sem[ch] = last_alpha * last_sem[ch] + (1.0 - last_alpha) * accum_sem[ch];
                    const double* rgb = v->rgb + 3 * idx;
                    const double diff[3] = {rgb[0] - acol[0], rgb[1] - acol[1], rgb[2] - acol[2]};
                    double dalpha = dot3(diff, dC) * T;
                    dalpha += (a->k - accum_k) * dK * T;
                    for (int ch = 0; ch < C; ++ch) dalpha += (a->sem[ch] - accum_sem[ch]) * dO[ch] * T;
                    dalpha -= (T_final / (1.0 - ae.alpha)) * bg_dot;
                    if (!ae.clamped) {
                        out->dopacity[idx] += ae.gauss * dalpha;
                        const double dpower = ae.alpha * dalpha;
                        const double cxx = sp->conic[0], cxy = sp->conic[1], cyy = sp->conic[3];
                        acc_dmean[2 * idx] += dpower * (cxx * ae.dx + cxy * ae.dy);
                        acc_dmean[2 * idx + 1] += dpower * (cxy * ae.dx + cyy * ae.dy);
                        acc_dconic[3 * idx] += dpower * (-0.5 * ae.dx * ae.dx);
                        acc_dconic[3 * idx + 1] += dpower * (-0.5 * ae.dx * ae.dy);
                        acc_dconic[3 * idx + 2] += dpower * (-0.5 * ae.dy * ae.dy);
                    }
                    for (int j = 0; j < 3; ++j) lcol[j] = rgb[j];
                    for (int ch = 0; ch < C; ++ch) last_sem[ch] = a->sem[ch];
                    last_k = a->k;
                    last_alpha = ae.alpha;
                }
            }
    }
    /* projection_backward (rasterizer_backward.cpp:57-123) */
    for (int64_t i = 0; i < n; ++i) {
        if (!v->vis[i]) continue;
        const act_t* a = &v->act[i];
        const splat_t* sp = &v->sp[i];
        const double* dc = acc_dconic + 3 * i;
        const double Gc[4] = {dc[0], dc[1], dc[1], dc[2]};
        const double nc_[4] = {-sp->conic[0], -sp->conic[1], -sp->conic[2], -sp->conic[3]};
        double t1[4], dcov[4];
        for (int r = 0; r < 2; ++r)
            for (int q = 0; q < 2; ++q) {
                double s = nc_[r * 2 + 0] * Gc[0 * 2 + q];
                s += nc_[r * 2 + 1] * Gc[1 * 2 + q];
                t1[r * 2 + q] = s;
            }
        for (int r = 0; r < 2; ++r)
            for (int q = 0; q < 2; ++q) {
                double s = t1[r * 2 + 0] * sp->conic[0 * 2 + q];
                s += t1[r * 2 + 1] * sp->conic[1 * 2 + q];
                dcov[r * 2 + q] = s;
            }
        double pc[3];
        mat3_vec(c->Rw2c, a->pos, pc);
        pc[0] += c->tw2c[0]; pc[1] += c->tw2c[1]; pc[2] += c->tw2c[2];
        const double x = pc[0], y = pc[1], z = pc[2];
        const double J[6] = {c->fx / z, 0, -c->fx * x / (z * z), 0, c->fy / z, -c->fy * y / (z * z)};
        double T[6];
        for (int r = 0; r < 2; ++r)
            for (int j = 0; j < 3; ++j) {
                double s = J[r * 3 + 0] * c->Rw2c[0 * 3 + j];
                s += J[r * 3 + 1] * c->Rw2c[1 * 3 + j];
                s += J[r * 3 + 2] * c->Rw2c[2 * 3 + j];
                T[r * 3 + j] = s;
            }
        double V[9];
        world_cov(a->R, a->s, V);
        /* dV = (T^T dcov) T */
        double TtD[6]; /* 3x2 */
        for (int r = 0; r < 3; ++r)
            for (int q = 0; q < 2; ++q) {
                double s = T[0 * 3 + r] * dcov[0 * 2 + q];
                s += T[1 * 3 + r] * dcov[1 * 2 + q];
                TtD[r * 2 + q] = s;
            }
        double dV[9];
        for (int r = 0; r < 3; ++r)
            for (int q = 0; q < 3; ++q) {
                double s = TtD[r * 2 + 0] * T[0 * 3 + q];
                s += TtD[r * 2 + 1] * T[1 * 3 + q];
                dV[r * 3 + q] = s;
            }
        /* dT = ((2 dcov) T) V */
        double D2[4] = {2.0 * dcov[0], 2.0 * dcov[1], 2.0 * dcov[2], 2.0 * dcov[3]};
        double D2T[6], dT[6], dJ[6];
        for (int r = 0; r < 2; ++r)
            for (int q = 0; q < 3; ++q) {
                double s = D2[r * 2 + 0] * T[0 * 3 + q];
                s += D2[r * 2 + 1] * T[1 * 3 + q];
                D2T[r * 3 + q] = s;
            }
        for (int r = 0; r < 2; ++r)
            for (int q = 0; q < 3; ++q) {
                double s = D2T[r * 3 + 0] * V[0 * 3 + q];
                s += D2T[r * 3 + 1] * V[1 * 3 + q];
                s += D2T[r * 3 + 2] * V[2 * 3 + q];
                dT[r * 3 + q] = s;
            }
        /* dJ = dT R_w2c^T */
        for (int r = 0; r < 2; ++r)
            for (int q = 0; q < 3; ++q) {
                double s = dT[r * 3 + 0] * c->Rw2c[q * 3 + 0];
                s += dT[r * 3 + 1] * c->Rw2c[q * 3 + 1];
                s += dT[r * 3 + 2] * c->Rw2c[q * 3 + 2];
                dJ[r * 3 + q] = s;
            }
        double dp[3] = {0, 0, 0};
        dp[0] += dJ[2] * (-c->fx / (z * z));
        dp[1] += dJ[5] * (-c->fy / (z * z));
        dp[2] += dJ[0] * (-c->fx / (z * z)) + dJ[4] * (-c->fy / (z * z)) +
                 dJ[2] * (2 * c->fx * x / (z * z * z)) + dJ[5] * (2 * c->fy * y / (z * z * z));
        const double* dm = acc_dmean + 2 * i;
        dp[0] += dm[0] * c->fx / z;
        dp[1] += dm[1] * c->fy / z;
        dp[2] += -dm[0] * c->fx * x / (z * z) - dm[1] * c->fy * y / (z * z);
        double dpw[3];
        mat3_vec(c->Rc2w, dp, dpw);
        for (int j = 0; j < 3; ++j) out->dposition[3 * i + j] += dpw[j];
        /* V = M M^T, M = R diag(s) */
        double M[9], dM[9], dR[9], dV2[9];
        for (int r = 0; r < 3; ++r)
            for (int q = 0; q < 3; ++q) M[r * 3 + q] = a->R[r * 3 + q] * a->s[q];
        for (int k2 = 0; k2 < 9; ++k2) dV2[k2] = 2.0 * dV[k2];
        for (int r = 0; r < 3; ++r)
            for (int q = 0; q < 3; ++q) {
                double s = dV2[r * 3 + 0] * M[0 * 3 + q];
                s += dV2[r * 3 + 1] * M[1 * 3 + q];
                s += dV2[r * 3 + 2] * M[2 * 3 + q];
                dM[r * 3 + q] = s;
            }
        for (int r = 0; r < 3; ++r)
            for (int q = 0; q < 3; ++q) dR[r * 3 + q] = dM[r * 3 + q] * a->s[q];
        double dq[4];
        quat_rotation_backward(a->q, dR, dq);
        for (int j = 0; j < 4; ++j) out->drotation[4 * i + j] += dq[j];
        for (int j = 0; j < 3; ++j) { /* diag(R^T dM) */
            double s = a->R[0 * 3 + j] * dM[0 * 3 + j];
            s += a->R[1 * 3 + j] * dM[1 * 3 + j];
            s += a->R[2 * 3 + j] * dM[2 * 3 + j];
            out->dscale[3 * i + j] += s;
        }
        const double* dcol = acc_dcolor + 3 * i;
        if (dot3(dcol, dcol) != 0) {
            const double tg[3] = {a->pos[0] - c->tc2w[0], a->pos[1] - c->tc2w[1], a->pos[2] - c->tc2w[2]};
            const double nrm = sqrt(dot3(tg, tg));
            if (nrm > 1e-12) {
                const double dir[3] = {tg[0] / nrm, tg[1] / nrm, tg[2] / nrm};
                double g3[3] = {dcol[0], dcol[1], dcol[2]};
                for (int ch = 0; ch < 3; ++ch) if (v->clamped[3 * i + ch]) g3[ch] = 0;
                double bs[16], Jb[48], shg[16];
                sh_basis(S->sh_degree, dir, bs);
                for (int ch = 0; ch < 3; ++ch)
                    for (int j = 0; j < K; ++j) out->dsh[(i * 3 + ch) * K + j] += g3[ch] * bs[j];
                sh_jacobian(S->sh_degree, dir, Jb);
                for (int j = 0; j < K; ++j) {
                    double s = a->sh[0 * K + j] * g3[0];
                    s += a->sh[1 * K + j] * g3[1];
                    s += a->sh[2 * K + j] * g3[2];
                    shg[j] = s;
                }
                double ddir[3];
                for (int q = 0; q < 3; ++q) {
                    double s = Jb[0 * 3 + q] * shg[0];
                    for (int j = 1; j < K; ++j) s += Jb[j * 3 + q] * shg[j];
                    ddir[q] = s;
                }
                const double dd = dot3(dir, ddir);
                for (int j = 0; j < 3; ++j) out->dposition[3 * i + j] += (ddir[j] - dir[j] * dd) / nrm;
            }
        }
    }
    free(acc_dcolor); free(acc_dmean); free(acc_dconic); free(accum_sem); free(last_sem);
    /* GradientBuffer::check_finite (core/src/scene.cpp:97-106) */
    for (int64_t i = 0; i < n; ++i) {
        int ok = 1;
        for (int j = 0; j < 3; ++j) ok &= isfinite(out->dposition[3 * i + j]) && isfinite(out->dscale[3 * i + j]);
        for (int j = 0; j < 4; ++j) ok &= isfinite(out->drotation[4 * i + j]);
        ok &= isfinite(out->dopacity[i]) && isfinite(out->dk[i]);
        for (int j = 0; j < 3 * K; ++j) ok &= isfinite(out->dsh[i * 3 * K + j]);
        for (int j = 0; j < C; ++j) ok &= isfinite(out->dsemantics[i * C + j]);
        if (!ok)
            return fail(2, "rasterize_backward: non-finite gradient for primitive %lld", (long long)i);
    }
    return 0;
}

int mo_backward(const mo_scene* S, const mo_camera* camera, const mo_render_cfg* cfg,
                const double* dcolor, const double* ddepth, const double* dsemantics,
                const double* dkmap, mo_grads* out) {
    cam_t c;
    int st = make_cam(camera, &c);
    if (st) return st;
    if ((st = validate(S))) return st;
    view_t v;
    if ((st = prepare_view(S, &c, &v))) return st;
    bins_t b;
    bin_and_sort(S->n, v.vis, v.sp, c.W, c.H, &b);
    const size_t HW = (size_t)c.W * c.H;
    double* T = (double*)malloc(HW * sizeof(double));
    int32_t* term = (int32_t*)malloc(HW * sizeof(int32_t));
    frame_out_t f = {NULL, NULL, NULL, NULL, T, NULL, term, NULL};
    st = render(S, &c, cfg, &v, &b, &f);
    if (!st) st = backward(S, &c, cfg, &v, &b, T, term, dcolor, ddepth, dsemantics, dkmap, out);
    free(T); free(term);
    free_bins(&b);
    free_view(&v);
    return st;
}

/* chain_activations (core/src/scene.cpp:108-129) */
int mo_chain(const mo_scene* S, mo_grads* g) {
    for (int64_t i = 0; i < S->n; ++i) {
        const double* q = S->quats + 4 * i;
        double n2 = q[0] * q[0];
        n2 += q[1] * q[1];
        n2 += q[2] * q[2];
        n2 += q[3] * q[3];
        const double norm = sqrt(n2);
        const double qh[4] = {q[0] / norm, q[1] / norm, q[2] / norm, q[3] / norm};
        double* dq = g->drotation + 4 * i;
        double qd = qh[0] * dq[0];
        qd += qh[1] * dq[1];
        qd += qh[2] * dq[2];
        qd += qh[3] * dq[3];
        for (int j = 0; j < 4; ++j) dq[j] = (dq[j] - qh[j] * qd) / norm;
        for (int j = 0; j < 3; ++j) g->dscale[3 * i + j] *= exp(S->log_scales[3 * i + j]);
        const double alpha = 1.0 / (1.0 + exp(-S->opacity_logits[i]));
        g->dopacity[i] *= alpha * (1.0 - alpha);
    }
    return 0;
}

static double now_ms(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

int mo_fwd_bwd(const mo_scene* S, const mo_camera* camera, const mo_render_cfg* cfg,
               const mo_normal_cfg* ncfg, const double* dcolor, const double* ddepth,
               const double* dsemantics, const double* dkmap, const double* dnormals,
               double* color, double* depth, double* semantics, double* kmap,
               double* transmittance, double* normals, mo_grads* out, double* ms_out) {
    cam_t c;
    int st = make_cam(camera, &c);
    if (st) return st;
    if ((st = validate(S))) return st;
    const double t0 = now_ms();
    view_t v;
    if ((st = prepare_view(S, &c, &v))) return st;
    bins_t b;
    bin_and_sort(S->n, v.vis, v.sp, c.W, c.H, &b);
    const size_t HW = (size_t)c.W * c.H;
    const int C = S->num_classes;
    double* Tl = transmittance ? transmittance : (double*)malloc(HW * sizeof(double));
    double* Dl = depth ? depth : (double*)malloc(HW * sizeof(double));
    int32_t* term = (int32_t*)malloc(HW * sizeof(int32_t));
    frame_out_t f = {color, Dl, semantics, kmap, Tl, NULL, term, NULL};
    st = render(S, &c, cfg, &v, &b, &f);
    const double t1 = now_ms();
    nstate_t ns;
    memset(&ns, 0, sizeof ns);
    double* dD_total = (double*)malloc(HW * sizeof(double));
    double t2 = t1, t3 = t1;
    if (!st) {
        double* nrm = normals ? normals : (double*)malloc(3 * HW * sizeof(double));
        st = estimate_normals(Dl, Tl, &c, ncfg, nrm, &ns);
        if (!normals) free(nrm);
        t2 = now_ms();
        if (!st) {
            normals_backward(dnormals, &ns, &c, ncfg, dD_total);
            for (size_t p = 0; p < HW; ++p) dD_total[p] = ddepth[p] + 1.0 * dD_total[p];
        }
        t3 = now_ms();
    }
    (void)C;
    if (!st) st = backward(S, &c, cfg, &v, &b, Tl, term, dcolor, dD_total, dsemantics, dkmap, out);
    const double t4 = now_ms();
    if (!st) st = mo_chain(S, out);
    const double t5 = now_ms();
    if (ms_out) {
        ms_out[0] = t1 - t0; ms_out[1] = t2 - t1; ms_out[2] = t3 - t2; ms_out[3] = t4 - t3;
        ms_out[4] = t5 - t4;
    }
    free_nstate(&ns);
    free(dD_total); free(term);
    if (!transmittance) free(Tl);
    if (!depth) free(Dl);
    free_bins(&b);
    free_view(&v);
    return st;
}

/* ---------------------------------------------------------- optimizer */
static inline double adam_update(double g, double* m, double* v, double lr, double bc1, double bc2) {
    *m = 0.9 * *m + (1 - 0.9) * g;
    *v = 0.999 * *v + (1 - 0.999) * g * g;
    return lr * (*m / bc1) / (sqrt(*v / bc2) + 1e-15);
}

/* adam_step (core/src/trainer.cpp:98-133) */
int mo_adam(int64_t n, int C, int deg, double* means, double* quats, double* log_scales,
            double* opacity_logits, double* sh, double* semantics, double* k, const mo_grads* g,
            mo_grads* m, mo_grads* v, int64_t step, const double* lr) {
    const int K = (deg + 1) * (deg + 1);
    const double bc1 = 1 - pow(0.9, (double)step);
    const double bc2 = 1 - pow(0.999, (double)step);
    for (int64_t i = 0; i < n; ++i) {
        for (int c = 0; c < 3; ++c)
            means[3 * i + c] -= adam_update(g->dposition[3 * i + c], &m->dposition[3 * i + c],
                                            &v->dposition[3 * i + c], lr[0], bc1, bc2);
        for (int c = 0; c < 4; ++c)
            quats[4 * i + c] -= adam_update(g->drotation[4 * i + c], &m->drotation[4 * i + c],
                                            &v->drotation[4 * i + c], lr[1], bc1, bc2);
        for (int c = 0; c < 3; ++c)
            log_scales[3 * i + c] -= adam_update(g->dscale[3 * i + c], &m->dscale[3 * i + c],
                                                 &v->dscale[3 * i + c], lr[2], bc1, bc2);
        opacity_logits[i] -= adam_update(g->dopacity[i], &m->dopacity[i], &v->dopacity[i], lr[3],
                                         bc1, bc2);
        /* ShMatrix (3 x K) is stored column-major in the reference; the update
         * is element-wise, so traversal order does not change the result. */
        for (int c = 0; c < 3; ++c)
            for (int j = 0; j < K; ++j) {
                const int64_t e = (i * 3 + c) * K + j;
                sh[e] -= adam_update(g->dsh[e], &m->dsh[e], &v->dsh[e], lr[4], bc1, bc2);
            }
        for (int c = 0; c < C; ++c) {
            const int64_t e = i * C + c;
            semantics[e] -= adam_update(g->dsemantics[e], &m->dsemantics[e], &v->dsemantics[e],
                                        lr[5], bc1, bc2);
        }
        k[i] -= adam_update(g->dk[i], &m->dk[i], &v->dk[i], lr[6], bc1, bc2);
    }
    return 0;
}

/* prune keep mask (core/src/trainer.cpp:135-147) */
int64_t mo_prune_mask(int64_t n, const double* k, double threshold, int keep_small, uint8_t* keep) {
    int64_t kept = 0;
    for (int64_t i = 0; i < n; ++i) {
        const double dev = fabs(k[i] - 1.0);
        const int anomalous = keep_small ? dev < threshold : dev > threshold;
        keep[i] = (uint8_t)!anomalous;
        kept += !anomalous;
    }
    if (kept == 0)
        return -fail(2, "prune: threshold %f would remove every gaussian", threshold);
    return kept;
}
