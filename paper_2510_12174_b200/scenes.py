"""Seeded synthetic scenes, cameras and pixel gradients.

"Room slab" scene: Gaussians lie on textured planar surfaces (back wall,
floor, ceiling, side walls, a table top) plus a few spheres, all 1.5-5 m in
front of a camera at the origin; every benchmark view jitters yaw/pitch by at
most 10 degrees.  Parameters are drawn as float32 (the oracle widens them
exactly to double).  Numbers follow the SURVEY recipe:
  tangential sigma = 0.8 h e^U(-.25,.25), h = sqrt(area / N)
  normal sigma     = 0.15 * tangential
  opacity logit    ~ U(-0.5, 3.0); SH DC from a smooth texture, higher U(-.05,.05)
  semantics        = 3 * onehot(surface id) + N(0, 0.3);  k ~ 0.9 + 0.2 U(-1, 1)
Gaussians with 0.01 < z_cam < 1.0 in any benchmark view are rejected (the
no-Jacobian-clamp near-plane tail).

Config table (BASELINE.json "configs"):
  cfg1/cfg2  100k Gaussians, 640x480,  f=500, C=16
  cfg3/cfg4  1M Gaussians,  1200x680, f=600, C=50 (cx=599.5, cy=339.5)
  cfg5       4M Gaussians,  1920x1080, f=960, C=50
"""
from __future__ import annotations

import math

import numpy as np

SH_C0 = 0.28209479177387814

CONFIGS = {
    "cfg1": dict(n=100_000, width=640, height=480, f=500.0, C=16, passes="fwd"),
    "cfg2": dict(n=100_000, width=640, height=480, f=500.0, C=16, passes="fwd+bwd"),
    "cfg3": dict(n=1_000_000, width=1200, height=680, f=600.0, C=50, passes="fwd+bwd"),
    "cfg4": dict(n=1_000_000, width=1200, height=680, f=600.0, C=50, passes="fwd+bwd+allreduce+adam"),
    "cfg5": dict(n=4_000_000, width=1920, height=1080, f=960.0, C=50, passes="fwd"),
}


def _rot_x(a):
    c, s = math.cos(a), math.sin(a)
    return np.array([[1, 0, 0], [0, c, -s], [0, s, c]])


def _rot_y(a):
    c, s = math.cos(a), math.sin(a)
    return np.array([[c, 0, s], [0, 1, 0], [-s, 0, c]])


def view_camera(view: int, width: int, height: int, f: float):
    """Camera `view` of the benchmark set: yaw/pitch jitter within +-10 deg
    (seeded by the view index), small translation jitter, pinhole f."""
    rng = np.random.default_rng(1000 + view)
    if view == 0:
        yaw = pitch = 0.0
        t = np.zeros(3)
    else:
        yaw, pitch = np.deg2rad(rng.uniform(-10, 10, 2))
        t = rng.uniform(-0.05, 0.05, 3)
    R = _rot_y(yaw) @ _rot_x(pitch)
    return {"fx": f, "fy": f, "cx": width / 2 - 0.5, "cy": height / 2 - 0.5, "width": width,
            "height": height, "R_c2w": R, "t_c2w": t}


def _quat_from_matrix(R):
    """Rotation matrices [n,3,3] -> unit quaternions (w,x,y,z) [n,4]."""
    m = R
    tr = m[:, 0, 0] + m[:, 1, 1] + m[:, 2, 2]
    q = np.zeros((len(R), 4))
    c0 = tr > 0
    s = np.sqrt(np.maximum(tr + 1.0, 1e-12)) * 2
    q[c0, 0] = 0.25 * s[c0]
    q[c0, 1] = (m[c0, 2, 1] - m[c0, 1, 2]) / s[c0]
    q[c0, 2] = (m[c0, 0, 2] - m[c0, 2, 0]) / s[c0]
    q[c0, 3] = (m[c0, 1, 0] - m[c0, 0, 1]) / s[c0]
    rest = ~c0
    for i in np.nonzero(rest)[0]:
        r = m[i]
        if r[0, 0] > r[1, 1] and r[0, 0] > r[2, 2]:
            s_ = math.sqrt(max(1.0 + r[0, 0] - r[1, 1] - r[2, 2], 1e-12)) * 2
            q[i] = [(r[2, 1] - r[1, 2]) / s_, 0.25 * s_, (r[0, 1] + r[1, 0]) / s_, (r[0, 2] + r[2, 0]) / s_]
        elif r[1, 1] > r[2, 2]:
            s_ = math.sqrt(max(1.0 + r[1, 1] - r[0, 0] - r[2, 2], 1e-12)) * 2
            q[i] = [(r[0, 2] - r[2, 0]) / s_, (r[0, 1] + r[1, 0]) / s_, 0.25 * s_, (r[1, 2] + r[2, 1]) / s_]
        else:
            s_ = math.sqrt(max(1.0 + r[2, 2] - r[0, 0] - r[1, 1], 1e-12)) * 2
            q[i] = [(r[1, 0] - r[0, 1]) / s_, (r[0, 2] + r[2, 0]) / s_, (r[1, 2] + r[2, 1]) / s_, 0.25 * s_]
    return q / np.linalg.norm(q, axis=1, keepdims=True)


# Surfaces: (kind, params).  World = camera-0 frame: x right, y down, z forward.
_PLANES = [
    # origin, edge u, edge v  (rectangles); normal = u x v (direction irrelevant)
    ("back", np.array([-4.5, -2.6, 4.6]), np.array([9.0, 0, 0]), np.array([0, 5.2, 0])),
    ("floor", np.array([-4.5, 1.3, 1.5]), np.array([9.0, 0, 0]), np.array([0, 0, 3.1])),
    ("ceiling", np.array([-4.5, -1.3, 1.5]), np.array([9.0, 0, 0]), np.array([0, 0, 3.1])),
    ("left", np.array([-2.2, -1.3, 1.5]), np.array([0, 2.6, 0]), np.array([0, 0, 3.1])),
    ("right", np.array([2.2, -1.3, 1.5]), np.array([0, 2.6, 0]), np.array([0, 0, 3.1])),
    ("table", np.array([-0.8, 0.5, 2.2]), np.array([1.6, 0, 0]), np.array([0, 0, 1.0])),
]
_SPHERES = [("sphere0", np.array([-0.9, 0.1, 2.9]), 0.35), ("sphere1", np.array([0.7, -0.2, 3.3]), 0.45),
            ("sphere2", np.array([0.1, 0.15, 2.6]), 0.25)]


def _texture(p, sid):
    return np.stack([0.5 + 0.25 * np.sin(1.3 * p[:, 0] + 0.7 * sid + 0.4 * p[:, 2]),
                     0.5 + 0.25 * np.sin(1.7 * p[:, 1] + 1.1 * sid + 0.3 * p[:, 0]),
                     0.5 + 0.25 * np.cos(0.9 * p[:, 2] + 0.5 * sid + 0.6 * p[:, 1])], axis=1)


def make_room_scene(n: int, num_classes: int, sh_degree: int = 2, seed: int = 0,
                    views=(0,), width=1200, height=680, f=600.0) -> dict:
    """Room-slab scene of exactly n Gaussians (float32-representable values)."""
    rng = np.random.default_rng(seed)
    K = (sh_degree + 1) ** 2
    areas = [np.linalg.norm(np.cross(u, v)) for _, _, u, v in _PLANES] + \
            [4 * math.pi * r * r for _, _, r in _SPHERES]
    total_area = float(sum(areas))
    h = math.sqrt(total_area / n)
    cams = [view_camera(v, width, height, f) for v in views]

    out_pos, out_R, out_sid = [], [], []
    have = 0
    while have < n:
        m = int((n - have) * 1.15) + 64
        surf = rng.choice(len(areas), size=m, p=np.array(areas) / total_area)
        pos = np.zeros((m, 3))
        nrm = np.zeros((m, 3))
        for sidx in range(len(areas)):
            sel = surf == sidx
            k = int(sel.sum())
            if k == 0:
                continue
            if sidx < len(_PLANES):
                _, o, u, v = _PLANES[sidx]
                a, b = rng.random(k), rng.random(k)
                pos[sel] = o + a[:, None] * u + b[:, None] * v
                nn = np.cross(u, v)
                nrm[sel] = nn / np.linalg.norm(nn)
            else:
                _, c, r = _SPHERES[sidx - len(_PLANES)]
                d = rng.normal(size=(k, 3))
                d /= np.linalg.norm(d, axis=1, keepdims=True)
                pos[sel] = c + r * d
                nrm[sel] = d
        # reject near-plane and behind-camera in any view
        ok = np.ones(m, bool)
        for cam in cams:
            zc = (pos - cam["t_c2w"]) @ cam["R_c2w"][:, 2]
            ok &= ~((zc > 0.01) & (zc < 1.0))
        pos, nrm, surf = pos[ok], nrm[ok], surf[ok]
        # frame: t1, t2 tangents, n normal; random twist about n
        helper = np.where(np.abs(nrm[:, :1]) < 0.9, np.array([[1.0, 0, 0]]), np.array([[0, 1.0, 0]]))
        t1 = np.cross(nrm, helper)
        t1 /= np.linalg.norm(t1, axis=1, keepdims=True)
        t2 = np.cross(nrm, t1)
        phi = rng.uniform(0, 2 * math.pi, len(pos))
        c, s = np.cos(phi)[:, None], np.sin(phi)[:, None]
        a1, a2 = c * t1 + s * t2, -s * t1 + c * t2
        out_pos.append(pos)
        out_R.append(np.stack([a1, a2, nrm], axis=2))  # columns: local x, y, z(normal)
        out_sid.append(surf)
        have += len(pos)
    pos = np.concatenate(out_pos)[:n]
    R = np.concatenate(out_R)[:n]
    sid = np.concatenate(out_sid)[:n]

    st = 0.8 * h * np.exp(rng.uniform(-0.25, 0.25, (n, 2)))
    sn = 0.15 * st.mean(axis=1, keepdims=True)
    scales = np.concatenate([st, sn], axis=1)
    quats = _quat_from_matrix(R)
    rgb = _texture(pos, sid)
    sh = np.zeros((n, 3, K))
    sh[:, :, 0] = (rgb - 0.5) / SH_C0
    if K > 1:
        sh[:, :, 1:] = rng.uniform(-0.05, 0.05, (n, 3, K - 1))
    sem = rng.normal(0, 0.3, (n, num_classes))
    if num_classes:
        sem[np.arange(n), sid % num_classes] += 3.0
    f32 = lambda a: np.ascontiguousarray(a, np.float32)  # noqa: E731
    return {
        "means": f32(pos), "quats": f32(quats), "log_scales": f32(np.log(scales)),
        "opacity_logits": f32(rng.uniform(-0.5, 3.0, n)), "sh": f32(sh), "semantics": f32(sem),
        "k": f32(0.9 + 0.2 * rng.uniform(-1, 1, n)), "num_classes": num_classes,
        "sh_degree": sh_degree,
    }


def make_random_scene(n: int, num_classes: int = 3, sh_degree: int = 1, seed: int = 0) -> dict:
    """Small generic scene in the style of the reference fixtures
    (tests/test_common.hpp:23-51): positions in a box in front of the camera,
    random rotations and anisotropic scales."""
    rng = np.random.default_rng(seed)
    K = (sh_degree + 1) ** 2
    u = lambda *s: rng.uniform(-1, 1, s)  # noqa: E731
    pos = np.stack([1.5 * u(n), 1.5 * u(n), 2.2 + 1.2 * u(n)], axis=1)
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    sh = np.zeros((n, 3, K))
    sh[:, :, 0] = 0.4 * u(n, 3)
    if K > 1:
        sh[:, :, 1:] = 0.1 * u(n, 3, K - 1)
    f32 = lambda a: np.ascontiguousarray(a, np.float32)  # noqa: E731
    return {"means": f32(pos), "quats": f32(q), "log_scales": f32(u(n, 3) * 0.7 - 1.3),
            "opacity_logits": f32(0.8 * u(n) + 0.3), "sh": f32(sh), "semantics": f32(u(n, num_classes)),
            "k": f32(0.9 + 0.2 * u(n)), "num_classes": num_classes, "sh_degree": sh_degree}


def simple_camera(w=16, h=16, f=20.0):
    """tests/test_common.hpp:53-55: identity pose, principal point at the centre."""
    return {"fx": f, "fy": f, "cx": w / 2.0, "cy": h / 2.0, "width": w, "height": h,
            "R_c2w": np.eye(3), "t_c2w": np.zeros(3)}


def pixel_grads(width: int, height: int, num_classes: int, seed: int = 0, scale=None) -> dict:
    """Dense seeded U(-1,1)/HW pixel gradients (planar [C,H,W]) for dC, dD, dO,
    dK and dN: dense seeds defeat the reference's all-zero skip
    (rasterizer_backward.cpp:167-171) -- the worst case."""
    rng = np.random.default_rng(10_000 + seed)
    s = 1.0 / (width * height) if scale is None else scale
    g = lambda c: np.ascontiguousarray(rng.uniform(-1, 1, (c, height, width)) * s, np.float32)  # noqa: E731
    return {"dcolor": g(3), "ddepth": g(1)[0], "dsemantics": g(num_classes), "dkmap": g(1)[0],
            "dnormals": g(3)}


def planar_to_hwc(a: np.ndarray) -> np.ndarray:
    """[C,H,W] -> [H,W,C] (reference Grid layout)."""
    return np.ascontiguousarray(np.moveaxis(a, 0, -1))
