"""ctypes front-end for the CPU parity oracle.  TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this module; the product package never
does.  ``load("port")`` opens ``oracle/liboracle.so`` (the plain-C
restatement, ``msplat_oracle.c``); ``load("reference")`` opens
``oracle/_ref/libmsplat_ref.so`` (the reference's own sources compiled
unmodified, ``ref_adapter.cpp``).  Both export the same flat ABI
(``msplat_oracle.h``), so every helper below works with either.

Arrays are numpy float64 in the reference layouts: per-Gaussian arrays
``[n, ...]`` and HWC pixel grids ``[H, W, C]``.
"""
from __future__ import annotations

import ctypes as ct
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PATHS = {
    "port": os.path.join(HERE, "liboracle.so"),
    "reference": os.path.join(HERE, "_ref", "libmsplat_ref.so"),
}

_dp = ct.POINTER(ct.c_double)
_u8p = ct.POINTER(ct.c_uint8)
_i32p = ct.POINTER(ct.c_int32)
_i64p = ct.POINTER(ct.c_int64)


class MoScene(ct.Structure):
    _fields_ = [("n", ct.c_int64), ("num_classes", ct.c_int), ("sh_degree", ct.c_int),
                ("means", _dp), ("quats", _dp), ("log_scales", _dp), ("opacity_logits", _dp),
                ("sh", _dp), ("semantics", _dp), ("k", _dp)]


class MoCamera(ct.Structure):
    _fields_ = [("fx", ct.c_double), ("fy", ct.c_double), ("cx", ct.c_double),
                ("cy", ct.c_double), ("width", ct.c_int), ("height", ct.c_int),
                ("R_c2w", ct.c_double * 9), ("t_c2w", ct.c_double * 3)]


class MoRenderCfg(ct.Structure):
    _fields_ = [("sigma_scale", ct.c_double), ("background", ct.c_double * 3),
                ("early_stop_transmittance", ct.c_double), ("early_termination", ct.c_int),
                ("threads", ct.c_int)]


class MoNormalCfg(ct.Structure):
    _fields_ = [("step1", ct.c_int), ("step2", ct.c_int), ("fuse_lambda", ct.c_double),
                ("mask_threshold", ct.c_double)]


class MoGrads(ct.Structure):
    _fields_ = [("dposition", _dp), ("drotation", _dp), ("dscale", _dp), ("dopacity", _dp),
                ("dsh", _dp), ("dsemantics", _dp), ("dk", _dp)]


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def _p(a, typ=_dp):
    return None if a is None else a.ctypes.data_as(typ)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class Oracle:
    kind: str
    lib: ct.CDLL

    # ------------------------------------------------------------ helpers
    def _check(self, st):
        if st != 0:
            raise OracleError(st, self.lib.mo_last_error().decode())

    @staticmethod
    def scene(s):
        """Keep-alive tuple (struct, arrays) from a scene dict of float arrays."""
        arrs = {k: _f64(s[k]) for k in ("means", "quats", "log_scales", "opacity_logits", "sh",
                                         "semantics", "k")}
        n = arrs["means"].shape[0]
        st = MoScene(n, int(s["num_classes"]), int(s["sh_degree"]),
                     *(_p(arrs[k]) for k in ("means", "quats", "log_scales", "opacity_logits",
                                             "sh", "semantics", "k")))
        return st, arrs

    @staticmethod
    def camera(c):
        R = np.asarray(c["R_c2w"], np.float64).reshape(9)
        t = np.asarray(c["t_c2w"], np.float64).reshape(3)
        return MoCamera(c["fx"], c["fy"], c["cx"], c["cy"], int(c["width"]), int(c["height"]),
                        (ct.c_double * 9)(*R), (ct.c_double * 3)(*t))

    @staticmethod
    def render_cfg(cfg=None, threads=1):
        cfg = cfg or {}
        bg = cfg.get("background", (0.0, 0.0, 0.0))
        return MoRenderCfg(cfg.get("sigma_scale", 1.0), (ct.c_double * 3)(*bg),
                           cfg.get("early_stop_transmittance", 1e-4),
                           int(cfg.get("early_termination", True)), int(threads))

    @staticmethod
    def normal_cfg(ncfg=None):
        ncfg = ncfg or {}
        return MoNormalCfg(ncfg.get("step1", 1), ncfg.get("step2", 4),
                           ncfg.get("fuse_lambda", 0.5), ncfg.get("mask_threshold", 0.5))

    @staticmethod
    def alloc_grads(n, K, C):
        g = {"dposition": np.zeros((n, 3)), "drotation": np.zeros((n, 4)),
             "dscale": np.zeros((n, 3)), "dopacity": np.zeros(n), "dsh": np.zeros((n, 3, K)),
             "dsemantics": np.zeros((n, max(C, 0))), "dk": np.zeros(n)}
        st = MoGrads(*(_p(g[k]) for k in ("dposition", "drotation", "dscale", "dopacity", "dsh",
                                          "dsemantics", "dk")))
        return st, g

    # ---------------------------------------------------------------- API
    def preprocess(self, s, cam):
        sc, keep = self.scene(s)
        n = sc.n
        out = {"visible": np.zeros(n, np.uint8), "center": np.zeros((n, 2)),
               "cov": np.zeros((n, 2, 2)), "conic": np.zeros((n, 3)), "depth": np.zeros(n),
               "radius": np.zeros(n), "rgb": np.zeros((n, 3)), "clamped": np.zeros((n, 3), np.uint8)}
        self._check(self.lib.mo_preprocess(
            ct.byref(sc), ct.byref(self.camera(cam)), _p(out["visible"], _u8p), _p(out["center"]),
            _p(out["cov"]), _p(out["conic"]), _p(out["depth"]), _p(out["radius"]), _p(out["rgb"]),
            _p(out["clamped"], _u8p)))
        return out

    def bin(self, visible, center, radius, depth, width, height):
        n = len(visible)
        tiles = ((width + 15) // 16) * ((height + 15) // 16)
        off = np.zeros(tiles + 1, np.int64)
        vis = np.ascontiguousarray(visible, np.uint8)
        c, r, d = _f64(center), _f64(radius), _f64(depth)
        cnt = self.lib.mo_bin(n, _p(vis, _u8p), _p(c), _p(r), _p(d), width, height, _p(off, _i64p),
                              None, 0)
        if cnt < 0:
            self._check(-cnt)
        vals = np.zeros(max(cnt, 1), np.int32)
        self.lib.mo_bin(n, _p(vis, _u8p), _p(c), _p(r), _p(d), width, height, _p(off, _i64p),
                        _p(vals, _i32p), cnt)
        return off, vals[:cnt]

    def render(self, s, cam, cfg=None, threads=1):
        sc, keep = self.scene(s)
        W, H, C, n = int(cam["width"]), int(cam["height"]), int(s["num_classes"]), sc.n
        out = {"color": np.zeros((H, W, 3)), "depth": np.zeros((H, W)),
               "semantics": np.zeros((H, W, C)), "kmap": np.zeros((H, W)),
               "transmittance": np.zeros((H, W)), "contributors": np.zeros((H, W), np.int32),
               "terminus": np.zeros((H, W), np.int32), "weight_sums": np.zeros(n)}
        self._check(self.lib.mo_render(
            ct.byref(sc), ct.byref(self.camera(cam)), ct.byref(self.render_cfg(cfg, threads)),
            _p(out["color"]), _p(out["depth"]), _p(out["semantics"]) if C else None,
            _p(out["kmap"]), _p(out["transmittance"]), _p(out["contributors"], _i32p),
            _p(out["terminus"], _i32p), _p(out["weight_sums"])))
        return out

    def normals(self, depth, T, cam, ncfg=None):
        W, H = int(cam["width"]), int(cam["height"])
        nrm = np.zeros((H, W, 3))
        valid = np.zeros((H, W), np.uint8)
        flipped = np.zeros((H, W), np.uint8)
        d, t = _f64(depth), _f64(T)
        self._check(self.lib.mo_normals(_p(d), _p(t), ct.byref(self.camera(cam)),
                                        ct.byref(self.normal_cfg(ncfg)), _p(nrm),
                                        _p(valid, _u8p), _p(flipped, _u8p)))
        return nrm, valid, flipped

    def normals_backward(self, dN, depth, T, cam, ncfg=None):
        W, H = int(cam["width"]), int(cam["height"])
        dD = np.zeros((H, W))
        g, d, t = _f64(dN), _f64(depth), _f64(T)
        self._check(self.lib.mo_normals_backward(_p(g), _p(d), _p(t), ct.byref(self.camera(cam)),
                                                 ct.byref(self.normal_cfg(ncfg)), _p(dD)))
        return dD

    LOSS_FIELDS = ("l1", "ssim", "depth", "normal", "seg", "k", "combined", "ratio_ssim", "ratio_normal",
                   "ratio_depth", "ratio_seg", "ratio_k", "seed_l1", "seed_ssim", "seed_depth", "seed_normal",
                   "seed_seg", "seed_k")

    def frame_losses(self, frame, gt, cam, lambdas, ncfg=None):
        """evaluate_frame_losses (trainer.cpp:171-264) after estimate_normals on
        the frame's depth/T.  frame: HWC color/depth/semantics/kmap/transmittance;
        gt: dict with optional rgb/depth/normal (HWC) and labels (uint8 HxW).
        Returns (report dict, pixel-gradient dict HWC, normals HWC)."""
        W, H = int(cam["width"]), int(cam["height"])
        C = int(frame["semantics"].shape[2]) if frame["semantics"].ndim == 3 else 0
        f = {k: _f64(frame[k]) for k in ("color", "depth", "kmap", "transmittance")}
        sem = _f64(frame["semantics"]) if C else None
        g = {k: (_f64(gt[k]) if gt.get(k) is not None else None) for k in ("rgb", "depth", "normal")}
        labels = np.ascontiguousarray(gt["labels"], np.uint8) if gt.get("labels") is not None else None
        rep = np.zeros(18)
        out = {"dcolor": np.zeros((H, W, 3)), "ddepth": np.zeros((H, W)), "dsemantics": np.zeros((H, W, C)),
               "dkmap": np.zeros((H, W))}
        nrm = np.zeros((H, W, 3))
        lam = np.asarray(lambdas, np.float64)
        pn = lambda a: _p(a) if a is not None else None  # noqa: E731
        self._check(self.lib.mo_frame_losses(
            W, H, C, ct.byref(self.camera(cam)), ct.byref(self.normal_cfg(ncfg)), _p(f["color"]), _p(f["depth"]),
            pn(sem), _p(f["kmap"]), _p(f["transmittance"]), pn(g["rgb"]), pn(g["depth"]), pn(g["normal"]),
            _p(labels, _u8p) if labels is not None else None, _p(lam), _p(rep), _p(out["dcolor"]),
            _p(out["ddepth"]), _p(out["dsemantics"]) if C else None, _p(out["dkmap"]), _p(nrm)))
        return dict(zip(self.LOSS_FIELDS, rep.tolist())), out, nrm

    METRIC_FIELDS = ("psnr", "ssim", "abs_rel", "rmse", "cos_simi", "miou")

    def metrics(self, W, H, C, color=None, gt_rgb=None, depth=None, gt_depth=None, depth_mask=None, normals=None,
                gt_normal=None, normal_mask=None, semantics=None, labels=None, label_mask=None):
        """metrics.cpp:68-187 on HWC arrays -> {name: value or None}."""
        args = [_f64(a) if a is not None else None
                for a in (color, gt_rgb, depth, gt_depth, normals, gt_normal, semantics)]
        um = [np.ascontiguousarray(a, np.uint8) if a is not None else None
              for a in (depth_mask, normal_mask, labels, label_mask)]
        vals = np.zeros(6)
        has = np.zeros(6, np.int32)
        pa = lambda a: _p(a) if a is not None else None  # noqa: E731
        pu = lambda a: _p(a, _u8p) if a is not None else None  # noqa: E731
        self._check(self.lib.mo_metrics(W, H, C, pa(args[0]), pa(args[1]), pa(args[2]), pa(args[3]), pu(um[0]),
                                        pa(args[4]), pa(args[5]), pu(um[1]), pa(args[6]), pu(um[2]), pu(um[3]),
                                        _p(vals), has.ctypes.data_as(ct.POINTER(ct.c_int))))
        return {k: (float(vals[i]) if has[i] else None) for i, k in enumerate(self.METRIC_FIELDS)}

    def backward(self, s, cam, pix, cfg=None, threads=1):
        sc, keep = self.scene(s)
        K = (int(s["sh_degree"]) + 1) ** 2
        gst, g = self.alloc_grads(sc.n, K, int(s["num_classes"]))
        arrs = [_f64(pix[k]) for k in ("dcolor", "ddepth", "dsemantics", "dkmap")]
        self._check(self.lib.mo_backward(
            ct.byref(sc), ct.byref(self.camera(cam)), ct.byref(self.render_cfg(cfg, threads)),
            *(_p(a) for a in arrs), ct.byref(gst)))
        return g

    def chain(self, s, grads):
        sc, keep = self.scene(s)
        g = {k: _f64(v).copy() for k, v in grads.items()}
        gst = MoGrads(*(_p(g[k]) for k in ("dposition", "drotation", "dscale", "dopacity", "dsh",
                                           "dsemantics", "dk")))
        self._check(self.lib.mo_chain(ct.byref(sc), ct.byref(gst)))
        return g

    def fwd_bwd(self, s, cam, pix, cfg=None, ncfg=None, threads=1, want_frame=True):
        sc, keep = self.scene(s)
        W, H, C, n = int(cam["width"]), int(cam["height"]), int(s["num_classes"]), sc.n
        K = (int(s["sh_degree"]) + 1) ** 2
        gst, g = self.alloc_grads(n, K, C)
        fr = {"color": np.zeros((H, W, 3)), "depth": np.zeros((H, W)),
              "semantics": np.zeros((H, W, C)), "kmap": np.zeros((H, W)),
              "transmittance": np.zeros((H, W)), "normals": np.zeros((H, W, 3))} if want_frame else None
        ms = np.zeros(5)
        arrs = [_f64(pix[k]) for k in ("dcolor", "ddepth", "dsemantics", "dkmap", "dnormals")]
        fp = (lambda k: _p(fr[k]) if fr is not None and (k != "semantics" or C) else None)
        self._check(self.lib.mo_fwd_bwd(
            ct.byref(sc), ct.byref(self.camera(cam)), ct.byref(self.render_cfg(cfg, threads)),
            ct.byref(self.normal_cfg(ncfg)), *(_p(a) for a in arrs), fp("color"), fp("depth"),
            fp("semantics"), fp("kmap"), fp("transmittance"), fp("normals"), ct.byref(gst),
            _p(ms)))
        return fr, g, ms

    def adam(self, s, grads, m, v, step, lr):
        p = {k: _f64(s[k]).copy() for k in ("means", "quats", "log_scales", "opacity_logits", "sh",
                                             "semantics", "k")}
        bufs = []
        for d in (grads, m, v):
            dd = {k: _f64(x).copy() for k, x in d.items()}
            bufs.append((dd, MoGrads(*(_p(dd[k]) for k in ("dposition", "drotation", "dscale",
                                                           "dopacity", "dsh", "dsemantics", "dk")))))
        lr = np.asarray(lr, np.float64)
        n = p["means"].shape[0]
        self._check(self.lib.mo_adam(n, int(s["num_classes"]), int(s["sh_degree"]),
                                     *(_p(p[k]) for k in ("means", "quats", "log_scales",
                                                          "opacity_logits", "sh", "semantics", "k")),
                                     ct.byref(bufs[0][1]), ct.byref(bufs[1][1]),
                                     ct.byref(bufs[2][1]), int(step), _p(lr)))
        return p, bufs[1][0], bufs[2][0]

    def prune_mask(self, k, threshold, keep_small=False):
        kk = _f64(k)
        keep = np.zeros(len(kk), np.uint8)
        r = self.lib.mo_prune_mask(len(kk), _p(kk), float(threshold), int(keep_small), _p(keep, _u8p))
        if r < 0:
            self._check(-r)
        return keep.astype(bool)


def _bind(lib):
    lib.mo_last_error.restype = ct.c_char_p
    lib.mo_impl_name.restype = ct.c_char_p
    lib.mo_bin.restype = ct.c_int64
    lib.mo_bin.argtypes = [ct.c_int64, _u8p, _dp, _dp, _dp, ct.c_int, ct.c_int, _i64p, _i32p,
                           ct.c_int64]
    lib.mo_prune_mask.restype = ct.c_int64
    lib.mo_prune_mask.argtypes = [ct.c_int64, _dp, ct.c_double, ct.c_int, _u8p]
    lib.mo_adam.argtypes = [ct.c_int64, ct.c_int, ct.c_int] + [_dp] * 7 + [ct.c_void_p] * 3 + \
        [ct.c_int64, _dp]
    return lib


_cache: dict[str, Oracle] = {}


def available(kind: str) -> bool:
    return os.path.exists(PATHS[kind])


def load(kind: str = "port") -> Oracle:
    if kind not in _cache:
        path = PATHS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library {path} not built (run make -C oracle)")
        _cache[kind] = Oracle(kind, _bind(ct.CDLL(path)))
    return _cache[kind]
