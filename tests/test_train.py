"""train() (core/src/trainer.cpp:266-331): the C++
drop-in's device-resident training loop (libmsplat_dropin.so,
msplat_train_flat) against the reference's own train() (oracle/_ref mo_train)
on a synthetic dataset: same view schedule (std::shuffle with mt19937_64),
same per-iteration losses, same prune decisions, same final scene.

Dataset: a random "true" scene rendered by the CPU port into ground truth
(rgb, depth, estimated normals, argmax labels) for 4 cameras, one of them a
test view; initial points = true centres + noise.
"""
import ctypes as ct
import os

import numpy as np
import pytest

from paper_2510_12174_b200 import scenes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DROPIN = os.path.join(ROOT, "paper_2510_12174_b200", "libmsplat_dropin.so")

CFG_KEYS = ["iterations", "lr_position", "lr_rotation", "lr_scale", "lr_opacity", "lr_sh", "lr_semantics", "lr_k",
            "l_l1", "l_ssim", "l_normal", "l_depth", "l_seg", "l_k", "prune_interval", "prune_threshold",
            "prune_enabled", "prune_keep_small", "k_reset", "step1", "step2", "lambda_fuse", "mask_threshold",
            "sigma_scale", "early_stop", "bg0", "bg1", "bg2", "sh_degree", "seed", "threads", "deterministic"]
DEFAULT = dict(iterations=6, lr_position=1.6e-4, lr_rotation=1e-3, lr_scale=5e-3, lr_opacity=5e-2, lr_sh=2.5e-3,
               lr_semantics=2.5e-2, lr_k=5e-2, l_l1=1.0, l_ssim=0.1, l_normal=0.1, l_depth=0.1, l_seg=0.1, l_k=0.1,
               prune_interval=3, prune_threshold=0.09, prune_enabled=1, prune_keep_small=1, k_reset=0.9, step1=1,
               step2=4, lambda_fuse=0.5, mask_threshold=0.5, sigma_scale=1.0, early_stop=1e-4, bg0=0.1, bg1=0.2,
               bg2=0.3, sh_degree=2, seed=7, threads=1, deterministic=1)


class Cam(ct.Structure):  # mo_camera == msplat_camera layout
    _fields_ = [("fx", ct.c_double), ("fy", ct.c_double), ("cx", ct.c_double), ("cy", ct.c_double),
                ("width", ct.c_int), ("height", ct.c_int), ("R_c2w", ct.c_double * 9), ("t_c2w", ct.c_double * 3)]


def make_dataset(port, W=48, H=40, C=3, n=300, seed=0):
    rng = np.random.default_rng(seed)
    truth = scenes.make_random_scene(n, C, 2, seed=500 + seed)
    cams = []
    for yaw in (-0.08, -0.03, 0.02, 0.07):
        cams.append({"fx": 45.0, "fy": 45.0, "cx": W / 2, "cy": H / 2, "width": W, "height": H,
                     "R_c2w": scenes._rot_y(yaw), "t_c2w": np.array([yaw, 0.0, -0.6])})
    rgb, depth, normal, labels = [], [], [], []
    for cam in cams:
        f = port.render(truth, cam, {"background": (0.1, 0.2, 0.3)})
        nrm, _, _ = port.normals(f["depth"], f["transmittance"], cam)
        rgb.append(np.clip(f["color"], 0, 1))
        depth.append(f["depth"])
        normal.append(nrm)
        labels.append(np.argmax(f["semantics"], axis=2).astype(np.uint8))
    pts = truth["means"] + 0.01 * rng.standard_normal(truth["means"].shape)
    cols = rng.random((n, 3))
    return {"points": np.ascontiguousarray(pts), "colors": cols, "C": C, "cams": cams,
            "rgb": np.ascontiguousarray(np.stack(rgb)), "depth": np.ascontiguousarray(np.stack(depth)),
            "normal": np.ascontiguousarray(np.stack(normal)), "labels": np.ascontiguousarray(np.stack(labels)),
            "is_test": np.array([0, 1, 0, 0], np.uint8)}


def run_train(fn, err_fn, ds, cfg):
    d = dict(DEFAULT, **cfg)
    c = np.array([float(d[k]) for k in CFG_KEYS])
    n, C = len(ds["points"]), ds["C"]
    P = 12 + 3 * (int(d["sh_degree"]) + 1) ** 2 + C
    cams = (Cam * len(ds["cams"]))()
    for i, cm in enumerate(ds["cams"]):
        cams[i] = Cam(cm["fx"], cm["fy"], cm["cx"], cm["cy"], cm["width"], cm["height"],
                      (ct.c_double * 9)(*np.asarray(cm["R_c2w"], float).ravel()),
                      (ct.c_double * 3)(*np.asarray(cm["t_c2w"], float)))
    params = np.zeros(n * P)
    n_out = ct.c_int64()
    log = np.zeros((int(d["iterations"]), 21))
    completed, halted = ct.c_int(), ct.c_int()
    dp = lambda a: a.ctypes.data_as(ct.c_void_p)  # noqa: E731
    st = fn(n, dp(ds["points"]), dp(ds["colors"]), C, len(ds["cams"]), cams, dp(ds["rgb"]), dp(ds["depth"]),
            dp(ds["normal"]), dp(ds["labels"]), dp(ds["is_test"]), dp(c), dp(params), ct.byref(n_out), dp(log),
            ct.byref(completed), ct.byref(halted))
    if st != 0:
        raise RuntimeError(f"status {st}: {err_fn().decode()}")
    k = int(n_out.value)
    return {"n": k, "params": params[: k * P], "log": log[: completed.value], "completed": completed.value,
            "halted": halted.value}


def _ref_fn(reference):
    fn = reference.lib.mo_train
    fn.restype = ct.c_int
    return fn, reference.lib.mo_last_error


def test_reference_train_runs_and_prunes(port, reference):
    ds = make_dataset(port)
    fn, err = _ref_fn(reference)
    r = run_train(fn, err, ds, {})
    assert r["completed"] == DEFAULT["iterations"] and r["halted"] == 0
    views = r["log"][:, 1].astype(int)
    assert 1 not in views.tolist()          # the test view is never trained on
    assert r["log"][2, 2] < len(ds["points"])  # the prune at iteration 3 removed some
    assert np.all(np.isfinite(r["params"]))


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [{}, {"l_ssim": 0.0, "l_seg": 0.3, "seed": 3}])
def test_dropin_train_matches_reference(port, reference, cfg):
    if not os.path.exists(DROPIN):
        pytest.skip("libmsplat_dropin.so not built")
    ds = make_dataset(port)
    lib = ct.CDLL(DROPIN)
    lib.msplat_train_flat.restype = ct.c_int
    lib.msplat_train_last_error.restype = ct.c_char_p
    got = run_train(lib.msplat_train_flat, lib.msplat_train_last_error, ds, cfg)
    fn, err = _ref_fn(reference)
    ref = run_train(fn, err, ds, cfg)
    assert got["completed"] == ref["completed"] and got["halted"] == ref["halted"]
    assert np.array_equal(got["log"][:, :3], ref["log"][:, :3])  # iteration, view, Gaussian count
    # The first iteration sees identical inputs: rounding-level agreement.
    assert np.allclose(got["log"][0, 3:], ref["log"][0, 3:], rtol=1e-12, atol=1e-15)
    # Later iterations: Adam's first steps move every parameter by ~lr * sign(g)
    # whatever |g| (eps = 1e-15), so components whose exact gradient is zero but
    # whose rounded gradient is +-1e-18 step differently in any two summation
    # orders.  The losses stay close; the parameters agree except on those.
    assert np.allclose(got["log"][:, 3:], ref["log"][:, 3:], rtol=1e-5, atol=1e-9)
    assert got["n"] == ref["n"]
    d = np.abs(got["params"] - ref["params"])
    scale = np.abs(ref["params"]).max()
    print("params: max |diff|", d.max(), "fraction > 1e-9 scale:", float((d > 1e-9 * scale).mean()))
    assert float((d > 1e-9 * scale).mean()) < 0.02
    lr_max = max(DEFAULT[k] for k in ("lr_position", "lr_rotation", "lr_scale", "lr_opacity", "lr_sh",
                                      "lr_semantics", "lr_k"))
    assert d.max() <= 2 * lr_max * DEFAULT["iterations"]
