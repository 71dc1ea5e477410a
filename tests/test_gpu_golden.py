"""GPU: the CUDA path against golden outputs of the REFERENCE ITSELF
(tests/golden/*.npz, made by tests/golden/make_golden.py from oracle/_ref).
Needs no /root/reference on the GPU box."""
import numpy as np
import pytest
import torch

from helpers import GRAD_NAMES, frame_np, gpu_forward, grad_parity, grads_np, hwc_pix, rel_l2_err, rel_max_err, torch_pix
from test_oracle import _load_golden

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("name", ["random150", "room2k"])
def test_cuda_path_matches_reference_golden(name, dtype):
    import paper_2510_12174_b200 as M
    z, s, cam, cfg, pix = _load_golden(name)
    scene, view, rc, replay, frame = gpu_forward(s, cam, cfg, dtype)
    # binning: bit-exact against the reference's bin_and_sort
    off, vals = replay.bins()
    assert np.array_equal(off, z["bins_offsets"]) and np.array_equal(vals, z["bins_values"])
    sp = replay.splats()
    vis = z["pre_visible"].astype(bool)
    assert np.array_equal(sp["visible"], z["pre_visible"])
    assert np.array_equal(sp["center"][vis], z["pre_center"][vis])
    assert np.array_equal(sp["depth"][vis], z["pre_depth"][vis])
    got = frame_np(frame)
    same = (got["contributors"] == z["fwd_contributors"]) & (replay.terminus() == z["fwd_terminus"])
    tol = 1e-10 if dtype == "float64" else 1e-4
    if dtype == "float64":
        assert same.all()
    assert 1 - same.mean() < 0.01
    for k in ("color", "depth", "kmap", "transmittance"):
        assert rel_max_err(got[k], z["fwd_" + k], same) < tol, k
    dt = torch.float64 if dtype == "float64" else torch.float32
    g = grads_np(M.rasterize_backward(scene, view, frame, replay, torch_pix(pix, dt)))
    gtol = 1e-8 if dtype == "float64" else 1e-3
    for k in GRAD_NAMES:
        if z["bwd_" + k].size:
            assert rel_l2_err(g[k], z["bwd_" + k]) < gtol, k
    if dtype == "float32" and same.all():  # no decision flips: the per-element bar on every Gaussian
        for k, r in grad_parity(g, {k: z["bwd_" + k] for k in GRAD_NAMES}).items():
            assert r["max_rel"] <= 1e-4 and r["p9999_floor"] <= 1e-3, (k, r)
    # the fused training-step unit, chained, against the reference's
    frame2 = M.MultimodalFrame.empty(cam["width"], cam["height"], s["num_classes"], dt, "cuda")
    grads = M.GradientBuffer.zeros_like_scene(scene)
    M.fwd_bwd(scene, view, rc, M.NormalConfig(), frame2, torch_pix(pix, dt), grads, M.ReplayState())
    gs = grads_np(grads)
    for k in GRAD_NAMES:
        if z["step_" + k].size:
            assert rel_l2_err(gs[k], z["step_" + k]) < gtol, k
