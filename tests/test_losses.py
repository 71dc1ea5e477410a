"""Frame losses and gradient-seed assembly:
evaluate_frame_losses (core/src/trainer.cpp:171-264) over core/src/losses.cpp.

CPU: the C restatement (oracle/msplat_oracle.c mo_frame_losses) equals the
reference's own evaluate_frame_losses (oracle/_ref) on rendered frames with
synthetic ground truth, and both keep the reference's error contract.
GPU: the device module (msplat_frame_losses, csrc/losses.cu) against the
reference on the same frame: report values and seeded pixel gradients.
"""
import numpy as np
import pytest

from helpers import rel_l2_err
from paper_2510_12174_b200 import scenes

LAMBDAS = {
    "default": (1.0, 0.1, 0.1, 0.1, 0.1, 0.1),
    "l1_ssim": (1.0, 0.2, 0.0, 0.0, 0.0, 0.0),
    "geometry": (1.0, 0.0, 0.3, 0.3, 0.0, 0.0),
    "seg_k": (0.5, 0.0, 0.0, 0.0, 0.4, 0.2),
}


def loss_case(port, seed=0, C=4, W=48, H=40):
    """A rendered frame (port) and synthetic ground truth of its shape."""
    s = scenes.make_random_scene(400, C, 2, seed=300 + seed)
    cam = {"fx": 45.0, "fy": 45.0, "cx": W / 2, "cy": H / 2, "width": W, "height": H,
           "R_c2w": scenes._rot_y(0.05), "t_c2w": np.array([0.0, 0.0, -0.6])}
    f = port.render(s, cam, {"background": (0.1, 0.2, 0.3)})
    rng = np.random.default_rng(seed)
    gt_depth = f["depth"] * (1 + 0.05 * rng.standard_normal((H, W)))
    gt_depth[rng.random((H, W)) < 0.2] = 0.0  # unsupervised pixels
    n = rng.standard_normal((H, W, 3))
    n /= np.linalg.norm(n, axis=2, keepdims=True)
    n[rng.random((H, W)) < 0.2] = 0.0
    gt = {"rgb": rng.random((H, W, 3)), "depth": gt_depth, "normal": n,
          "labels": rng.integers(0, max(C, 1), (H, W)).astype(np.uint8)}
    return s, cam, f, gt


@pytest.mark.parametrize("lam", sorted(LAMBDAS))
@pytest.mark.parametrize("seed", [0, 1])
def test_port_frame_losses_equal_reference(port, reference, lam, seed):
    s, cam, f, gt = loss_case(port, seed)
    rp, gp, npo = port.frame_losses(f, gt, cam, LAMBDAS[lam])
    rr, gr, nre = reference.frame_losses(f, gt, cam, LAMBDAS[lam])
    assert np.array_equal(npo, nre)
    for k in rp:
        assert rp[k] == pytest.approx(rr[k], rel=1e-12, abs=1e-15), k
    for k in gp:
        assert np.allclose(gp[k], gr[k], rtol=1e-10, atol=1e-15), k
    # every enabled modality contributes
    if LAMBDAS[lam][0] > 0:
        assert np.abs(gp["dcolor"]).max() > 0


def test_loss_error_contract(port, reference):
    """Status 2 = std::runtime_error, 1 = std::invalid_argument (oracle convention)."""
    from oracle.oracle import OracleError
    s, cam, f, gt = loss_case(port, 0)
    for impl in (port, reference):
        with pytest.raises(OracleError, match="rgb loss enabled but the frame has no rgb ground truth") as e:
            impl.frame_losses(f, dict(gt, rgb=None), cam, LAMBDAS["default"])
        assert e.value.code == 2
        with pytest.raises(OracleError, match="depth loss enabled") as e:
            impl.frame_losses(f, dict(gt, depth=None), cam, LAMBDAS["default"])
        assert e.value.code == 2
        bad = gt["labels"].copy()
        bad[3, 7] = 9
        with pytest.raises(OracleError, match=r"label 9 out of range at pixel \(7,3\)") as e:
            impl.frame_losses(f, dict(gt, labels=bad), cam, LAMBDAS["default"])
        assert e.value.code == 1
        # disabled modalities need no ground truth
        impl.frame_losses(f, dict(gt, normal=None, labels=None), cam, (1.0, 0.1, 0.0, 0.1, 0.0, 0.1))


def _planar(a, dt, device="cuda"):
    import torch
    a = np.asarray(a)
    if a.ndim == 3:
        a = np.transpose(a, (2, 0, 1))
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=device)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,vtol,gtol", [("float64", 1e-10, 1e-8), ("float32", 2e-5, 1e-4)])
@pytest.mark.parametrize("lam", sorted(LAMBDAS))
def test_device_frame_losses_match_reference(port, reference, dtype, vtol, gtol, lam):
    import torch
    import paper_2510_12174_b200 as M
    s, cam, f, gt = loss_case(port, 1)
    dt = torch.float64 if dtype == "float64" else torch.float32
    W, H, C = cam["width"], cam["height"], int(s["num_classes"])
    frame = M.MultimodalFrame(W, H, C, _planar(f["color"], dt), _planar(f["depth"], dt), _planar(f["semantics"], dt),
                              _planar(f["kmap"], dt), _planar(f["transmittance"], dt),
                              torch.zeros(3, H, W, dtype=dt, device="cuda"),
                              torch.zeros(H, W, dtype=torch.int32, device="cuda"))
    view = M.make_camera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], W, H, cam["R_c2w"], cam["t_c2w"])
    ncfg = M.NormalConfig()
    M.estimate_normals(frame.depth, frame.transmittance, view, ncfg, frame.normals)
    g = M.GroundTruth(_planar(gt["rgb"], dt), _planar(gt["depth"], dt), _planar(gt["normal"], dt),
                      torch.as_tensor(gt["labels"], device="cuda"))
    rep, pix = M.frame_losses(frame, g, view, ncfg, LAMBDAS[lam])
    rr, gr, _ = reference.frame_losses(f, gt, cam, LAMBDAS[lam])
    for k, v in rr.items():
        assert getattr(rep, k) == pytest.approx(v, rel=vtol, abs=1e-12), k
    got = {"dcolor": pix.dcolor.double().cpu().numpy().transpose(1, 2, 0),
           "ddepth": pix.ddepth.double().cpu().numpy(),
           "dsemantics": pix.dsemantics.double().cpu().numpy().transpose(1, 2, 0),
           "dkmap": pix.dkmap.double().cpu().numpy()}
    for k in got:
        if np.abs(gr[k]).max() > 0:
            assert rel_l2_err(got[k], gr[k]) < gtol, k
        else:
            assert np.abs(got[k]).max() == 0, k


@pytest.mark.gpu
def test_device_frame_losses_errors(port):
    import torch
    import paper_2510_12174_b200 as M
    s, cam, f, gt = loss_case(port, 0)
    dt = torch.float32
    W, H, C = cam["width"], cam["height"], int(s["num_classes"])
    frame = M.MultimodalFrame(W, H, C, _planar(f["color"], dt), _planar(f["depth"], dt), _planar(f["semantics"], dt),
                              _planar(f["kmap"], dt), _planar(f["transmittance"], dt),
                              torch.zeros(3, H, W, dtype=dt, device="cuda"),
                              torch.zeros(H, W, dtype=torch.int32, device="cuda"))
    view = M.make_camera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], W, H, cam["R_c2w"], cam["t_c2w"])
    ncfg = M.NormalConfig()
    bad = gt["labels"].copy()
    bad[3, 7] = 9
    g = M.GroundTruth(_planar(gt["rgb"], dt), _planar(gt["depth"], dt), _planar(gt["normal"], dt),
                      torch.as_tensor(bad, device="cuda"))
    with pytest.raises(ValueError, match=r"label 9 out of range at pixel \(7,3\)"):
        M.frame_losses(frame, g, view, ncfg)
    with pytest.raises(RuntimeError, match="rgb loss enabled"):
        M.frame_losses(frame, M.GroundTruth(None, g.depth, g.normal, g.labels), view, ncfg)


# ------------------------------------------------------------ metrics
def metric_case(port, seed=0):
    """Rendered frame + ground truth + the masks evaluation uses."""
    s, cam, f, gt = loss_case(port, seed)
    nrm, valid, _ = port.normals(f["depth"], f["transmittance"], cam)
    H, W = f["depth"].shape
    rng = np.random.default_rng(10 + seed)
    masks = {"depth_mask": (gt["depth"] > 0).astype(np.uint8), "normal_mask": valid,
             "label_mask": (rng.random((H, W)) < 0.8).astype(np.uint8)}
    return s, cam, f, gt, nrm, masks


def _metric_inputs(f, gt, nrm, masks):
    return dict(color=f["color"], gt_rgb=gt["rgb"], depth=f["depth"], gt_depth=gt["depth"], normals=nrm,
                gt_normal=gt["normal"], semantics=f["semantics"], labels=gt["labels"], **masks)


@pytest.mark.parametrize("seed", [0, 1])
def test_port_metrics_equal_reference(port, reference, seed):
    s, cam, f, gt, nrm, masks = metric_case(port, seed)
    H, W = f["depth"].shape
    kw = _metric_inputs(f, gt, nrm, masks)
    mp = port.metrics(W, H, int(s["num_classes"]), **kw)
    mr = reference.metrics(W, H, int(s["num_classes"]), **kw)
    assert all(v is not None for v in mr.values())  # every metric evaluated
    for k in mr:
        assert mp[k] == pytest.approx(mr[k], rel=1e-12, abs=1e-15), k
    # an empty mask is nullopt, as in the reference
    z = np.zeros((H, W), np.uint8)
    e = reference.metrics(W, H, int(s["num_classes"]), depth=f["depth"], gt_depth=gt["depth"], depth_mask=z)
    assert e["abs_rel"] is None and e["rmse"] is None
    assert port.metrics(W, H, 0, depth=f["depth"], gt_depth=gt["depth"], depth_mask=z)["rmse"] is None


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,tol", [("float64", 1e-11), ("float32", 1e-5)])
def test_device_metrics_match_reference(port, reference, dtype, tol):
    import torch
    import paper_2510_12174_b200 as M
    s, cam, f, gt, nrm, masks = metric_case(port, 1)
    H, W = f["depth"].shape
    C = int(s["num_classes"])
    dt = torch.float64 if dtype == "float64" else torch.float32
    frame = M.MultimodalFrame(W, H, C, _planar(f["color"], dt), _planar(f["depth"], dt), _planar(f["semantics"], dt),
                              _planar(f["kmap"], dt), _planar(f["transmittance"], dt), _planar(nrm, dt),
                              torch.zeros(H, W, dtype=torch.int32, device="cuda"))
    g = M.GroundTruth(_planar(gt["rgb"], dt), _planar(gt["depth"], dt), _planar(gt["normal"], dt),
                      torch.as_tensor(gt["labels"], device="cuda"))
    u8 = lambda a: torch.as_tensor(a, dtype=torch.uint8, device="cuda")  # noqa: E731
    got = M.frame_metrics(frame, g, u8(masks["depth_mask"]), u8(masks["normal_mask"]), u8(masks["label_mask"]))
    ref = reference.metrics(W, H, C, **_metric_inputs(f, gt, nrm, masks))
    for k, v in ref.items():
        assert v is not None and got[k] is not None, k
        assert got[k] == pytest.approx(v, rel=tol, abs=1e-12), k
