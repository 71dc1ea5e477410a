"""Shared helpers: run the CUDA path through the public Python API and compare
it with the CPU oracle (reference layouts: HWC grids, per-Gaussian arrays)."""
from __future__ import annotations

import numpy as np

from paper_2510_12174_b200 import scenes

GRAD_NAMES = ("dposition", "drotation", "dscale", "dopacity", "dsh", "dsemantics", "dk")


def hwc_pix(pix):
    """Planar pixel gradients -> the oracle's HWC float64 layout."""
    out = {"dcolor": scenes.planar_to_hwc(pix["dcolor"]).astype(np.float64),
           "ddepth": np.asarray(pix["ddepth"], np.float64),
           "dsemantics": scenes.planar_to_hwc(pix["dsemantics"]).astype(np.float64),
           "dkmap": np.asarray(pix["dkmap"], np.float64)}
    if "dnormals" in pix:
        out["dnormals"] = scenes.planar_to_hwc(pix["dnormals"]).astype(np.float64)
    return out


def gpu_forward(s_np, cam, cfg=None, dtype="float32", capture=3):
    import torch
    import paper_2510_12174_b200 as M
    dt = torch.float64 if dtype == "float64" else torch.float32
    scene = M.Scene.from_numpy(s_np, dtype=dt)
    view = M.make_camera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], cam["width"], cam["height"],
                         cam["R_c2w"], cam["t_c2w"])
    rc = M.RenderConfig(**(cfg or {}))
    replay = M.ReplayState(capture=capture)
    frame = M.rasterize(scene, view, rc, replay)
    return scene, view, rc, replay, frame


def frame_np(frame):
    return {"color": scenes.planar_to_hwc(frame.color.double().cpu().numpy()),
            "depth": frame.depth.double().cpu().numpy(),
            "semantics": scenes.planar_to_hwc(frame.semantics.double().cpu().numpy()),
            "kmap": frame.kmap.double().cpu().numpy(),
            "transmittance": frame.transmittance.double().cpu().numpy(),
            "contributors": frame.contributors.cpu().numpy()}


def torch_pix(pix, dtype):
    import torch
    import paper_2510_12174_b200 as M
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device="cuda")  # noqa: E731
    return M.PixelGradients(t(pix["dcolor"]), t(pix["ddepth"]), t(pix["dsemantics"]), t(pix["dkmap"]),
                            t(pix["dnormals"]) if "dnormals" in pix else None)


def grads_np(g):
    return {k: getattr(g, k).double().cpu().numpy() for k in GRAD_NAMES}


def rel_max_err(a, b, mask=None):
    """max |a-b| over the kept entries, relative to the array's max |b|."""
    d = np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64))
    if mask is not None:
        d = d[mask]
    scale = max(np.abs(b).max() if np.size(b) else 0.0, 1e-12)
    return float(d.max() / scale) if d.size else 0.0


def rel_l2_err(a, b):
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-30))


def touched_gaussians(bins, pre, flip, width, height, tile=16):
    """Gaussians that may blend at a decision-flip pixel (contributor count or
    terminus differing from the reference): every Gaussian in that pixel's tile
    list whose centre lies within 1.2 x its 3-sigma radius + 1 px (alpha >= 1/255
    reaches ~3.33 sigma, rasterizer.cpp:139 vs geometry.cpp:132-134).  A
    superset, used to report flip-driven gradient differences separately."""
    off, vals = bins
    n = len(pre["visible"])
    touched = np.zeros(n, bool)
    ys, xs = np.nonzero(flip)
    tiles_x = (width + tile - 1) // tile
    for y, x in zip(ys.tolist(), xs.tolist()):
        t = (y // tile) * tiles_x + x // tile
        ids = np.asarray(vals[off[t]:off[t + 1]], np.int64)
        if ids.size == 0:
            continue
        c = pre["center"][ids]
        r = pre["radius"][ids]
        d = np.hypot(c[:, 0] - (x + 0.5), c[:, 1] - (y + 0.5))
        touched[ids[d <= 1.2 * r + 1.0]] = True
    return touched


def grad_parity(got, ref, touched=None, floor_frac=1e-3):
    """Per-element gradient parity (floors in the style of
    proj/tests/test_common.hpp:57-64).  Per attribute:
      max_rel        max |a-b| / max|b|                   (over every Gaussian)
      max_rel_clean  the same without the flip-touched Gaussians
      p9999_floor    99.99th percentile of |a-b| / max(|a|, |b|, floor_frac max|b|)
    Returns {name: {...}} for the attributes the reference fills."""
    out = {}
    for k in GRAD_NAMES:
        b = np.asarray(ref[k], np.float64)
        if not b.size:
            continue
        a = np.asarray(got[k], np.float64)
        d = np.abs(a - b)
        scale = max(np.abs(b).max(), 1e-30)
        per = d.reshape(d.shape[0], -1).max(axis=1) if d.ndim > 1 else d
        rel = d / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor_frac * scale)
        rec = {"max_rel": float(per.max() / scale),
               "p9999_floor": float(np.quantile(rel, 0.9999))}
        if touched is not None:
            keep = ~touched
            rec["max_rel_clean"] = float(per[keep].max() / scale) if keep.any() else 0.0
            rec["touched"] = int(touched.sum())
        out[k] = rec
    return out
