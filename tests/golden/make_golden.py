"""Generate tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref: the
reference's own sources compiled unmodified against third_party/eigen_subset).

Run here (where /root/reference exists and `make -C oracle` built _ref):
    python tests/golden/make_golden.py
The fixtures travel with the repo so the GPU box (which has no /root/reference)
checks the CUDA path against reference outputs, not only against the port.
Inputs are float32-representable; the reference widens them exactly to double.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2510_12174_b200 import scenes  # noqa: E402

LR = [1.6e-4, 1e-3, 5e-3, 5e-2, 2.5e-3, 2.5e-2, 5e-2]  # trainer.hpp:18-24 order (pos, rot, scale, opac, sh, sem, k)


def hwc(pix):
    return {"dcolor": scenes.planar_to_hwc(pix["dcolor"]).astype(np.float64), "ddepth": pix["ddepth"].astype(np.float64),
            "dsemantics": scenes.planar_to_hwc(pix["dsemantics"]).astype(np.float64),
            "dkmap": pix["dkmap"].astype(np.float64), "dnormals": scenes.planar_to_hwc(pix["dnormals"]).astype(np.float64)}


def make(name, s, cam, cfg, ref):
    out = {}
    for k in ("means", "quats", "log_scales", "opacity_logits", "sh", "semantics", "k"):
        out["in_" + k] = np.asarray(s[k], np.float32)
    out["in_num_classes"] = np.int64(s["num_classes"])
    out["in_sh_degree"] = np.int64(s["sh_degree"])
    for k in ("fx", "fy", "cx", "cy", "width", "height"):
        out["cam_" + k] = np.float64(cam[k])
    out["cam_R_c2w"] = np.asarray(cam["R_c2w"], np.float64)
    out["cam_t_c2w"] = np.asarray(cam["t_c2w"], np.float64)
    out["cfg_background"] = np.asarray(cfg["background"], np.float64)
    W, H, C = cam["width"], cam["height"], s["num_classes"]
    pix = scenes.pixel_grads(W, H, C, seed=5, scale=1.0)
    for k, v in pix.items():
        out["pix_" + k] = v
    pre = ref.preprocess(s, cam)
    for k, v in pre.items():
        out["pre_" + k] = v
    off, vals = ref.bin(pre["visible"], pre["center"], pre["radius"], pre["depth"], W, H)
    out["bins_offsets"], out["bins_values"] = off, vals
    r = ref.render(s, cam, cfg)
    for k, v in r.items():
        out["fwd_" + k] = v
    nrm, valid, flipped = ref.normals(r["depth"], r["transmittance"], cam)
    out["nrm_normals"], out["nrm_valid"], out["nrm_flipped"] = nrm, valid, flipped
    ph = hwc(pix)
    out["nbwd_dD"] = ref.normals_backward(ph["dnormals"], r["depth"], r["transmittance"], cam)
    g = ref.backward(s, cam, ph, cfg)
    for k, v in g.items():
        out["bwd_" + k] = v
    fr, gc, _ = ref.fwd_bwd(s, cam, ph, cfg)
    for k, v in gc.items():
        out["step_" + k] = v
    zeros = {k: np.zeros_like(v) for k, v in gc.items()}
    p, m, v = ref.adam(s, gc, zeros, zeros, 1, LR)
    for k, x in p.items():
        out["adam_" + k] = x
    kk = np.random.default_rng(1).uniform(0, 2, len(s["k"]))
    out["prune_k"] = kk
    out["prune_keep"] = ref.prune_mask(kk, 0.5)
    out["prune_keep_small"] = ref.prune_mask(kk, 0.5, True)
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path) // 1024, "KiB")


def main():
    ref = O.load("reference")
    cam0 = {"fx": 30.0, "fy": 30.0, "cx": 16.0, "cy": 16.0, "width": 32, "height": 32, "R_c2w": np.eye(3),
            "t_c2w": np.array([0.1, 0.0, -0.5])}
    make("random150", scenes.make_random_scene(150, 3, 1, seed=101), cam0, {"background": (0.1, 0.2, 0.3)}, ref)
    cam1 = scenes.view_camera(2, 64, 48, 40.0)
    make("room2k", scenes.make_room_scene(2500, 5, 2, seed=3, views=(2,), width=64, height=48, f=40.0), cam1,
         {"background": (0.1, 0.2, 0.3)}, ref)


if __name__ == "__main__":
    main()
