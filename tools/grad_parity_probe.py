"""Per-element FP32 gradient parity against the reference (oracle/_ref) at the
golden cases, the small cases and cfg2 / cfg3: prints helpers.grad_parity for
each, so the test bars are set from measurements.  GPU box only."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_12174_b200 as M  # noqa: E402
from helpers import frame_np, gpu_forward, grad_parity, grads_np, hwc_pix, torch_pix, touched_gaussians  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2510_12174_b200 import scenes  # noqa: E402

BG = {"background": (0.1, 0.2, 0.3)}
ref = O.load("reference")
T = os.cpu_count() or 8


def run(name, s, cam, pix, seed_cfg=BG):
    pre = ref.preprocess(s, cam)
    z = ref.render(s, cam, seed_cfg, threads=T)
    scene, view, rc, replay, frame = gpu_forward(s, cam, seed_cfg, "float32")
    got = frame_np(frame)
    flip = ~((got["contributors"] == z["contributors"]) & (replay.terminus() == z["terminus"]))
    g = grads_np(M.rasterize_backward(scene, view, frame, replay, torch_pix(pix, torch.float32)))
    r = ref.backward(s, cam, hwc_pix(pix), seed_cfg, threads=T)
    touched = touched_gaussians(replay.bins(), pre, flip, cam["width"], cam["height"])
    rep = grad_parity(g, r, touched)
    print(json.dumps({"case": name, "flip_pixels": int(flip.sum()), "report": rep}), flush=True)


sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_gpu_parity import CASES  # noqa: E402
for i, (s, cam) in enumerate(CASES):
    pix = scenes.pixel_grads(cam["width"], cam["height"], s["num_classes"], seed=5, scale=1.0)
    run(f"small{i}", s, cam, pix)
for cfg in sys.argv[1:] or ["cfg2", "cfg3"]:
    c = scenes.CONFIGS[cfg]
    s = scenes.make_room_scene(c["n"], c["C"], 2, seed=0, views=(0,), width=c["width"], height=c["height"], f=c["f"])
    cam = scenes.view_camera(0, c["width"], c["height"], c["f"])
    pix = scenes.pixel_grads(cam["width"], cam["height"], s["num_classes"], seed=4, scale=1.0)
    run(cfg, s, cam, pix)
