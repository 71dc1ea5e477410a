"""Minimal driver for ncu: builds the cfg3 scene (or a smaller one) and runs
`--iters` eager msplat_fwd_bwd calls on cuda:0.  Usage:
  python tools/profile_render.py [--n 1000000] [--width 1200] [--height 680] [--classes 50] [--iters 2]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2510_12174_b200 as M  # noqa: E402
from paper_2510_12174_b200 import rasterizer as R, scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--width", type=int, default=1200)
ap.add_argument("--height", type=int, default=680)
ap.add_argument("--focal", type=float, default=600.0)
ap.add_argument("--classes", type=int, default=50)
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--timing", action="store_true")
a = ap.parse_args()
s = scenes.make_room_scene(a.n, a.classes, 2, seed=0, views=(0,), width=a.width, height=a.height, f=a.focal)
scene = M.Scene.from_numpy(s)
c = scenes.view_camera(0, a.width, a.height, a.focal)
view = M.make_camera(c["fx"], c["fy"], c["cx"], c["cy"], a.width, a.height, c["R_c2w"], c["t_c2w"])
g = torch.Generator(device="cuda").manual_seed(0)
sc = 1.0 / (a.width * a.height)
r = lambda *sh: (torch.rand(*sh, generator=g, device="cuda") * 2 - 1) * sc  # noqa: E731
pix = M.PixelGradients(r(3, a.height, a.width), r(a.height, a.width), r(a.classes, a.height, a.width),
                       r(a.height, a.width), r(3, a.height, a.width))
frame = M.MultimodalFrame.empty(a.width, a.height, a.classes, torch.float32, "cuda")
grads = M.GradientBuffer.zeros_like_scene(scene)
replay = M.ReplayState()
rc, nc = M.RenderConfig(background=(0.1, 0.2, 0.3)), M.NormalConfig()
for i in range(a.iters):
    if a.timing and i == a.iters - 1:
        R.set_stage_timing(True)
    M.fwd_bwd(scene, view, rc, nc, frame, pix, grads, replay)
torch.cuda.synchronize()
R.check_device_errors()
print("counters", replay.counters())
if a.timing:
    print("stages", R.stage_timings())
