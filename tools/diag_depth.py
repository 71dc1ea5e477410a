"""Diagnostic: FP32/FP64 depth error distribution vs the reference at a config."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from helpers import frame_np, gpu_forward  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2510_12174_b200 import scenes  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
c = scenes.CONFIGS[cfg]
s = scenes.make_room_scene(c["n"], c["C"], 2, seed=0, views=(0,), width=c["width"], height=c["height"], f=c["f"])
cam = scenes.view_camera(0, c["width"], c["height"], c["f"])
ref = O.load("reference")
z = ref.render(s, cam, {"background": (0.1, 0.2, 0.3)}, threads=os.cpu_count())
for dt in ("float32", "float64"):
    sc, view, rc, replay, frame = gpu_forward(s, cam, {"background": (0.1, 0.2, 0.3)}, dt)
    got = frame_np(frame)
    same = (got["contributors"] == z["contributors"]) & (replay.terminus() == z["terminus"])
    d = np.abs(got["depth"] - z["depth"]) / np.abs(z["depth"]).max()
    d[~same] = 0
    order = np.argsort(d.ravel())[::-1][:8]
    print(dt, "same", same.mean(), "max", d.max(), "n>1e-4", int((d > 1e-4).sum()), "n>3e-5", int((d > 3e-5).sum()),
          "p99.99", np.quantile(d, 0.9999))
    for o in order[:5]:
        y, x = divmod(int(o), c["width"])
        print("   px", x, y, "err", d[y, x], "depth", z["depth"][y, x], got["depth"][y, x], "contrib",
              z["contributors"][y, x], "T", z["transmittance"][y, x])
