"""The C++ drop-in at the reference API boundary (tools/dropin_bench.cpp over
libmsplat_dropin.so): msplat::rasterize + msplat::rasterize_backward with host
Eigen AoS data in and out, at a BASELINE config (default cfg3), in the four
modes FP32 / FP64 x deterministic on / off.  Writes the scene as an extended
PLY (the reference's format) for the C++ program.  GPU box only.

    python tools/dropin_bench.py [--config cfg3] [--iters 3] [--warmup 1]

Prints one JSON object per mode, then a summary object {"dropin_e2e": [...]}.
"""
import argparse
import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
BIN = os.path.join(ROOT, "tools", "_bin", "dropin_bench")


def run_modes(config="cfg3", iters=3, warmup=1, modes=(("32", "0"), ("32", "1"), ("64", "0"), ("64", "1")),
              timeout=600):
    import torch
    import paper_2510_12174_b200 as M
    from paper_2510_12174_b200 import scenes
    if not os.path.exists(BIN):
        raise RuntimeError(f"{BIN} not built (make -C paper_2510_12174_b200/cpp)")
    c = scenes.CONFIGS[config]
    s = scenes.make_room_scene(c["n"], c["C"], 2, seed=0, views=tuple(range(8)), width=c["width"],
                               height=c["height"], f=c["f"])
    cam = scenes.view_camera(0, c["width"], c["height"], c["f"])
    out = []
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "scene.ply")
        M.save_scene_ply(path, M.Scene.from_numpy(s, dtype=torch.float32))
        torch.cuda.synchronize()
        args = [BIN, path, *(repr(float(cam[k])) for k in ("fx", "fy", "cx", "cy")), str(cam["width"]),
                str(cam["height"]), *(repr(float(v)) for v in cam["R_c2w"].reshape(-1)),
                *(repr(float(v)) for v in cam["t_c2w"]), str(warmup), str(iters)]
        for prec, det in modes:
            env = dict(os.environ, MSPLAT_PRECISION=prec, MSPLAT_DETERMINISTIC=det)
            r = subprocess.run(args, capture_output=True, text=True, env=env, timeout=timeout)
            if os.environ.get("MSPLAT_DROPIN_PROFILE") == "1":
                sys.stderr.write(f"--- f{prec} deterministic={det}\n" + r.stderr)
            if r.returncode != 0:
                out.append({"precision": "f" + prec, "deterministic": det == "1",
                            "error": (r.stderr or r.stdout).strip()[-300:]})
                continue
            rec = json.loads(r.stdout.strip().splitlines()[-1])
            rec["config"] = config
            out.append(rec)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    a = ap.parse_args()
    recs = run_modes(a.config, a.iters, a.warmup)
    for r in recs:
        print(json.dumps(r), flush=True)
    print(json.dumps({"dropin_e2e": recs}))


if __name__ == "__main__":
    main()
