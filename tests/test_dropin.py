"""The C++ drop-in (paper_2510_12174_b200/cpp, libmsplat_dropin.so) judged by
the reference's OWN test suite: proj/tests/*.cpp compiled unmodified against
the drop-in headers (oracle/_ref/msplat_dropin_tests, built by `make -C
paper_2510_12174_b200/cpp tests` while /root/reference is present).

CPU: the host-only cases (scene / geometry) pass and every render-path case
fails LOUDLY with a CUDA error -- the drop-in has no CPU fallback.
GPU: FP64 reproduces the reference binary's result exactly (26 of 28, the same
two algorithmic failures, see test_oracle.py); FP32 (MSPLAT_PRECISION=32)
must pass every case whose tolerance is looser than FP32 resolution."""
import ctypes
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "msplat_dropin_tests")
LIB = os.path.join(ROOT, "paper_2510_12174_b200", "libmsplat_dropin.so")
REF_FAILS = ["[FAIL] early termination changes outputs by at most 1e-4",
             "[FAIL] tile rasterizer equals the brute-force oracle"]


def _run(env_extra=None):
    if not os.path.exists(EXE):
        pytest.skip("drop-in test binary not built (needs /root/reference at build time)")
    env = dict(os.environ, **(env_extra or {}))
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=900, env=env)
    lines = (r.stdout + r.stderr).splitlines()
    summary = [l for l in lines if l.startswith("test cases:")][-1]
    return lines, summary


def test_dropin_library_exports_reference_api():
    if not os.path.exists(LIB):
        pytest.skip("libmsplat_dropin.so not built")
    out = subprocess.run(["nm", "-DC", "--defined-only", LIB], capture_output=True, text=True).stdout
    for sym in ("msplat::rasterize(", "msplat::rasterize_backward(", "msplat::bin_and_sort(",
                "msplat::estimate_normals(", "msplat::normals_backward(", "msplat::chain_activations(",
                "msplat::project_gaussian(", "msplat::brute_force_render(", "msplat::Scene::validate("):
        assert sym in out, sym
    ctypes.CDLL(LIB)  # loads next to libmsplat_b200.so via $ORIGIN


def test_dropin_has_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu tests")
    lines, summary = _run()
    assert "test cases: 28" in summary, summary
    fails = [l for l in lines if l.startswith("[FAIL]")]
    # every render-path case fails, and only them; each with a CUDA error
    assert len(fails) == 15, summary
    assert sum("CUDA error" in l for l in lines if "threw" in l) == 15


@pytest.mark.gpu
def test_dropin_fp64_matches_reference_test_results():
    lines, summary = _run()
    assert "test cases: 28 | 2 failed" in summary, "\n".join(lines[-40:])
    assert sorted(l for l in lines if l.startswith("[FAIL]")) == REF_FAILS


@pytest.mark.gpu
def test_dropin_fp32_reference_tests():
    lines, summary = _run({"MSPLAT_PRECISION": "32"})
    fails = sorted(l for l in lines if l.startswith("[FAIL]"))
    # The reference's tolerances are written for doubles; these cases assert
    # bounds below FP32 resolution (1e-9 .. 1e-14) and are allowed to fail; every
    # other case must pass.
    allowed = set(REF_FAILS) | {
        "[FAIL] backward trivial cases for k and semantics",                  # eps 1e-12 / 1e-9
        "[FAIL] projected quaternion gradient is tangent to the unit sphere",  # |g.q| < 1e-14
        "[FAIL] two-contributor blend matches the closed form",
        "[FAIL] per-pixel blending weights sum to 1 - T_final",
        "[FAIL] gradient-factor map is linear in k",
        "[FAIL] depth-loss gradients match frozen-weight finite differences",
        "[FAIL] dk against dL/dK=1 reproduces recorded per-gaussian weight sums",
    }
    assert set(fails) <= allowed, "\n".join(lines[-60:])


@pytest.mark.gpu
def test_dropin_boundary_benchmark_runs(tmp_path):
    """tools/dropin_bench (the reference API timed with host Eigen AoS data)
    on a small scene, in all four precision x determinism modes: same frame
    and gradient checksum up to the precision."""
    import json
    import numpy as np
    import torch
    import paper_2510_12174_b200 as M
    from paper_2510_12174_b200 import scenes
    exe = os.path.join(ROOT, "tools", "_bin", "dropin_bench")
    if not os.path.exists(exe):
        pytest.skip("dropin_bench not built")
    s = scenes.make_random_scene(2000, 5, 2, seed=3)
    path = str(tmp_path / "s.ply")
    M.save_scene_ply(path, M.Scene.from_numpy(s, dtype=torch.float32))
    cam = scenes.simple_camera(96, 64, 60.0)
    args = [exe, path, *(repr(float(cam[k])) for k in ("fx", "fy", "cx", "cy")), "96", "64",
            *(repr(float(v)) for v in np.eye(3).reshape(-1)), "0.0", "0.0", "-0.5", "0", "1"]
    recs = []
    for prec in ("32", "64"):
        for det in ("0", "1"):
            r = subprocess.run(args, capture_output=True, text=True, timeout=300,
                               env=dict(os.environ, MSPLAT_PRECISION=prec, MSPLAT_DETERMINISTIC=det))
            assert r.returncode == 0, r.stderr
            recs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert [x["precision"] for x in recs] == ["f32", "f32", "f64", "f64"]
    assert [x["deterministic"] for x in recs] == [False, True, False, True]
    c = [x["checksum"] for x in recs]
    assert c[2] == c[3] and abs(c[0] - c[2]) <= 1e-4 * max(abs(c[2]), 1e-6), c
    assert all(x["fwd_bwd_ms"] > 0 for x in recs)
