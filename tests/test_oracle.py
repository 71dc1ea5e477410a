"""CPU: pin the oracle.

1. The reference's own unit tests (proj/tests, doctest) run against the
   reference sources built here (oracle/_ref/msplat_ref_tests).
2. The C restatement (oracle/msplat_oracle.c) is BITWISE identical to the
   compiled reference on every output of the hot path, over scenes that cover
   SH degrees 0-3, C = 0..5, background, early termination on/off.
3. Both reproduce the committed golden fixtures (tests/golden, generated from
   the reference by tests/golden/make_golden.py) bit for bit.
4. KATs of the reference tests restated against the port.
"""
import os
import subprocess

import numpy as np
import pytest

from helpers import GRAD_NAMES, hwc_pix
from paper_2510_12174_b200 import scenes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def _scenes():
    cams = [
        {"fx": 30.0, "fy": 30.0, "cx": 16.0, "cy": 16.0, "width": 32, "height": 32, "R_c2w": np.eye(3),
         "t_c2w": np.array([0.1, 0.0, -0.5])},
        {"fx": 40.0, "fy": 36.0, "cx": 33.0, "cy": 21.0, "width": 50, "height": 40,
         "R_c2w": scenes._rot_y(0.1) @ scenes._rot_x(-0.05), "t_c2w": np.array([-0.1, 0.05, -0.4])},
    ]
    out = []
    for i, (n, C, deg) in enumerate([(120, 3, 1), (200, 5, 2), (90, 0, 0), (150, 2, 3)]):
        out.append((scenes.make_random_scene(n, C, deg, seed=200 + i), cams[i % 2]))
    return out


CASES = _scenes()
CFGS = [{"background": (0.1, 0.2, 0.3)}, {"early_termination": False}]


def test_reference_own_unit_tests_run():
    """The reference's doctest suite, compiled against the shims: 26 of 28 test
    cases pass.  The two failures are properties of the reference algorithm
    (explained in DESIGN.md), not of the shims:
      * 'tile rasterizer equals the brute-force oracle': the tile rect uses the
        3-sigma radius (geometry.cpp:132-134) while alpha >= 1/255 reaches
        sqrt(2 ln 255) = 3.33 sigma, so brute force sees contributions the tiles
        drop (max |diff| 1e-3 in trial 3);
      * 'early termination changes outputs by at most 1e-4': after the break
        T < 1e-4 but T * depth (depth ~ 1-3) exceeds 1e-4."""
    exe = os.path.join(ROOT, "oracle", "_ref", "msplat_ref_tests")
    if not os.path.exists(exe):
        pytest.skip("reference test binary not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    summary = r.stderr.strip().splitlines()[-1]
    assert "test cases: 28 | 2 failed" in summary, summary
    failed = [l for l in r.stderr.splitlines() if l.startswith("[FAIL]")]
    assert sorted(failed) == ["[FAIL] early termination changes outputs by at most 1e-4",
                              "[FAIL] tile rasterizer equals the brute-force oracle"]


@pytest.mark.parametrize("cfg", range(len(CFGS)))
@pytest.mark.parametrize("case", range(len(CASES)))
def test_port_is_bitwise_the_reference(port, reference, case, cfg):
    s, cam = CASES[case]
    c = CFGS[cfg]
    a, b = port.preprocess(s, cam), reference.preprocess(s, cam)
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    oa = port.bin(a["visible"], a["center"], a["radius"], a["depth"], cam["width"], cam["height"])
    ob = reference.bin(b["visible"], b["center"], b["radius"], b["depth"], cam["width"], cam["height"])
    assert np.array_equal(oa[0], ob[0]) and np.array_equal(oa[1], ob[1])
    ra, rb = port.render(s, cam, c), reference.render(s, cam, c)
    for k in ra:
        assert np.array_equal(ra[k], rb[k]), k
    pix = hwc_pix(scenes.pixel_grads(cam["width"], cam["height"], s["num_classes"], seed=case, scale=1.0))
    ga, gb = port.backward(s, cam, pix, c), reference.backward(s, cam, pix, c)
    for k in GRAD_NAMES:
        assert np.array_equal(ga[k], gb[k]), k
    fa, gfa, _ = port.fwd_bwd(s, cam, pix, c)
    fb, gfb, _ = reference.fwd_bwd(s, cam, pix, c)
    for k in GRAD_NAMES:
        assert np.array_equal(gfa[k], gfb[k]), k
    for k in fa:
        assert np.array_equal(fa[k], fb[k]), k


def _load_golden(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    s = {k[3:]: z[k] for k in z.files if k.startswith("in_")}
    s["num_classes"], s["sh_degree"] = int(s["num_classes"]), int(s["sh_degree"])
    cam = {k[4:]: z[k] for k in z.files if k.startswith("cam_")}
    cam["width"], cam["height"] = int(cam["width"]), int(cam["height"])
    for k in ("fx", "fy", "cx", "cy"):
        cam[k] = float(cam[k])
    cfg = {"background": tuple(z["cfg_background"])}
    pix = {k[4:]: z[k] for k in z.files if k.startswith("pix_")}
    return z, s, cam, cfg, pix


@pytest.mark.parametrize("name", ["random150", "room2k"])
def test_port_reproduces_reference_golden_fixtures(port, name):
    z, s, cam, cfg, pix = _load_golden(name)
    pre = port.preprocess(s, cam)
    for k, v in pre.items():
        assert np.array_equal(v, z["pre_" + k]), k
    off, vals = port.bin(pre["visible"], pre["center"], pre["radius"], pre["depth"], cam["width"], cam["height"])
    assert np.array_equal(off, z["bins_offsets"]) and np.array_equal(vals, z["bins_values"])
    r = port.render(s, cam, cfg)
    for k, v in r.items():
        assert np.array_equal(v, z["fwd_" + k]), k
    nrm, valid, flipped = port.normals(r["depth"], r["transmittance"], cam)
    assert np.array_equal(nrm, z["nrm_normals"]) and np.array_equal(valid, z["nrm_valid"])
    ph = hwc_pix(pix)
    assert np.array_equal(port.normals_backward(ph["dnormals"], r["depth"], r["transmittance"], cam), z["nbwd_dD"])
    g = port.backward(s, cam, ph, cfg)
    for k in GRAD_NAMES:
        assert np.array_equal(g[k], z["bwd_" + k]), k
    _, gc, _ = port.fwd_bwd(s, cam, ph, cfg)
    for k in GRAD_NAMES:
        assert np.array_equal(gc[k], z["step_" + k]), k
    assert np.array_equal(port.prune_mask(z["prune_k"], 0.5), z["prune_keep"])
    assert np.array_equal(port.prune_mask(z["prune_k"], 0.5, True), z["prune_keep_small"])


def test_bin_and_sort_kat_on_port(port):
    """tests/test_rasterizer.cpp:35-56: wide splat in every tile, nearer first."""
    vis = np.array([1, 1], np.uint8)
    center = np.array([[16.0, 16.0], [4.0, 4.0]])
    off, vals = port.bin(vis, center, np.array([100.0, 2.0]), np.array([2.0, 1.0]), 32, 32)
    bins = [vals[off[t]:off[t + 1]].tolist() for t in range(4)]
    assert all(0 in b for b in bins)
    assert bins[0] == [1, 0]


def _axis_scene(specs, C):
    n = len(specs)
    s = {"means": np.array([[0, 0, z] for z, _, _ in specs], float), "quats": np.tile([1.0, 0, 0, 0], (n, 1)),
         "log_scales": np.array([[np.log(sc)] * 3 for _, sc, _ in specs]), "opacity_logits": np.zeros(n),
         "sh": np.zeros((n, 3, 1)), "semantics": np.zeros((n, C)), "k": np.array([k for _, _, k in specs], float),
         "num_classes": C, "sh_degree": 0}
    return s


def test_two_contributor_closed_form_on_port(port):
    """tests/test_rasterizer.cpp:90-106."""
    s = _axis_scene([(1.0, 0.2, 1.0), (2.0, 0.4, 1.0)], 1)
    cam = {"fx": 20.0, "fy": 20.0, "cx": 7.5, "cy": 7.5, "width": 16, "height": 16, "R_c2w": np.eye(3),
           "t_c2w": np.zeros(3)}
    r = port.render(s, cam)
    assert abs(r["depth"][7, 7] - (0.5 * 1.0 + 0.25 * 2.0)) < 1e-12
    assert abs(r["kmap"][7, 7] - 0.75) < 1e-12
    assert abs(r["transmittance"][7, 7] - 0.25) < 1e-12
    assert r["contributors"][7, 7] == 2


def test_empty_scene_renders_background_on_port(port):
    """tests/test_rasterizer.cpp:108-125."""
    s = _axis_scene([], 2)
    s = {k: (np.zeros((0,) + np.shape(v)[1:]) if isinstance(v, np.ndarray) else v) for k, v in s.items()}
    s["sh"] = np.zeros((0, 3, 1))
    cam = scenes.simple_camera()
    r = port.render(s, cam, {"background": (0.2, 0.4, 0.6)})
    assert np.allclose(r["color"][..., 0], 0.2) and np.allclose(r["color"][..., 2], 0.6)
    assert (r["transmittance"] == 1).all() and (r["depth"] == 0).all()


def test_dk_equals_weight_sums_on_port(port):
    """tests/test_rasterizer.cpp:264-276: dL/dK = 1 gives dk = recorded weight sums."""
    s = scenes.make_random_scene(50, 2, 0, seed=113)
    cam = {"fx": 18.0, "fy": 18.0, "cx": 8.0, "cy": 8.0, "width": 16, "height": 16, "R_c2w": np.eye(3),
           "t_c2w": np.zeros(3)}
    r = port.render(s, cam)
    pix = {"dcolor": np.zeros((16, 16, 3)), "ddepth": np.zeros((16, 16)), "dsemantics": np.zeros((16, 16, 2)),
           "dkmap": np.ones((16, 16))}
    g = port.backward(s, cam, pix)
    assert np.allclose(g["dk"], r["weight_sums"], rtol=1e-5, atol=1e-12)


def test_oracle_error_contract(port):
    s = scenes.make_random_scene(10, 2, 1, seed=1)
    s["means"] = s["means"].copy()
    s["means"][7, 2] = np.nan
    from oracle.oracle import OracleError
    with pytest.raises(OracleError, match="primitive 7"):
        port.render(s, scenes.simple_camera())
    with pytest.raises(OracleError, match="remove every gaussian"):
        port.prune_mask(np.full(5, 3.0), 0.5)
