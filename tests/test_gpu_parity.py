"""Parity of the CUDA path (through the public API / C ABI) against the CPU
oracle on identical inputs.

Bars (BASELINE.json north star):
  * tile key lists, per-tile order and ranges, prune masks: bit-exact;
  * FP64 kernels: images ~1e-10, gradients ~1e-8 (rounding-order only);
  * FP32 kernels: rendered channels max-abs <= 1e-4 relative to the channel's
    range, gradients <= 1e-3 relative; pixels whose blend decisions flip
    between FP32 and FP64 (alpha >= 1/255, T < 1e-4; visible as a different
    contributor count or terminus) are counted and bounded separately.
"""
import numpy as np
import pytest

from helpers import GRAD_NAMES, frame_np, gpu_forward, grad_parity, grads_np, hwc_pix, rel_l2_err, rel_max_err, torch_pix
from paper_2510_12174_b200 import scenes

pytestmark = pytest.mark.gpu

BG = {"background": (0.1, 0.2, 0.3)}


def small_cases():
    cams = [
        {"fx": 30.0, "fy": 30.0, "cx": 16.0, "cy": 16.0, "width": 32, "height": 32, "R_c2w": np.eye(3),
         "t_c2w": np.array([0.1, 0.0, -0.5])},
        {"fx": 40.0, "fy": 36.0, "cx": 33.0, "cy": 21.0, "width": 70, "height": 45,
         "R_c2w": scenes._rot_y(0.1) @ scenes._rot_x(-0.05), "t_c2w": np.array([-0.1, 0.05, -0.4])},
    ]
    out = []
    for i, (n, C, deg) in enumerate([(150, 3, 1), (400, 5, 2), (250, 0, 0), (300, 2, 3)]):
        out.append((scenes.make_random_scene(n, C, deg, seed=100 + i), cams[i % 2]))
    return out


CASES = small_cases()


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_preprocess_and_binning_bit_exact(port, case, dtype):
    s, cam = CASES[case]
    _, _, _, replay, _ = gpu_forward(s, cam, BG, dtype)
    ref = port.preprocess(s, cam)
    got = replay.splats()
    assert np.array_equal(got["visible"], ref["visible"])
    vis = ref["visible"].astype(bool)
    # centre and depth involve no transcendental: identical FP64 op order -> identical bits
    for k in ("center", "depth"):
        assert np.array_equal(got[k][vis], ref[k][vis]), k
    # radius and conic go through s = exp(log_scale): CUDA's and glibc's exp may
    # round the last bit differently, so allow a few ulp (a tile-rect flip would
    # need centre +- radius within 1 ulp of an integer; binning is checked exactly below)
    for k in ("radius", "conic"):
        a, b = got[k][vis], ref[k][vis]
        rel = np.abs(a - b) / np.maximum(np.abs(b), 1e-300)
        print(f"{k}: {np.count_nonzero(rel)} of {rel.size} differ, max rel {rel.max():.2e}")
        assert rel.max() <= 1e-12, k  # 1-ulp exp differences amplified by det cancellation
    off, vals = port.bin(ref["visible"], ref["center"], ref["radius"], ref["depth"], cam["width"], cam["height"])
    goff, gvals = replay.bins()
    assert np.array_equal(goff, off)
    assert np.array_equal(gvals, vals)


@pytest.mark.parametrize("case", range(len(CASES)))
def test_forward_fp64_matches_oracle(port, case):
    s, cam = CASES[case]
    _, _, _, replay, frame = gpu_forward(s, cam, BG, "float64")
    ref = port.render(s, cam, BG)
    got = frame_np(frame)
    assert np.array_equal(got["contributors"], ref["contributors"])
    assert np.array_equal(replay.terminus(), ref["terminus"])
    for k in ("color", "depth", "semantics", "kmap", "transmittance"):
        assert rel_max_err(got[k], ref[k]) < 1e-10, k
    ws = replay.weight_sums()
    assert rel_max_err(ws, ref["weight_sums"]) < 1e-10


@pytest.mark.parametrize("case", range(len(CASES)))
def test_forward_fp32_within_tolerance(port, case):
    s, cam = CASES[case]
    _, _, _, replay, frame = gpu_forward(s, cam, BG, "float32")
    ref = port.render(s, cam, BG)
    got = frame_np(frame)
    same = (got["contributors"] == ref["contributors"]) & (replay.terminus() == ref["terminus"])
    flips = 1.0 - same.mean()
    print(f"case {case}: decision-flip pixels {flips:.4%}")
    assert flips < 0.01
    for k in ("color", "depth", "kmap", "transmittance"):
        e = rel_max_err(got[k], ref[k], same)
        print(f"  {k}: {e:.2e}")
        assert e < 1e-4, k
    if s["num_classes"]:
        e = rel_max_err(got["semantics"], ref["semantics"], np.broadcast_to(same[..., None], got["semantics"].shape))
        assert e < 1e-4


@pytest.mark.parametrize("dtype,tol", [("float64", 1e-8), ("float32", 1e-3)])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_backward_matches_oracle(port, case, dtype, tol):
    import torch
    import paper_2510_12174_b200 as M
    s, cam = CASES[case]
    scene, view, rc, replay, frame = gpu_forward(s, cam, BG, dtype)
    pix = scenes.pixel_grads(cam["width"], cam["height"], s["num_classes"], seed=case, scale=1.0)
    dt = torch.float64 if dtype == "float64" else torch.float32
    g = grads_np(M.rasterize_backward(scene, view, frame, replay, torch_pix(pix, dt)))
    ref = port.backward(s, cam, hwc_pix(pix), BG)
    for k in GRAD_NAMES:
        if ref[k].size == 0:
            continue
        e = rel_l2_err(g[k], ref[k])
        print(f"case {case} {dtype} {k}: rel L2 {e:.2e}")
        assert e < tol, k
    if dtype == "float32":  # per element (no decision flips at these sizes): max |a-b| <= 1e-3 max|b|
        for k, r in grad_parity(g, ref).items():
            assert r["max_rel"] <= 1e-3 and r["p9999_floor"] <= 1e-3, (k, r)


@pytest.mark.parametrize("dtype,tol", [("float64", 1e-8), ("float32", 1e-3)])
def test_deterministic_backward_is_bitwise_reproducible(port, dtype, tol):
    """tests/test_rasterizer.cpp:386-419: repeated backward passes are bitwise
    equal (fixed-order reduction), and match the oracle like the atomic path."""
    import torch
    import paper_2510_12174_b200 as M
    s = scenes.make_random_scene(3000, 6, 2, seed=77)
    cam = {"fx": 120.0, "fy": 120.0, "cx": 80.0, "cy": 60.0, "width": 160, "height": 120,
           "R_c2w": np.eye(3), "t_c2w": np.array([0.0, 0.0, -1.2])}
    dt = torch.float64 if dtype == "float64" else torch.float32
    pix = scenes.pixel_grads(cam["width"], cam["height"], s["num_classes"], seed=5, scale=1.0)
    M.set_deterministic(True)
    try:
        runs = []
        for _ in range(3):
            scene, view, rc, replay, frame = gpu_forward(s, cam, BG, dtype)
            runs.append(grads_np(M.rasterize_backward(scene, view, frame, replay, torch_pix(pix, dt))))
    finally:
        M.set_deterministic(False)
    for k in GRAD_NAMES:
        assert np.array_equal(runs[0][k], runs[1][k]) and np.array_equal(runs[0][k], runs[2][k]), k
    ref = port.backward(s, cam, hwc_pix(pix), BG)
    for k in GRAD_NAMES:
        if ref[k].size:
            assert rel_l2_err(runs[0][k], ref[k]) < tol, k


def test_degenerate_axes_fp32(port):
    """Splats with an axis below kDegenerateScale never intersect
    (geometry.cpp:37-43): the FP32 depth forms (DepthRec E = (-1, 0..)) give the
    centre depth in the forward and route the depth gradient to the centre in
    the backward's moments, as the reference does."""
    import torch
    import paper_2510_12174_b200 as M
    s = scenes.make_random_scene(1500, 4, 1, seed=91)
    s["log_scales"][::3, 2] = -25.0  # one axis ~1e-11: degenerate
    cam = {"fx": 120.0, "fy": 120.0, "cx": 80.0, "cy": 60.0, "width": 160, "height": 120,
           "R_c2w": np.eye(3), "t_c2w": np.array([0.0, 0.0, -1.2])}
    scene, view, rc, replay, frame = gpu_forward(s, cam, BG, "float32")
    ref = port.render(s, cam, BG)
    got = frame_np(frame)
    same = (got["contributors"] == ref["contributors"]) & (replay.terminus() == ref["terminus"])
    assert 1.0 - same.mean() < 0.01
    for k in ("color", "depth", "transmittance"):
        assert rel_max_err(got[k], ref[k], same) < 1e-4, k
    pix = scenes.pixel_grads(cam["width"], cam["height"], s["num_classes"], seed=9, scale=1.0)
    g = grads_np(M.rasterize_backward(scene, view, frame, replay, torch_pix(pix, torch.float32)))
    rb = port.backward(s, cam, hwc_pix(pix), BG)
    for k, r in grad_parity(g, rb).items():
        assert r["max_rel"] <= 1e-3, (k, r)


def test_bin_and_sort_beyond_shared_counters():
    """More tiles than the shared-memory tile counters hold (31,250 > 24,576):
    the binning falls back to global atomics; lists and order as the reference
    (rasterizer.cpp:14-45)."""
    import paper_2510_12174_b200 as M
    rng = np.random.default_rng(5)
    W, H, n = 4000, 2000, 3000
    cx, cy, rad = rng.random(n) * W, rng.random(n) * H, rng.random(n) * 40
    dep = rng.random(n)
    splats = [{"center": (float(cx[i]), float(cy[i])), "radius": float(rad[i]), "sort_depth": float(dep[i])}
              for i in range(n)]
    rb = M.bin_and_sort(splats, W, H)
    x0 = np.maximum(0, np.floor(cx - rad)).astype(int) // 16
    x1 = np.minimum(W - 1, np.floor(cx + rad)).astype(int) // 16
    y0 = np.maximum(0, np.floor(cy - rad)).astype(int) // 16
    y1 = np.minimum(H - 1, np.floor(cy + rad)).astype(int) // 16
    lists = {}
    for i in np.lexsort((np.arange(n), dep)):
        for ty in range(y0[i], y1[i] + 1):
            for tx in range(x0[i], x1[i] + 1):
                lists.setdefault((tx, ty), []).append(int(i))
    assert (rb.tiles_x, rb.tiles_y) == (250, 125)
    for (tx, ty), want in lists.items():
        assert rb.tile(tx, ty) == want, (tx, ty)
    assert sum(len(v) for v in lists.values()) == len(rb.values)


def test_deterministic_mode_switched_between_forward_and_backward():
    """The FP32 forward skips the BlendRecs when no backward of this mode reads
    them; a deterministic backward after a non-deterministic forward re-runs
    K1 for them and gives the same bits as an all-deterministic pass."""
    import torch
    import paper_2510_12174_b200 as M
    s = scenes.make_random_scene(3000, 6, 2, seed=78)
    cam = {"fx": 120.0, "fy": 120.0, "cx": 80.0, "cy": 60.0, "width": 160, "height": 120,
           "R_c2w": np.eye(3), "t_c2w": np.array([0.0, 0.0, -1.2])}
    pix = scenes.pixel_grads(cam["width"], cam["height"], s["num_classes"], seed=6, scale=1.0)
    M.set_deterministic(True)
    try:
        scene, view, rc, replay, frame = gpu_forward(s, cam, BG, "float32")
        want = grads_np(M.rasterize_backward(scene, view, frame, replay, torch_pix(pix, torch.float32)))
    finally:
        M.set_deterministic(False)
    scene, view, rc, replay, frame = gpu_forward(s, cam, BG, "float32")
    M.set_deterministic(True)
    try:
        got = grads_np(M.rasterize_backward(scene, view, frame, replay, torch_pix(pix, torch.float32)))
    finally:
        M.set_deterministic(False)
    for k in GRAD_NAMES:
        assert np.array_equal(got[k], want[k]), k


@pytest.mark.parametrize("dtype,tol", [("float64", 1e-10), ("float32", 1e-4)])
def test_normals_forward_and_backward(port, dtype, tol):
    import torch
    import paper_2510_12174_b200 as M
    s = scenes.make_room_scene(20000, 3, 1, seed=5, width=96, height=64, f=60.0)
    cam = scenes.view_camera(0, 96, 64, 60.0)
    scene, view, rc, replay, frame = gpu_forward(s, cam, BG, dtype)
    ref = port.render(s, cam, BG)
    # feed the oracle's own depth/T so the comparison isolates the normal kernels
    dt = torch.float64 if dtype == "float64" else torch.float32
    depth = torch.as_tensor(ref["depth"], dtype=dt, device="cuda")
    T = torch.as_tensor(ref["transmittance"], dtype=dt, device="cuda")
    nc = M.NormalConfig()
    nrm = torch.zeros(3, 64, 96, dtype=dt, device="cuda")
    M.estimate_normals(depth, T, view, nc, nrm)
    rn, valid, flipped = port.normals(ref["depth"], ref["transmittance"], cam)
    got = scenes.planar_to_hwc(nrm.double().cpu().numpy())
    assert valid.sum() > 1000
    assert np.array_equal(np.abs(got).sum(-1) > 0, valid.astype(bool))
    assert np.abs(got - rn).max() < (1e-10 if dtype == "float64" else 2e-4)
    dN = scenes.pixel_grads(96, 64, 0, seed=3, scale=1.0)["dnormals"]
    dD = M.normals_backward(torch.as_tensor(dN, dtype=dt, device="cuda"), depth, T, view, nc)
    rdD = port.normals_backward(scenes.planar_to_hwc(dN).astype(np.float64), ref["depth"], ref["transmittance"], cam)
    assert rel_max_err(dD.double().cpu().numpy(), rdD) < tol


@pytest.mark.parametrize("dtype,tol", [("float64", 1e-8), ("float32", 1e-3)])
def test_fused_fwd_bwd_unit(port, dtype, tol):
    """msplat_fwd_bwd == rasterize, estimate_normals, normals_backward merged
    into ddepth, rasterize_backward, chain_activations (trainer.cpp:295-309)."""
    import torch
    import paper_2510_12174_b200 as M
    s = scenes.make_room_scene(30000, 6, 2, seed=11, width=128, height=96, f=90.0)
    cam = scenes.view_camera(1, 128, 96, 90.0)
    dt = torch.float64 if dtype == "float64" else torch.float32
    scene = M.Scene.from_numpy(s, dtype=dt)
    view = M.make_camera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], 128, 96, cam["R_c2w"], cam["t_c2w"])
    pix = scenes.pixel_grads(128, 96, 6, seed=4, scale=1.0)
    frame = M.MultimodalFrame.empty(128, 96, 6, dt, "cuda")
    grads = M.GradientBuffer.zeros_like_scene(scene)
    replay = M.ReplayState()
    for _ in range(2):  # second call takes the asynchronous path
        M.fwd_bwd(scene, view, M.RenderConfig(**BG), M.NormalConfig(), frame, torch_pix(pix, dt), grads, replay)
    M.rasterizer.check_device_errors()
    fr, g_ref, _ = port.fwd_bwd(s, cam, hwc_pix(pix), BG)
    g = grads_np(grads)
    for k in GRAD_NAMES:
        e = rel_l2_err(g[k], g_ref[k])
        print(f"{dtype} {k}: rel L2 {e:.2e}")
        assert e < tol, k
    got_n = scenes.planar_to_hwc(frame.normals.double().cpu().numpy())
    same = frame.contributors.cpu().numpy() == port.render(s, cam, BG)["contributors"]
    assert np.abs(got_n - fr["normals"])[same].max() < (1e-9 if dtype == "float64" else 5e-3)


def test_multiview_accumulation_is_sum_of_views(port):
    """cfg4 semantics: the step gradient is the sum over views of per-view
    rasterize_backward, chained once (chain_activations is linear)."""
    import torch
    import paper_2510_12174_b200 as M
    s = scenes.make_room_scene(20000, 4, 1, seed=2, views=(0, 1, 2), width=96, height=64, f=70.0)
    scene = M.Scene.from_numpy(s, dtype=torch.float64)
    frame = M.MultimodalFrame.empty(96, 64, 4, torch.float64, "cuda")
    grads = M.GradientBuffer.zeros_like_scene(scene)
    replay = M.ReplayState()
    total = None
    for v in range(3):
        cam = scenes.view_camera(v, 96, 64, 70.0)
        view = M.make_camera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], 96, 64, cam["R_c2w"], cam["t_c2w"])
        pix = scenes.pixel_grads(96, 64, 4, seed=v, scale=1.0)
        M.fwd_bwd(scene, view, M.RenderConfig(), M.NormalConfig(), frame, torch_pix(pix, torch.float64), grads,
                  replay, chain=False, accumulate=v > 0)
        _, gv, _ = port.fwd_bwd(s, cam, hwc_pix(pix), {})
        gv = {k: x for k, x in gv.items()}
        total = gv if total is None else {k: total[k] + gv[k] for k in total}
    M.chain_activations(grads, scene)
    g = grads_np(grads)
    # oracle: per-view fwd_bwd already chained; chain is linear so sums agree
    for k in GRAD_NAMES:
        assert rel_l2_err(g[k], total[k]) < 1e-8, k


@pytest.mark.parametrize("graph", [False, True])
def test_multilane_step_gradients_equal_sum_of_views(port, graph):
    """The view-sharded step with its views split over two context lanes on two
    streams (ViewShardedStep(lanes=2): separate replays / frames / gradient
    buffers, summed by msplat_accumulate) gives the oracle's summed, chained
    gradients; also when the step is captured into a CUDA graph."""
    import torch
    import paper_2510_12174_b200 as M
    from paper_2510_12174_b200.distributed import ViewShardedStep
    V, W, H, C = 4, 96, 64, 4
    s = scenes.make_room_scene(20000, C, 1, seed=3, views=tuple(range(V)), width=W, height=H, f=70.0)
    scene = M.Scene.from_numpy(s, dtype=torch.float64)
    n = scene.size()
    off = M.param_layout(n, C, 1)
    flat = M.pack_scene(scene)
    gflat = torch.zeros(off[-1], dtype=torch.float64, device="cuda")
    grads = M.GradientBuffer.from_packed(gflat, n, C, 1)
    cams, pixs, total = [], [], None
    for v in range(V):
        cam = scenes.view_camera(v, W, H, 70.0)
        cams.append(M.make_camera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], W, H, cam["R_c2w"], cam["t_c2w"]))
        pix = scenes.pixel_grads(W, H, C, seed=10 + v, scale=1.0)
        pixs.append(torch_pix(pix, torch.float64))
        _, gv, _ = port.fwd_bwd(s, cam, hwc_pix(pix), {})
        total = dict(gv) if total is None else {k: total[k] + gv[k] for k in total}
    frame = M.MultimodalFrame.empty(W, H, C, torch.float64, "cuda")
    step = ViewShardedStep(scene, flat, gflat, grads, M.OptimizerState(torch.zeros_like(flat), torch.zeros_like(flat), 0),
                           M.TrainConfig(), M.RenderConfig(), M.NormalConfig(), cams, pixs, frame, M.ReplayState(),
                           lanes=2, optimizer=False)  # no Adam: the packed buffer keeps the chained gradients
    assert step.lanes == 2 and step.blocks == [[0, 1], [2, 3]]
    seen = {}
    step()  # sizes the replays (eager)
    if graph:
        torch.cuda.synchronize()
        gflat.zero_()
        g = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        cap.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(g, stream=cap):
            step()
        g.replay()
    torch.cuda.synchronize()
    seen["g"] = gflat.clone()
    from paper_2510_12174_b200.distributed import pack_grad_dict
    assert rel_l2_err(seen["g"].cpu().numpy(), pack_grad_dict(total)) < 1e-8


@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_sharded_adam_ranges_equal_one_full_step(dtype):
    """msplat_adam_step_range over the shards of a sharded optimizer step (the
    ranks' [begin, begin+count) ranges, distributed.shard_range, and ranges
    that start off the 16-byte vector grid) leaves exactly the bits of one
    full adam_step (trainer.cpp:98-133) -- params and both moments."""
    import torch
    import paper_2510_12174_b200 as M
    from paper_2510_12174_b200.distributed import shard_range
    dt = torch.float64 if dtype == "float64" else torch.float32
    n, C, deg = 3001, 5, 2
    s = scenes.make_random_scene(n, num_classes=C, sh_degree=deg, seed=11)
    scene = M.Scene.from_numpy(s, dtype=dt)
    total = M.param_layout(n, C, deg)[-1]
    gen = torch.Generator(device="cuda").manual_seed(3)
    g = torch.randn(total, generator=gen, device="cuda", dtype=dt)
    m0 = torch.randn(total, generator=gen, device="cuda", dtype=dt) * 0.1
    v0 = torch.rand(total, generator=gen, device="cuda", dtype=dt) * 0.01
    grads = M.GradientBuffer.from_packed(g.clone(), n, C, deg)
    grads.raw_space = True
    tc = M.TrainConfig()
    p_full = M.pack_scene(scene)
    st_full = M.OptimizerState(m0.clone(), v0.clone(), 4)
    M.adam_step(scene, grads, st_full, tc, packed_params=p_full, packed_grads=g)  # step 5
    for ranges in ([shard_range(total, r, 3) for r in range(3)], [(0, 7), (7, 1234), (1241, total - 1241)]):
        p = M.pack_scene(scene)
        st = M.OptimizerState(m0.clone(), v0.clone(), 5)
        for b, c in ranges:
            M.rasterizer.adam_step_range(scene, grads, st, tc, p, g, b, c)
        torch.cuda.synchronize()
        assert torch.equal(p, p_full) and torch.equal(st.m, st_full.m) and torch.equal(st.v, st_full.v)
    with pytest.raises(ValueError):
        M.rasterizer.adam_step_range(scene, grads, st, tc, p, g, total - 3, 4)


def test_bin_and_sort_reference_kat():
    """tests/test_rasterizer.cpp:35-88 on the device binning path."""
    import paper_2510_12174_b200 as M
    splats = [{"center": (16.0, 16.0), "radius": 100.0, "sort_depth": 2.0},
              {"center": (4.0, 4.0), "radius": 2.0, "sort_depth": 1.0}]
    bins = M.bin_and_sort(splats, 32, 32)
    assert (bins.tiles_x, bins.tiles_y) == (2, 2)
    assert all(0 in b for b in bins.bins)
    assert bins.tile(0, 0) == [1, 0]
    rng = np.random.default_rng(7)
    rs = [{"center": (40 * rng.random() - 4, 40 * rng.random() - 4), "radius": 6 * rng.random(),
           "sort_depth": rng.random()} for _ in range(100)]
    rb = M.bin_and_sort(rs, 32, 32)
    for ty in range(2):
        for tx in range(2):
            exp = []
            for i, s in enumerate(rs):
                x0 = max(0, int(np.floor(s["center"][0] - s["radius"])))
                x1 = min(31, int(np.floor(s["center"][0] + s["radius"])))
                y0 = max(0, int(np.floor(s["center"][1] - s["radius"])))
                y1 = min(31, int(np.floor(s["center"][1] + s["radius"])))
                if x1 < x0 or y1 < y0:
                    continue
                if x0 // 16 <= tx <= x1 // 16 and y0 // 16 <= ty <= y1 // 16:
                    exp.append(i)
            exp.sort(key=lambda i: (rs[i]["sort_depth"], i))
            assert rb.tile(tx, ty) == exp


@pytest.mark.parametrize("n", [6000, 40000])
def test_bin_and_sort_long_lists_and_depth_ties(n):
    """Per-tile (depth, index) order (rasterizer.cpp:25-28) on tile lists longer
    than one CTA's register sort (2048: the persistent large-list sort; 8192:
    its in-place global-memory network), with many exactly equal depths (index
    tie-break), equal high words (the full-key fix-up) and negative depths."""
    import paper_2510_12174_b200 as M
    rng = np.random.default_rng(n)
    W, H = 64, 48
    cx = rng.random(n) * 80 - 8
    cy = rng.random(n) * 60 - 6
    rad = rng.random(n) * 30
    dep = rng.choice(np.array([-1.5, -0.0, 0.0, 0.25, 0.5, 2.0, 1e-300, 7.0]), n) + \
        np.where(rng.random(n) < 0.5, 0.0, rng.random(n))
    splats = [{"center": (float(cx[i]), float(cy[i])), "radius": float(rad[i]), "sort_depth": float(dep[i])}
              for i in range(n)]
    x0 = np.maximum(0, np.floor(cx - rad)).astype(int)
    x1 = np.minimum(W - 1, np.floor(cx + rad)).astype(int)
    y0 = np.maximum(0, np.floor(cy - rad)).astype(int)
    y1 = np.minimum(H - 1, np.floor(cy + rad)).astype(int)
    ok = (x1 >= x0) & (y1 >= y0)
    for _ in range(2):  # repeatable
        rb = M.bin_and_sort(splats, W, H)
        longest = 0
        for ty in range(3):
            for tx in range(4):
                m = ok & (x0 // 16 <= tx) & (tx <= x1 // 16) & (y0 // 16 <= ty) & (ty <= y1 // 16)
                idx = np.nonzero(m)[0]
                # -0.0 == 0.0 for the reference's std::sort comparator
                exp = idx[np.lexsort((idx, dep[idx] + 0.0))]
                got = rb.tile(tx, ty)
                longest = max(longest, len(got))
                assert got == exp.tolist(), (tx, ty)
        assert longest > 2048


def test_scene_modified_since_forward_is_detected():
    import torch
    import paper_2510_12174_b200 as M
    s = scenes.make_random_scene(5, 1, 0, seed=117)
    cam = scenes.simple_camera()
    scene, view, rc, replay, frame = gpu_forward(s, cam, {}, "float64")
    scene.means[2, 0] += 0.5
    pix = M.PixelGradients.zero(16, 16, 1, dtype=torch.float64)
    with pytest.raises(RuntimeError, match="modified"):
        M.rasterize_backward(scene, view, frame, replay, pix)


def test_non_finite_and_zero_quaternion_primitives_raise():
    import paper_2510_12174_b200 as M
    s = scenes.make_random_scene(10, 2, 1, seed=1)
    s["means"][7, 2] = np.nan
    with pytest.raises(ValueError, match="primitive 7"):
        gpu_forward(s, scenes.simple_camera(), {}, "float32")
    s = scenes.make_random_scene(10, 2, 1, seed=1)
    s["quats"][3] = 0
    with pytest.raises(ValueError, match="primitive 3"):
        gpu_forward(s, scenes.simple_camera(), {}, "float32")
    with pytest.raises(ValueError, match="sh_degree"):
        M.Scene.from_numpy(dict(scenes.make_random_scene(3, 1, 1), sh_degree=4))._abi()
    # SH and semantic rows (scanned block-wide by K1): the first bad primitive
    # is reported, also past the first 256-Gaussian block and at a row tail
    for dtype in ("float32", "float64"):
        for field, idx, val in (("sh", (300, 2, 8), np.inf), ("semantics", (517, 4), np.nan),
                                ("sh", (0, 0, 0), -np.inf), ("semantics", (599, 0), np.inf)):
            s = scenes.make_random_scene(600, 5, 2, seed=2)
            s[field] = np.array(s[field])
            s[field][idx] = val
            with pytest.raises(ValueError, match=f"primitive {idx[0]}"):
                gpu_forward(s, scenes.simple_camera(), {}, dtype)


def test_adam_and_prune_match_oracle(port):
    import torch
    import paper_2510_12174_b200 as M
    s = scenes.make_random_scene(500, 5, 2, seed=9)
    scene = M.Scene.from_numpy(s, dtype=torch.float64)
    rng = np.random.default_rng(0)
    gd = {k: rng.normal(size=getattr(scene, f).shape) for k, f in
          zip(GRAD_NAMES, ("means", "quats", "log_scales", "opacity_logits", "sh", "semantics", "k"))}
    g = M.GradientBuffer(*(torch.as_tensor(gd[k], device="cuda") for k in GRAD_NAMES), raw_space=True)
    st = M.OptimizerState.init(scene)
    tc = M.TrainConfig()
    zeros = {k: np.zeros_like(v) for k, v in gd.items()}
    p_ref, m_ref, v_ref = port.adam(s, gd, zeros, zeros, 1, [tc.lr_position, tc.lr_rotation, tc.lr_scale,
                                                             tc.lr_opacity, tc.lr_sh, tc.lr_semantics, tc.lr_k])
    M.adam_step(scene, g, st, tc)
    for f in ("means", "quats", "log_scales", "opacity_logits", "sh", "semantics", "k"):
        assert np.allclose(getattr(scene, f).cpu().numpy(), p_ref[f], rtol=1e-13, atol=1e-15), f
    # FP32: same step within single-precision rounding
    scene32 = M.Scene.from_numpy(s, dtype=torch.float32)
    g32 = M.GradientBuffer(*(torch.as_tensor(gd[k], device="cuda", dtype=torch.float32) for k in GRAD_NAMES),
                           raw_space=True)
    M.adam_step(scene32, g32, M.OptimizerState.init(scene32), tc)
    for f in ("means", "quats", "log_scales", "opacity_logits", "sh", "semantics", "k"):
        assert np.allclose(getattr(scene32, f).cpu().numpy(), p_ref[f], rtol=2e-6, atol=1e-6), f
    k = rng.uniform(0, 2, 5000)
    for keep_small in (False, True):
        sc = M.Scene.from_numpy(dict(scenes.make_random_scene(5000, 1, 0, seed=3), k=k), dtype=torch.float64)
        st2 = M.OptimizerState.init(sc)
        mask_ref = port.prune_mask(k, 0.5, keep_small)
        removed = M.prune(sc, st2, M.TrainConfig(prune_keep_small=keep_small))
        assert removed == int((~mask_ref).sum())
        assert sc.size() == int(mask_ref.sum())
        assert np.all(sc.k.cpu().numpy() == 0.9)


@pytest.mark.parametrize("dtype", ["float32", "float64"])
@pytest.mark.parametrize("count,offset", [(1, 0), (7, 0), (4096 + 3, 0), (1000, 1)])
def test_accumulate_packed(dtype, count, offset):
    """msplat_accumulate (dst += src) on vector and scalar-tail paths, aligned
    and misaligned views, against the host sum."""
    import torch
    import paper_2510_12174_b200 as M
    dt = getattr(torch, dtype)
    g = torch.Generator().manual_seed(count)
    a = torch.randn(count + offset, generator=g, dtype=torch.float64)
    b = torch.randn(count + offset, generator=g, dtype=torch.float64)
    dst = a.to(dt).cuda()[offset:]
    src = b.to(dt).cuda()[offset:]
    want = (a.to(dt)[offset:] + b.to(dt)[offset:]).numpy()
    M.accumulate_packed(dst, src)
    torch.cuda.synchronize()
    assert np.array_equal(dst.cpu().numpy(), want)
    with pytest.raises(ValueError):
        M.accumulate_packed(dst, src[:-1] if count > 1 else src.double() if dtype == "float32" else src.float())


@pytest.mark.parametrize("deg,C", [(2, 4), (0, 6), (2, 50)])
def test_fp32_packed_scene_and_gradients_odd_n(port, deg, C):
    """FP32 fused step (msplat_fwd_bwd) with the scene AND the gradients as views
    of packed n*P buffers (msplat_param_layout order) at odd n: the semantic
    blocks start at n*(12 + 3K) floats, only 4-byte aligned.
    The 16-byte row staging (K6b, phase A) and the vector gradient adds must
    handle that base; gradients equal the unpacked oracle's."""
    import torch
    import paper_2510_12174_b200 as M
    W, H, n = 96, 64, 4001
    s = scenes.make_room_scene(n, C, deg, seed=7 + C, width=W, height=H, f=70.0)
    cam = scenes.view_camera(2, W, H, 70.0)
    flat = M.pack_scene(M.Scene.from_numpy(s, dtype=torch.float32))
    off = M.param_layout(n, C, deg)
    K = (deg + 1) ** 2
    v = lambda i, *shape: flat[off[i]:off[i + 1]].view(*shape)  # noqa: E731
    scene = M.Scene(v(0, n, 3), v(1, n, 4), v(2, n, 3), v(3, n), v(5, n, 3, K), v(6, n, C), v(4, n),
                    num_classes=C, sh_degree=deg)
    assert scene.semantics.data_ptr() % 8 != 0  # the case under test: a 4-byte aligned semantic base
    view = M.make_camera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], W, H, cam["R_c2w"], cam["t_c2w"])
    pix = scenes.pixel_grads(W, H, C, seed=4, scale=1.0)
    frame = M.MultimodalFrame.empty(W, H, C, torch.float32, "cuda")
    gflat = torch.zeros(off[-1], dtype=torch.float32, device="cuda")
    grads = M.GradientBuffer.from_packed(gflat, n, C, deg)
    assert grads.dsemantics.data_ptr() % 8 != 0
    M.fwd_bwd(scene, view, M.RenderConfig(**BG), M.NormalConfig(), frame, torch_pix(pix, torch.float32),
              grads, M.ReplayState())
    M.rasterizer.check_device_errors()
    fr, g_ref, _ = port.fwd_bwd(s, cam, hwc_pix(pix), BG)
    g = grads_np(grads)
    for k in GRAD_NAMES:
        if g_ref[k].size:
            e = rel_l2_err(g[k], g_ref[k])
            print(f"deg {deg} C {C} {k}: rel L2 {e:.2e}")
            assert e < 1e-3, k
    same = frame.contributors.cpu().numpy() == port.render(s, cam, BG)["contributors"]
    assert same.mean() > 0.99
    if C:
        sem = scenes.planar_to_hwc(frame.semantics.double().cpu().numpy())
        assert rel_max_err(sem, fr["semantics"], np.broadcast_to(same[..., None], sem.shape)) < 1e-4


def test_fp32_prune_mask_bit_exact(port):
    """FP32 scenes: the prune mask (trainer.cpp:135-147) and the compaction
    (:150-168) keep exactly the reference's Gaussians -- the reference's test
    on the float-rounded k values, including values at the threshold edge."""
    import torch
    import paper_2510_12174_b200 as M
    rng = np.random.default_rng(21)
    n = 7001
    k = rng.uniform(0, 2, n).astype(np.float32)
    k[:6] = np.float32([0.5, 1.5, 1.5000001, 0.49999997, 1.0, 0.0])  # edges of |k - 1| > 0.5
    for keep_small in (False, True):
        s = dict(scenes.make_random_scene(n, 2, 1, seed=4), k=k.astype(np.float64))
        sc = M.Scene.from_numpy(s, dtype=torch.float32)
        ids = torch.arange(n, dtype=torch.float32, device="cuda")
        sc.opacity_logits.copy_(ids)  # carries each Gaussian's index through the compaction
        st = M.OptimizerState.init(sc)
        mask_ref = port.prune_mask(k.astype(np.float64), 0.5, keep_small)
        removed = M.prune(sc, st, M.TrainConfig(prune_keep_small=keep_small))
        assert removed == int((~mask_ref).sum())
        assert np.array_equal(sc.opacity_logits.cpu().numpy().astype(np.int64), np.nonzero(mask_ref)[0])


def test_non_finite_output_raises():
    """rasterize: non-finite output at pixel (x,y) (rasterizer.cpp:179-183)."""
    s = scenes.make_random_scene(40, 2, 1, seed=5)
    for dtype in ("float32", "float64"):
        with pytest.raises(RuntimeError, match=r"non-finite output at pixel \(\d+,\d+\)"):
            gpu_forward(s, scenes.simple_camera(), {"background": (float("inf"), 0.0, 0.0)}, dtype)


@pytest.mark.parametrize("dtype", ["float32", "float64"])
@pytest.mark.parametrize("field", ["dcolor", "dsemantics", "ddepth"])
def test_non_finite_pixel_gradient_names_reference_primitive(port, dtype, field):
    """A non-finite pixel gradient makes check_finite (scene.cpp:97-106) throw
    'non-finite gradient for primitive i' with i the LOWEST primitive whose
    gradient is non-finite in the reference -- the primitives blending at that
    pixel, and no others (the FP32 tensor-core products must not spread NaN)."""
    import torch
    import paper_2510_12174_b200 as M
    s, cam = CASES[1]
    scene, view, rc, replay, frame = gpu_forward(s, cam, BG, dtype)
    cont = frame.contributors.cpu().numpy()
    y, x = np.unravel_index(np.argmax(cont), cont.shape)
    pix = scenes.pixel_grads(cam["width"], cam["height"], s["num_classes"], seed=5, scale=1.0)
    pix = {k: np.array(v) for k, v in pix.items()}
    if field == "ddepth":
        pix["ddepth"][y, x] = np.inf
    else:
        pix[field][1, y, x] = np.nan
    import re
    with pytest.raises(Exception) as ei:  # the oracle restates check_finite
        port.backward(s, cam, hwc_pix(pix), BG)
    first = int(re.search(r"non-finite gradient for primitive (\d+)", str(ei.value)).group(1))
    dt = torch.float64 if dtype == "float64" else torch.float32
    with pytest.raises(RuntimeError, match=f"non-finite gradient for primitive {first}$"):
        M.rasterize_backward(scene, view, frame, replay, torch_pix(pix, dt))


@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_deterministic_step_is_graph_capturable(dtype):
    """The deterministic backward (fixed-order reduction, tests/test_rasterizer.cpp:
    386-419) sizes its partial slots from a capacity, so the training step can
    be captured into a CUDA graph: every replay gives the eager step's bits."""
    import torch
    import paper_2510_12174_b200 as M
    from paper_2510_12174_b200.distributed import ViewShardedStep
    dt = torch.float64 if dtype == "float64" else torch.float32
    V, W, H, C = 2, 96, 64, 4
    s = scenes.make_room_scene(20000, C, 1, seed=5, views=tuple(range(V)), width=W, height=H, f=70.0)
    scene = M.Scene.from_numpy(s, dtype=dt)
    n = scene.size()
    flat = M.pack_scene(scene)
    gflat = torch.zeros(M.param_layout(n, C, 1)[-1], dtype=dt, device="cuda")
    grads = M.GradientBuffer.from_packed(gflat, n, C, 1)
    cams, pixs = [], []
    for v in range(V):
        cam = scenes.view_camera(v, W, H, 70.0)
        cams.append(M.make_camera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], W, H, cam["R_c2w"], cam["t_c2w"]))
        pixs.append(torch_pix(scenes.pixel_grads(W, H, C, seed=20 + v, scale=1.0), dt))
    frame = M.MultimodalFrame.empty(W, H, C, dt, "cuda")
    M.set_deterministic(True)
    try:
        step = ViewShardedStep(scene, flat, gflat, grads, M.OptimizerState(torch.zeros_like(flat),
                               torch.zeros_like(flat), 0), M.TrainConfig(), M.RenderConfig(), M.NormalConfig(),
                               cams, pixs, frame, M.ReplayState(), lanes=1, optimizer=False)
        gflat.zero_()
        step()  # eager: sizes the replay, the pair records and the deterministic slots
        torch.cuda.synchronize()
        eager = gflat.clone()
        g = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        cap.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(g, stream=cap):
            step()
        for _ in range(2):
            gflat.zero_()
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
            assert torch.equal(gflat, eager)
        M.rasterizer.check_device_errors()
    finally:
        M.set_deterministic(False)


@pytest.mark.parametrize("C", [0, 1, 8, 9, 57, 64, 65, 72])
def test_forward_paths_across_class_counts(port, C):
    """Both FP32 forward paths against the oracle: the split forward (blend +
    tensor-core semantic pass, C <= 64, n-tile count a template parameter:
    C = 1, 8, 9, 57, 64 cover NT = 1, 1, 2, 8, 8 and partial tiles) and the
    fused kernel (C > 64); C = 0 has no semantic pass.  Then the backward on
    top (weight-row replay after the split forward, the alpha test after the
    fused one) against the oracle's gradients."""
    import torch
    import paper_2510_12174_b200 as M
    cam = {"fx": 40.0, "fy": 36.0, "cx": 33.0, "cy": 21.0, "width": 70, "height": 45,
           "R_c2w": scenes._rot_y(0.1) @ scenes._rot_x(-0.05), "t_c2w": np.array([-0.1, 0.05, -0.4])}
    s = scenes.make_random_scene(400, C, 2, seed=300 + C)
    scene, view, rc, replay, frame = gpu_forward(s, cam, BG, "float32")
    ref = port.render(s, cam, BG)
    got = frame_np(frame)
    same = (got["contributors"] == ref["contributors"]) & (replay.terminus() == ref["terminus"])
    assert 1.0 - same.mean() < 0.01
    for k in ("color", "depth", "kmap", "transmittance"):
        assert rel_max_err(got[k], ref[k], same) < 1e-4, k
    if C:
        assert rel_max_err(got["semantics"], ref["semantics"],
                           np.broadcast_to(same[..., None], got["semantics"].shape)) < 1e-4
    pix = scenes.pixel_grads(cam["width"], cam["height"], C, seed=9, scale=1.0)
    g = grads_np(M.rasterize_backward(scene, view, frame, replay, torch_pix(pix, torch.float32)))
    gref = port.backward(s, cam, hwc_pix(pix), BG)
    for k, r in grad_parity(g, gref).items():
        assert r["max_rel"] <= 1e-3, (k, r)


@pytest.mark.parametrize("frame_per_view", [False, True])
def test_view_sharded_render_matches_single_renders(port, frame_per_view):
    """ViewShardedRender (the forward configs' multi-view driver, two lanes,
    after_view hooks; frame_per_view=True gives every view its own frame) gives
    each view the frame of a plain rasterize + estimate_normals, in FP64 equal to
    the oracle's render; also when the step is captured into a CUDA graph."""
    import torch
    import paper_2510_12174_b200 as M
    from paper_2510_12174_b200.distributed import ViewShardedRender
    V, W, H, C = 4, 80, 56, 3
    s = scenes.make_room_scene(8000, C, 1, seed=21, views=tuple(range(V)), width=W, height=H, f=60.0)
    scene = M.Scene.from_numpy(s, dtype=torch.float64)
    cams_np = [scenes.view_camera(v, W, H, 60.0) for v in range(V)]
    cams = [M.make_camera(c["fx"], c["fy"], c["cx"], c["cy"], W, H, c["R_c2w"], c["t_c2w"]) for c in cams_np]
    head = ViewShardedRender(scene, cams, M.RenderConfig(**BG), M.NormalConfig(), lanes=2,
                             frame_per_view=frame_per_view)
    assert len(head.frames) == (V if frame_per_view else 2)
    got = {}

    def after(k, j, frame):
        got[j] = frame.color.clone()

    head(after)  # eager: sizes the replays
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=cap):
        head(after)
    for t in got.values():
        t.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert sorted(got) == list(range(V))
    for j in range(V):
        ref = port.render(s, cams_np[j], BG)
        assert rel_max_err(scenes.planar_to_hwc(got[j].cpu().numpy()), ref["color"]) < 1e-10, j
        if frame_per_view:
            assert rel_max_err(scenes.planar_to_hwc(head.frames[j].color.cpu().numpy()), ref["color"]) < 1e-10


def test_rasterize_backward_into_packed_out(port):
    """rasterize_backward(out=GradientBuffer.from_packed(...)) writes the same
    gradients as a fresh buffer into the packed views (stale contents are
    overwritten: the library zeroes before accumulating), and rejects an out
    buffer of the wrong shape."""
    import torch
    import paper_2510_12174_b200 as M
    s, cam = CASES[1]
    scene, view, rc, replay, frame = gpu_forward(s, cam, BG, "float32")
    pix = torch_pix(scenes.pixel_grads(cam["width"], cam["height"], s["num_classes"], seed=9, scale=1.0),
                    torch.float32)
    fresh = grads_np(M.rasterize_backward(scene, view, frame, replay, pix))
    n, C, deg = scene.size(), scene.num_classes, scene.sh_degree
    gflat = torch.full((M.param_layout(n, C, deg)[-1],), 7.0, device="cuda")  # stale
    out = M.GradientBuffer.from_packed(gflat, n, C, deg)
    out.raw_space = True
    got = M.rasterize_backward(scene, view, frame, replay, pix, out=out)
    assert got is out and not out.raw_space
    g = grads_np(out)
    for k in GRAD_NAMES:
        assert np.array_equal(g[k], fresh[k]) or rel_l2_err(g[k], fresh[k]) < 1e-6, k
    bad = M.GradientBuffer.from_packed(torch.zeros(M.param_layout(n - 1, C, deg)[-1], device="cuda"), n - 1, C, deg)
    with pytest.raises(ValueError):
        M.rasterize_backward(scene, view, frame, replay, pix, out=bad)
