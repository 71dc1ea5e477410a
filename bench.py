#!/usr/bin/env python
"""Benchmark: fwd+bwd multimodal renders/sec, 1M Gaussians @1200x680 (BASELINE.json).

One STEP = one view-sharded training step (BASELINE configs 3/4): each rank
renders V views (default 8) of the 1M-Gaussian, 50-class room scene through
the fused unit msplat_fwd_bwd (rasterize -> estimate_normals ->
normals_backward merged into ddepth -> rasterize_backward), accumulating the
gradients of its views; chain_activations once; with N>1 one NCCL all-reduce
of the packed gradient buffer; then Adam on every rank (identical bits).
value = all ranks' renders / max-over-ranks device time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--views V] [--impl ours|reference]

Under torchrun (N>1) every rank runs; rank 0 prints one JSON line.
--impl reference times the reference's own CPU implementation (oracle/_ref:
the reference sources compiled unmodified) on rank 0 on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fwd+bwd multimodal renders/sec, 1M Gaussians @1200×680; % of HBM roofline"
UNIT = "renders/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--views", type=int, default=8, help="views per rank per step")
    p.add_argument("--lanes", type=int, default=2, help="context lanes (concurrent streams) per rank")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--n", type=int, default=1_000_000)
    p.add_argument("--width", type=int, default=1200)
    p.add_argument("--height", type=int, default=680)
    p.add_argument("--focal", type=float, default=600.0)
    p.add_argument("--classes", type=int, default=50)
    p.add_argument("--sh-degree", type=int, default=2)
    p.add_argument("--no-graph", action="store_true", help="eager launches instead of a CUDA graph")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-train-step", action="store_true", help="skip the full training-iteration measurement")
    p.add_argument("--ref-budget-s", type=float, default=150.0, help="wall budget of the reference arm")
    return p.parse_args()


def pair_counters(frame, replay, early_stop):
    """SURVEY.md section 8d pair counts of one render (view of `frame`):
    Pc = blended pairs (sum of contributors), Pb = backward-visited pairs (sum
    of terminus), Pf = forward-visited pairs (terminus where the pixel
    terminated early, else its tile's whole list)."""
    import numpy as np
    W, H = frame.width, frame.height
    term = replay.terminus().astype(np.int64)
    off, _ = replay.bins()
    tiles_x = (W + 15) // 16
    ty, tx = np.meshgrid(np.arange(H) // 16, np.arange(W) // 16, indexing="ij")
    t = ty * tiles_x + tx
    L = (off[t + 1] - off[t]).astype(np.int64)
    T = frame.transmittance.double().cpu().numpy()
    Pc = int(frame.contributors.long().sum().item())
    Pb = int(term.sum())
    Pf = int(np.where(T < early_stop, term, L).sum())
    return Pc, Pb, Pf


def fp32_peak_tflops():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mhz = float(json.load(f)["sm_max_mhz"])
    except Exception:
        mhz = 1965.0
    return 148 * 128 * 2 * mhz * 1e6 / 1e12, f"nominal: 148 SM x 128 FP32 lanes x 2 x {mhz:.0f} MHz"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md recipe)."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ byte models
def alg_bytes(stage: str, N: int, P: int, HW: int, C: int, I: int) -> float:
    """Algorithmic HBM bytes per launch (per view) of each stage (DESIGN.md,
    following SURVEY.md section 8d's per-unit terms)."""
    f = 4
    if stage == "preprocess":   # params in, alpha+blend records, keys, rects out
        return f * N * P + N * (32 + 128 + 8 + 4 + 4 + 8 + 2)
    if stage == "forward":      # per-instance gathers + list in, 8+C planar outputs
        return f * I * (21 + C) + 4 * I + f * HW * (8 + C)
    if stage == "backward":     # pixel seeds/T/terminus + per-instance gathers in, grads out
        return f * HW * (7 + C) + f * I * (21 + C) + 4 * I + f * N * (20 + C)
    if stage == "binning":      # 12 B per instance written once, read once (key + value)
        return 2 * 12 * I
    if stage == "normals":
        return f * HW * (2 + 3)
    if stage == "normals_bwd":
        return f * HW * (2 + 3 + 12 + 12 + 1)
    if stage == "proj_bwd":
        return f * N * (P + 8 + 7 + 12)
    return 0.0


def render_alg_bytes(N, P, HW, C, I):
    """SURVEY.md 8d B_alg(fwd+bwd) per render."""
    return 4 * 3 * N * P + 4 * HW * (10 + C) + 4 * HW * (10 + C) + 2 * 4 * I * (21 + C) + 2 * 12 * I


# --------------------------------------------------------------- reference
def run_reference_arm(args, rank, world):
    if rank != 0:
        return None
    import numpy as np
    from oracle import oracle as O
    from paper_2510_12174_b200 import scenes
    kind = "reference" if O.available("reference") else "port"
    ora = O.load(kind)
    threads = ref_threads() if kind == "reference" else 1
    s = scenes.make_room_scene(args.n, args.classes, args.sh_degree, seed=0,
                               views=tuple(range(max(args.views * world, 1))), width=args.width,
                               height=args.height, f=args.focal)
    t_start = time.time()
    times, done = [], 0
    total = args.warmup + args.steps
    for it in range(total):
        if it > 0 and time.time() - t_start > args.ref_budget_s:
            break
        cam = scenes.view_camera(it % max(args.views, 1), args.width, args.height, args.focal)
        pix = scenes.pixel_grads(args.width, args.height, args.classes, seed=it)
        pixh = {"dcolor": scenes.planar_to_hwc(pix["dcolor"]).astype(np.float64),
                "ddepth": pix["ddepth"].astype(np.float64),
                "dsemantics": scenes.planar_to_hwc(pix["dsemantics"]).astype(np.float64),
                "dkmap": pix["dkmap"].astype(np.float64),
                "dnormals": scenes.planar_to_hwc(pix["dnormals"]).astype(np.float64)}
        _, _, ms = ora.fwd_bwd(s, cam, pixh, {"background": (0.1, 0.2, 0.3)}, threads=threads, want_frame=False)
        if it >= min(args.warmup, 1):   # CPU needs no warm-up beyond the first call
            times.append(float(sum(ms)))
            done += 1
    ms_per = statistics.mean(times) if times else float("nan")
    value = 1000.0 / ms_per
    sample = (f"{done} full fwd+bwd render(s) of the {args.n}-Gaussian {args.width}x{args.height} "
              f"C={args.classes} scene (rasterize, estimate_normals, normals_backward, rasterize_backward, "
              f"chain_activations; steady_clock around the reference calls)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": done, "warmup": min(args.warmup, 1), "ms_per_step": ms_per, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, world, graph=False),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    return line


def ref_threads():
    n = os.cpu_count() or 1
    try:  # the reference keeps one full gradient buffer per thread (~0.8 KB/Gaussian)
        with open("/proc/meminfo") as f:
            avail_kb = next(int(l.split()[1]) for l in f if l.startswith("MemAvailable"))
        n = min(n, max(1, int(avail_kb / 1.6e6)))
    except Exception:
        pass
    return max(1, min(n, 32))


def cpu_baseline(args):
    import numpy as np
    from oracle import oracle as O
    from paper_2510_12174_b200 import scenes
    kind = "reference" if O.available("reference") else "port"
    ora = O.load(kind)
    threads = ref_threads() if kind == "reference" else 1
    s = scenes.make_room_scene(args.n, args.classes, args.sh_degree, seed=0, views=tuple(range(args.views)),
                               width=args.width, height=args.height, f=args.focal)
    cam = scenes.view_camera(0, args.width, args.height, args.focal)
    pix = scenes.pixel_grads(args.width, args.height, args.classes, seed=0)
    pixh = {"dcolor": scenes.planar_to_hwc(pix["dcolor"]).astype(np.float64),
            "ddepth": pix["ddepth"].astype(np.float64),
            "dsemantics": scenes.planar_to_hwc(pix["dsemantics"]).astype(np.float64),
            "dkmap": pix["dkmap"].astype(np.float64), "dnormals": scenes.planar_to_hwc(pix["dnormals"]).astype(np.float64)}
    _, _, ms = ora.fwd_bwd(s, cam, pixh, {"background": (0.1, 0.2, 0.3)}, threads=threads, want_frame=False)
    total = float(sum(ms))
    return {"value": 1000.0 / total, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"1 full fwd+bwd render (view 0) of the same scene, {total / 1000:.1f} s; stage ms "
                      f"rasterize/normals/normals_bwd/backward/chain = {[round(float(x), 1) for x in ms]}"}


def workload_config(args, world, graph):
    return {"workload": f"cfg3/cfg4: {args.n} Gaussians, {args.width}x{args.height}, C={args.classes}, "
                        f"SH deg {args.sh_degree}; fwd+bwd (+normals, +normal-chain) x{args.views} views/rank, "
                        f"grad all-reduce (N>1) + Adam per step",
            "n_gaussians": args.n, "width": args.width, "height": args.height, "num_classes": args.classes,
            "sh_degree": args.sh_degree, "views_per_rank": args.views, "parallelism": f"view-sharded dp{world}",
            "l2": "inputs larger than L2 (scene 356 MB + 189 MB of pixel gradients per view)",
            "cuda_graph": bool(graph), "lanes": args.lanes,
            "stage_timing": "per-stage CUDA-event brackets from a single-lane replay of the same step"}


# ---------------------------------------------------------------------- ours
def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2510_12174_b200 as M
    from paper_2510_12174_b200 import rasterizer as R, scenes

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    V, C, Wd, Ht = args.views, args.classes, args.width, args.height
    s_np = scenes.make_room_scene(args.n, C, args.sh_degree, seed=0, views=tuple(range(V * world)),
                                  width=Wd, height=Ht, f=args.focal)
    n = args.n
    off = M.param_layout(n, C, args.sh_degree)
    P_total = off[-1]
    P = P_total // n
    K = (args.sh_degree + 1) ** 2
    # Packed parameter buffer; the Scene's tensors are views into it so Adam
    # updates it in place.
    flat = torch.empty(P_total, dtype=torch.float32, device=dev)
    pieces = [s_np["means"], s_np["quats"], s_np["log_scales"], s_np["opacity_logits"], s_np["k"], s_np["sh"],
              s_np["semantics"]]
    for i, a in enumerate(pieces):
        flat[off[i]:off[i + 1]].copy_(torch.from_numpy(np.ascontiguousarray(a).reshape(-1)))
    v = lambda i, *shape: flat[off[i]:off[i + 1]].view(*shape)  # noqa: E731
    scene = M.Scene(v(0, n, 3), v(1, n, 4), v(2, n, 3), v(3, n), v(5, n, 3, K), v(6, n, C), v(4, n), C,
                    args.sh_degree)
    gflat = torch.zeros(P_total, dtype=torch.float32, device=dev)
    grads = M.GradientBuffer.from_packed(gflat, n, C, args.sh_degree)
    opt = M.OptimizerState(torch.zeros_like(flat), torch.zeros_like(flat), 0)
    tc = M.TrainConfig()
    rc = M.RenderConfig(background=(0.1, 0.2, 0.3))
    nc = M.NormalConfig()
    cams = []
    for j in range(V):
        c = scenes.view_camera(rank * V + j, Wd, Ht, args.focal)
        cams.append(M.make_camera(c["fx"], c["fy"], c["cx"], c["cy"], Wd, Ht, c["R_c2w"], c["t_c2w"]))
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    scale = 1.0 / (Wd * Ht)

    def rand(*shape):
        return (torch.rand(*shape, generator=gen, device=dev) * 2 - 1) * scale

    pixs = [M.PixelGradients(rand(3, Ht, Wd), rand(Ht, Wd), rand(C, Ht, Wd), rand(Ht, Wd), rand(3, Ht, Wd))
            for _ in range(V)]
    frame = M.MultimodalFrame.empty(Wd, Ht, C, torch.float32, dev)
    replay = M.ReplayState(device=local_rank)

    from paper_2510_12174_b200.distributed import ViewShardedStep
    sharded = ViewShardedStep(scene, flat, gflat, grads, opt, tc, rc, nc, cams, pixs, frame, replay, world,
                              lanes=args.lanes)

    # Single-lane twin sharing lane 0's frame / replay / gradients: its graph
    # carries the per-stage event brackets (stage times of concurrent lanes
    # would include each other's interference).
    single = ViewShardedStep(scene, flat, gflat, grads, opt, tc, rc, nc, cams, pixs, frame, replay, world, lanes=1)

    def step(pix_list):
        sharded(pix_list)

    stream = torch.cuda.current_stream(dev)
    for _ in range(max(args.warmup, 1)):
        step(pixs)
    torch.cuda.synchronize(dev)
    R.check_device_errors(local_rank)
    counters = replay.counters()
    Pc, Pb, Pf = pair_counters(frame, replay, rc.early_stop_transmittance)

    def capture(fn, timing):
        g = torch.cuda.CUDAGraph()
        s_cap = torch.cuda.Stream(dev)
        s_cap.wait_stream(stream)
        R.set_stage_timing(timing, local_rank)
        try:
            with torch.cuda.graph(g, stream=s_cap):
                fn(pixs)
        finally:
            R.set_stage_timing(False, local_rank)
        torch.cuda.synchronize(dev)
        return g

    graph = stage_graph = None
    if not args.no_graph:
        try:
            graph = capture(step, False)
            stage_graph = capture(single, True)
        except Exception as e:  # noqa: BLE001
            if rank == 0:
                print(f"# cuda graph capture failed ({e}); timing eager launches", file=sys.stderr)
            graph = stage_graph = None
            torch.cuda.synchronize(dev)
    if graph is None:
        R.set_stage_timing(True, local_rank)

    launches0 = R.kernel_launches()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local_rank)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        if graph is not None:
            graph.replay()
        else:
            step(pixs)
    t1.record(stream)
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    ms = t0.elapsed_time(t1)
    launches = R.kernel_launches() - launches0  # 0 under graph replay (no host launches)
    if stage_graph is not None:  # per-stage brackets from a single-lane replay, after the timed region
        stage_graph.replay()
        torch.cuda.synchronize(dev)
    stage = R.stage_timings(local_rank)
    R.set_stage_timing(False, local_rank)
    R.check_device_errors(local_rank)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())

    # kernels per step: count one eager step's launches
    before = R.kernel_launches()
    step(pixs)
    torch.cuda.synchronize(dev)
    kernels_per_step = R.kernel_launches() - before
    if graph is None:
        kernels_per_step = launches // max(args.steps, 1)

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, rank, world, dev, scene, grads, gflat, flat, opt, tc, rc, nc, cams, frame, replay,
                      pixs, step_fn=None)

    train_step = None
    if rank == 0 and world == 1 and not args.no_train_step:
        try:
            train_step = run_train_step(args, dev, scene, flat, opt, tc, rc, nc, cams)
        except Exception as e:  # noqa: BLE001
            train_step = {"error": str(e)}
    if rank != 0:
        return None
    HW = Wd * Ht
    I = counters["instances"]
    renders = world * V * args.steps
    value = renders / (ms_max / 1000.0)
    peak, peak_src = peaks()
    # stage durations: per view-launch averages (graph: last replay; eager: all timed steps)
    per_launch = {k: (t / c if c else 0.0) for k, (t, c) in stage.items()}
    dom = max((k for k in per_launch if k != "optim"), key=lambda k: stage[k][0])
    bytes_dom = alg_bytes(dom, n, P, HW, C, I)
    ach = bytes_dom / (per_launch[dom] / 1000.0) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(dom)
    except Exception:
        pass
    render_ms = sum(per_launch[k] for k in per_launch if k != "optim")
    rb = render_alg_bytes(n, P, HW, C, I)
    # SURVEY.md 8d algorithmic FP32 flops per fwd+bwd render (FMA = 2)
    F_alg = 12 * (Pf + Pb) + Pc * (53 + 2 * C) + Pc * (264 + 8 * C)
    fpk, fpk_src = fp32_peak_tflops()
    t_hbm, t_fp32 = rb / (peak * 1e9), F_alg / (fpk * 1e12)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded room-slab scene, dense U(-1,1)/HW seeds)",
        "config": workload_config(args, world, graph is not None),
        "clocks": clk,
        "e2e": e2e,
        "gpu_launches": int(kernels_per_step * args.steps),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "unit": "GB/s",
                     "frac": ach / peak, "traffic": traffic, "peak_source": peak_src,
                     "alg_bytes_per_launch": bytes_dom, "avg_launch_ms": per_launch[dom]},
        "render_roofline": {"alg_bytes_per_render": rb, "render_device_ms": render_ms,
                            "achieved_gbs": rb / (render_ms / 1000.0) / 1e9,
                            "frac_of_hbm": rb / (render_ms / 1000.0) / 1e9 / peak,
                            "alg_fp32_flops_per_render": F_alg,
                            "achieved_tflops": F_alg / (render_ms / 1000.0) / 1e12,
                            "fp32_peak_tflops": fpk, "fp32_peak_source": fpk_src,
                            "frac_of_fp32": F_alg / (render_ms / 1000.0) / 1e12 / fpk,
                            "roofline_bound_frac": max(t_hbm, t_fp32) / (render_ms / 1000.0)},
        "stage_ms_per_view": {k: round(v, 4) for k, v in per_launch.items()},
        "train_step": train_step,
        "counters": dict(counters, pixels=HW, P=P, Pc_blended_pairs=Pc, Pb_backward_pairs=Pb,
                         Pf_forward_pairs=Pf),
    }
    return line


def run_train_step(args, dev, scene, flat, opt, tc, rc, nc, cams, iters=8, warm=2):
    """One full device-resident training iteration per view, as trainer.cpp:289-328
    (SURVEY.md 8f #1-#2): rasterize, estimate_normals, frame_losses (the six
    losses, combine, seed assembly and the normal chain), rasterize_backward,
    chain_activations and adam_step, through the public API on synthetic ground
    truth.  Timed with CUDA events on the launching stream (informational; the
    headline metric is the reference-comparable fwd+bwd step)."""
    import torch
    import paper_2510_12174_b200 as M
    W, H, C = args.width, args.height, args.classes
    g = torch.Generator(device=dev).manual_seed(5)
    gts = []
    for _ in range(2):
        normal = torch.randn(3, H, W, generator=g, device=dev)
        normal = normal / normal.norm(dim=0, keepdim=True)
        gts.append(M.GroundTruth(torch.rand(3, H, W, generator=g, device=dev),
                                 1.5 + 3.0 * torch.rand(H, W, generator=g, device=dev), normal,
                                 torch.randint(0, C, (H, W), generator=g, device=dev).to(torch.uint8)))
    replay = M.ReplayState()
    lambdas = (1.0, 0.1, 0.1, 0.1, 0.1, 0.1)

    def one(i):
        view = cams[i % len(cams)]
        frame = M.rasterize(scene, view, rc, replay)
        M.estimate_normals(frame.depth, frame.transmittance, view, nc, frame.normals)
        _, pix = M.frame_losses(frame, gts[i % 2], view, nc, lambdas, sync=False)
        gb = M.rasterize_backward(scene, view, frame, replay, pix)
        M.chain_activations(gb, scene)
        M.adam_step(scene, gb, opt, tc, packed_params=flat, packed_grads=M.rasterizer.pack_grads(gb))

    for i in range(warm):
        one(i)
    torch.cuda.synchronize(dev)
    st = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(iters):
        one(warm + i)
    e1.record(st)
    torch.cuda.synchronize(dev)
    M.rasterizer.check_device_errors(dev.index)
    ms = e0.elapsed_time(e1) / iters
    return {"ms_per_iteration": ms, "iterations_per_s": 1000.0 / ms, "iterations": iters,
            "includes": "rasterize, estimate_normals, frame_losses (l1, ssim, normal, depth, seg, k + combine + "
                        "seed assembly + normal chain), rasterize_backward, chain_activations, adam_step; one view "
                        "per iteration (trainer.cpp:289-328), public Python API, synthetic ground truth"}


def run_e2e(args, rank, world, dev, scene, grads, gflat, flat, opt, tc, rc, nc, cams, frame, replay, pixs,
            step_fn=None):
    """Same step through the public API with HOST inputs.  Every step's pixel
    gradients (all views) are copied from pinned host memory and the step's
    result (|grad|_1 of the reduced gradient) is read back to the host.  The
    copies are software-pipelined one step ahead over two device buffer sets:
    while step k renders from set k%2, a copy stream uploads step k+1's inputs
    into the other set (the first step's inputs are uploaded at the start of
    the timed region).  Each step is a CUDA graph of public-API calls
    (ViewShardedStep is capturable); wall-clock timed."""
    import torch
    import torch.distributed as dist

    import paper_2510_12174_b200 as M
    from paper_2510_12174_b200.distributed import ViewShardedStep

    V = len(cams)
    fields = ("dcolor", "ddepth", "dsemantics", "dkmap", "dnormals")
    host = [[getattr(p, f).cpu().pin_memory() for f in fields] for p in pixs]
    sets = [[M.PixelGradients(*(torch.empty_like(getattr(p, f)) for f in fields)) for p in pixs] for _ in range(2)]
    h2d = sum(t.numel() * t.element_size() for t in host[0]) * V
    step = ViewShardedStep(scene, flat, gflat, grads, opt, tc, rc, nc, cams, sets[0], frame, replay, world,
                           lanes=args.lanes)
    copy = torch.cuda.Stream(dev)

    def upload(dst, stream):
        with torch.cuda.stream(stream):
            for j in step.issue_order():
                for f, src in zip(fields, host[j]):
                    getattr(dst[j], f).copy_(src, non_blocking=True)

    def body(k):  # render from set k, upload the next step's inputs into set 1 - k
        main = torch.cuda.current_stream(dev)
        copy.wait_stream(main)
        upload(sets[1 - k], copy)
        step(sets[k])
        main.wait_stream(copy)

    main0 = torch.cuda.current_stream(dev)
    upload(sets[0], main0)
    body(0)  # sizes the lanes' replays (eager)
    torch.cuda.synchronize(dev)
    graphs = None
    if not args.no_graph and world == 1:
        try:
            graphs = []
            for k in range(2):
                g = torch.cuda.CUDAGraph()
                cap = torch.cuda.Stream(dev)
                cap.wait_stream(torch.cuda.current_stream(dev))
                with torch.cuda.graph(g, stream=cap):
                    body(k)
                graphs.append(g)
            torch.cuda.synchronize(dev)
        except Exception as e:  # noqa: BLE001
            print(f"# e2e graph capture failed ({e}); eager", file=sys.stderr)
            graphs = None
            torch.cuda.synchronize(dev)

    def e2e_step(i):
        if graphs is not None:
            graphs[i & 1].replay()
        else:
            body(i & 1)
        return float(gflat.abs().sum().item())  # device -> host read of the step's result

    for i in range(max(1, min(args.warmup, 2))):
        upload(sets[0], main0)
        e2e_step(0)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t = time.perf_counter()
    upload(sets[0], main0)  # the first step's inputs
    for i in range(args.steps):
        e2e_step(i)
    torch.cuda.synchronize(dev)
    dt = time.perf_counter() - t
    if world > 1:
        tt = torch.tensor([dt], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
    return {"value": world * V * args.steps / dt, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": 4,
            "note": f"public Python API (ViewShardedStep over msplat_fwd_bwd, {args.lanes} lanes); every step's "
                    "pixel gradients (all views) copied from pinned host memory, software-pipelined one step "
                    "ahead on a copy stream (first step's upload inside the timed region), |grad|_1 read back "
                    f"every step; steps as CUDA graphs ({'yes' if graphs is not None else 'no, eager'}); wall clock"}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        line = run_reference_arm(args, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    import torch
    import torch.distributed as dist
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    line = run_ours(args, rank, world, local_rank)
    if rank == 0 and line is not None:
        if world == 1 and not args.no_cpu_baseline:
            try:
                line["cpu_baseline"] = cpu_baseline(args)
            except Exception as e:  # noqa: BLE001
                line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "port",
                                        "sample": f"unavailable: {e}"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
