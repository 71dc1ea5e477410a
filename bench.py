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


PRESETS = {  # BASELINE.json configs (scenes.CONFIGS); cfg4 = cfg3's scene as the view-sharded step
    "cfg1": dict(n=100_000, width=640, height=480, focal=500.0, classes=16, mode="fwd"),
    "cfg2": dict(n=100_000, width=640, height=480, focal=500.0, classes=16, mode="fwdbwd"),
    "cfg3": dict(n=1_000_000, width=1200, height=680, focal=600.0, classes=50, mode="fwdbwd"),
    "cfg5": dict(n=4_000_000, width=1920, height=1080, focal=960.0, classes=50, mode="fwd"),
}


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--repeats", type=int, default=3, help="timed repeats of --steps steps; value = median")
    p.add_argument("--config", default="cfg3", choices=sorted(PRESETS),
                   help="BASELINE config preset (cfg3 = the headline; with --gpus N it is cfg4)")
    p.add_argument("--views", type=int, default=8, help="views per rank per step")
    p.add_argument("--lanes", type=int, default=2, help="context lanes (concurrent streams) per rank")
    p.add_argument("--exchange", default="sharded", choices=["allreduce", "sharded"],
                   help="gradient exchange of the training step (N>1)")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--n", type=int, default=None)
    p.add_argument("--width", type=int, default=None)
    p.add_argument("--height", type=int, default=None)
    p.add_argument("--focal", type=float, default=None)
    p.add_argument("--classes", type=int, default=None)
    p.add_argument("--mode", default=None, choices=["fwd", "fwdbwd"])
    p.add_argument("--sh-degree", type=int, default=2)
    p.add_argument("--no-graph", action="store_true", help="eager launches instead of a CUDA graph")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-dropin", action="store_true",
                   help="skip the C++ drop-in record (msplat::rasterize + rasterize_backward with host Eigen AoS "
                        "data at the reference API, tools/dropin_bench.cpp)")
    p.add_argument("--no-train-step", action="store_true", help="skip the training-step measurements")
    p.add_argument("--dry-run", action="store_true",
                   help="no CUDA: launcher + gloo exchange of the packed buffer only (no render, no value)")
    p.add_argument("--ref-threads", type=int, default=0, help="reference arm threads (0 = all it can use)")
    p.add_argument("--ref-budget-s", type=float, default=420.0, help="wall budget of the reference arm")
    a = p.parse_args(argv)
    for k, v in PRESETS[a.config].items():
        if getattr(a, k) is None:
            setattr(a, k, v)
    return a


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


def render_alg_bytes(N, P, HW, C, I, mode="fwdbwd"):
    """SURVEY.md 8d B_alg per render (fwd+bwd, or forward only)."""
    if mode == "fwd":
        return 4 * N * P + 4 * HW * (10 + C) + 4 * I * (21 + C) + 2 * 12 * I
    return 4 * 3 * N * P + 4 * HW * (10 + C) + 4 * HW * (10 + C) + 2 * 4 * I * (21 + C) + 2 * 12 * I


def render_alg_flops(Pf, Pb, Pc, C, mode="fwdbwd"):
    """SURVEY.md 8d algorithmic FP32 flops per render (FMA = 2)."""
    if mode == "fwd":
        return 12 * Pf + Pc * (53 + 2 * C)
    return 12 * (Pf + Pb) + Pc * (53 + 2 * C) + Pc * (264 + 8 * C)


# --------------------------------------------------------------- reference
def _ref_pix(args, seed):
    import numpy as np
    from paper_2510_12174_b200 import scenes
    pix = scenes.pixel_grads(args.width, args.height, args.classes, seed=seed)
    return {"dcolor": scenes.planar_to_hwc(pix["dcolor"]).astype(np.float64),
            "ddepth": pix["ddepth"].astype(np.float64),
            "dsemantics": scenes.planar_to_hwc(pix["dsemantics"]).astype(np.float64),
            "dkmap": pix["dkmap"].astype(np.float64),
            "dnormals": scenes.planar_to_hwc(pix["dnormals"]).astype(np.float64)}


def _ref_render(ora, s, cam, args, threads, it):
    """One render of the reference CPU path; returns its wall ms.  fwd:
    rasterize + estimate_normals.  fwdbwd: rasterize, estimate_normals,
    normals_backward, rasterize_backward, chain_activations (steady_clock
    around the reference calls, inside the adapter)."""
    if args.mode == "fwd":
        t = time.perf_counter()
        fr = ora.render(s, cam, {"background": (0.1, 0.2, 0.3)}, threads=threads)
        ora.normals(fr["depth"], fr["transmittance"], cam)
        return (time.perf_counter() - t) * 1000.0
    _, _, ms = ora.fwd_bwd(s, cam, _ref_pix(args, it), {"background": (0.1, 0.2, 0.3)}, threads=threads,
                           want_frame=False)
    return float(sum(ms))


def _ref_scene(args, views):
    from paper_2510_12174_b200 import scenes
    return scenes.make_room_scene(args.n, args.classes, args.sh_degree, seed=0, views=tuple(range(max(views, 1))),
                                  width=args.width, height=args.height, f=args.focal)


def run_reference_arm(args, rank, world):
    if rank != 0:
        return None
    from oracle import oracle as O
    from paper_2510_12174_b200 import scenes
    kind = "reference" if O.available("reference") else "port"
    ora = O.load(kind)
    threads = (args.ref_threads or ref_threads()) if kind == "reference" else 1
    s = _ref_scene(args, args.views * world)
    # --steps K --warmup W as asked when the projected run fits the wall
    # budget (--ref-budget-s); otherwise one warm-up and as many timed renders
    # as fit (reported in `steps` / `warmup`)
    t_start = time.time()
    times, done, warm = [], 0, 0
    it = 0
    while done < args.steps:
        elapsed = time.time() - t_start
        if it > 0:
            per = elapsed / it
            if elapsed + per > args.ref_budget_s and done > 0:
                break
        cam = scenes.view_camera(it % max(args.views, 1), args.width, args.height, args.focal)
        ms = _ref_render(ora, s, cam, args, threads, it)
        it += 1
        per = (time.time() - t_start) / it
        if warm < args.warmup and (warm == 0 or per * (args.warmup - warm + args.steps - done) <= args.ref_budget_s):
            warm += 1
            continue
        times.append(ms)
        done += 1
    ms_per = statistics.median(times) if times else float("nan")
    value = 1000.0 / ms_per
    what = ("rasterize, estimate_normals" if args.mode == "fwd" else
            "rasterize, estimate_normals, normals_backward, rasterize_backward, chain_activations")
    sample = (f"{done} full {'forward' if args.mode == 'fwd' else 'fwd+bwd'} render(s) of the {args.n}-Gaussian "
              f"{args.width}x{args.height} C={args.classes} scene ({what}), median; {threads} thread(s)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": done, "warmup": warm, "ms_per_step": ms_per, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, world, graph=False),
            "repeats": [round(1000.0 / t, 6) for t in times],
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
    from oracle import oracle as O
    from paper_2510_12174_b200 import scenes
    kind = "reference" if O.available("reference") else "port"
    ora = O.load(kind)
    threads = (args.ref_threads or ref_threads()) if kind == "reference" else 1
    s = _ref_scene(args, args.views)
    cam = scenes.view_camera(0, args.width, args.height, args.focal)
    total = _ref_render(ora, s, cam, args, threads, 0)
    return {"value": 1000.0 / total, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"1 full {'forward' if args.mode == 'fwd' else 'fwd+bwd'} render (view 0) of the same scene, "
                      f"{total / 1000:.2f} s"}


def workload_config(args, world, graph):
    name = {"cfg3": "cfg4" if world > 1 else "cfg3"}.get(args.config, args.config)
    passes = ("forward (rasterize + estimate_normals)" if args.mode == "fwd" else
              "fwd+bwd (+normals, +normal-chain), chain once, grad all-reduce (N>1)")
    N, HW, C = args.n, args.width * args.height, args.classes
    K = (args.sh_degree + 1) ** 2
    big = 4 * N * (12 + 3 * K + C) + 4 * HW * (10 + C) * (2 if args.mode == "fwdbwd" else 1)
    return {"workload": f"{name}: {N} Gaussians, {args.width}x{args.height}, C={C}, SH deg {args.sh_degree}; "
                        f"{passes} x{args.views} views/rank; frozen scene (no optimizer in the timed step)",
            "name": name, "mode": args.mode,
            "n_gaussians": N, "width": args.width, "height": args.height, "num_classes": C,
            "sh_degree": args.sh_degree, "views_per_rank": args.views,
            "parallelism": f"view-sharded dp{world}" + (" (replicas, no collective)" if args.mode == "fwd" else ""),
            "l2": (f"inputs larger than L2 ({big / 1e6:.0f} MB of scene + per-view pixel buffers per render)"
                   if big > 126e6 else f"working set {big / 1e6:.0f} MB fits the 126 MB L2 (no flush; L2-resident "
                   "config, HBM fraction not meaningful)")}


def execution_detail(args, graph):
    """How our arm runs the workload (kept out of `config`, which names the
    workload only and is identical on both arms)."""
    return {"cuda_graph": bool(graph), "lanes": args.lanes,
            "stage_timing": "per-stage CUDA-event brackets from a single-lane replay of the same step"}


# ---------------------------------------------------------------------- ours
def build_state(args, rank, world, dev, padded):
    """Scene (views into one packed, optionally padded, parameter buffer),
    gradient buffer, Adam state, cameras and per-view pixel gradients."""
    import numpy as np
    import torch
    import paper_2510_12174_b200 as M
    from paper_2510_12174_b200 import scenes
    from paper_2510_12174_b200.distributed import padded_size
    V, C, Wd, Ht = args.views, args.classes, args.width, args.height
    s_np = scenes.make_room_scene(args.n, C, args.sh_degree, seed=0, views=tuple(range(V * world)),
                                  width=Wd, height=Ht, f=args.focal)
    n = args.n
    off = M.param_layout(n, C, args.sh_degree)
    P_total = off[-1]
    L = padded_size(P_total, world) if padded else P_total
    K = (args.sh_degree + 1) ** 2
    flat = torch.zeros(L, dtype=torch.float32, device=dev)
    pieces = [s_np["means"], s_np["quats"], s_np["log_scales"], s_np["opacity_logits"], s_np["k"], s_np["sh"],
              s_np["semantics"]]
    for i, a in enumerate(pieces):
        flat[off[i]:off[i + 1]].copy_(torch.from_numpy(np.ascontiguousarray(a).reshape(-1)))
    v = lambda i, *shape: flat[off[i]:off[i + 1]].view(*shape)  # noqa: E731
    scene = M.Scene(v(0, n, 3), v(1, n, 4), v(2, n, 3), v(3, n), v(5, n, 3, K), v(6, n, C), v(4, n), C,
                    args.sh_degree)
    cams = []
    for j in range(V):
        c = scenes.view_camera(rank * V + j, Wd, Ht, args.focal)
        cams.append(M.make_camera(c["fx"], c["fy"], c["cx"], c["cy"], Wd, Ht, c["R_c2w"], c["t_c2w"]))
    st = {"scene": scene, "flat": flat, "cams": cams, "n": n, "P": P_total // n, "P_total": P_total}
    if args.mode == "fwdbwd":
        gflat = torch.zeros(L, dtype=torch.float32, device=dev)
        gen = torch.Generator(device=dev).manual_seed(1234 + rank)
        scale = 1.0 / (Wd * Ht)
        rand = lambda *shape: (torch.rand(*shape, generator=gen, device=dev) * 2 - 1) * scale  # noqa: E731
        st.update(gflat=gflat, grads=M.GradientBuffer.from_packed(gflat[:P_total], n, C, args.sh_degree),
                  opt=M.OptimizerState(torch.zeros_like(flat), torch.zeros_like(flat), 0),
                  pixs=[M.PixelGradients(rand(3, Ht, Wd), rand(Ht, Wd), rand(C, Ht, Wd), rand(Ht, Wd),
                                         rand(3, Ht, Wd)) for _ in range(V)],
                  frame=M.MultimodalFrame.empty(Wd, Ht, C, torch.float32, dev),
                  replay=M.ReplayState(device=dev.index))
    return st


def _capture(fn, dev, timing=False):
    import torch
    from paper_2510_12174_b200 import rasterizer as R
    g = torch.cuda.CUDAGraph()
    s_cap = torch.cuda.Stream(dev)
    s_cap.wait_stream(torch.cuda.current_stream(dev))
    R.set_stage_timing(timing, dev.index)
    try:
        with torch.cuda.graph(g, stream=s_cap):
            fn()
    finally:
        R.set_stage_timing(False, dev.index)
    torch.cuda.synchronize(dev)
    return g


def _time_steps(run, steps, repeats, dev, world, clocks_for=None):
    """repeats x (K steps between CUDA events on the launching stream, barrier +
    synchronize on both sides); max over ranks per repeat.  Returns the list of
    per-repeat ms (max over ranks) and the clock record."""
    import torch
    import torch.distributed as dist
    stream = torch.cuda.current_stream(dev)
    out = []
    clocks = ClockSampler(dev.index) if clocks_for else None
    for _ in range(repeats):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(steps):
            run()
        t1.record(stream)
        torch.cuda.synchronize(dev)
        ms = torch.tensor([t0.elapsed_time(t1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        out.append(float(ms.item()))
    clk = clocks.stop() if clocks is not None else None
    return out, clk


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2510_12174_b200 as M
    from paper_2510_12174_b200 import rasterizer as R
    from paper_2510_12174_b200.distributed import ViewShardedRender, ViewShardedStep

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    V, C, Wd, Ht = args.views, args.classes, args.width, args.height
    fwd_only = args.mode == "fwd"
    st = build_state(args, rank, world, dev, padded=not fwd_only and args.exchange == "sharded")
    scene, flat, cams, n, P = st["scene"], st["flat"], st["cams"], st["n"], st["P"]
    rc = M.RenderConfig(background=(0.1, 0.2, 0.3))
    nc = M.NormalConfig()
    tc = M.TrainConfig()

    if fwd_only:
        head = ViewShardedRender(scene, cams, rc, nc, lanes=args.lanes)
        single = ViewShardedRender(scene, cams, rc, nc, lanes=1)
        single.frames, single.replays = head.frames[:1], head.replays[:1]
        frame, replay = head.frames[0], head.replays[0]
        step, stage_fn = (lambda: head()), (lambda: single())
    else:
        gflat, grads, opt, pixs = st["gflat"], st["grads"], st["opt"], st["pixs"]
        frame, replay = st["frame"], st["replay"]
        # headline: render + chain + all-reduce (N>1), no optimizer: the scene stays frozen
        head = ViewShardedStep(scene, flat, gflat, grads, opt, tc, rc, nc, cams, pixs, frame, replay, world,
                               lanes=args.lanes, exchange="allreduce", rank=rank, optimizer=False)
        # single-lane twin sharing lane 0's frame / replay / gradients: its graph carries the per-stage
        # event brackets (stage times of concurrent lanes would include each other's interference)
        single = ViewShardedStep(scene, flat, gflat, grads, opt, tc, rc, nc, cams, pixs, frame, replay, world,
                                 lanes=1, exchange="allreduce", rank=rank, optimizer=False)
        step, stage_fn = (lambda: head()), (lambda: single())

    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize(dev)
    R.check_device_errors(local_rank)
    counters = replay.counters()  # the frozen scene's counters (view 0 of lane 0)
    Pc, Pb, Pf = pair_counters(frame, replay, rc.early_stop_transmittance)
    graph = stage_graph = None
    if not args.no_graph:
        try:
            graph = _capture(step, dev)
            stage_graph = _capture(stage_fn, dev, timing=True)
        except Exception as e:  # noqa: BLE001
            if rank == 0:
                print(f"# cuda graph capture failed ({e}); timing eager launches", file=sys.stderr)
            graph = stage_graph = None
            torch.cuda.synchronize(dev)
    if graph is None:
        R.set_stage_timing(True, local_rank)
    run = graph.replay if graph is not None else step
    for _ in range(2):  # settle the graph before the timed region
        run()
    launches0 = R.kernel_launches()
    reps, clk = _time_steps(run, args.steps, max(1, args.repeats), dev, world, clocks_for=True)
    launches = R.kernel_launches() - launches0  # 0 under graph replay (no host launches)
    if stage_graph is not None:  # per-stage brackets from a single-lane replay, after the timed region
        stage_graph.replay()  # its event-record nodes are the only brackets held
        torch.cuda.synchronize(dev)
    stage = R.stage_timings(local_rank)
    R.set_stage_timing(False, local_rank)
    R.check_device_errors(local_rank)
    ms_med = statistics.median(reps)

    # kernels per step: count one eager step's launches
    before = R.kernel_launches()
    step()
    torch.cuda.synchronize(dev)
    kernels_per_step = R.kernel_launches() - before
    if graph is None:
        kernels_per_step = launches // max(args.steps * max(1, args.repeats), 1)

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        if fwd_only:
            e2e = run_e2e_fwd(args, rank, world, dev, head)
        else:
            e2e = run_e2e(args, rank, world, dev, st, tc, rc, nc)

    # ---- the training step (exchange + Adam: the scene drifts, so it runs after the headline)
    training = None
    if not fwd_only and not args.no_train_step:
        try:
            training = run_training_step(args, rank, world, dev, st, tc, rc, nc, frame, replay)
        except Exception as e:  # noqa: BLE001
            training = {"error": str(e)}
    train_iter = None
    if rank == 0 and world == 1 and not fwd_only and not args.no_train_step:
        try:
            train_iter = run_train_step(args, dev, scene, flat[:st["P_total"]], tc, rc, nc, cams)
        except Exception as e:  # noqa: BLE001
            train_iter = {"error": str(e)}
    comm = None
    if world > 1:
        ones = torch.ones(1, device=dev)
        dist.all_reduce(ones)
        comm = {"backend": dist.get_backend(), "ranks_reporting": int(ones.item()),
                "nccl_version": ".".join(map(str, torch.cuda.nccl.version())),
                "collectives_per_step": ("1 all-reduce of the packed n*P gradient (headline); training step: "
                                         f"{args.exchange}")}
    if rank != 0:
        return None
    HW = Wd * Ht
    I = counters["instances"]
    renders = world * V * args.steps
    value = renders / (ms_med / 1000.0)
    peak, peak_src = peaks()
    per_launch = {k: (t / c if c else 0.0) for k, (t, c) in stage.items()}
    dom = max((k for k in per_launch if k != "optim"), key=lambda k: stage[k][0])
    bytes_dom = alg_bytes(dom, n, P, HW, C, I)
    ach = bytes_dom / (per_launch[dom] / 1000.0) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tj = json.load(f)
        traffic = tj.get(args.config, tj).get(dom) if isinstance(tj.get(args.config, tj), dict) else None
    except Exception:
        pass
    render_ms = sum(per_launch[k] for k in per_launch if k != "optim")
    rb = render_alg_bytes(n, P, HW, C, I, args.mode)
    F_alg = render_alg_flops(Pf, Pb, Pc, C, args.mode)
    fpk, fpk_src = fp32_peak_tflops()
    t_hbm, t_fp32 = rb / (peak * 1e9), F_alg / (fpk * 1e12)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_med / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded room-slab scene, dense U(-1,1)/HW seeds)",
        "config": workload_config(args, world, graph is not None),
        "execution": execution_detail(args, graph is not None),
        "repeats": [round(renders / (m / 1000.0), 3) for m in reps],
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
        "training_step": training,
        "train_iteration": train_iter,
        "comm": comm,
        "counters": dict(counters, pixels=HW, P=P, Pc_blended_pairs=Pc, Pb_backward_pairs=Pb,
                         Pf_forward_pairs=Pf),
    }
    return line


def run_training_step(args, rank, world, dev, st, tc, rc, nc, frame, replay):
    """The full view-sharded training step (BASELINE cfg4): render + chain +
    exchange (--exchange: all-reduce + replicated Adam, or reduce-scatter ->
    Adam on the shard -> all-gather) + Adam, as a CUDA graph.  Timed after the
    headline because Adam moves the scene."""
    import torch
    from paper_2510_12174_b200.distributed import ViewShardedStep
    exch = args.exchange if world > 1 else "allreduce"
    if exch == "sharded" and st["flat"].numel() == st["P_total"] and world > 1:
        exch = "allreduce"
    step = ViewShardedStep(st["scene"], st["flat"], st["gflat"], st["grads"], st["opt"], tc, rc, nc, st["cams"],
                           st["pixs"], frame, replay, world, lanes=args.lanes, exchange=exch, rank=rank,
                           optimizer=True)
    step()
    torch.cuda.synchronize(dev)
    run = step
    if not args.no_graph:
        try:
            g = _capture(step, dev)
            run = g.replay
        except Exception:  # noqa: BLE001
            torch.cuda.synchronize(dev)
    run()
    reps, _ = _time_steps(run, args.steps, 1, dev, world)
    ms = reps[0] / args.steps
    return {"value": world * args.views / (ms / 1000.0), "unit": UNIT, "ms_per_step": ms,
            "exchange": exch if world > 1 else "none (N=1)",
            "includes": f"{args.views} views/rank fwd+bwd, lane sum, chain, "
                        f"{'exchange, ' if world > 1 else ''}Adam on the packed buffer"}


def run_train_step(args, dev, scene, flat, tc, rc, nc, cams, iters=8, warm=2):
    """One full device-resident training iteration per view, as trainer.cpp:289-328
    (SURVEY.md 8f #1-#2): rasterize, estimate_normals, frame_losses (the six
    losses, combine, seed assembly and the normal chain), rasterize_backward,
    chain_activations and adam_step, through the public API on synthetic ground
    truth.  Timed with CUDA events on the launching stream (informational; the
    headline metric is the reference-comparable fwd+bwd step)."""
    import torch
    import paper_2510_12174_b200 as M
    W, H, C = args.width, args.height, args.classes
    opt = M.OptimizerState(torch.zeros_like(flat), torch.zeros_like(flat), 0)
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
    gflat = torch.empty_like(flat)  # the packed gradient buffer, written in place by the backward
    gb = M.GradientBuffer.from_packed(gflat, scene.size(), scene.num_classes, scene.sh_degree)

    def one(i):
        view = cams[i % len(cams)]
        frame = M.rasterize(scene, view, rc, replay)
        M.estimate_normals(frame.depth, frame.transmittance, view, nc, frame.normals)
        _, pix = M.frame_losses(frame, gts[i % 2], view, nc, lambdas, sync=False)
        M.rasterize_backward(scene, view, frame, replay, pix, out=gb)
        M.chain_activations(gb, scene)
        M.adam_step(scene, gb, opt, tc, packed_params=flat, packed_grads=gflat)

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


def run_e2e(args, rank, world, dev, st, tc, rc, nc):
    """The headline step through the public API with HOST inputs.  Every step's
    pixel gradients (all views) are copied from pinned host memory and the
    step's result (|grad|_1 of the reduced gradient) is read back to the host.
    The copies run on a copy stream, software-pipelined over two device buffer
    sets: while step k renders from set k%2, step k+1's inputs are uploaded
    into the other set (K steps, K uploads, the first one inside the timed
    region too).  Each view of a step renders as soon as its own inputs have
    landed (per-view external events waited on inside the step's CUDA graph),
    so the link stays busy and the renders trail it.  Each step is a CUDA
    graph of public-API calls (ViewShardedStep is capturable); wall-clock
    timed, max over ranks."""
    import torch
    import torch.distributed as dist

    import paper_2510_12174_b200 as M
    from paper_2510_12174_b200.distributed import ViewShardedStep

    pixs, cams, gflat = st["pixs"], st["cams"], st["gflat"]
    V = len(cams)
    fields = ("dcolor", "ddepth", "dsemantics", "dkmap", "dnormals")
    host = [[getattr(p, f).cpu().pin_memory() for f in fields] for p in pixs]
    sets = [[M.PixelGradients(*(torch.empty_like(getattr(p, f)) for f in fields)) for p in pixs] for _ in range(2)]
    h2d = sum(t.numel() * t.element_size() for t in host[0]) * V
    step = ViewShardedStep(st["scene"], st["flat"], gflat, st["grads"], st["opt"], tc, rc, nc, cams, sets[0],
                           st["frame"], st["replay"], world, lanes=args.lanes, exchange="allreduce", rank=rank,
                           optimizer=False)
    copy = torch.cuda.Stream(dev)
    result = torch.empty(1, dtype=torch.float32, device=dev)
    res_host = torch.empty(1, dtype=torch.float32).pin_memory()

    # ready[k][j]: view j's inputs in set k have landed.  External events: the
    # step graphs below contain a wait node per view on them, so a view renders
    # as soon as its own inputs are on the device -- also across the graph
    # boundary, while the copy stream keeps the link busy with the next step.
    ready = [[torch.cuda.Event(external=True) for _ in range(V)] for _ in range(2)]

    def upload(k):
        """Step inputs into set k on the copy stream (eager, asynchronous)."""
        with torch.cuda.stream(copy):
            for j in step.issue_order():
                for f, src in zip(fields, host[j]):
                    getattr(sets[k][j], f).copy_(src, non_blocking=True)
                ready[k][j].record(copy)

    def body(k):  # one step rendering from set k, each view after its inputs' event
        step(sets[k], before_view=lambda j: torch.cuda.current_stream(dev).wait_event(ready[k][j]))
        torch.sum(gflat[:st["P_total"]].abs(), dim=0, keepdim=True, out=result)

    upload(0)
    upload(1)
    body(0)  # sizes the lanes' replays (eager)
    body(1)
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

    def run_steps(K):
        """K steps; step i's inputs are uploaded inside the call: set 0 before
        the first step, step i + 1's while step i renders (its set was last read
        by step i - 1, which has completed: its result was read back)."""
        upload(0)
        out = 0.0
        for i in range(K):
            k = i & 1
            if graphs is not None:
                graphs[k].replay()
            else:
                body(k)
            if i + 1 < K:  # queued behind step i's own uploads on the copy stream
                upload(1 - k)
            res_host.copy_(result)  # device -> host read of the step's result (synchronizes the step)
            out = float(res_host.item())
        return out

    for _ in range(max(1, min(args.warmup, 2))):
        run_steps(2)
    vals = []
    for _ in range(max(1, args.repeats)):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t = time.perf_counter()
        run_steps(args.steps)
        torch.cuda.synchronize(dev)
        dt = time.perf_counter() - t
        if world > 1:
            tt = torch.tensor([dt], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt = float(tt.item())
        vals.append(world * V * args.steps / dt)
    return {"value": statistics.median(vals), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": 4, "repeats": [round(v, 3) for v in vals],
            "note": f"public Python API (ViewShardedStep over msplat_fwd_bwd, {args.lanes} lanes); every step's "
                    "pixel gradients (all views) copied from pinned host memory inside the timed region on a copy "
                    "stream, software-pipelined one step ahead; each view renders once its own inputs have "
                    "landed (per-view events); |grad|_1 read back "
                    f"every step; steps as CUDA graphs ({'yes' if graphs is not None else 'no, eager'}); wall clock"}


def run_e2e_fwd(args, rank, world, dev, head):
    """Forward configs end to end through the public API: every view's
    rendered modalities (colour, depth, normals, semantic logits, k map; the
    frame's FP32 planes) are copied to pinned host memory.  The views render
    into their own frames (ViewShardedRender(frame_per_view=True), same lanes
    and scene as `head`), and each view's copy runs on a copy stream as soon as
    the view is rendered, so the lanes keep rendering while the link drains the
    finished views; a step ends when its last copy has landed.  The inputs of a
    render are its camera (host struct, a few hundred bytes) and the resident
    scene, so h2d is 0 tensor bytes.  Wall-clock timed."""
    import torch
    import torch.distributed as dist

    from paper_2510_12174_b200.distributed import ViewShardedRender
    e2e_head = ViewShardedRender(head.scene, head.cameras, head.rc, head.nc, lanes=head.lanes,
                                 frame_per_view=True)
    e2e_head.replays = head.replays  # the lanes' sized replays
    fields = ("color", "depth", "normals", "semantics", "kmap")
    f0 = e2e_head.frames[0]
    V = len(head.cameras)
    host = [[torch.empty(getattr(f0, f).shape, dtype=getattr(f0, f).dtype).pin_memory() for f in fields]
            for _ in range(V)]
    d2h = sum(t.numel() * t.element_size() for t in host[0]) * V
    copy = torch.cuda.Stream(dev)

    def after(k, j, frame):  # on the lane's stream, right after view j's render
        copy.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(copy):
            for f, dst in zip(fields, host[j]):
                dst.copy_(getattr(frame, f), non_blocking=True)

    def run_step():
        e2e_head(after)
        torch.cuda.current_stream(dev).wait_stream(copy)

    run_step()  # eager: sizes the replays
    torch.cuda.synchronize(dev)
    graph = None
    if not args.no_graph and world == 1:  # eager renders read their counters back, queued behind the copies
        try:
            graph = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream(dev)
            cap.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.graph(graph, stream=cap):
                run_step()
            torch.cuda.synchronize(dev)
            graph.replay()
            torch.cuda.synchronize(dev)
        except Exception as e:  # noqa: BLE001
            print(f"# e2e graph capture failed ({e}); eager", file=sys.stderr)
            graph = None
            torch.cuda.synchronize(dev)
    vals = []
    for _ in range(max(1, args.repeats)):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t = time.perf_counter()
        for _ in range(args.steps):
            if graph is not None:
                graph.replay()
            else:
                run_step()
        torch.cuda.synchronize(dev)
        dt = time.perf_counter() - t
        if world > 1:
            tt = torch.tensor([dt], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt = float(tt.item())
        vals.append(world * V * args.steps / dt)
    return {"value": statistics.median(vals), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": int(d2h),
            "repeats": [round(v, 3) for v in vals],
            "note": "public Python API (ViewShardedRender(frame_per_view=True): rasterize + estimate_normals per "
                    "view); every view's colour, depth, normals, semantic logits and k map copied to pinned host "
                    "memory on a copy stream as soon as the view is rendered; steps as CUDA graphs "
                    f"({'yes' if graph is not None else 'no, eager'}); wall clock"}


def relaunch_under_torchrun(args_argv, n):
    """--gpus N without a torchrun environment: start N ranks ourselves (one
    process per GPU, rendezvous on 127.0.0.1) and pass rank 0's line through."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")               # communicator-init lines (nranks) ...
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")   # ... on stderr: stdout carries only the JSON line
    # the ranks read their arguments from the environment: torchrun's own parser
    # would take abbreviations such as --n for its options
    env["MSPLAT_BENCH_ARGV"] = json.dumps(list(args_argv))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)]
    return subprocess.call(cmd, env=env)


def run_dry(args, rank, world):
    """No CUDA device: the launcher and the exchange plumbing only.  Every rank
    joins a gloo group, all-reduces and reduce-scatters / all-gathers a packed
    buffer of the workload's n*P length, and rank 0 reports how many ranks
    took part.  No render runs, so there is no throughput value."""
    import torch
    import torch.distributed as dist
    from paper_2510_12174_b200.distributed import padded_size
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("gloo")
    K = (args.sh_degree + 1) ** 2
    total = args.n * (12 + 3 * K + args.classes)
    L = padded_size(total, world)
    g = torch.full((L,), float(rank + 1))
    t = time.perf_counter()
    if world > 1:
        dist.all_reduce(g)
        shard = torch.empty(L // world)
        dist.reduce_scatter_tensor(shard, g)
        dist.all_gather_into_tensor(g, shard)
    dt = time.perf_counter() - t
    ones = torch.ones(1)
    if world > 1:
        dist.all_reduce(ones)
    expect = world * (world + 1) / 2 * (world if world > 1 else 1)
    ok = bool(torch.all(g == expect).item())
    if rank != 0:
        return None
    return {"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": world, "steps": 0, "warmup": 0,
            "ms_per_step": None, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": workload_config(args, world, graph=False),
            "dry_run": "no CUDA device: launcher + gloo exchange of the packed buffer only, no render, no value",
            "comm": {"backend": "gloo" if world > 1 else None, "ranks_reporting": int(ones.item()),
                     "exchange_ok": ok, "exchange_s": dt, "packed_elements": total, "padded_elements": L}}


def main(argv=None):
    if argv is None:
        argv = json.loads(os.environ["MSPLAT_BENCH_ARGV"]) if "MSPLAT_BENCH_ARGV" in os.environ else sys.argv[1:]
    args = parse(argv)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(argv, args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and "--gpus" in " ".join(argv):
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        line = run_reference_arm(args, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    import torch
    import torch.distributed as dist
    if args.dry_run or not torch.cuda.is_available():
        line = run_dry(args, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
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
        if world == 1 and not args.no_dropin and args.config in ("cfg2", "cfg3"):
            # the plugin boundary: the reference API (rasterizer.hpp:67-83) through the C++ drop-in, host
            # AoS in and out, one render per call (view 0 of the same scene), FP32 / FP64 x deterministic
            try:
                sys.path.insert(0, os.path.join(ROOT, "tools"))
                import dropin_bench
                line["dropin_e2e"] = {"unit": "renders/s (one fwd+bwd per call, wall clock)",
                                      "records": dropin_bench.run_modes(args.config, iters=2, warmup=1)}
            except Exception as e:  # noqa: BLE001
                line["dropin_e2e"] = {"unavailable": str(e)[:300]}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
