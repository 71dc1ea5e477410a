"""Probe: do two context lanes on two streams (views 0..V/2-1 and V/2..V-1,
separate replays / frames / gradient buffers) beat one lane issuing all V
views in order?  Eager launches, CUDA events around the whole set."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2510_12174_b200 as M  # noqa: E402
from paper_2510_12174_b200 import rasterizer as R, scenes  # noqa: E402

V, Wd, Ht, C, n, f = 8, 1200, 680, 50, 1_000_000, 600.0
s = scenes.make_room_scene(n, C, 2, seed=0, views=tuple(range(V)), width=Wd, height=Ht, f=f)
scene = M.Scene.from_numpy(s)
cams = []
for j in range(V):
    c = scenes.view_camera(j, Wd, Ht, f)
    cams.append(M.make_camera(c["fx"], c["fy"], c["cx"], c["cy"], Wd, Ht, c["R_c2w"], c["t_c2w"]))
g = torch.Generator(device="cuda").manual_seed(0)
sc = 1.0 / (Wd * Ht)
r = lambda *sh: (torch.rand(*sh, generator=g, device="cuda") * 2 - 1) * sc  # noqa: E731
pixs = [M.PixelGradients(r(3, Ht, Wd), r(Ht, Wd), r(C, Ht, Wd), r(Ht, Wd), r(3, Ht, Wd)) for _ in range(V)]
rc, nc = M.RenderConfig(background=(0.1, 0.2, 0.3)), M.NormalConfig()
lanes = 4
frames = [M.MultimodalFrame.empty(Wd, Ht, C, torch.float32, "cuda") for _ in range(lanes)]
grads = [M.GradientBuffer.zeros_like_scene(scene) for _ in range(lanes)]
replays = [M.ReplayState(lane=k) for k in range(lanes)]
main = torch.cuda.current_stream()
sides = [torch.cuda.Stream() for _ in range(lanes)]


def one_lane():
    for j in range(V):
        R.fwd_bwd(scene, cams[j], rc, nc, frames[0], pixs[j], grads[0], replays[0], chain=False, accumulate=j > 0)


def k_lanes(k):
    def fn():
        main = torch.cuda.current_stream()
        for st in sides[1:k]:
            st.wait_stream(main)
        per = V // k
        for j in range(per):
            for l in range(k):
                with torch.cuda.stream(main if l == 0 else sides[l]):
                    R.fwd_bwd(scene, cams[l * per + j], rc, nc, frames[l], pixs[l * per + j], grads[l], replays[l],
                              chain=False, accumulate=j > 0)
        for st in sides[1:k]:
            main.wait_stream(st)
    return fn


def graphed(fn):
    fn()  # sizes the replays (eager)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(main)
    with torch.cuda.graph(gr, stream=cap):
        fn()
    torch.cuda.synchronize()
    return gr.replay


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main)
        fn()
        b.record(main)
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


g1, g2, g4 = graphed(one_lane), graphed(k_lanes(2)), graphed(k_lanes(4))
for _ in range(2):
    t1, t2, t4 = timeit(g1), timeit(g2), timeit(g4)
    print(f"per view: one lane {t1 / V:.3f} ms, two lanes {t2 / V:.3f} ({t1 / t2:.3f}x), four lanes {t4 / V:.3f} ({t1 / t4:.3f}x)")
