"""CPU, world size 2 over gloo: the view-sharded step's host logic.

Each rank computes the chained gradients of its shard of views with the CPU
oracle (the GPU kernels are covered by the gpu tests), packs them in
msplat_param_layout order and runs the step's one collective
(distributed.reduce_gradients).  The reduced buffer must equal the
single-process sum over all views, and be identical on both ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _views_grads(views):
    import sys
    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    from paper_2510_12174_b200 import distributed as D, scenes
    from helpers import hwc_pix
    port = O.load("port")
    s = scenes.make_room_scene(3000, 4, 1, seed=4, views=tuple(range(4)), width=48, height=32, f=30.0)
    total = None
    for v in views:
        cam = scenes.view_camera(v, 48, 32, 30.0)
        pix = scenes.pixel_grads(48, 32, 4, seed=v, scale=1.0)
        _, g, _ = port.fwd_bwd(s, cam, hwc_pix(pix), {})
        p = D.pack_grad_dict(g)
        total = p if total is None else total + p
    return total


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2510_12174_b200 import distributed as D
    mine = D.shard_views(4, rank, world)
    flat = torch.from_numpy(_views_grads(mine))
    D.reduce_gradients(flat, world)
    q.put((rank, mine, flat.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_lane_views_partitions_a_ranks_views():
    from paper_2510_12174_b200.distributed import lane_views
    assert lane_views(8, 2) == [[0, 1, 2, 3], [4, 5, 6, 7]]
    assert lane_views(5, 2) == [[0, 1], [2, 3, 4]]
    assert lane_views(3, 1) == [[0, 1, 2]]
    for V in range(1, 12):
        for L in range(1, 5):
            parts = lane_views(V, L)
            assert sum(parts, []) == list(range(V)) and len(parts) == L
    with pytest.raises(ValueError):
        lane_views(4, 0)


def test_shard_views_partitions_all_views():
    from paper_2510_12174_b200.distributed import shard_views
    for total in (1, 7, 8, 64):
        for world in (1, 2, 3, 8):
            parts = [shard_views(total, r, world) for r in range(world)]
            assert sum(parts, []) == list(range(total))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1


@pytest.mark.timeout(600)
def test_two_rank_gradient_allreduce_equals_single_process_sum():
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert res[0][1] == [0, 1] and res[1][1] == [2, 3]
    assert np.array_equal(res[0][2], res[1][2])          # identical bits on every rank
    ref = _views_grads([0, 1, 2, 3])
    assert np.allclose(res[0][2], ref, rtol=1e-12, atol=1e-18)


# ---------------------------------------------------------------------------
# ViewShardedStep itself on CPU tensors over gloo: the step order (per-view
# accumulation -> chain once -> exchange -> Adam) with the oracle doing the
# per-view math (tests/oracle_ops.py).  Both exchanges must leave identical
# bits on every rank, and the sharded exchange (reduce-scatter -> Adam on the
# shard -> all-gather) must equal the all-reduce + replicated Adam bitwise.
N_G, C_S, DEG, W_S, H_S = 1500, 3, 1, 40, 32


def _step_setup(total_views, rank, world, exchange):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle import oracle as O
    from paper_2510_12174_b200 import distributed as D, scenes
    from paper_2510_12174_b200.rasterizer import OptimizerState, TrainConfig
    from helpers import hwc_pix
    import oracle_ops as OO
    port = O.load("port")
    ops = OO.OracleOps(port)
    s = scenes.make_room_scene(N_G, C_S, DEG, seed=4, views=tuple(range(total_views)), width=W_S, height=H_S,
                               f=25.0)
    total = ops.packed_total(s)
    L = D.padded_size(total, world) if exchange == "sharded" else total
    flat = torch.zeros(L, dtype=torch.float64)
    flat[:total] = torch.from_numpy(OO.pack_scene(s))
    gflat = torch.zeros(L, dtype=torch.float64)
    opt = OptimizerState(torch.zeros(L, dtype=torch.float64), torch.zeros(L, dtype=torch.float64), 0)
    mine = D.shard_views(total_views, rank, world)
    cams = [scenes.view_camera(v, W_S, H_S, 25.0) for v in mine]
    pixs = [hwc_pix(scenes.pixel_grads(W_S, H_S, C_S, seed=v, scale=1.0)) for v in mine]
    grads = OO.GradView(gflat)
    step = D.ViewShardedStep((s, flat), flat, gflat, grads, opt, TrainConfig(), {}, {}, cams, pixs, None, None,
                             world=world, lanes=1, exchange=exchange, rank=rank, ops=ops)
    return step, flat, total


def _step_worker(rank, world, port, exchange, steps, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    step, flat, total = _step_setup(4, rank, world, exchange)
    for _ in range(steps):
        step()
    q.put((rank, flat[:total].numpy().copy(), step.gflat[:total].numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


def _run_two_ranks(exchange, steps):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_step_worker, args=(r, 2, port, exchange, steps, q)) for r in range(2)]
    for p in procs:
        p.start()
    import queue
    import time
    res, t0 = [], time.time()
    while len(res) < 2:  # fail fast if a rank dies instead of waiting out the queue
        try:
            res.append(q.get(timeout=2))
        except queue.Empty:
            assert all(p.exitcode in (None, 0) for p in procs), "a rank failed"
            assert time.time() - t0 < 600, "ranks timed out"
    res.sort(key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.timeout(900)
def test_view_sharded_step_exchanges_agree_bitwise_across_ranks():
    ar = _run_two_ranks("allreduce", 2)
    sh = _run_two_ranks("sharded", 2)
    assert np.array_equal(ar[0][1], ar[1][1])        # all-reduce: identical parameters on every rank
    assert np.array_equal(sh[0][1], sh[1][1])        # sharded: identical parameters on every rank
    assert np.array_equal(sh[0][1], ar[0][1])        # sharded Adam == replicated Adam, bit for bit
    # the single-process sequence: all four views on one rank, same order of operations up to
    # the (linear) chain being applied to per-rank sums
    step, flat, total = _step_setup(4, 0, 1, "allreduce")
    for _ in range(2):
        step()
    assert np.allclose(ar[0][1], flat[:total].numpy(), rtol=1e-12, atol=1e-15)
    assert not np.array_equal(flat[:total].numpy(), _step_setup(4, 0, 1, "allreduce")[1][:total].numpy())


def test_shard_ranges_cover_the_buffer():
    from paper_2510_12174_b200.distributed import padded_size, shard_range
    for total in (0, 1, 7, 89, 89_000_001):
        for world in (1, 2, 3, 8):
            L = padded_size(total, world)
            assert L >= total and L % (4 * world) == 0 and L - total < 4 * world
            parts = [shard_range(total, r, world) for r in range(world)]
            covered = [i for b, c in parts for i in range(b, b + c)] if total < 1000 else None
            if covered is not None:
                assert covered == list(range(total))
            assert sum(c for _, c in parts) == total
            assert all(b % 4 == 0 for b, c in parts if c)
