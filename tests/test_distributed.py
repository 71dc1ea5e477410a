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
