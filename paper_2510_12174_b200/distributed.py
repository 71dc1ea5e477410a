"""View-sharded training step across GPUs (BASELINE config 4).

The path shards by view: every rank holds a replica of the scene, renders its
own views through msplat_fwd_bwd, sums their gradients locally, and the ranks
exchange exactly one collective per step -- an all-reduce (sum) of the packed
n*P gradient buffer (msplat_param_layout order).  chain_activations is linear
per Gaussian, so it is applied once to the local sum before the reduction; the
replicated Adam step then leaves identical parameters on every rank.

Only the reduction touches torch.distributed (NCCL on GPUs, gloo in the CPU
tests); the kernels never wait on another rank.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def shard_views(total_views: int, rank: int, world: int) -> list[int]:
    """Contiguous block of view indices owned by `rank` (sizes differ by <= 1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("shard_views: bad rank/world")
    lo = total_views * rank // world
    hi = total_views * (rank + 1) // world
    return list(range(lo, hi))


GRAD_ORDER = ("dposition", "drotation", "dscale", "dopacity", "dk", "dsh", "dsemantics")


def pack_grad_dict(g: dict) -> np.ndarray:
    """Pack a per-attribute gradient dict (reference layouts) into the
    msplat_param_layout order: means, quats, log_scales, opacity, k, sh, semantics."""
    return np.concatenate([np.asarray(g[k], np.float64).reshape(-1) for k in GRAD_ORDER])


def reduce_gradients(flat: torch.Tensor, world: int | None = None) -> torch.Tensor:
    """The step's one collective: in-place sum over ranks of the packed buffer."""
    world = dist.get_world_size() if world is None and dist.is_initialized() else (world or 1)
    if world > 1:
        dist.all_reduce(flat, op=dist.ReduceOp.SUM)
    return flat


def lane_views(num_views: int, lanes: int) -> list[list[int]]:
    """Contiguous blocks of this rank's view indices, one per context lane."""
    if lanes < 1:
        raise ValueError("lane_views: lanes must be >= 1")
    return [list(range(num_views * k // lanes, num_views * (k + 1) // lanes)) for k in range(lanes)]


class ViewShardedStep:
    """One training step of `views` on this rank: fused fwd+bwd per view with
    gradient accumulation, chain once, all-reduce, Adam.  All tensors live on
    the rank's GPU; the call is asynchronous and CUDA-graph capturable once the
    replay buffers are sized (first call).

    lanes > 1 splits the rank's views over that many context lanes, each with
    its own stream, replay, frame and packed gradient buffer (lane 0 uses
    `packed_grads`): the lanes' renders overlap on the GPU (one lane's
    latency-bound preprocess / binning / kernel tails run beside another's
    blend kernels), and their buffers are summed (msplat_accumulate) before
    chain / all-reduce / Adam.  Same gradients up to float summation order."""

    def __init__(self, scene, packed_params, packed_grads, grads, opt, train_cfg, render_cfg, normal_cfg,
                 cameras, pixel_grads, frame, replay, world: int = 1, lanes: int = 1):
        from . import rasterizer as R
        self.scene, self.flat, self.gflat, self.grads = scene, packed_params, packed_grads, grads
        self.opt, self.tc, self.rc, self.nc = opt, train_cfg, render_cfg, normal_cfg
        self.cameras, self.pixel_grads, self.frame, self.replay = cameras, pixel_grads, frame, replay
        self.world = world
        self.lanes = max(1, min(int(lanes), len(cameras)))
        self.blocks = lane_views(len(cameras), self.lanes)
        self.lane_state = [(frame, replay, grads, packed_grads)]
        dev = packed_grads.device
        for k in range(1, self.lanes):
            g = torch.zeros_like(packed_grads)
            self.lane_state.append((R.MultimodalFrame.empty(frame.width, frame.height, frame.num_classes,
                                                            frame.color.dtype, dev),
                                    R.ReplayState(device=dev.index, lane=k),
                                    R.GradientBuffer.from_packed(g, scene.size(), scene.num_classes,
                                                                 scene.sh_degree), g))
        self.streams = [None] + [torch.cuda.Stream(dev) for _ in range(1, self.lanes)] if dev.type == "cuda" else []

    def issue_order(self) -> list[int]:
        """Views in the order __call__ issues them (lanes interleaved)."""
        return [b[i] for i in range(max(len(b) for b in self.blocks)) for b in self.blocks if i < len(b)]

    def __call__(self, pixel_grads=None, before_view=None):
        """before_view(j), when given, runs on view j's stream right before its
        render is issued (e.g. to wait for that view's upload)."""
        from . import rasterizer as R
        pix = self.pixel_grads if pixel_grads is None else pixel_grads
        if self.lanes == 1:
            for j, cam in enumerate(self.cameras):
                if before_view is not None:
                    before_view(j)
                R.fwd_bwd(self.scene, cam, self.rc, self.nc, self.frame, pix[j], self.grads, self.replay,
                          chain=False, accumulate=j > 0)
        else:
            main = torch.cuda.current_stream(self.gflat.device)
            for st in self.streams[1:]:
                st.wait_stream(main)
            for i in range(max(len(b) for b in self.blocks)):  # interleaved issue: lanes advance together
                for k, views in enumerate(self.blocks):
                    if i >= len(views):
                        continue
                    frame, replay, grads, _ = self.lane_state[k]
                    with torch.cuda.stream(main if k == 0 else self.streams[k]):
                        if before_view is not None:
                            before_view(views[i])
                        R.fwd_bwd(self.scene, self.cameras[views[i]], self.rc, self.nc, frame, pix[views[i]], grads,
                                  replay, chain=False, accumulate=i > 0)
            for st in self.streams[1:]:
                main.wait_stream(st)
            for k in range(1, self.lanes):
                R.accumulate_packed(self.gflat, self.lane_state[k][3])
        self.grads.raw_space = False
        R.chain_activations(self.grads, self.scene)
        reduce_gradients(self.gflat, self.world)
        R.adam_step(self.scene, self.grads, self.opt, self.tc, packed_params=self.flat, packed_grads=self.gflat)
