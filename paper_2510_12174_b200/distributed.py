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


class ViewShardedStep:
    """One training step of `views` on this rank: fused fwd+bwd per view with
    gradient accumulation, chain once, all-reduce, Adam.  All tensors live on
    the rank's GPU; the call is asynchronous and CUDA-graph capturable once the
    replay buffers are sized (first call)."""

    def __init__(self, scene, packed_params, packed_grads, grads, opt, train_cfg, render_cfg, normal_cfg,
                 cameras, pixel_grads, frame, replay, world: int = 1):
        self.scene, self.flat, self.gflat, self.grads = scene, packed_params, packed_grads, grads
        self.opt, self.tc, self.rc, self.nc = opt, train_cfg, render_cfg, normal_cfg
        self.cameras, self.pixel_grads, self.frame, self.replay = cameras, pixel_grads, frame, replay
        self.world = world

    def __call__(self, pixel_grads=None):
        from . import rasterizer as R
        pix = self.pixel_grads if pixel_grads is None else pixel_grads
        for j, cam in enumerate(self.cameras):
            R.fwd_bwd(self.scene, cam, self.rc, self.nc, self.frame, pix[j], self.grads, self.replay,
                      chain=False, accumulate=j > 0)
        self.grads.raw_space = False
        R.chain_activations(self.grads, self.scene)
        reduce_gradients(self.gflat, self.world)
        R.adam_step(self.scene, self.grads, self.opt, self.tc, packed_params=self.flat, packed_grads=self.gflat)
