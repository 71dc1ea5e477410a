"""View-sharded training step across GPUs (BASELINE config 4).

The path shards by view: every rank holds a replica of the scene, renders its
own views through msplat_fwd_bwd, sums their gradients locally (train()
accumulates every view of a step into one Gradients, core/src/trainer.cpp:
295-309), and the ranks then exchange the packed n*P gradient buffer
(msplat_param_layout order).  chain_activations is linear per Gaussian, so it
is applied once to the local sum before the exchange.  Two exchanges:

  "allreduce"  one all-reduce (sum) of the packed buffer, then a replicated
               Adam step on every rank (adam_step, trainer.cpp:98-133);
  "sharded"    reduce-scatter of the packed buffer, Adam on this rank's
               contiguous shard only (msplat_adam_step_range), all-gather of
               the updated parameters.  Adam is elementwise, so the shards
               together are one full step bit for bit; each rank's optimizer
               work and moment traffic drop to 1/N and the two collectives
               together move the same bytes as the all-reduce.

Both leave identical parameters on every rank.  Only the exchange touches
torch.distributed (NCCL on GPUs, gloo in the CPU tests); the kernels never
wait on another rank.  The step's device work goes through an `ops` object
(default: the CUDA library); the CPU tests substitute one backed by the
reference restatement to drive this exact step order over gloo.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

EXCHANGES = ("allreduce", "sharded")
SHARD_ALIGN = 4  # elements: every shard starts on a 16-byte boundary (FP32 vector path)


def shard_views(total_views: int, rank: int, world: int) -> list[int]:
    """Contiguous block of view indices owned by `rank` (sizes differ by <= 1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("shard_views: bad rank/world")
    lo = total_views * rank // world
    hi = total_views * (rank + 1) // world
    return list(range(lo, hi))


def padded_size(total: int, world: int, align: int = SHARD_ALIGN) -> int:
    """Length of a packed buffer padded so that `world` equal shards of a
    multiple of `align` elements cover it (reduce-scatter / all-gather need
    equal shards)."""
    if world < 1 or total < 0:
        raise ValueError("padded_size: bad total/world")
    per = -(-total // world)
    per = -(-per // align) * align
    return per * world


def shard_range(total: int, rank: int, world: int, align: int = SHARD_ALIGN) -> tuple[int, int]:
    """(begin, count) of the real (unpadded) elements of `rank`'s shard."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("shard_range: bad rank/world")
    per = padded_size(total, world, align) // world
    begin = min(total, rank * per)
    return begin, min(total, begin + per) - begin


GRAD_ORDER = ("dposition", "drotation", "dscale", "dopacity", "dk", "dsh", "dsemantics")


def pack_grad_dict(g: dict) -> np.ndarray:
    """Pack a per-attribute gradient dict (reference layouts) into the
    msplat_param_layout order: means, quats, log_scales, opacity, k, sh, semantics."""
    return np.concatenate([np.asarray(g[k], np.float64).reshape(-1) for k in GRAD_ORDER])


def reduce_gradients(flat: torch.Tensor, world: int | None = None) -> torch.Tensor:
    """The all-reduce exchange: in-place sum over ranks of the packed buffer."""
    world = dist.get_world_size() if world is None and dist.is_initialized() else (world or 1)
    if world > 1:
        dist.all_reduce(flat, op=dist.ReduceOp.SUM)
    return flat


def lane_views(num_views: int, lanes: int) -> list[list[int]]:
    """Contiguous blocks of this rank's view indices, one per context lane."""
    if lanes < 1:
        raise ValueError("lane_views: lanes must be >= 1")
    return [list(range(num_views * k // lanes, num_views * (k + 1) // lanes)) for k in range(lanes)]


class DeviceOps:
    """The step's device work through the CUDA library (msplat_fwd_bwd,
    msplat_accumulate, msplat_chain_activations, msplat_adam_step[_range])."""

    def packed_total(self, scene) -> int:
        from . import rasterizer as R
        return R.param_layout(scene.size(), scene.num_classes, scene.sh_degree)[-1]

    def fwd_bwd(self, scene, cam, rc, nc, frame, pix, grads, replay, accumulate):
        from . import rasterizer as R
        R.fwd_bwd(scene, cam, rc, nc, frame, pix, grads, replay, chain=False, accumulate=accumulate)

    def accumulate(self, dst, src):
        from . import rasterizer as R
        R.accumulate_packed(dst, src)

    def chain(self, grads, scene):
        from . import rasterizer as R
        grads.raw_space = False
        R.chain_activations(grads, scene)

    def adam(self, scene, grads, opt, tc, flat, gflat, begin, count):
        """Adam on packed elements [begin, begin+count) of the full packed
        buffers flat/gflat; opt.step is already advanced."""
        from . import rasterizer as R
        R.adam_step_range(scene, grads, opt, tc, flat, gflat, begin, count)


class ViewShardedStep:
    """One training step of `views` on this rank: fused fwd+bwd per view with
    gradient accumulation, chain once, the exchange, Adam.  All tensors live on
    the rank's GPU; the call is asynchronous and CUDA-graph capturable once the
    replay buffers are sized (first call).

    lanes > 1 splits the rank's views over that many context lanes, each with
    its own stream, replay, frame and packed gradient buffer (lane 0 uses
    `packed_grads`): the lanes' renders overlap on the GPU (one lane's
    latency-bound preprocess / binning / kernel tails run beside another's
    blend kernels), and their buffers are summed (msplat_accumulate) before
    chain / exchange / Adam.  Same gradients up to float summation order.

    exchange="sharded" needs packed_params / packed_grads of at least
    padded_size(n*P, world) elements (the tail is padding)."""

    def __init__(self, scene, packed_params, packed_grads, grads, opt, train_cfg, render_cfg, normal_cfg,
                 cameras, pixel_grads, frame, replay, world: int = 1, lanes: int = 1,
                 exchange: str = "allreduce", rank: int | None = None, ops=None, optimizer: bool = True):
        if exchange not in EXCHANGES:
            raise ValueError(f"ViewShardedStep: exchange must be one of {EXCHANGES}")
        self.scene, self.flat, self.gflat, self.grads = scene, packed_params, packed_grads, grads
        self.opt, self.tc, self.rc, self.nc = opt, train_cfg, render_cfg, normal_cfg
        self.cameras, self.pixel_grads, self.frame, self.replay = cameras, pixel_grads, frame, replay
        self.world, self.exchange_kind, self.optimizer = world, exchange, optimizer
        self.rank = (dist.get_rank() if dist.is_initialized() else 0) if rank is None else rank
        self.ops = DeviceOps() if ops is None else ops
        self.total = int(self.ops.packed_total(scene))
        if exchange == "sharded":
            need = padded_size(self.total, world)
            if packed_grads.numel() < need or packed_params.numel() < need:
                raise ValueError(f"ViewShardedStep: sharded exchange needs packed buffers of "
                                 f"padded_size = {need} elements")
            self.padded = need
            self.per = need // world
            self.shard = torch.empty(self.per, dtype=packed_grads.dtype, device=packed_grads.device)
        self.lanes = max(1, min(int(lanes), len(cameras)))
        self.blocks = lane_views(len(cameras), self.lanes)
        self.lane_state = [(frame, replay, grads, packed_grads)]
        dev = packed_grads.device
        if self.lanes > 1:
            from . import rasterizer as R
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

    def render(self, pixel_grads=None, before_view=None):
        """fwd+bwd of every view of this rank, gradients summed into packed_grads
        (lane buffers added in).  before_view(j), when given, runs on view j's
        stream right before its render is issued (e.g. to wait for its upload)."""
        pix = self.pixel_grads if pixel_grads is None else pixel_grads
        if self.lanes == 1:
            for j, cam in enumerate(self.cameras):
                if before_view is not None:
                    before_view(j)
                self.ops.fwd_bwd(self.scene, cam, self.rc, self.nc, self.frame, pix[j], self.grads, self.replay,
                                 accumulate=j > 0)
            return
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
                    self.ops.fwd_bwd(self.scene, self.cameras[views[i]], self.rc, self.nc, frame, pix[views[i]],
                                     grads, replay, accumulate=i > 0)
        for st in self.streams[1:]:
            main.wait_stream(st)
        for k in range(1, self.lanes):
            self.ops.accumulate(self.gflat, self.lane_state[k][3])

    def exchange(self):
        """chain once -> exchange -> Adam (trainer.cpp:308-310 summed over views)."""
        self.ops.chain(self.grads, self.scene)
        if self.exchange_kind == "allreduce" or self.world == 1:
            reduce_gradients(self.gflat, self.world)
            if self.optimizer:
                self.opt.step += 1
                self.ops.adam(self.scene, self.grads, self.opt, self.tc, self.flat, self.gflat, 0, self.total)
            return
        # sharded: reduce-scatter -> Adam on the shard -> all-gather
        g = self.gflat[:self.padded]
        if self.padded > self.total:
            g[self.total:].zero_()
        dist.reduce_scatter_tensor(self.shard, g, op=dist.ReduceOp.SUM)
        lo = self.rank * self.per
        begin, count = shard_range(self.total, self.rank, self.world)
        self.gflat[lo:lo + self.per].copy_(self.shard)  # the reduced shard, in place in the packed buffer
        if self.optimizer:
            self.opt.step += 1
            if count > 0:
                self.ops.adam(self.scene, self.grads, self.opt, self.tc, self.flat, self.gflat, begin, count)
            p = self.flat[:self.padded]
            dist.all_gather_into_tensor(p, p[lo:lo + self.per].clone() if p.device.type == "cpu"
                                        else p[lo:lo + self.per])

    def __call__(self, pixel_grads=None, before_view=None):
        self.render(pixel_grads, before_view)
        self.exchange()


class ViewShardedRender:
    """Forward render throughput (BASELINE configs 1 and 5): each rank renders
    its own views -- rasterize (rasterizer.cpp:87-205) + estimate_normals
    (normals.cpp:28-101) per view -- into per-lane frames.  Replicas only: the
    views are independent, so there is no collective.  lanes > 1 issues the
    views interleaved over that many context lanes on their own streams.
    Asynchronous and CUDA-graph capturable once the replays are sized.
    frame_per_view=True renders every view into its own frame (frames[j])
    instead of one frame per lane, so a view's frame can still be read out
    while the lane renders its next view."""

    def __init__(self, scene, cameras, render_cfg, normal_cfg, lanes: int = 1, dtype=None,
                 frame_per_view: bool = False):
        from . import rasterizer as R
        self.scene, self.cameras, self.rc, self.nc = scene, cameras, render_cfg, normal_cfg
        self.lanes = max(1, min(int(lanes), len(cameras)))
        self.blocks = lane_views(len(cameras), self.lanes)
        self.frame_per_view = bool(frame_per_view)
        dev = scene.means.device
        W, H = cameras[0].width, cameras[0].height
        self.frames = [R.MultimodalFrame.empty(W, H, scene.num_classes, dtype or scene.dtype, dev)
                       for _ in range(len(cameras) if self.frame_per_view else self.lanes)]
        self.replays = [R.ReplayState(device=dev.index, lane=k) for k in range(self.lanes)]
        self.streams = [None] + [torch.cuda.Stream(dev) for _ in range(1, self.lanes)]
        self.device = dev

    def render_view(self, k, j, after=None):
        from . import rasterizer as R
        f = self.frames[j if self.frame_per_view else k]
        R.rasterize(self.scene, self.cameras[j], self.rc, self.replays[k], out=f)
        R.estimate_normals(f.depth, f.transmittance, self.cameras[j], self.nc, f.normals, lane=k)
        if after is not None:
            after(k, j, f)

    def __call__(self, after_view=None):
        """after_view(lane, view, frame), when given, runs on the lane's stream
        right after the view is rendered (e.g. to copy the frame out)."""
        main = torch.cuda.current_stream(self.device)
        for st in self.streams[1:]:
            st.wait_stream(main)
        for i in range(max(len(b) for b in self.blocks)):
            for k, views in enumerate(self.blocks):
                if i < len(views):
                    with torch.cuda.stream(main if k == 0 else self.streams[k]):
                        self.render_view(k, views[i], after_view)
        for st in self.streams[1:]:
            main.wait_stream(st)
