"""Test-only `ops` for distributed.ViewShardedStep backed by the CPU oracle
(the reference restatement), so that the step's exact order -- per-view
gradient accumulation, lane sums, chain once, all-reduce or reduce-scatter ->
Adam on the shard -> all-gather -- runs over gloo on CPU tensors.  The product
path uses distributed.DeviceOps (the CUDA library); nothing here ships."""
from __future__ import annotations

import numpy as np
import torch

SEG_KEYS = (("means", "dposition"), ("quats", "drotation"), ("log_scales", "dscale"),
            ("opacity_logits", "dopacity"), ("k", "dk"), ("sh", "dsh"), ("semantics", "dsemantics"))


def shapes(s):
    n, C, K = s["means"].shape[0], int(s["num_classes"]), (int(s["sh_degree"]) + 1) ** 2
    return [(n, 3), (n, 4), (n, 3), (n,), (n,), (n, 3, K), (n, C)]


def unpack(flat: np.ndarray, s) -> list[np.ndarray]:
    out, o = [], 0
    for shp in shapes(s):
        m = int(np.prod(shp))
        out.append(flat[o:o + m].reshape(shp))
        o += m
    return out


def pack_scene(s) -> np.ndarray:
    return np.concatenate([np.asarray(s[k], np.float64).reshape(-1) for k, _ in SEG_KEYS])


class GradView:
    """Stands in for GradientBuffer: the packed float64 CPU buffer."""

    def __init__(self, flat: torch.Tensor):
        self.flat = flat
        self.raw_space = False


class OracleOps:
    def __init__(self, port):
        self.port = port

    def packed_total(self, s) -> int:
        s = s[0] if isinstance(s, tuple) else s
        return int(sum(int(np.prod(x)) for x in shapes(s)))

    def _scene(self, s, flat):
        """The scene dict with parameters taken from the packed buffer (Adam
        updates the packed buffer, as on the GPU)."""
        d = dict(s)
        for (k, _), a in zip(SEG_KEYS, unpack(flat.numpy()[:self.packed_total(s)], s)):
            d[k] = a
        return d

    def fwd_bwd(self, scene, cam, rc, nc, frame, pix, grads, replay, accumulate):
        s, pflat = scene
        g = self.port.backward(self._scene(s, pflat), cam, pix, rc)
        p = np.concatenate([np.asarray(g[gk], np.float64).reshape(-1) for _, gk in SEG_KEYS])
        n = p.size
        if accumulate:
            grads.flat[:n] += torch.from_numpy(p)
        else:
            grads.flat[:n] = torch.from_numpy(p)

    def accumulate(self, dst, src):
        dst += src

    def chain(self, grads, scene):
        s, pflat = scene
        n = self.packed_total(s)
        parts = unpack(grads.flat.numpy()[:n].copy(), s)
        g = self.port.chain(self._scene(s, pflat), {gk: a for (_, gk), a in zip(SEG_KEYS, parts)})
        grads.flat[:n] = torch.from_numpy(np.concatenate([g[gk].reshape(-1) for _, gk in SEG_KEYS]))
        grads.raw_space = True

    def adam(self, scene, grads, opt, tc, flat, gflat, begin, count):
        """Reference adam_step on the whole packed state, written back on
        [begin, begin+count) only: a shard of the step."""
        s, _ = scene
        n = self.packed_total(s)
        ss = self._scene(s, flat)
        keyed = lambda buf: {gk: a for (_, gk), a in zip(SEG_KEYS, unpack(buf.numpy()[:n].copy(), s))}  # noqa
        lr = (tc.lr_position, tc.lr_rotation, tc.lr_scale, tc.lr_opacity, tc.lr_sh, tc.lr_semantics, tc.lr_k)
        p, m, v = self.port.adam(ss, keyed(gflat), keyed(opt.m), keyed(opt.v), opt.step, lr)  # reference lr order
        newp = np.concatenate([p[k].reshape(-1) for k, _ in SEG_KEYS])
        newm = np.concatenate([m[gk].reshape(-1) for _, gk in SEG_KEYS])
        newv = np.concatenate([v[gk].reshape(-1) for _, gk in SEG_KEYS])
        sl = slice(begin, begin + count)
        flat[sl] = torch.from_numpy(newp[sl])
        opt.m[sl] = torch.from_numpy(newm[sl])
        opt.v[sl] = torch.from_numpy(newv[sl])
