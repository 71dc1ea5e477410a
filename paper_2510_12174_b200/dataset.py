"""Dataset ingestion: cameras.json + PNG/PFM ground truth -> device tensors.

Mirrors msplat::load_dataset (core/src/dataset.cpp:53-145): the manifest, the
per-frame poses (q_cam_to_world w,x,y,z + t_cam_to_world), RGB PNG / depth PFM
/ normal PFM / label PNG maps with the reference's validation and error texts,
and the optional initial point cloud.  Parsing and decoding run in the C++
drop-in (libmsplat_dropin.so: src/dataset_io.cpp, src/io_image.cpp); the maps
come back planar and go to the device as GroundTruth for frame_losses /
frame_metrics.
"""
from __future__ import annotations

import ctypes as ct
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from .rasterizer import CameraView, GroundTruth, make_camera

_HERE = os.path.dirname(os.path.abspath(__file__))
_DROPIN = None


def _dropin():
    global _DROPIN
    if _DROPIN is None:
        path = os.path.join(_HERE, "libmsplat_dropin.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} is missing: build it with __graft_entry__.build()")
        lib = ct.CDLL(path)
        lib.msplat_dataset_last_error.restype = ct.c_char_p
        lib.msplat_dataset_load.argtypes = [ct.c_char_p, ct.POINTER(ct.c_void_p)]
        lib.msplat_dataset_load.restype = ct.c_int
        lib.msplat_dataset_free.argtypes = [ct.c_void_p]
        lib.msplat_dataset_dims.argtypes = [ct.c_void_p, ct.POINTER(ct.c_int64)]
        lib.msplat_dataset_frame.argtypes = [ct.c_void_p, ct.c_int64, ct.POINTER(ct.c_double), ct.POINTER(ct.c_int),
                                             ct.c_void_p, ct.c_void_p, ct.c_void_p, ct.c_void_p]
        lib.msplat_dataset_frame.restype = ct.c_int
        lib.msplat_dataset_points.argtypes = [ct.c_void_p, ct.c_void_p, ct.c_void_p]
        _DROPIN = lib
    return _DROPIN


@dataclass
class DatasetFrame:
    """msplat::FrameRecord (dataset.hpp:13-22) with its maps on the device."""
    view: CameraView
    split: str
    truth: GroundTruth


@dataclass
class SceneDataset:
    """msplat::SceneDataset (dataset.hpp:24-35)."""
    width: int
    height: int
    num_classes: int
    frames: list = field(default_factory=list)
    points: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    point_colors: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))

    def train_indices(self):
        return [i for i, f in enumerate(self.frames) if f.split != "test"]

    def test_indices(self):
        return [i for i, f in enumerate(self.frames) if f.split == "test"]


def load_dataset(root, dtype=torch.float32, device=None) -> SceneDataset:
    """load_dataset (dataset.cpp:53-145); maps land on `device` (default: the
    current CUDA device) as planar tensors of `dtype` (labels uint8)."""
    lib = _dropin()
    h = ct.c_void_p()
    if lib.msplat_dataset_load(os.fspath(root).encode(), ct.byref(h)) != 0:
        raise RuntimeError(lib.msplat_dataset_last_error().decode())
    try:
        dims = (ct.c_int64 * 5)()
        lib.msplat_dataset_dims(h, dims)
        W, H, C, nf, npts = (int(v) for v in dims)
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        ds = SceneDataset(W, H, C)
        pin = dev.type == "cuda"
        cam = (ct.c_double * 16)()
        flags = ct.c_int()
        for i in range(nf):
            rgb = torch.empty((3, H, W), dtype=torch.float32, pin_memory=pin)
            depth = torch.empty((H, W), dtype=torch.float32, pin_memory=pin)
            normal = torch.empty((3, H, W), dtype=torch.float32, pin_memory=pin)
            labels = torch.empty((H, W), dtype=torch.uint8, pin_memory=pin)
            if lib.msplat_dataset_frame(h, i, cam, ct.byref(flags), rgb.data_ptr(), depth.data_ptr(), normal.data_ptr(),
                                        labels.data_ptr()) != 0:
                raise RuntimeError(lib.msplat_dataset_last_error().decode())
            f = flags.value
            up = lambda t, on: t.to(dev, dtype if t.dtype != torch.uint8 else torch.uint8, non_blocking=True) if on else None  # noqa: E731,E501
            truth = GroundTruth(up(rgb, f & 1), up(depth, f & 2), up(normal, f & 4), up(labels, f & 8))
            c = list(cam)
            view = make_camera(c[0], c[1], c[2], c[3], W, H, np.array(c[4:13]).reshape(3, 3), np.array(c[13:16]))
            ds.frames.append(DatasetFrame(view, "test" if f & 16 else "train", truth))
        if npts:
            pts, cols = np.zeros((npts, 3)), np.zeros((npts, 3))
            lib.msplat_dataset_points(h, pts.ctypes.data, cols.ctypes.data)
            ds.points, ds.point_colors = pts, cols
        if dev.type == "cuda":
            torch.cuda.current_stream(dev).synchronize()  # pinned staging buffers die with this call
        return ds
    finally:
        lib.msplat_dataset_free(h)
