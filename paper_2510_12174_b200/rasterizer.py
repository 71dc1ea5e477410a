"""Python mirror of the reference render API (proj/core, namespace msplat).

Same function names, argument meaning and error behaviour as the reference
C++ API, over torch device tensors:

    rasterize(scene, view, cfg, replay=None) -> MultimodalFrame     rasterizer.hpp:67-68
    estimate_normals(depth, T, view, ncfg, normals) -> None          normals.hpp:37-38
    normals_backward(dL_dN, depth, T, view, ncfg) -> dD              normals.hpp:42-43
    rasterize_backward(scene, view, frame, replay, pix) -> GradientBuffer   rasterizer.hpp:81-83
    chain_activations(buf, scene) -> None                            scene.hpp:74
    adam_step(scene, grads, state, cfg) -> None                      trainer.hpp:85-86
    prune(scene, state, cfg) -> removed                              trainer.hpp:90
    bin_and_sort(splats, width, height) -> TileBins                  rasterizer.hpp:52

Differences forced by the device: pixel grids are planar ([C, H, W]) torch
tensors instead of HWC Grids; scene/gradient buffers are SoA tensors.  The
element type of the scene (float32 or float64) selects the kernel precision.
Exceptions: ValueError for std::invalid_argument, RuntimeError for
std::runtime_error, LogicError for std::logic_error, with the reference's
message text.
"""
from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import LogicError, check

__all__ = [
    "Scene", "CameraView", "make_camera", "make_lookat_camera", "RenderConfig", "NormalConfig",
    "MultimodalFrame", "ReplayState", "PixelGradients", "GradientBuffer", "TileBins",
    "OptimizerState", "TrainConfig", "rasterize", "rasterize_backward", "estimate_normals",
    "normals_backward", "chain_activations", "adam_step", "prune", "bin_and_sort", "fwd_bwd",
    "LogicError", "param_layout", "GroundTruth", "LossReport", "frame_losses", "frame_metrics",
    "load_scene_ply", "save_scene_ply",
]


# ----------------------------------------------------------------- scene
@dataclass
class Scene:
    """SoA device copy of msplat::Scene (scene.hpp:14-34)."""
    means: torch.Tensor          # [n, 3]
    quats: torch.Tensor          # [n, 4] (w, x, y, z), raw
    log_scales: torch.Tensor     # [n, 3]
    opacity_logits: torch.Tensor  # [n]
    sh: torch.Tensor             # [n, 3, K]
    semantics: torch.Tensor      # [n, C]
    k: torch.Tensor              # [n] gradient factor
    num_classes: int = 0
    sh_degree: int = 2

    def size(self) -> int:
        return int(self.means.shape[0])

    def sh_coeff_count(self) -> int:
        return (self.sh_degree + 1) ** 2

    @property
    def dtype(self):
        return self.means.dtype

    def tensors(self):
        return [self.means, self.quats, self.log_scales, self.opacity_logits, self.sh,
                self.semantics, self.k]

    def validate(self):
        """Shape checks of Scene::validate (scene.cpp:22-40); finiteness is
        checked on the device by the preprocess kernel."""
        if self.sh_degree < 0 or self.sh_degree > 3:
            raise ValueError("Scene: sh_degree must be in [0,3]")
        if self.num_classes < 0:
            raise ValueError("Scene: num_classes must be >= 0")
        n, K, C = self.size(), self.sh_coeff_count(), self.num_classes
        expect = {"means": (n, 3), "quats": (n, 4), "log_scales": (n, 3), "opacity_logits": (n,),
                  "sh": (n, 3, K), "semantics": (n, C), "k": (n,)}
        for name, shp in expect.items():
            t = getattr(self, name)
            if tuple(t.shape) != shp:
                what = "SH coefficient count" if name == "sh" else (
                    "semantic channel count" if name == "semantics" else name + " shape")
                raise ValueError(f"Scene: wrong {what}: {tuple(t.shape)} != {shp}")
        for name in expect:
            t = getattr(self, name)
            if t.dtype != self.dtype or not t.is_cuda or not t.is_contiguous():
                raise ValueError(f"Scene: {name} must be a contiguous CUDA tensor of one dtype")
        if self.dtype not in (torch.float32, torch.float64):
            raise ValueError("Scene: dtype must be float32 or float64")

    def _abi(self) -> _lib.MsplatScene:
        self.validate()
        return _lib.MsplatScene(
            self.size(), self.num_classes, self.sh_degree, _dtype_code(self.dtype),
            self.means.data_ptr(), self.quats.data_ptr(), self.log_scales.data_ptr(),
            self.opacity_logits.data_ptr(), self.k.data_ptr(), self.sh.data_ptr(),
            self.semantics.data_ptr() if self.num_classes else None)

    @staticmethod
    def from_numpy(arrs: dict, device="cuda", dtype=torch.float32) -> "Scene":
        def t(a):
            return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device=device).contiguous()
        n = len(arrs["means"])
        C = int(arrs["num_classes"])
        sem = arrs["semantics"] if C else np.zeros((n, 0))
        return Scene(t(arrs["means"]), t(arrs["quats"]), t(arrs["log_scales"]),
                     t(arrs["opacity_logits"]), t(arrs["sh"]), t(sem), t(arrs["k"]), C,
                     int(arrs["sh_degree"]))


def _dtype_code(dt):
    if dt == torch.float64:
        return _lib.MSPLAT_F64
    if dt == torch.float32:
        return _lib.MSPLAT_F32
    raise ValueError("dtype must be float32 or float64")


# ----------------------------------------------------------------- camera
@dataclass
class CameraView:
    """msplat::CameraView (camera.hpp:8-32); R is cam->world."""
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    R_cam_to_world: np.ndarray = field(default_factory=lambda: np.eye(3))
    t_cam_to_world: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def finalize(self):
        """CameraView::finalize checks (camera.cpp:8-21)."""
        if self.width < 1 or self.height < 1:
            raise ValueError("CameraView: width and height must be >= 1")
        if not (self.fx > 0) or not (self.fy > 0):
            raise ValueError("CameraView: focal lengths must be positive")
        R = np.asarray(self.R_cam_to_world, np.float64)
        if np.abs(R.T @ R - np.eye(3)).max() > 1e-6:
            raise ValueError("CameraView: rotation is not orthonormal (tol 1e-6)")
        if abs(np.linalg.det(R) - 1.0) > 1e-6:
            raise ValueError("CameraView: rotation determinant is not +1 (tol 1e-6)")
        return self

    @property
    def R_world_to_cam(self):
        return np.asarray(self.R_cam_to_world, np.float64).T

    @property
    def t_world_to_cam(self):
        return -(self.R_world_to_cam @ np.asarray(self.t_cam_to_world, np.float64))

    def _abi(self) -> _lib.MsplatCamera:
        R = np.asarray(self.R_cam_to_world, np.float64).reshape(9)
        t = np.asarray(self.t_cam_to_world, np.float64).reshape(3)
        return _lib.MsplatCamera(float(self.fx), float(self.fy), float(self.cx), float(self.cy),
                                 int(self.width), int(self.height), (ct.c_double * 9)(*R),
                                 (ct.c_double * 3)(*t))

    def as_dict(self):
        return {"fx": self.fx, "fy": self.fy, "cx": self.cx, "cy": self.cy, "width": self.width,
                "height": self.height, "R_c2w": np.asarray(self.R_cam_to_world, np.float64),
                "t_c2w": np.asarray(self.t_cam_to_world, np.float64)}


def make_camera(fx, fy, cx, cy, width, height, R_cam_to_world, t_cam_to_world) -> CameraView:
    """make_camera (camera.cpp:23-36)."""
    return CameraView(fx, fy, cx, cy, width, height, np.asarray(R_cam_to_world, np.float64),
                      np.asarray(t_cam_to_world, np.float64)).finalize()


def make_lookat_camera(fx, fy, cx, cy, width, height, eye, target, up_hint=(0, -1, 0)):
    """make_lookat_camera (camera.cpp:38-59): +z forward, y down, x right."""
    eye, target, up = (np.asarray(v, np.float64) for v in (eye, target, up_hint))
    fwd = target - eye
    n = np.linalg.norm(fwd)
    if n < 1e-12:
        raise ValueError("make_lookat_camera: eye and target coincide")
    fwd = fwd / n
    right = np.cross(fwd, up)
    if np.linalg.norm(right) < 1e-9:
        right = np.cross(fwd, [1.0, 0, 0])
        if np.linalg.norm(right) < 1e-9:
            right = np.cross(fwd, [0, 0, 1.0])
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    return make_camera(fx, fy, cx, cy, width, height, np.stack([right, down, fwd], axis=1), eye)


# ---------------------------------------------------------------- configs
@dataclass
class RenderConfig:
    """msplat::RenderConfig (rasterizer.hpp:13-19)."""
    sigma_scale: float = 1.0
    background: tuple = (0.0, 0.0, 0.0)
    early_stop_transmittance: float = 1e-4
    early_termination: bool = True
    threads: int = 1  # accepted, ignored (the CUDA grid replaces host threads)

    def _abi(self):
        return _lib.MsplatRenderConfig(float(self.sigma_scale),
                                       (ct.c_double * 3)(*[float(b) for b in self.background]),
                                       float(self.early_stop_transmittance),
                                       int(bool(self.early_termination)), int(self.threads))


@dataclass
class NormalConfig:
    """msplat::NormalConfig (normals.hpp:10-15)."""
    step1: int = 1
    step2: int = 4
    fuse_lambda: float = 0.5
    mask_threshold: float = 0.5

    def _abi(self):
        return _lib.MsplatNormalConfig(int(self.step1), int(self.step2), float(self.fuse_lambda),
                                       float(self.mask_threshold))


# ----------------------------------------------------------------- frames
@dataclass
class MultimodalFrame:
    """msplat::MultimodalFrame (rasterizer.hpp:22-31), planar device tensors."""
    width: int
    height: int
    num_classes: int
    color: torch.Tensor          # [3, H, W], background composited
    depth: torch.Tensor          # [H, W]
    semantics: torch.Tensor      # [C, H, W]
    kmap: torch.Tensor           # [H, W]
    transmittance: torch.Tensor  # [H, W]
    normals: torch.Tensor        # [3, H, W]
    contributors: torch.Tensor   # [H, W] int32

    @staticmethod
    def empty(W, H, C, dtype, device):
        z = lambda *s: torch.zeros(*s, dtype=dtype, device=device)  # noqa: E731
        return MultimodalFrame(W, H, C, z(3, H, W), z(H, W), z(C, H, W), z(H, W), z(H, W),
                               z(3, H, W), torch.zeros(H, W, dtype=torch.int32, device=device))

    def _abi(self):
        return _lib.MsplatFrame(self.color.data_ptr(), self.depth.data_ptr(),
                                self.semantics.data_ptr() if self.num_classes else None,
                                self.kmap.data_ptr(), self.transmittance.data_ptr(),
                                self.normals.data_ptr(), self.contributors.data_ptr())


@dataclass
class PixelGradients:
    """msplat::PixelGradients (rasterizer.hpp:72-79) planar, + optional dnormals."""
    dcolor: torch.Tensor
    ddepth: torch.Tensor
    dsemantics: torch.Tensor
    dkmap: torch.Tensor
    dnormals: torch.Tensor | None = None

    @staticmethod
    def zero(width, height, num_classes, dtype=torch.float32, device="cuda"):
        z = lambda *s: torch.zeros(*s, dtype=dtype, device=device)  # noqa: E731
        return PixelGradients(z(3, height, width), z(height, width), z(num_classes, height, width),
                              z(height, width))

    def _abi(self):
        return _lib.MsplatPixelGrads(
            self.dcolor.data_ptr(), self.ddepth.data_ptr(),
            self.dsemantics.data_ptr() if self.dsemantics.numel() else None,
            self.dkmap.data_ptr(), self.dnormals.data_ptr() if self.dnormals is not None else None)


@dataclass
class GradientBuffer:
    """msplat::GradientBuffer (scene.hpp:54-68), SoA device tensors."""
    dposition: torch.Tensor
    drotation: torch.Tensor
    dscale: torch.Tensor
    dopacity: torch.Tensor
    dsh: torch.Tensor
    dsemantics: torch.Tensor
    dk: torch.Tensor
    raw_space: bool = False

    @staticmethod
    def zeros_like_scene(scene: Scene) -> "GradientBuffer":
        return GradientBuffer(*(torch.zeros_like(t) for t in (
            scene.means, scene.quats, scene.log_scales, scene.opacity_logits, scene.sh,
            scene.semantics, scene.k)))

    @staticmethod
    def from_packed(flat: torch.Tensor, n: int, C: int, deg: int) -> "GradientBuffer":
        """Views into one packed n*P buffer (msplat_param_layout order)."""
        off = param_layout(n, C, deg)
        K = (deg + 1) ** 2
        v = lambda i, *shape: flat[off[i]:off[i + 1]].view(*shape)  # noqa: E731
        return GradientBuffer(v(0, n, 3), v(1, n, 4), v(2, n, 3), v(3, n), v(5, n, 3, K),
                              v(6, n, C), v(4, n))

    def size(self):
        return int(self.dposition.shape[0])

    def _abi(self):
        return _lib.MsplatGrads(self.dposition.data_ptr(), self.drotation.data_ptr(),
                                self.dscale.data_ptr(), self.dopacity.data_ptr(),
                                self.dk.data_ptr(), self.dsh.data_ptr(),
                                self.dsemantics.data_ptr() if self.dsemantics.numel() else None)

    def check_finite(self, where="GradientBuffer"):
        for t in (self.dposition, self.drotation, self.dscale, self.dopacity, self.dsh,
                  self.dsemantics, self.dk):
            if t.numel() and not torch.isfinite(t).all():
                bad = (~torch.isfinite(t.reshape(t.shape[0], -1))).any(dim=1).nonzero()[0, 0]
                raise RuntimeError(f"{where}: non-finite gradient for primitive {int(bad)}")


def param_layout(n: int, C: int, deg: int):
    off = (ct.c_int64 * 8)()
    check(_lib.lib().msplat_param_layout(n, C, deg, off))
    return list(off)


# ---------------------------------------------------------------- context
_deferred_replays: list = []


def _capturing() -> bool:
    try:
        return bool(torch.cuda.is_current_stream_capturing())
    except Exception:
        return False


def _release_deferred() -> None:
    """Destroys replays whose finalizer ran during a CUDA-graph capture."""
    while _deferred_replays and not _capturing():
        _lib.lib().msplat_replay_destroy(_deferred_replays.pop())


class _Context:
    """One msplat_context per (device, lane); follows torch's current stream.
    Lanes are independent contexts (own scratch and error word) so that
    renders on different streams of one device can run concurrently."""
    _per_device: dict[tuple, "_Context"] = {}
    # Per-device settings every lane follows (also lanes created later):
    # {device: {"deterministic": bool, "timing": bool}}
    _settings: dict[int, dict] = {}

    def __init__(self, device: int):
        self.device = device
        h = ct.c_void_p()
        check(_lib.lib().msplat_context_create(device, ct.c_void_p(torch.cuda.current_stream(device).cuda_stream),
                                               ct.byref(h)))
        self.h = h
        st = self._settings.get(device, {})
        if st.get("deterministic"):
            check(_lib.lib().msplat_context_set_deterministic(h, 1))
        if st.get("timing"):
            check(_lib.lib().msplat_context_set_timing(h, 1))

    @classmethod
    def get(cls, device=None, lane: int = 0) -> "_Context":
        dev = torch.cuda.current_device() if device is None else int(device)
        c = cls._per_device.get((dev, lane))
        if c is None:
            c = cls._per_device[(dev, lane)] = _Context(dev)
        check(_lib.lib().msplat_context_set_stream(c.h, ct.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
        if _deferred_replays:
            _release_deferred()
        return c

    @classmethod
    def apply(cls, device, key: str, value: bool, fn) -> None:
        """Set a per-device flag on every existing lane and remember it for
        lanes created later."""
        dev = torch.cuda.current_device() if device is None else int(device)
        cls.get(dev)
        cls._settings.setdefault(dev, {})[key] = bool(value)
        for (d, _lane), c in sorted(cls._per_device.items()):
            if d == dev:
                check(fn(c.h, int(value)))


class ReplayState:
    """Device-resident msplat::ReplayState (rasterizer.hpp:55-65).

    capture: 1 keeps FP64 splats (for parity checks), 2 records weight_sums."""

    def __init__(self, capture: int = 0, device=None, lane: int = 0):
        self._ctx = _Context.get(device, lane)
        self.lane = lane
        h = ct.c_void_p()
        check(_lib.lib().msplat_replay_create(self._ctx.h, ct.byref(h)))
        self.h = h
        self.capture = capture
        check(_lib.lib().msplat_replay_set_capture(h, capture))
        self.num_gaussians = 0
        self.width = self.height = 0

    def __del__(self):
        # Freeing device memory (cudaFree) inside a CUDA-graph capture would
        # invalidate the capture, and the garbage collector may run here at
        # any point: during a capture the handle is parked and released by
        # the next non-capturing ReplayState / context call.
        try:
            if getattr(self, "h", None):
                if _capturing():
                    _deferred_replays.append(self.h)
                else:
                    _lib.lib().msplat_replay_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def counters(self) -> dict:
        c = _lib.MsplatCounters()
        check(_lib.lib().msplat_replay_counters(self.h, ct.byref(c)))
        return {k: int(getattr(c, k)) for k, _ in c._fields_}

    def bins(self):
        """(tile_offsets[tiles+1], values[I]) as numpy arrays."""
        c = self.counters()
        off = np.zeros(c["tiles"] + 1, np.int64)
        vals = np.zeros(max(c["instances"], 1), np.int32)
        check(_lib.lib().msplat_replay_bins(self.h, off.ctypes.data_as(ct.POINTER(ct.c_int64)),
                                            vals.ctypes.data_as(ct.POINTER(ct.c_int32)), len(vals)))
        return off, vals[:c["instances"]]

    def splats(self) -> dict:
        n = self.num_gaussians
        out = {"visible": np.zeros(n, np.uint8), "center": np.zeros((n, 2)), "conic": np.zeros((n, 3)),
               "depth": np.zeros(n), "radius": np.zeros(n), "rgb": np.zeros((n, 3)),
               "clamped": np.zeros((n, 3), np.uint8)}
        p = lambda a: a.ctypes.data  # noqa: E731
        check(_lib.lib().msplat_replay_splats(self.h, p(out["visible"]), p(out["center"]), p(out["conic"]),
                                              p(out["depth"]), p(out["radius"]), p(out["rgb"]),
                                              p(out["clamped"])))
        return out

    def terminus(self) -> np.ndarray:
        t = np.zeros((self.height, self.width), np.int32)
        check(_lib.lib().msplat_replay_terminus(self.h, t.ctypes.data_as(ct.POINTER(ct.c_int32))))
        return t

    def weight_sums(self) -> np.ndarray:
        w = np.zeros(self.num_gaussians)
        check(_lib.lib().msplat_replay_weight_sums(self.h, w.ctypes.data_as(ct.POINTER(ct.c_double))))
        return w


# ------------------------------------------------------------- hot path API
def rasterize(scene: Scene, view: CameraView, cfg: RenderConfig | None = None,
              replay: ReplayState | None = None, out: MultimodalFrame | None = None) -> MultimodalFrame:
    """rasterize (rasterizer.cpp:87-205).  frame.normals stays zero until
    estimate_normals, exactly like the reference (rasterizer.cpp:101).  `out`
    reuses a caller-owned frame of the view's size (every channel is
    overwritten; no allocation, so the call is CUDA-graph capturable once the
    replay is sized)."""
    cfg = cfg or RenderConfig()
    ctx = _Context.get(scene.means.device.index, replay.lane if replay is not None else 0)
    if out is None:
        frame = MultimodalFrame.empty(view.width, view.height, scene.num_classes, scene.dtype,
                                      scene.means.device)
        frame.transmittance.fill_(1.0)
    else:
        if (out.width, out.height, out.num_classes) != (view.width, view.height, scene.num_classes) or \
                out.color.dtype != scene.dtype:
            raise ValueError("rasterize: output frame does not match the view / scene")
        frame = out
    check(_lib.lib().msplat_rasterize(ctx.h, ct.byref(scene._abi()), ct.byref(view._abi()),
                                      ct.byref(cfg._abi()), ct.byref(frame._abi()),
                                      replay.h if replay is not None else None))
    if replay is not None:
        replay.num_gaussians, replay.width, replay.height = scene.size(), view.width, view.height
        replay.sh_degree, replay.num_classes, replay.cfg = scene.sh_degree, scene.num_classes, cfg
    return frame


def estimate_normals(depth: torch.Tensor, transmittance: torch.Tensor, view: CameraView,
                     ncfg: NormalConfig, normals: torch.Tensor, lane: int = 0) -> None:
    """estimate_normals (normals.cpp:28-101): writes unit normals [3, H, W]
    (on context lane `lane`, torch's current stream)."""
    if depth.shape != (view.height, view.width) or transmittance.shape != depth.shape:
        raise ValueError("backproject: depth map does not match the view")
    ctx = _Context.get(depth.device.index, lane)
    check(_lib.lib().msplat_estimate_normals(ctx.h, _dtype_code(depth.dtype), depth.data_ptr(),
                                             transmittance.data_ptr(), ct.byref(view._abi()),
                                             ct.byref(ncfg._abi()), normals.data_ptr()))


def normals_backward(dL_dnormals: torch.Tensor, depth: torch.Tensor, transmittance: torch.Tensor,
                     view: CameraView, ncfg: NormalConfig) -> torch.Tensor:
    """normals_backward (normals.cpp:103-152) -> dL/ddepth [H, W].  The
    NormalState is recomputed from depth/T instead of being stored."""
    if dL_dnormals.shape != (3, view.height, view.width):
        raise ValueError("normals_backward: gradient shape mismatch")
    ctx = _Context.get(depth.device.index)
    dD = torch.zeros_like(depth)
    check(_lib.lib().msplat_normals_backward(ctx.h, _dtype_code(depth.dtype), dL_dnormals.data_ptr(),
                                             depth.data_ptr(), transmittance.data_ptr(),
                                             ct.byref(view._abi()), ct.byref(ncfg._abi()), 1.0,
                                             dD.data_ptr()))
    return dD


# ----------------------------------------------------------------- losses
@dataclass
class GroundTruth:
    """The supervision of one frame (dataset.hpp FrameRecord), planar device
    tensors in the frame's dtype; None = modality absent."""
    rgb: torch.Tensor | None = None       # [3, H, W]
    depth: torch.Tensor | None = None     # [H, W], pixels with depth > 0 supervised
    normal: torch.Tensor | None = None    # [3, H, W], non-zero normals supervised
    labels: torch.Tensor | None = None    # [H, W] uint8 class ids

    def _abi(self):
        p = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
        if self.labels is not None and self.labels.dtype != torch.uint8:
            raise ValueError("GroundTruth: labels must be uint8")
        return _lib.MsplatGroundTruth(p(self.rgb), p(self.depth), p(self.normal), p(self.labels))


@dataclass
class LossReport:
    """msplat::LossReport (losses.hpp:40-50)."""
    l1: float = 0.0
    ssim: float = 0.0
    depth: float = 0.0
    normal: float = 0.0
    seg: float = 0.0
    k: float = 0.0
    combined: float = 0.0
    ratio_ssim: float = 0.0
    ratio_normal: float = 0.0
    ratio_depth: float = 0.0
    ratio_seg: float = 0.0
    ratio_k: float = 0.0
    seed_l1: float = 0.0
    seed_ssim: float = 0.0
    seed_depth: float = 0.0
    seed_normal: float = 0.0
    seed_seg: float = 0.0
    seed_k: float = 0.0


def frame_losses(frame: MultimodalFrame, gt: GroundTruth, view: CameraView, ncfg: NormalConfig,
                 lambdas=(1.0, 0.1, 0.1, 0.1, 0.1, 0.1), out: PixelGradients | None = None,
                 sync: bool = True):
    """evaluate_frame_losses (trainer.cpp:171-264) on the device.

    `frame.normals` must come from estimate_normals (a non-zero normal marks a
    valid pixel).  lambdas = (l1, ssim, normal, depth, seg, k).  Returns
    (LossReport, PixelGradients); the normal term is already pushed through
    normals_backward into ddepth.  sync=False keeps the report on the device
    (LossReport is then None) -- the call is graph-capturable."""
    dev = frame.color.device
    if out is None:
        out = PixelGradients.zero(frame.width, frame.height, frame.num_classes, frame.color.dtype, dev)
    ctx = _Context.get(dev.index)
    lam = (ct.c_double * 6)(*[float(x) for x in lambdas])
    rep = _lib.MsplatLossReport()
    check(_lib.lib().msplat_frame_losses(ctx.h, _dtype_code(frame.color.dtype), frame.num_classes,
                                         ct.byref(view._abi()), ct.byref(ncfg._abi()), ct.byref(frame._abi()),
                                         ct.byref(gt._abi()), lam, ct.byref(out._abi()),
                                         ct.byref(rep) if sync else None))
    report = LossReport(**{f: getattr(rep, f) for f in _lib.LOSS_REPORT_FIELDS}) if sync else None
    return report, out


def frame_metrics(frame: MultimodalFrame, gt: GroundTruth, depth_mask: torch.Tensor | None = None,
                  normal_mask: torch.Tensor | None = None, label_mask: torch.Tensor | None = None) -> dict:
    """Image metrics of metrics.cpp:68-187 on the device: psnr, ssim (against
    gt.rgb), abs_rel, rmse (depth, masked), cos_simi (normals, masked), miou
    (argmax of the semantic logits vs gt.labels, masked).  A metric without its
    inputs (ground truth or mask) is None, as is an empty mask."""
    ctx = _Context.get(frame.color.device.index)
    p = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
    for m in (depth_mask, normal_mask, label_mask):
        if m is not None and m.dtype != torch.uint8:
            raise ValueError("frame_metrics: masks must be uint8")
    rep = _lib.MsplatMetricReport()
    have_sem = frame.num_classes > 0 and gt.labels is not None and label_mask is not None
    check(_lib.lib().msplat_frame_metrics(
        ctx.h, _dtype_code(frame.color.dtype), frame.width, frame.height, frame.num_classes,
        p(frame.color) if gt.rgb is not None else None, p(gt.rgb),
        p(frame.depth) if gt.depth is not None else None, p(gt.depth), p(depth_mask),
        p(frame.normals) if gt.normal is not None else None, p(gt.normal), p(normal_mask),
        p(frame.semantics) if have_sem else None, p(gt.labels), p(label_mask), ct.byref(rep)))
    return {f: (getattr(rep, f) if getattr(rep, "has_" + f) else None) for f in _lib.METRIC_FIELDS}


# ------------------------------------------------------------ scene I/O
def load_scene_ply(path: str, dtype=torch.float32, device="cuda") -> Scene:
    """load_scene_ply (io_ply.hpp, io_ply.cpp:165-263): the payload is decoded
    on the device straight into one packed parameter buffer; the Scene fields
    are views of it."""
    n, C, deg = ct.c_int64(), ct.c_int(), ct.c_int()
    check(_lib.lib().msplat_ply_scene_info(str(path).encode(), ct.byref(n), ct.byref(C), ct.byref(deg)))
    n, C, deg = n.value, C.value, deg.value
    off = param_layout(n, C, deg)
    dev = torch.device(device)
    flat = torch.empty(max(off[7], 1), dtype=dtype, device=dev)
    ctx = _Context.get(dev.index)
    check(_lib.lib().msplat_load_scene_ply(ctx.h, str(path).encode(), _dtype_code(dtype), flat.data_ptr()))
    K = (deg + 1) ** 2
    seg = lambda i, *shape: flat[off[i]:off[i + 1]].view(*shape)  # noqa: E731
    return Scene(means=seg(0, n, 3), quats=seg(1, n, 4), log_scales=seg(2, n, 3), opacity_logits=seg(3, n),
                 k=seg(4, n), sh=seg(5, n, 3, K), semantics=seg(6, n, C), num_classes=C, sh_degree=deg)


def save_scene_ply(path: str, scene: Scene) -> None:
    """save_scene_ply (io_ply.cpp:122-163): float64 rows encoded on the device."""
    n = scene.size()
    flat = pack_scene(scene) if n else torch.zeros(1, dtype=scene.dtype, device=scene.means.device)
    ctx = _Context.get(scene.means.device.index)
    check(_lib.lib().msplat_save_scene_ply(ctx.h, str(path).encode(), _dtype_code(scene.dtype), n,
                                           scene.num_classes, scene.sh_degree, flat.data_ptr()))


def rasterize_backward(scene: Scene, view: CameraView, frame: MultimodalFrame, replay: ReplayState,
                       pix: PixelGradients, out: GradientBuffer | None = None) -> GradientBuffer:
    """rasterize_backward (rasterizer_backward.cpp:127-264); activated space.
    The library zeroes the gradient arrays before accumulating, so the result
    is a fresh buffer's; `out` (e.g. GradientBuffer.from_packed views of the
    optimizer's packed gradient buffer) is written in place instead of a new
    allocation."""
    ctx = _Context.get(scene.means.device.index, replay.lane)
    if out is None:
        grads = GradientBuffer(*(torch.empty_like(t) for t in (
            scene.means, scene.quats, scene.log_scales, scene.opacity_logits, scene.sh,
            scene.semantics, scene.k)))
    else:
        want = (scene.means, scene.quats, scene.log_scales, scene.opacity_logits, scene.sh, scene.semantics, scene.k)
        have = (out.dposition, out.drotation, out.dscale, out.dopacity, out.dsh, out.dsemantics, out.dk)
        if any(h.shape != w.shape or h.dtype != w.dtype or h.device != w.device for h, w in zip(have, want)):
            raise ValueError("rasterize_backward: out does not match the scene")
        grads = out
        grads.raw_space = False
    for t in (pix.dcolor, pix.ddepth, pix.dsemantics, pix.dkmap):
        if t.dtype != scene.dtype or not t.is_contiguous():
            raise RuntimeError("rasterize_backward: pixel-gradient shape mismatch")
    ok = (tuple(pix.dcolor.shape) == (3, frame.height, frame.width)
          and tuple(pix.ddepth.shape) == (frame.height, frame.width)
          and tuple(pix.dsemantics.shape) == (frame.num_classes, frame.height, frame.width)
          and tuple(pix.dkmap.shape) == (frame.height, frame.width))
    if not ok:
        raise RuntimeError("rasterize_backward: pixel-gradient shape mismatch")
    check(_lib.lib().msplat_rasterize_backward(ctx.h, ct.byref(scene._abi()), ct.byref(view._abi()),
                                               ct.byref(frame._abi()), replay.h, ct.byref(pix._abi()),
                                               ct.byref(grads._abi())))
    return grads


def chain_activations(buf: GradientBuffer, scene: Scene) -> None:
    """chain_activations (scene.cpp:108-129), in place."""
    if buf.size() != scene.size():
        raise ValueError("chain_activations: buffer/scene size mismatch")
    if buf.raw_space:
        raise LogicError("chain_activations: buffer already in raw-parameter space")
    ctx = _Context.get(scene.means.device.index)
    check(_lib.lib().msplat_chain_activations(ctx.h, ct.byref(scene._abi()), ct.byref(buf._abi())))
    buf.raw_space = True


def fwd_bwd(scene: Scene, view: CameraView, cfg: RenderConfig, ncfg: NormalConfig,
            frame: MultimodalFrame, pix: PixelGradients, grads: GradientBuffer, replay: ReplayState,
            chain: bool = True, accumulate: bool = False) -> None:
    """The fused training-step unit (msplat_fwd_bwd): rasterize, estimate_normals,
    normals_backward merged into ddepth, rasterize_backward, chain_activations.
    Asynchronous on torch's current stream once the replay is sized.  Runs on
    the replay's context lane (ReplayState(lane=k)): renders of different lanes
    may be issued on different streams concurrently."""
    ctx = _Context.get(scene.means.device.index, replay.lane)
    check(_lib.lib().msplat_fwd_bwd(ctx.h, ct.byref(scene._abi()), ct.byref(view._abi()),
                                    ct.byref(cfg._abi()), ct.byref(ncfg._abi()), ct.byref(frame._abi()),
                                    ct.byref(pix._abi()), ct.byref(grads._abi()), int(chain),
                                    int(accumulate), replay.h))
    replay.num_gaussians, replay.width, replay.height = scene.size(), view.width, view.height
    grads.raw_space = bool(chain) and not accumulate


def check_device_errors(device=None):
    """Surface a latched device-side error of any context lane of the device
    (synchronizing)."""
    dev = torch.cuda.current_device() if device is None else int(device)
    _Context.get(dev)
    for (d, _lane), c in sorted(_Context._per_device.items()):
        if d == dev:
            check(_lib.lib().msplat_context_check(c.h))


def set_stage_timing(enable: bool, device=None):
    """Bracket every stage with CUDA events on the launching stream (every
    context lane of the device)."""
    _Context.apply(device, "timing", enable, _lib.lib().msplat_context_set_timing)


def set_deterministic(enable: bool, device=None):
    """Bitwise-reproducible backward (TrainConfig::deterministic,
    msplat/trainer.hpp:48-63): per-(instance, warp) partial slots reduced in a
    fixed order instead of float atomics.  Applies to every context lane of
    the device, including lanes created later."""
    _Context.apply(device, "deterministic", enable, _lib.lib().msplat_context_set_deterministic)


def stage_timings(device=None) -> dict:
    """{stage: (device ms summed since the last call, launches of the stage)},
    summed over every context lane of the device; synchronizing."""
    dev = torch.cuda.current_device() if device is None else int(device)
    _Context.get(dev)
    tot = {name: [0.0, 0] for name in _lib.STAGES}
    for (d, _lane), c in sorted(_Context._per_device.items()):
        if d != dev:
            continue
        ms = (ct.c_double * 8)()
        calls = (ct.c_int64 * 8)()
        check(_lib.lib().msplat_context_timings(c.h, ms, calls))
        for i, name in enumerate(_lib.STAGES):
            tot[name][0] += ms[i]
            tot[name][1] += int(calls[i])
    return {name: (v[0], v[1]) for name, v in tot.items()}


def kernel_launches() -> int:
    """Process-wide count of kernels this library has launched."""
    return int(_lib.lib().msplat_kernel_launches())


# ------------------------------------------------------------ optimizer
@dataclass
class TrainConfig:
    """The optimizer/prune subset of msplat::TrainConfig (trainer.hpp:15-65)."""
    lr_position: float = 1.6e-4
    lr_rotation: float = 1e-3
    lr_scale: float = 5e-3
    lr_opacity: float = 5e-2
    lr_sh: float = 2.5e-3
    lr_semantics: float = 2.5e-2
    lr_k: float = 5e-2
    prune_threshold: float = 0.5
    prune_keep_small: bool = False
    k_reset: float = 0.9

    def lrs_packed(self):
        # packed segment order: means, quats, log_scales, opacity, k, sh, semantics
        return [self.lr_position, self.lr_rotation, self.lr_scale, self.lr_opacity, self.lr_k,
                self.lr_sh, self.lr_semantics]


@dataclass
class OptimizerState:
    """Adam moments (trainer.hpp:67-73) as packed n*P buffers."""
    m: torch.Tensor
    v: torch.Tensor
    step: int = 0

    @staticmethod
    def init(scene: Scene) -> "OptimizerState":
        P = param_layout(scene.size(), scene.num_classes, scene.sh_degree)[-1]
        z = torch.zeros(P, dtype=scene.dtype, device=scene.means.device)
        return OptimizerState(z, z.clone(), 0)


def pack_scene(scene: Scene) -> torch.Tensor:
    return torch.cat([t.reshape(-1) for t in (scene.means, scene.quats, scene.log_scales,
                                              scene.opacity_logits, scene.k, scene.sh,
                                              scene.semantics)])


def unpack_into_scene(flat: torch.Tensor, scene: Scene) -> None:
    off = param_layout(scene.size(), scene.num_classes, scene.sh_degree)
    for i, t in enumerate((scene.means, scene.quats, scene.log_scales, scene.opacity_logits,
                           scene.k, scene.sh, scene.semantics)):
        t.copy_(flat[off[i]:off[i + 1]].view_as(t))


def pack_grads(g: GradientBuffer) -> torch.Tensor:
    return torch.cat([t.reshape(-1) for t in (g.dposition, g.drotation, g.dscale, g.dopacity, g.dk,
                                              g.dsh, g.dsemantics)])


def adam_step(scene: Scene, grads: GradientBuffer, state: OptimizerState, cfg: TrainConfig,
              packed_params: torch.Tensor | None = None, packed_grads: torch.Tensor | None = None):
    """adam_step (trainer.cpp:98-133).  Works on packed buffers; when the caller
    keeps the scene as views of one packed tensor it can pass it to avoid the
    pack/unpack copies."""
    if not grads.raw_space:
        raise LogicError("adam_step: gradients not chained to raw parameters")
    if grads.size() != scene.size() or state.m.numel() != param_layout(
            scene.size(), scene.num_classes, scene.sh_degree)[-1]:
        raise ValueError("adam_step: size mismatch")
    state.step += 1
    p = pack_scene(scene) if packed_params is None else packed_params
    g = pack_grads(grads) if packed_grads is None else packed_grads
    ctx = _Context.get(scene.means.device.index)
    lr = (ct.c_double * 7)(*cfg.lrs_packed())
    check(_lib.lib().msplat_adam_step(ctx.h, _dtype_code(scene.dtype), scene.size(), scene.num_classes,
                                      scene.sh_degree, p.data_ptr(), g.data_ptr(), state.m.data_ptr(),
                                      state.v.data_ptr(), state.step, lr))
    if packed_params is None:
        unpack_into_scene(p, scene)


def adam_step_range(scene: Scene, grads: GradientBuffer, state: OptimizerState, cfg: TrainConfig,
                    packed_params: torch.Tensor, packed_grads: torch.Tensor, begin: int, count: int) -> None:
    """adam_step (trainer.cpp:98-133) on the packed elements [begin, begin+count)
    only (msplat_adam_step_range): one rank's shard of a sharded optimizer step.
    state.step is used as is (the caller advances it once per step); the packed
    buffers and state.m / state.v are full length (n*P, or padded beyond)."""
    if not grads.raw_space:
        raise LogicError("adam_step: gradients not chained to raw parameters")
    total = param_layout(scene.size(), scene.num_classes, scene.sh_degree)[-1]
    if begin < 0 or count < 0 or begin + count > total:
        raise ValueError("adam_step_range: range outside the packed buffer")
    if min(packed_params.numel(), packed_grads.numel(), state.m.numel(), state.v.numel()) < total:
        raise ValueError("adam_step_range: packed buffers shorter than n*P")
    if state.step < 1:
        raise ValueError("adam_step_range: state.step must be >= 1")
    ctx = _Context.get(scene.means.device.index)
    lr = (ct.c_double * 7)(*cfg.lrs_packed())
    es = packed_params.element_size()
    check(_lib.lib().msplat_adam_step_range(
        ctx.h, _dtype_code(scene.dtype), scene.size(), scene.num_classes, scene.sh_degree, int(begin), int(count),
        packed_params.data_ptr() + begin * es, packed_grads.data_ptr() + begin * es,
        state.m.data_ptr() + begin * es, state.v.data_ptr() + begin * es, state.step, lr))


def accumulate_packed(dst: torch.Tensor, src: torch.Tensor) -> None:
    """dst += src (msplat_accumulate) on two packed buffers of one device, on
    torch's current stream: sums per-lane gradient buffers of a multi-lane step."""
    if dst.shape != src.shape or dst.dtype != src.dtype or dst.device != src.device:
        raise ValueError("accumulate: buffers differ in shape, dtype or device")
    if not (dst.is_contiguous() and src.is_contiguous()):
        raise ValueError("accumulate: buffers must be contiguous")
    ctx = _Context.get(dst.device.index)
    check(_lib.lib().msplat_accumulate(ctx.h, _dtype_code(dst.dtype), dst.numel(), dst.data_ptr(), src.data_ptr()))


def prune(scene: Scene, state: OptimizerState, cfg: TrainConfig) -> int:
    """prune (trainer.cpp:135-169): device mask (msplat_prune_mask), then one
    stable device compaction of the packed parameters and both Adam moments
    with the k reset (msplat_prune_compact, trainer.cpp:150-168).  The scene's
    tensors become views of the compacted packed buffer.  Returns the number
    removed."""
    n = scene.size()
    dev = scene.means.device
    keep = torch.empty(n, dtype=torch.uint8, device=dev)
    kept = ct.c_int64()
    ctx = _Context.get(dev.index)
    code = _dtype_code(scene.dtype)
    check(_lib.lib().msplat_prune_mask(ctx.h, code, n, scene.k.data_ptr(), float(cfg.prune_threshold),
                                       int(cfg.prune_keep_small), keep.data_ptr(), ct.byref(kept)))
    k = int(kept.value)
    C, deg = scene.num_classes, scene.sh_degree
    P_in = param_layout(n, C, deg)[-1]
    P_out = param_layout(k, C, deg)[-1]
    params = pack_scene(scene)
    if state.m.numel() != P_in or state.v.numel() != P_in:
        raise ValueError("prune: optimizer state does not match the scene")
    out = [torch.empty(P_out, dtype=scene.dtype, device=dev) for _ in range(3)]
    ins = (ct.c_void_p * 3)(params.data_ptr(), state.m.data_ptr(), state.v.data_ptr())
    outs = (ct.c_void_p * 3)(*(t.data_ptr() for t in out))
    check(_lib.lib().msplat_prune_compact(ctx.h, code, n, C, deg, keep.data_ptr(), k, ins, outs,
                                          float(cfg.k_reset)))
    off = param_layout(k, C, deg)
    shapes = {"means": (k, 3), "quats": (k, 4), "log_scales": (k, 3), "opacity_logits": (k,), "k": (k,),
              "sh": tuple(scene.sh.shape[1:]), "semantics": (k, C)}
    for i, name in enumerate(("means", "quats", "log_scales", "opacity_logits", "k", "sh", "semantics")):
        shp = shapes[name] if name != "sh" else (k, *shapes["sh"])
        setattr(scene, name, out[0][off[i]:off[i + 1]].view(shp))
    state.m, state.v = out[1], out[2]
    return n - k


# --------------------------------------------------------------- binning
@dataclass
class TileBins:
    """msplat::TileBins (rasterizer.hpp:33-39) as CSR: offsets + values."""
    tiles_x: int
    tiles_y: int
    offsets: np.ndarray
    values: np.ndarray

    def tile(self, tx, ty):
        t = ty * self.tiles_x + tx
        return self.values[self.offsets[t]:self.offsets[t + 1]].tolist()

    @property
    def bins(self):
        return [self.values[self.offsets[t]:self.offsets[t + 1]].tolist()
                for t in range(self.tiles_x * self.tiles_y)]


def bin_and_sort(splats, width: int, height: int, device=None) -> TileBins:
    """bin_and_sort (rasterizer.cpp:14-45) on explicit splats: a list of
    None or dicts with center (2,), radius, sort_depth -- runs the device
    radix-sort binning (K2-K5)."""
    n = len(splats)
    vis = np.array([s is not None for s in splats], np.uint8)
    center = np.array([s["center"] if s is not None else (0.0, 0.0) for s in splats], np.float64).reshape(n, 2)
    radius = np.array([s["radius"] if s is not None else 0.0 for s in splats], np.float64)
    depth = np.array([s["sort_depth"] if s is not None else 0.0 for s in splats], np.float64)
    tiles_x, tiles_y = (width + 15) // 16, (height + 15) // 16
    off = np.zeros(tiles_x * tiles_y + 1, np.int64)
    ctx = _Context.get(device)
    cap = 1 << 16
    while True:
        vals = np.zeros(cap, np.int32)
        count = ct.c_int64()
        check(_lib.lib().msplat_bin_and_sort_host(
            ctx.h, n, vis.ctypes.data, center.ctypes.data, radius.ctypes.data, depth.ctypes.data, width,
            height, off.ctypes.data_as(ct.POINTER(ct.c_int64)), vals.ctypes.data_as(ct.POINTER(ct.c_int32)),
            cap, ct.byref(count)))
        if count.value <= cap:
            return TileBins(tiles_x, tiles_y, off, vals[:count.value])
        cap = int(count.value)
