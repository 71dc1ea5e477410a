"""ctypes binding of the C ABI in include/msplat_b200.h.

The shared library is built in-tree (``make -C paper_2510_12174_b200/csrc``,
or ``__graft_entry__.build()``) as ``paper_2510_12174_b200/libmsplat_b200.so``.
There is no fallback: if the library is missing or fails to load, every entry
point raises -- the CUDA path is the only implementation of the product.
"""
from __future__ import annotations

import ctypes as ct
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# MSPLAT_LIB overrides the path (A/B timing of two in-tree builds).
LIB_PATH = os.environ.get("MSPLAT_LIB") or os.path.join(HERE, "libmsplat_b200.so")

MSPLAT_OK = 0
MSPLAT_ERR_INVALID_ARGUMENT = 1
MSPLAT_ERR_RUNTIME = 2
MSPLAT_ERR_LOGIC = 3
MSPLAT_ERR_CUDA = 4
MSPLAT_ERR_OUT_OF_MEMORY = 5
MSPLAT_F32 = 0
MSPLAT_F64 = 1
STAGES = ("preprocess", "binning", "forward", "normals", "normals_bwd", "backward", "proj_bwd", "optim")

_vp = ct.c_void_p
_i64 = ct.c_int64


class MsplatScene(ct.Structure):
    _fields_ = [("n", ct.c_int64), ("num_classes", ct.c_int), ("sh_degree", ct.c_int),
                ("dtype", ct.c_int), ("means", _vp), ("quats", _vp), ("log_scales", _vp),
                ("opacity_logits", _vp), ("k", _vp), ("sh", _vp), ("semantics", _vp)]


class MsplatCamera(ct.Structure):
    _fields_ = [("fx", ct.c_double), ("fy", ct.c_double), ("cx", ct.c_double), ("cy", ct.c_double),
                ("width", ct.c_int), ("height", ct.c_int), ("R_c2w", ct.c_double * 9),
                ("t_c2w", ct.c_double * 3)]


class MsplatRenderConfig(ct.Structure):
    _fields_ = [("sigma_scale", ct.c_double), ("background", ct.c_double * 3),
                ("early_stop_transmittance", ct.c_double), ("early_termination", ct.c_int),
                ("threads", ct.c_int)]


class MsplatNormalConfig(ct.Structure):
    _fields_ = [("step1", ct.c_int), ("step2", ct.c_int), ("fuse_lambda", ct.c_double),
                ("mask_threshold", ct.c_double)]


class MsplatFrame(ct.Structure):
    _fields_ = [("color", _vp), ("depth", _vp), ("semantics", _vp), ("kmap", _vp),
                ("transmittance", _vp), ("normals", _vp), ("contributors", _vp)]


class MsplatPixelGrads(ct.Structure):
    _fields_ = [("dcolor", _vp), ("ddepth", _vp), ("dsemantics", _vp), ("dkmap", _vp),
                ("dnormals", _vp)]


class MsplatGrads(ct.Structure):
    _fields_ = [("dposition", _vp), ("drotation", _vp), ("dscale", _vp), ("dopacity", _vp),
                ("dk", _vp), ("dsh", _vp), ("dsemantics", _vp)]


class MsplatCounters(ct.Structure):
    _fields_ = [("n", ct.c_int64), ("visible", ct.c_int64), ("instances", ct.c_int64),
                ("tiles", ct.c_int64), ("max_tile_list", ct.c_int64)]


class MsplatGroundTruth(ct.Structure):
    _fields_ = [("rgb", _vp), ("depth", _vp), ("normal", _vp), ("labels", _vp)]


LOSS_REPORT_FIELDS = ("l1", "ssim", "depth", "normal", "seg", "k", "combined", "ratio_ssim", "ratio_normal",
                      "ratio_depth", "ratio_seg", "ratio_k", "seed_l1", "seed_ssim", "seed_depth", "seed_normal",
                      "seed_seg", "seed_k")


class MsplatLossReport(ct.Structure):
    _fields_ = [(f, ct.c_double) for f in LOSS_REPORT_FIELDS]


METRIC_FIELDS = ("psnr", "ssim", "abs_rel", "rmse", "cos_simi", "miou")


class MsplatMetricReport(ct.Structure):
    _fields_ = [(f, ct.c_double) for f in METRIC_FIELDS] + [("has_" + f, ct.c_int) for f in METRIC_FIELDS]


class LogicError(RuntimeError):
    """std::logic_error of the reference (e.g. chaining an already-raw buffer)."""


def _sig(lib):
    P = ct.POINTER
    S = [
        ("msplat_last_error", ct.c_char_p, []),
        ("msplat_abi_version", ct.c_int, []),
        ("msplat_context_create", ct.c_int, [ct.c_int, _vp, P(_vp)]),
        ("msplat_context_destroy", None, [_vp]),
        ("msplat_context_set_stream", ct.c_int, [_vp, _vp]),
        ("msplat_context_check", ct.c_int, [_vp]),
        ("msplat_replay_create", ct.c_int, [_vp, P(_vp)]),
        ("msplat_replay_destroy", None, [_vp]),
        ("msplat_replay_set_capture", ct.c_int, [_vp, ct.c_int]),
        ("msplat_param_layout", ct.c_int, [_i64, ct.c_int, ct.c_int, P(_i64)]),
        ("msplat_rasterize", ct.c_int, [_vp, P(MsplatScene), P(MsplatCamera), P(MsplatRenderConfig),
                                        P(MsplatFrame), _vp]),
        ("msplat_estimate_normals", ct.c_int, [_vp, ct.c_int, _vp, _vp, P(MsplatCamera),
                                               P(MsplatNormalConfig), _vp]),
        ("msplat_normals_backward", ct.c_int, [_vp, ct.c_int, _vp, _vp, _vp, P(MsplatCamera),
                                               P(MsplatNormalConfig), ct.c_double, _vp]),
        ("msplat_rasterize_backward", ct.c_int, [_vp, P(MsplatScene), P(MsplatCamera), P(MsplatFrame),
                                                 _vp, P(MsplatPixelGrads), P(MsplatGrads)]),
        ("msplat_chain_activations", ct.c_int, [_vp, P(MsplatScene), P(MsplatGrads)]),
        ("msplat_fwd_bwd", ct.c_int, [_vp, P(MsplatScene), P(MsplatCamera), P(MsplatRenderConfig),
                                      P(MsplatNormalConfig), P(MsplatFrame), P(MsplatPixelGrads),
                                      P(MsplatGrads), ct.c_int, ct.c_int, _vp]),
        ("msplat_adam_step", ct.c_int, [_vp, ct.c_int, _i64, ct.c_int, ct.c_int, _vp, _vp, _vp, _vp,
                                        _i64, P(ct.c_double)]),
        ("msplat_adam_step_range", ct.c_int, [_vp, ct.c_int, _i64, ct.c_int, ct.c_int, _i64, _i64, _vp, _vp,
                                              _vp, _vp, _i64, P(ct.c_double)]),
        ("msplat_accumulate", ct.c_int, [_vp, ct.c_int, _i64, _vp, _vp]),
        ("msplat_prune_mask", ct.c_int, [_vp, ct.c_int, _i64, _vp, ct.c_double, ct.c_int, _vp,
                                         P(_i64)]),
        ("msplat_prune_compact", ct.c_int, [_vp, ct.c_int, _i64, ct.c_int, ct.c_int, _vp, _i64, P(_vp), P(_vp),
                                            ct.c_double]),
        ("msplat_replay_counters", ct.c_int, [_vp, P(MsplatCounters)]),
        ("msplat_replay_bins", ct.c_int, [_vp, P(_i64), P(ct.c_int32), _i64]),
        ("msplat_replay_splats", ct.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
        ("msplat_replay_terminus", ct.c_int, [_vp, P(ct.c_int32)]),
        ("msplat_replay_weight_sums", ct.c_int, [_vp, P(ct.c_double)]),
        ("msplat_bin_and_sort_host", ct.c_int, [_vp, _i64, _vp, _vp, _vp, _vp, ct.c_int, ct.c_int,
                                                P(_i64), P(ct.c_int32), _i64, P(_i64)]),
        ("msplat_context_set_timing", ct.c_int, [_vp, ct.c_int]),
        ("msplat_context_set_deterministic", ct.c_int, [_vp, ct.c_int]),
        ("msplat_frame_losses", ct.c_int, [_vp, ct.c_int, ct.c_int, P(MsplatCamera), P(MsplatNormalConfig),
                                           P(MsplatFrame), P(MsplatGroundTruth), P(ct.c_double),
                                           P(MsplatPixelGrads), P(MsplatLossReport)]),
        ("msplat_loss_report_device", _vp, [_vp]),
        ("msplat_frame_metrics", ct.c_int, [_vp, ct.c_int, ct.c_int, ct.c_int, ct.c_int, _vp, _vp, _vp, _vp, _vp,
                                            _vp, _vp, _vp, _vp, _vp, _vp, P(MsplatMetricReport)]),
        ("msplat_ply_scene_info", ct.c_int, [ct.c_char_p, P(_i64), P(ct.c_int), P(ct.c_int)]),
        ("msplat_load_scene_ply", ct.c_int, [_vp, ct.c_char_p, ct.c_int, _vp]),
        ("msplat_save_scene_ply", ct.c_int, [_vp, ct.c_char_p, ct.c_int, _i64, ct.c_int, ct.c_int, _vp]),
        ("msplat_init_scene", ct.c_int, [_vp, ct.c_int, _i64, _vp, _vp, ct.c_int, ct.c_int, ct.c_double, _vp]),
        ("msplat_context_timings", ct.c_int, [_vp, P(ct.c_double), P(_i64)]),
        ("msplat_kernel_launches", _i64, []),
    ]
    for name, res, args in S:
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_LIB = None


def lib():
    """The loaded CUDA library (raises if it was not built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"msplat CUDA library not found at {LIB_PATH}; build it with "
                "`make -C paper_2510_12174_b200/csrc` (there is no CPU fallback)")
        _LIB = _sig(ct.CDLL(LIB_PATH))
        if _LIB.msplat_abi_version() != 1:
            raise RuntimeError("msplat ABI version mismatch")
    return _LIB


def check(status: int):
    """Raise the exception type the reference would throw for a status."""
    if status == MSPLAT_OK:
        return
    msg = lib().msplat_last_error().decode()
    if status == MSPLAT_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == MSPLAT_ERR_LOGIC:
        raise LogicError(msg)
    if status == MSPLAT_ERR_OUT_OF_MEMORY:
        raise MemoryError(msg)
    raise RuntimeError(msg)
