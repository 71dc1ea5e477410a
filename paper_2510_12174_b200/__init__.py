"""B200-native UniGS multimodal rasterizer (arXiv 2510.12174).

A drop-in for the reference's render path (proj/core, namespace msplat):
hand-written sm_100a kernels behind the C ABI in include/msplat_b200.h.
`rasterizer` mirrors the reference API over torch device tensors;
`scenes` generates the seeded synthetic benchmark scenes.
"""
from . import _lib  # noqa: F401
from .rasterizer import (  # noqa: F401
    CameraView, GradientBuffer, GroundTruth, LogicError, LossReport, MultimodalFrame, NormalConfig, OptimizerState,
    PixelGradients, RenderConfig, ReplayState, Scene, TileBins, TrainConfig, accumulate_packed, adam_step, bin_and_sort,
    chain_activations, estimate_normals, frame_losses, frame_metrics, fwd_bwd, load_scene_ply, pack_scene, save_scene_ply, make_camera, make_lookat_camera, normals_backward,
    param_layout, prune, rasterize, rasterize_backward, set_deterministic, set_stage_timing, stage_timings,
)

from .dataset import DatasetFrame, SceneDataset, load_dataset  # noqa: F401,E402

__version__ = "0.1.0"
