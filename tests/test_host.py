"""CPU: host-side logic -- scene generator, camera contract, Python API
validation (everything that runs before a kernel launch)."""
import numpy as np
import pytest
import torch

import paper_2510_12174_b200 as M
from paper_2510_12174_b200 import scenes


def test_room_scene_is_deterministic_float32_and_rejects_near_plane():
    a = scenes.make_room_scene(5000, 7, 2, seed=1, views=(0, 1, 2))
    b = scenes.make_room_scene(5000, 7, 2, seed=1, views=(0, 1, 2))
    for k in ("means", "quats", "log_scales", "opacity_logits", "sh", "semantics", "k"):
        assert a[k].dtype == np.float32
        assert np.array_equal(a[k], b[k])
    assert a["sh"].shape == (5000, 3, 9) and a["semantics"].shape == (5000, 7)
    assert np.allclose(np.linalg.norm(a["quats"], axis=1), 1, atol=1e-6)
    for v in (0, 1, 2):
        cam = scenes.view_camera(v, 1200, 680, 600.0)
        zc = (a["means"] - cam["t_c2w"]) @ cam["R_c2w"][:, 2]
        assert not np.any((zc > 0.01) & (zc < 1.0))
    # surface normal is the short axis
    s = np.exp(a["log_scales"])
    assert np.all(s[:, 2] < s[:, :2].min(axis=1))


def test_view_cameras_are_rotations_with_bounded_jitter():
    for v in range(16):
        c = scenes.view_camera(v, 1200, 680, 600.0)
        R = c["R_c2w"]
        assert np.allclose(R.T @ R, np.eye(3), atol=1e-12) and abs(np.linalg.det(R) - 1) < 1e-12
        assert np.degrees(np.arccos(np.clip(R[2, 2], -1, 1))) <= 14.2  # yaw, pitch within +-10 deg
        M.make_camera(c["fx"], c["fy"], c["cx"], c["cy"], 1200, 680, R, c["t_c2w"])  # finalize passes


def test_camera_finalize_contract():
    """CameraView::finalize (camera.cpp:8-21)."""
    with pytest.raises(ValueError, match="focal"):
        M.make_camera(0, 1, 0, 0, 4, 4, np.eye(3), np.zeros(3))
    with pytest.raises(ValueError, match="width and height"):
        M.make_camera(1, 1, 0, 0, 0, 4, np.eye(3), np.zeros(3))
    with pytest.raises(ValueError, match="orthonormal"):
        M.make_camera(1, 1, 0, 0, 4, 4, np.diag([1, 1, 2.0]), np.zeros(3))
    with pytest.raises(ValueError, match="determinant"):
        M.make_camera(1, 1, 0, 0, 4, 4, np.diag([1, 1, -1.0]), np.zeros(3))
    cam = M.make_lookat_camera(10, 10, 5, 5, 10, 10, eye=(0, 0, -3), target=(0, 0, 0))
    assert np.allclose(cam.R_cam_to_world[:, 2], [0, 0, 1])


def test_scene_validation_mirrors_reference_messages():
    s = scenes.make_random_scene(4, 3, 1, seed=0)
    sc = M.Scene(*(torch.as_tensor(s[k]) for k in ("means", "quats", "log_scales", "opacity_logits", "sh",
                                                  "semantics", "k")), num_classes=3, sh_degree=1)
    with pytest.raises(ValueError, match="CUDA"):
        sc.validate()  # host tensors never reach the kernels (no CPU fallback)
    sc.sh_degree = 2
    with pytest.raises(ValueError, match="SH coefficient count"):
        sc.validate()
    sc.sh_degree, sc.num_classes = 1, 4
    with pytest.raises(ValueError, match="semantic channel count"):
        sc.validate()
    sc.sh_degree = 5
    with pytest.raises(ValueError, match="sh_degree"):
        sc.validate()


def test_packed_gradient_views_follow_param_layout():
    n, C, deg = 7, 3, 2
    off = M.param_layout(n, C, deg)
    flat = torch.arange(off[-1], dtype=torch.float32)
    g = M.GradientBuffer.from_packed(flat, n, C, deg)
    assert g.dposition.shape == (n, 3) and g.dsh.shape == (n, 3, 9) and g.dsemantics.shape == (n, 3)
    assert g.dposition.data_ptr() == flat.data_ptr()
    assert int(g.dk[0]) == off[4] and int(g.dsh[0, 0, 0]) == off[5] and int(g.dsemantics[0, 0]) == off[6]


def test_pixel_grads_are_dense_and_seeded():
    p = scenes.pixel_grads(40, 30, 5, seed=3)
    q = scenes.pixel_grads(40, 30, 5, seed=3)
    assert p["dsemantics"].shape == (5, 30, 40) and p["dnormals"].shape == (3, 30, 40)
    for k in p:
        assert np.array_equal(p[k], q[k]) and np.count_nonzero(p[k]) == p[k].size
        assert np.abs(p[k]).max() <= 1.0 / (40 * 30)
