"""Extended-PLY scene I/O (core/src/io_ply.cpp)
against the reference's own save_scene_ply / load_scene_ply (oracle/_ref).

CPU: the header interpretation (msplat_ply_scene_info, host code) and every
header error text equal the reference's.
GPU: the device decode/encode: loading a reference-written file reproduces the
scene bit for bit; saving writes a byte-identical file; float32 files from other
tools (no semantics, no grad_k) load with the reference's defaults; payload
errors (truncation, non-finite values) carry the reference's messages.
"""
import ctypes as ct
import os
import struct

import numpy as np
import pytest

from paper_2510_12174_b200 import scenes

TYPES = {"double": "d", "float": "f", "uchar": "B", "char": "b", "ushort": "H", "short": "h", "int": "i",
         "uint": "I"}


def write_ply(path, props, rows, header_extra=""):
    """props: [(type, name)], rows: list of value tuples (binary little endian)."""
    hdr = "ply\nformat binary_little_endian 1.0\n" + header_extra + f"element vertex {len(rows)}\n"
    hdr += "".join(f"property {t} {n}\n" for t, n in props) + "end_header\n"
    fmt = "<" + "".join(TYPES[t] for t, _ in props)
    with open(path, "wb") as f:
        f.write(hdr.encode())
        for r in rows:
            f.write(struct.pack(fmt, *r))


def scene_props(deg, C, k=True, t="double"):
    K = (deg + 1) ** 2
    names = ["x", "y", "z"] + [f"f_dc_{i}" for i in range(3)] + [f"f_rest_{i}" for i in range(3 * (K - 1))]
    names += ["opacity"] + [f"scale_{i}" for i in range(3)] + [f"rot_{i}" for i in range(4)]
    names += [f"sem_{i}" for i in range(C)] + (["grad_k"] if k else [])
    return [(t, n) for n in names]


def packed(s):
    n, C, K = len(s["means"]), int(s["num_classes"]), (int(s["sh_degree"]) + 1) ** 2
    return np.concatenate([np.asarray(s["means"]).ravel(), np.asarray(s["quats"]).ravel(),
                           np.asarray(s["log_scales"]).ravel(), np.asarray(s["opacity_logits"]).ravel(),
                           np.asarray(s["k"]).ravel(), np.asarray(s["sh"]).reshape(n, 3, K).ravel(),
                           np.asarray(s["semantics"]).reshape(n, C).ravel()])


def ref_load(reference, path):
    lib = reference.lib
    n, C, deg = ct.c_int64(), ct.c_int(), ct.c_int()
    st = lib.mo_ply_load(str(path).encode(), ct.c_int64(0), None, ct.byref(n), ct.byref(C), ct.byref(deg))
    if st:
        return None, lib.mo_last_error().decode()
    P = 12 + 3 * (deg.value + 1) ** 2 + C.value
    out = np.zeros(max(n.value * P, 1))
    lib.mo_ply_load(str(path).encode(), ct.c_int64(out.size), out.ctypes.data_as(ct.c_void_p), ct.byref(n),
                    ct.byref(C), ct.byref(deg))
    return (out[: n.value * P], n.value, C.value, deg.value), None


def ref_save(reference, path, s):
    sc, keep = reference.scene(s)
    st = reference.lib.mo_ply_save(str(path).encode(), ct.byref(sc))
    assert st == 0, reference.lib.mo_last_error().decode()


def our_info(path):
    from paper_2510_12174_b200 import _lib
    n, C, deg = ct.c_int64(), ct.c_int(), ct.c_int()
    st = _lib.lib().msplat_ply_scene_info(str(path).encode(), ct.byref(n), ct.byref(C), ct.byref(deg))
    if st:
        return None, _lib.lib().msplat_last_error().decode()
    return (n.value, C.value, deg.value), None


def test_header_interpretation_matches_reference(tmp_path, reference):
    for deg, C in ((0, 0), (2, 5), (3, 2)):
        s = scenes.make_random_scene(20, C, deg, seed=deg + C)
        p = tmp_path / f"s{deg}{C}.ply"
        ref_save(reference, p, s)
        (_, n, rc, rdeg), _ = ref_load(reference, p)
        assert our_info(p)[0] == (n, rc, rdeg) == (20, C, deg)
    bad = {
        "magic": (b"plx\n", None),
        "format": (b"ply\nformat ascii 1.0\nend_header\n", None),
    }
    for name, (blob, _) in bad.items():
        p = tmp_path / f"{name}.ply"
        p.write_bytes(blob)
        assert our_info(p)[1] == ref_load(reference, p)[1], name
    cases = {
        "missing": scene_props(1, 0)[1:],  # no x
        "rest": scene_props(1, 0) + [("double", "f_rest_9")],
        "rest_deg": [p for p in scene_props(2, 0) if p[1] not in ("f_rest_21", "f_rest_22", "f_rest_23")],
        "type": [("long", "x")] + scene_props(0, 0)[1:],
    }
    for name, props in cases.items():
        p = tmp_path / f"{name}.ply"
        hdr = "ply\nformat binary_little_endian 1.0\nelement vertex 0\n"
        hdr += "".join(f"property {t} {n}\n" for t, n in props) + "end_header\n"
        p.write_bytes(hdr.encode())
        ours, ref = our_info(p), ref_load(reference, p)
        assert ours[1] is not None and ours[1] == ref[1], (name, ours, ref)
    p = tmp_path / "face.ply"
    p.write_bytes(b"ply\nformat binary_little_endian 1.0\nelement vertex 0\nproperty double x\n"
                  b"element face 1\nproperty list uchar int vertex_indices\nend_header\n")
    assert our_info(p)[1] == ref_load(reference, p)[1]


@pytest.mark.gpu
@pytest.mark.parametrize("deg,C", [(0, 0), (1, 3), (2, 5), (3, 2)])
def test_device_load_save_match_reference(tmp_path, reference, deg, C):
    import torch
    import paper_2510_12174_b200 as M
    s = scenes.make_random_scene(300, C, deg, seed=10 * deg + C)
    pr = tmp_path / "ref.ply"
    ref_save(reference, pr, s)
    sc = M.load_scene_ply(pr, dtype=torch.float64)
    (want, n, _, _), _ = ref_load(reference, pr)
    got = M.pack_scene(sc).cpu().numpy()
    assert np.array_equal(got, want) and np.array_equal(want, packed(s))
    ours = tmp_path / "ours.ply"
    M.save_scene_ply(ours, sc)
    assert ours.read_bytes() == pr.read_bytes()
    s32 = M.load_scene_ply(pr, dtype=torch.float32)
    assert np.array_equal(M.pack_scene(s32).cpu().numpy(), want.astype(np.float32))


@pytest.mark.gpu
def test_device_load_float32_and_defaults(tmp_path, reference):
    import torch
    import paper_2510_12174_b200 as M
    rng = np.random.default_rng(3)
    props = scene_props(1, 0, k=False, t="float") + [("uchar", "red")]  # unknown column tolerated
    rows = [tuple(rng.standard_normal(len(props) - 1).astype(np.float32).tolist()) + (7,) for _ in range(50)]
    p = tmp_path / "f32.ply"
    write_ply(p, props, rows, header_extra="comment written by another tool\n")
    sc = M.load_scene_ply(p, dtype=torch.float64)
    (want, n, C, deg), _ = ref_load(reference, p)
    assert (n, C, deg) == (50, 0, 1)
    assert np.array_equal(M.pack_scene(sc).cpu().numpy(), want)
    assert np.all(sc.k.cpu().numpy() == 0.9)


@pytest.mark.gpu
def test_device_load_errors_match_reference(tmp_path, reference):
    import paper_2510_12174_b200 as M
    props = scene_props(0, 1)
    good = tuple([0.1] * len(props))
    p = tmp_path / "trunc.ply"
    write_ply(p, props, [good] * 5)
    p.write_bytes(p.read_bytes()[:-20])
    with pytest.raises(RuntimeError) as e:
        M.load_scene_ply(p)
    assert str(e.value) == ref_load(reference, p)[1]
    p = tmp_path / "nan.ply"
    bad = list(good)
    bad[4] = float("nan")
    write_ply(p, props, [good, good, tuple(bad), good])
    with pytest.raises(ValueError) as e:
        M.load_scene_ply(p)
    assert str(e.value) == ref_load(reference, p)[1] == "Scene: primitive 2 has non-finite fields"
