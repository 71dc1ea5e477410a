"""Ground-truth ingestion: the dataset manifest
(core/src/dataset.cpp:53-208), PNG / PFM maps (core/src/io_image.cpp:28-187)
and the training config (dataset.cpp:210-284), against the reference's own
code compiled unmodified into oracle/_ref/libmsplat_ref_io.so (real libpng
1.6.56 from Pillow's wheel, nlohmann/json 3.11.3).

Decoding and parsing are host work in both implementations, so these are CPU
tests; the last one (gpu) takes the maps to cuda:0 and through frame_losses /
frame_metrics.
"""
import ctypes as ct
import json
import os
import struct
import zlib

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_IO = os.path.join(REPO, "oracle", "_ref", "libmsplat_ref_io.so")
OURS = os.path.join(REPO, "paper_2510_12174_b200", "libmsplat_dropin.so")


class Lib:
    """The same flat shapes over either library (prefix mo_io_ / msplat_)."""

    def __init__(self, path, ref):
        self.lib = ct.CDLL(path)
        self.ref = ref
        n = (lambda s: "mo_io_" + s) if ref else (lambda s: {"last_error": "msplat_dataset_last_error"}.get(
            s, "msplat_" + s.replace("read_png", "image_read_png").replace("write_png", "image_write_png")
            .replace("read_pfm", "image_read_pfm").replace("write_pfm", "image_write_pfm")))
        self.f = {k: getattr(self.lib, n(k)) for k in (
            "last_error", "dataset_load", "dataset_free", "dataset_dims", "dataset_frame", "dataset_points",
            "dataset_save", "read_png", "write_png", "read_pfm", "write_pfm", "config_load")}
        self.f["last_error"].restype = ct.c_char_p
        self.f["dataset_load"].argtypes = [ct.c_char_p, ct.POINTER(ct.c_void_p)]
        for k in ("dataset_free",):
            self.f[k].argtypes = [ct.c_void_p]
        self.f["dataset_dims"].argtypes = [ct.c_void_p, ct.c_void_p]
        self.f["dataset_frame"].argtypes = [ct.c_void_p, ct.c_int64, ct.c_void_p, ct.c_void_p, ct.c_void_p,
                                            ct.c_void_p, ct.c_void_p, ct.c_void_p]
        self.f["dataset_points"].argtypes = [ct.c_void_p, ct.c_void_p, ct.c_void_p]
        self.f["dataset_save"].argtypes = [ct.c_void_p, ct.c_char_p]

    def err(self):
        return self.f["last_error"]().decode()

    def read_png(self, path):
        w, h, c = ct.c_int(), ct.c_int(), ct.c_int()
        if self.f["read_png"](str(path).encode(), ct.byref(w), ct.byref(h), ct.byref(c), None):
            return None, self.err()
        out = np.zeros((h.value, w.value, c.value), np.uint8)
        self.f["read_png"](str(path).encode(), ct.byref(w), ct.byref(h), ct.byref(c), out.ctypes.data_as(ct.c_void_p))
        return out, None

    def write_png(self, path, a):
        a = np.ascontiguousarray(a, np.uint8)
        h, w, c = a.shape
        if self.f["write_png"](str(path).encode(), w, h, c, a.ctypes.data_as(ct.c_void_p)):
            return self.err()
        return None

    def read_pfm(self, path):
        w, h, c = ct.c_int(), ct.c_int(), ct.c_int()
        if self.f["read_pfm"](str(path).encode(), ct.byref(w), ct.byref(h), ct.byref(c), None):
            return None, self.err()
        out = np.zeros((h.value, w.value, c.value))
        self.f["read_pfm"](str(path).encode(), ct.byref(w), ct.byref(h), ct.byref(c), out.ctypes.data_as(ct.c_void_p))
        return out, None

    def write_pfm(self, path, a):
        a = np.ascontiguousarray(a, np.float64)
        h, w, c = a.shape
        if self.f["write_pfm"](str(path).encode(), w, h, c, a.ctypes.data_as(ct.c_void_p)):
            return self.err()
        return None

    def config(self, path):
        out = np.zeros(33)
        if self.f["config_load"](str(path).encode(), out.ctypes.data_as(ct.c_void_p)):
            return None, self.err()
        return out, None

    def dataset(self, root):
        h = ct.c_void_p()
        if self.f["dataset_load"](str(root).encode(), ct.byref(h)):
            return None, self.err()
        try:
            dims = np.zeros(5, np.int64)
            self.f["dataset_dims"](h, dims.ctypes.data_as(ct.c_void_p))
            W, H, C, nf, npts = (int(v) for v in dims)
            frames = []
            for i in range(nf):
                cam, flags = np.zeros(16), ct.c_int()
                rgb, dep = np.zeros((3, H, W), np.float32), np.zeros((H, W), np.float32)
                nrm, lab = np.zeros((3, H, W), np.float32), np.zeros((H, W), np.uint8)
                st = self.f["dataset_frame"](h, i, cam.ctypes.data_as(ct.c_void_p), ct.byref(flags),
                                             *(x.ctypes.data_as(ct.c_void_p) for x in (rgb, dep, nrm, lab)))
                assert st == 0
                frames.append(dict(cam=cam, flags=flags.value, rgb=rgb, depth=dep, normal=nrm, labels=lab))
            pts, cols = np.zeros((npts, 3)), np.zeros((npts, 3))
            self.f["dataset_points"](h, pts.ctypes.data_as(ct.c_void_p), cols.ctypes.data_as(ct.c_void_p))
            return dict(dims=(W, H, C, nf, npts), frames=frames, points=pts, colors=cols), None
        finally:
            self.f["dataset_free"](h)

    def resave(self, root, out):
        h = ct.c_void_p()
        assert self.f["dataset_load"](str(root).encode(), ct.byref(h)) == 0, self.err()
        try:
            assert self.f["dataset_save"](h, str(out).encode()) == 0, self.err()
        finally:
            self.f["dataset_free"](h)


@pytest.fixture(scope="module")
def libs():
    if not os.path.exists(REF_IO):
        pytest.skip("oracle/_ref/libmsplat_ref_io.so not built (needs /root/reference)")
    return Lib(REF_IO, True), Lib(OURS, False)


# ---- PNG writers for cases Pillow cannot produce -------------------------------------------------
def _chunk(t, d):
    return struct.pack(">I", len(d)) + t + d + struct.pack(">I", zlib.crc32(t + d) & 0xFFFFFFFF)


def _filter_rows(rows, bpp, rng):
    """Applies a random PNG filter (0-4) to each packed row."""
    out, prev = b"", np.zeros(len(rows[0]), np.int32)
    for r in rows:
        x = np.frombuffer(r, np.uint8).astype(np.int32)
        a = np.concatenate([np.zeros(bpp, np.int32), x[:-bpp]])
        c = np.concatenate([np.zeros(bpp, np.int32), prev[:-bpp]])
        ft = int(rng.integers(0, 5))
        if ft == 0:
            f = x
        elif ft == 1:
            f = x - a
        elif ft == 2:
            f = x - prev
        elif ft == 3:
            f = x - (a + prev) // 2
        else:
            p = a + prev - c
            pa, pb, pc = np.abs(p - a), np.abs(p - prev), np.abs(p - c)
            pred = np.where((pa <= pb) & (pa <= pc), a, np.where(pb <= pc, prev, c))
            f = x - pred
        out += bytes([ft]) + (f & 0xFF).astype(np.uint8).tobytes()
        prev = x
    return out


def png_bytes(samples, depth, ctype, rng, palette=None, trns=None, interlace=False, idat_split=1):
    """samples: [H, W, ch] integer samples at `depth` bits."""
    H, W, ch = samples.shape

    def pack(sub):
        rows = []
        for r in sub:
            v = r.reshape(-1).astype(np.uint32)
            if depth == 8:
                rows.append(v.astype(np.uint8).tobytes())
            else:
                bits = np.zeros(((len(v) * depth + 7) // 8) * 8, np.uint8)
                for i, s in enumerate(v):
                    for b in range(depth):
                        bits[i * depth + b] = (s >> (depth - 1 - b)) & 1
                rows.append(np.packbits(bits).tobytes())
        return rows

    bpp = max(1, ch * depth // 8)
    raw = b""
    if interlace:
        for x0, y0, dx, dy in [(0, 0, 8, 8), (4, 0, 8, 8), (0, 4, 4, 8), (2, 0, 4, 4), (0, 2, 2, 4), (1, 0, 2, 2),
                               (0, 1, 1, 2)]:
            sub = samples[y0::dy, x0::dx]
            if sub.size:
                raw += _filter_rows(pack(sub), bpp, rng)
    else:
        raw = _filter_rows(pack(samples), bpp, rng)
    z = zlib.compress(raw)
    out = b"\x89PNG\r\n\x1a\n" + _chunk(b"IHDR", struct.pack(">IIBBBBB", W, H, depth, ctype, 0, 0, int(interlace)))
    if palette is not None:
        out += _chunk(b"PLTE", np.asarray(palette, np.uint8).tobytes())
    if trns is not None:
        out += _chunk(b"tRNS", bytes(trns))
    step = (len(z) + idat_split - 1) // idat_split
    for k in range(0, len(z), step):
        out += _chunk(b"IDAT", z[k:k + step])
    return out + _chunk(b"IEND", b"")


def png_cases(tmp_path):
    from PIL import Image
    rng = np.random.default_rng(7)
    a = rng.integers(0, 256, (29, 41, 3), dtype=np.uint8)
    cases = {}

    def put(name, writer):
        p = tmp_path / f"{name}.png"
        writer(p)
        cases[name] = p

    put("pil_rgb", lambda p: Image.fromarray(a).save(p))
    put("pil_gray", lambda p: Image.fromarray(a[..., 0]).save(p))
    put("pil_rgba", lambda p: Image.fromarray(np.concatenate([a, a[..., :1]], 2)).save(p))
    put("pil_la", lambda p: Image.fromarray(a[..., 0]).convert("LA").save(p))
    put("pil_pal", lambda p: Image.fromarray(a).convert("P", palette=Image.ADAPTIVE, colors=13).save(p))
    put("pil_pal4", lambda p: Image.fromarray(a).convert("P", palette=Image.ADAPTIVE, colors=13).save(p, bits=4))
    put("pil_1bit", lambda p: Image.fromarray(a[..., 0]).convert("1").save(p))
    put("pil_16bit", lambda p: Image.fromarray(a[..., 0].astype(np.uint16) * 200).save(p))
    put("pil_pal_trns", lambda p: Image.fromarray(a).convert("P", palette=Image.ADAPTIVE, colors=13).save(
        p, transparency=3))
    for depth in (1, 2, 4, 8):  # gray at every bit depth, all five filters
        g = rng.integers(0, 1 << depth, (23, 37, 1))
        put(f"gray{depth}", lambda p, g=g, d=depth: p.write_bytes(png_bytes(g, d, 0, rng)))
        put(f"gray{depth}_trns", lambda p, g=g, d=depth: p.write_bytes(png_bytes(g, d, 0, rng, trns=[0, 1])))
    pal = rng.integers(0, 256, (11, 3))
    for depth in (1, 2, 4, 8):  # palette indices, incl. ones past the palette
        idx = rng.integers(0, min(1 << depth, 14), (19, 33, 1))
        put(f"pal{depth}", lambda p, i=idx, d=depth: p.write_bytes(png_bytes(i, d, 3, rng, palette=pal)))
    put("rgb_filters", lambda p: p.write_bytes(png_bytes(a, 8, 2, rng, idat_split=5)))
    put("rgba_filters", lambda p: p.write_bytes(png_bytes(np.concatenate([a, a[..., :1]], 2), 8, 6, rng)))
    put("la_filters", lambda p: p.write_bytes(png_bytes(a[..., :2], 8, 4, rng)))
    put("rgb_trns", lambda p: p.write_bytes(png_bytes(a, 8, 2, rng, trns=[0, 1, 0, 2, 0, 3])))
    # errors
    put("bad_sig", lambda p: p.write_bytes(b"GIF89a\0\0"))
    put("truncated", lambda p: p.write_bytes(cases["pil_rgb"].read_bytes()[:300]))
    good = bytearray(cases["pil_rgb"].read_bytes())
    good[40] ^= 0x55  # inside IDAT: CRC mismatch
    put("bad_crc", lambda p: p.write_bytes(bytes(good)))
    return cases


def test_png_decode_matches_reference(tmp_path, libs):
    ref, ours = libs
    for name, path in png_cases(tmp_path).items():
        (r, re_), (o, oe) = ref.read_png(path), ours.read_png(path)
        if r is None:
            assert oe is not None, (name, re_)
            assert oe == re_, (name, oe, re_)
        else:
            assert o is not None, (name, oe)
            assert r.shape == o.shape and np.array_equal(r, o), name


def test_png_interlaced_decodes_like_pillow(tmp_path, libs):
    """Adam7 files: decoded in full (Pillow agrees).  The reference reads them
    without png_set_interlace_handling, so it returns the passes' rows -- a
    documented deviation."""
    from PIL import Image
    ref, ours = libs
    rng = np.random.default_rng(3)
    for shape, depth, ctype in (((13, 11, 3), 8, 2), ((9, 17, 1), 8, 0), ((21, 5, 1), 4, 0)):
        s = rng.integers(0, 1 << depth, shape)
        p = tmp_path / f"adam7_{ctype}_{depth}.png"
        p.write_bytes(png_bytes(s, depth, ctype, rng, interlace=True))
        o, oe = ours.read_png(p)
        assert oe is None
        want = np.asarray(Image.open(p).convert("RGB" if ctype == 2 else "L"))
        assert np.array_equal(o.reshape(want.shape), want)


def test_png_write_roundtrip(tmp_path, libs):
    from PIL import Image
    ref, ours = libs
    rng = np.random.default_rng(11)
    for c in (1, 3):
        a = rng.integers(0, 256, (17, 23, c), dtype=np.uint8)
        p = tmp_path / f"w{c}.png"
        assert ours.write_png(p, a) is None
        r, _ = ref.read_png(p)
        assert np.array_equal(r, a)
        assert np.array_equal(np.asarray(Image.open(p)).reshape(a.shape), a)
    bad = np.zeros((4, 4, 2), np.uint8)
    assert ours.write_png(tmp_path / "x.png", bad) == ref.write_png(tmp_path / "y.png", bad) == \
        "write_png: only 1 or 3 channels supported"


def test_pfm_matches_reference(tmp_path, libs):
    ref, ours = libs
    rng = np.random.default_rng(5)
    for c in (1, 3):
        a = rng.standard_normal((13, 19, c))
        pr, po = tmp_path / f"r{c}.pfm", tmp_path / f"o{c}.pfm"
        assert ref.write_pfm(pr, a) is None and ours.write_pfm(po, a) is None
        assert pr.read_bytes() == po.read_bytes()
        (x, _), (y, _) = ref.read_pfm(pr), ours.read_pfm(pr)
        assert np.array_equal(x, y) and np.array_equal(x, a.astype(np.float32).astype(np.float64))
    # big-endian file (positive scale)
    a = rng.standard_normal((5, 7, 1)).astype(np.float32)
    p = tmp_path / "be.pfm"
    p.write_bytes(b"Pf\n7 5\n1.0\n" + a[::-1].astype(">f4").tobytes())
    (x, _), (y, _) = ref.read_pfm(p), ours.read_pfm(p)
    assert np.array_equal(x, y) and np.array_equal(y, a.astype(np.float64))
    for name, blob in {"magic": b"P6\n1 1\n-1\n", "header": b"PF\n0 3\n-1.0\n", "scale": b"Pf\n2 2\n0\n",
                       "trunc": b"PF\n4 4\n-1.0\n" + b"\0" * 40}.items():
        p = tmp_path / f"bad_{name}.pfm"
        p.write_bytes(blob)
        (x, re_), (y, oe) = ref.read_pfm(p), ours.read_pfm(p)
        assert x is None and y is None and re_ == oe, (name, re_, oe)
    assert ours.read_pfm(tmp_path / "missing.pfm")[1] == ref.read_pfm(tmp_path / "missing.pfm")[1]


def _quat(rng):
    q = rng.standard_normal(4)
    return (q / np.linalg.norm(q) * rng.uniform(0.5, 2.0)).tolist()


def make_dataset(root, rng, W=24, H=16, C=5, nframes=3, points=True, mutate=None):
    from PIL import Image
    root.mkdir(parents=True, exist_ok=True)
    (root / "maps").mkdir(exist_ok=True)
    doc = {"width": W, "height": H, "num_classes": C, "fx": 21.5, "fy": 20.25, "cx": 11.5, "cy": 7.75, "frames": []}
    if points:
        pts = rng.standard_normal((9, 3))
        cols = rng.integers(0, 256, (9, 3))
        hdr = (f"ply\nformat binary_little_endian 1.0\nelement vertex {len(pts)}\nproperty double x\n"
               "property double y\nproperty double z\nproperty uchar red\nproperty uchar green\n"
               "property uchar blue\nend_header\n").encode()
        body = b"".join(struct.pack("<dddBBB", *p, *c) for p, c in zip(pts.tolist(), cols.tolist()))
        (root / "pts.ply").write_bytes(hdr + body)
        doc["points"] = "pts.ply"
    for i in range(nframes):
        f = {"q_cam_to_world": _quat(rng), "t_cam_to_world": rng.standard_normal(3).tolist()}
        if i == nframes - 1:
            f["split"] = "test"
        if i != 1:  # frame 1 has no rgb
            Image.fromarray(rng.integers(0, 256, (H, W, 3), dtype=np.uint8)).save(root / "maps" / f"{i}_rgb.png")
            f["rgb"] = f"maps/{i}_rgb.png"
        dep = np.abs(rng.standard_normal((H, W))).astype(np.float32)
        (root / "maps" / f"{i}_d.pfm").write_bytes(f"Pf\n{W} {H}\n-1.0\n".encode() + dep[::-1].astype("<f4").tobytes())
        f["depth"] = f"maps/{i}_d.pfm"
        nrm = rng.standard_normal((H, W, 3)).astype(np.float32)
        (root / "maps" / f"{i}_n.pfm").write_bytes(f"PF\n{W} {H}\n-1.0\n".encode() + nrm[::-1].astype("<f4").tobytes())
        f["normal"] = f"maps/{i}_n.pfm"
        Image.fromarray(rng.integers(0, C, (H, W), dtype=np.uint8)).save(root / "maps" / f"{i}_sem.png")
        f["sem"] = f"maps/{i}_sem.png"
        doc["frames"].append(f)
    if mutate:
        mutate(doc, root)
    (root / "cameras.json").write_text(json.dumps(doc, indent=1))
    return doc


def _same_dataset(a, b):
    assert a["dims"] == b["dims"]
    for fa, fb in zip(a["frames"], b["frames"]):
        assert fa["flags"] == fb["flags"]
        assert np.array_equal(fa["cam"], fb["cam"])
        for k in ("rgb", "depth", "normal", "labels"):
            assert np.array_equal(fa[k], fb[k]), k
    assert np.array_equal(a["points"], b["points"]) and np.array_equal(a["colors"], b["colors"])


def test_load_dataset_matches_reference(tmp_path, libs):
    ref, ours = libs
    rng = np.random.default_rng(1)
    make_dataset(tmp_path / "ds", rng)
    r, re_ = ref.dataset(tmp_path / "ds")
    o, oe = ours.dataset(tmp_path / "ds")
    assert re_ is None and oe is None, (re_, oe)
    assert r["dims"] == (24, 16, 5, 3, 9)
    _same_dataset(r, o)


def test_load_dataset_errors_match_reference(tmp_path, libs):
    ref, ours = libs

    def bad_size(doc, root):
        from PIL import Image
        Image.fromarray(np.zeros((5, 5, 3), np.uint8)).save(root / "maps" / "0_rgb.png")

    def bad_label(doc, root):
        from PIL import Image
        Image.fromarray(np.full((16, 24), 9, np.uint8)).save(root / "maps" / "2_sem.png")

    def neg_depth(doc, root):
        (root / "maps" / "0_d.pfm").write_bytes(b"Pf\n24 16\n-1.0\n" + np.full((16, 24), -1, "<f4").tobytes())

    def gray_rgb(doc, root):
        from PIL import Image
        Image.fromarray(np.zeros((16, 24), np.uint8)).save(root / "maps" / "0_rgb.png")

    def rgb_labels(doc, root):
        from PIL import Image
        Image.fromarray(np.zeros((16, 24, 3), np.uint8)).save(root / "maps" / "0_sem.png")

    def one_ch_normal(doc, root):
        (root / "maps" / "0_n.pfm").write_bytes(b"Pf\n24 16\n-1.0\n" + np.zeros((16, 24), "<f4").tobytes())

    cases = {
        "size": bad_size, "label": bad_label, "depth": neg_depth, "rgb_channels": gray_rgb,
        "label_channels": rgb_labels, "normal_channels": one_ch_normal,
        "pose": lambda d, r: d["frames"][0].update(q_cam_to_world=[1, 0, 0]),
        "no_frames": lambda d, r: d.update(frames=[]),
        "missing_png": lambda d, r: d["frames"][0].update(rgb="maps/none.png"),
    }
    for name, mut in cases.items():
        rng = np.random.default_rng(2)
        make_dataset(tmp_path / name, rng, mutate=mut)
        (r, re_), (o, oe) = ref.dataset(tmp_path / name), ours.dataset(tmp_path / name)
        assert r is None and o is None, name
        assert re_ == oe, (name, re_, oe)
    assert ours.dataset(tmp_path / "nowhere")[1] == ref.dataset(tmp_path / "nowhere")[1]
    # malformed JSON: the wrapper text is the reference's; the parser detail is nlohmann's there
    (tmp_path / "js").mkdir()
    (tmp_path / "js" / "cameras.json").write_text('{"width": 4, "height": tru }')
    (_, re_), (_, oe) = ref.dataset(tmp_path / "js"), ours.dataset(tmp_path / "js")
    prefix = f"load_dataset: {tmp_path / 'js' / 'cameras.json'}: [json.exception.parse_error.101] parse error at line 1"
    assert re_.startswith(prefix) and oe.startswith(prefix), (re_, oe)


def test_save_dataset_roundtrip_matches_reference(tmp_path, libs):
    ref, ours = libs
    rng = np.random.default_rng(4)
    make_dataset(tmp_path / "src", rng)
    ref.resave(tmp_path / "src", tmp_path / "by_ref")
    ours.resave(tmp_path / "src", tmp_path / "by_ours")
    jr = json.loads((tmp_path / "by_ref" / "cameras.json").read_text())
    jo = json.loads((tmp_path / "by_ours" / "cameras.json").read_text())
    assert jr == jo  # same keys, same numbers (shortest round-trip text on both sides)
    for f in jr["frames"]:
        for k in ("depth", "normal"):
            assert (tmp_path / "by_ref" / f[k]).read_bytes() == (tmp_path / "by_ours" / f[k]).read_bytes()
        for k in ("rgb", "sem"):
            if k in f:
                assert np.array_equal(ref.read_png(tmp_path / "by_ref" / f[k])[0],
                                      ref.read_png(tmp_path / "by_ours" / f[k])[0])
    assert (tmp_path / "by_ref" / "points.ply").read_bytes() == (tmp_path / "by_ours" / "points.ply").read_bytes()
    # and the saved datasets load back identically through both
    _same_dataset(ref.dataset(tmp_path / "by_ref")[0], ours.dataset(tmp_path / "by_ours")[0])


def test_load_config_matches_reference(tmp_path, libs):
    ref, ours = libs
    good = {
        "defaults": {},
        "full": {"iterations": 17, "lr_position": 1e-3, "lambdas": [1, 0.5, 0, 0.25, 0.125, 0], "prune_interval": 5,
                 "prune_threshold": 0.25, "prune_enabled": False, "prune_keep_small": True, "k_reset": 0.8,
                 "step1": 2, "step2": 6, "lambda_fuse": 0.75, "mask_threshold": 0.4, "sigma_scale": 1.5,
                 "early_stop_transmittance": 1e-3, "background": [0.1, 0.2, 0.3], "sh_degree": 3, "seed": 99,
                 "threads": 4, "deterministic": True, "lr_k": 0.5},
        "float_int": {"iterations": 12.0},
    }
    for name, doc in good.items():
        p = tmp_path / f"{name}.json"
        p.write_text(json.dumps(doc))
        (r, re_), (o, oe) = ref.config(p), ours.config(p)
        assert re_ is None and oe is None, (name, re_, oe)
        assert np.array_equal(r, o), name
    bad = {
        "unknown": {"iterations": 3, "bogus": 1},
        "lambdas": {"lambdas": [1, 2]},
        "background": {"background": 0.5},
        "validate": {"iterations": -4},
        "type": {"iterations": "many"},
    }
    for name, doc in bad.items():
        p = tmp_path / f"bad_{name}.json"
        p.write_text(json.dumps(doc))
        (r, re_), (o, oe) = ref.config(p), ours.config(p)
        assert r is None and o is None, name
        assert re_ == oe, (name, re_, oe)
    assert ours.config(tmp_path / "none.json")[1] == ref.config(tmp_path / "none.json")[1]


def test_python_load_dataset_to_tensors(tmp_path, libs):
    """The Python front end (paper_2510_12174_b200.dataset) returns the
    reference's maps as planar GroundTruth tensors and its cameras."""
    import torch
    from paper_2510_12174_b200 import dataset as D
    ref, _ = libs
    rng = np.random.default_rng(9)
    make_dataset(tmp_path / "py", rng)
    r, _ = ref.dataset(tmp_path / "py")
    ds = D.load_dataset(tmp_path / "py", device="cpu")
    assert (ds.width, ds.height, ds.num_classes, len(ds.frames)) == r["dims"][:4]
    assert ds.train_indices() == [0, 1] and ds.test_indices() == [2]
    for f, fr in zip(ds.frames, r["frames"]):
        assert np.array_equal(np.asarray(f.view.R_cam_to_world).ravel(), fr["cam"][4:13])
        assert (f.truth.rgb is None) == (fr["flags"] & 1 == 0)
        if f.truth.rgb is not None:
            assert torch.equal(f.truth.rgb, torch.from_numpy(fr["rgb"]))
        assert torch.equal(f.truth.depth, torch.from_numpy(fr["depth"]))
        assert torch.equal(f.truth.normal, torch.from_numpy(fr["normal"]))
        assert torch.equal(f.truth.labels, torch.from_numpy(fr["labels"]))
    assert np.array_equal(ds.points, r["points"]) and np.array_equal(ds.point_colors, r["colors"])
    with pytest.raises(RuntimeError, match="cannot open"):
        D.load_dataset(tmp_path / "absent", device="cpu")


@pytest.mark.gpu
def test_dataset_ground_truth_on_device_feeds_losses(tmp_path, libs):
    """load_dataset onto cuda:0: the maps equal the reference's, and a frame
    rendered from the dataset's camera goes through frame_losses /
    frame_metrics with that ground truth."""
    import torch
    import paper_2510_12174_b200 as M
    from paper_2510_12174_b200 import scenes
    ref, _ = libs
    rng = np.random.default_rng(12)
    make_dataset(tmp_path / "g", rng, W=40, H=32, C=3, nframes=2, points=False)
    r, _ = ref.dataset(tmp_path / "g")
    ds = M.load_dataset(tmp_path / "g")
    f = ds.frames[0]
    assert f.truth.rgb.is_cuda and torch.equal(f.truth.rgb.cpu(), torch.from_numpy(r["frames"][0]["rgb"]))
    assert torch.equal(f.truth.labels.cpu(), torch.from_numpy(r["frames"][0]["labels"]))
    s = scenes.make_random_scene(200, 3, 1, seed=1)
    scene = M.Scene.from_numpy(s, dtype=torch.float32)
    # a camera looking at the random scene, with the dataset's intrinsics and size
    view = M.make_camera(f.view.fx, f.view.fy, f.view.cx, f.view.cy, ds.width, ds.height, np.eye(3), np.zeros(3))
    frame = M.rasterize(scene, view, M.RenderConfig(), M.ReplayState())
    M.estimate_normals(frame.depth, frame.transmittance, view, M.NormalConfig(), frame.normals)
    report, pix = M.frame_losses(frame, f.truth, view, M.NormalConfig())
    assert np.isfinite(report.combined) and report.l1 > 0
    met = M.frame_metrics(frame, f.truth)
    assert met["psnr"] is not None and np.isfinite(met["psnr"])
