"""CPU: the C-ABI library builds for sm_100a, loads, and exports every symbol
include/msplat_b200.h declares; host-only entry points behave (no GPU calls)."""
import ctypes as ct
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "msplat_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"MSPLAT_API\s+[\w\s\*]+?\b(msplat_\w+)\s*\(", src)))


def test_header_declares_the_abi():
    syms = declared_symbols()
    for required in ("msplat_rasterize", "msplat_rasterize_backward", "msplat_estimate_normals",
                     "msplat_normals_backward", "msplat_chain_activations", "msplat_fwd_bwd", "msplat_adam_step",
                     "msplat_prune_mask", "msplat_bin_and_sort_host", "msplat_context_create"):
        assert required in syms


def test_library_exports_every_declared_symbol():
    from paper_2510_12174_b200 import _lib
    lib = _lib.lib()  # loads without creating a CUDA context
    for name in declared_symbols():
        assert hasattr(lib, name), name
    nm = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (msplat_\w+)", nm))
    assert set(declared_symbols()) <= exported
    assert all(s.startswith("msplat_") for s in exported)  # nothing else leaks


def test_library_is_sm100a_only():
    from paper_2510_12174_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_\d+a?", out))
    assert arches == {"sm_100a"}, arches


def test_param_layout_and_errors_host_only():
    from paper_2510_12174_b200 import _lib
    lib = _lib.lib()
    off = (ct.c_int64 * 8)()
    assert lib.msplat_param_layout(1000, 50, 2, off) == 0
    assert list(off) == [0, 3000, 7000, 10000, 11000, 12000, 39000, 89000]  # P = 89 at C=50
    assert lib.msplat_param_layout(10, 1, 4, off) == _lib.MSPLAT_ERR_INVALID_ARGUMENT
    assert b"bad layout" in lib.msplat_last_error()
    assert lib.msplat_abi_version() == 1


def test_python_errors_map_to_reference_exception_types():
    from paper_2510_12174_b200 import _lib
    with pytest.raises(ValueError):
        _lib.check(_lib.MSPLAT_ERR_INVALID_ARGUMENT)
    with pytest.raises(_lib.LogicError):
        _lib.check(_lib.MSPLAT_ERR_LOGIC)
    with pytest.raises(RuntimeError):
        _lib.check(_lib.MSPLAT_ERR_RUNTIME)


def test_dropin_exports_the_io_header():
    """include/msplat_io.h (dataset / image / config I/O) is exported by the
    C++ drop-in library."""
    hdr = open(os.path.join(ROOT, "include", "msplat_io.h")).read()
    syms = set(re.findall(r"MSPLAT_IO_API\s+[\w\s\*]+?\b(msplat_\w+)\s*\(", hdr))
    assert "msplat_dataset_load" in syms and "msplat_image_read_png" in syms
    lib = os.path.join(ROOT, "paper_2510_12174_b200", "libmsplat_dropin.so")
    nm = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True).stdout
    assert syms <= set(re.findall(r" T (msplat_\w+)", nm))
