"""The C ABI library loads and exports every entry point include/hogb200.h
declares (CPU only: no CUDA calls are made)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
HEADER = os.path.join(ROOT, "include", "hogb200.h")
LIB = os.path.join(ROOT, "paper_1703_06256_b200", "libhogb200.so")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(hog_[a-z_0-9]+)\s*\(",
                                 text, re.M)))


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for s in ("hog_grad_bin", "hog_integral", "hog_pipeline", "hog_cell_grid",
              "hog_cell_norm", "hog_window_features", "hog_resize_bilinear",
              "hog_scratch_bytes", "hog_last_error", "hog_plane_pitch", "hog_version"):
        assert s in syms


@pytest.mark.skipif(not os.path.exists(LIB), reason="libhogb200.so not built")
def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert missing == []


@pytest.mark.skipif(not os.path.exists(LIB), reason="libhogb200.so not built")
def test_python_binding_matches_header():
    from paper_1703_06256_b200 import _native

    assert set(_native.SIGNATURES) == set(declared_symbols())
    lib = _native.load()
    assert lib.hog_version().decode().startswith("hogb200")
    assert lib.hog_plane_pitch(640) % 8 == 0 and lib.hog_plane_pitch(640) >= 644
    # pure host arithmetic: scratch sizing is deterministic and non-zero
    assert lib.hog_scratch_bytes(512, 480, 640, 8, 4, 8) > 0
    assert lib.hog_scratch_bytes(1, 480, 640, 8, 0, 0) > 0


def test_library_is_sm100a_only():
    if not os.path.exists(LIB):
        pytest.skip("libhogb200.so not built")
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


IO_HEADER = os.path.join(ROOT, "include", "hogio.h")
IO_LIB = os.path.join(ROOT, "paper_1703_06256_b200", "libhogio.so")


@pytest.mark.skipif(not os.path.exists(IO_LIB), reason="libhogio.so not built")
def test_io_library_exports_every_declared_symbol():
    text = open(IO_HEADER).read()
    syms = sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(hogio_[a-z_0-9]+)\s*\(",
                                 text, re.M)))
    assert {"hogio_pnm_decode", "hogio_decode_batch", "hogio_format_descriptors"} <= set(syms)
    lib = ctypes.CDLL(IO_LIB)
    assert [s for s in syms if not hasattr(lib, s)] == []


@pytest.mark.skipif(not os.path.exists(LIB), reason="libhogb200.so not built")
def test_abi_rejects_bad_arguments_before_touching_the_gpu():
    # argument checks are host code: each call returns HOG_EINVAL and sets the
    # error text without launching anything (safe without a GPU)
    from paper_1703_06256_b200 import _native

    lib = _native.load()
    EINVAL = _native.HOG_EINVAL
    # frames too small / bins out of range (gradient.py:62-63, 104-105)
    assert lib.hog_grad_bin(None, 1, 1, 2, 2, 4, 0, 0, None, 8, None, 4, 0, None) == EINVAL
    assert b"3x3" in lib.hog_last_error()
    assert lib.hog_grad_bin(None, 1, 1, 8, 8, 8, 0, 0, None, 65, None, 8, 0, None) == EINVAL
    assert b"bins" in lib.hog_last_error()
    assert lib.hog_grad_bin(None, 1, 2, 8, 8, 8, 0, 0, None, 8, None, 8, 0, None) == EINVAL
    # fused lattice constraints
    rc = lib.hog_pipeline(None, 1, 1, 64, 64, 64, 0, 0, None, 8, None, 64, 0, None, 72, 0, 0,
                          8, 3, 4, 4, 1, None, 0, 0, None, None)
    assert rc == EINVAL
    # 16-bit accumulators: the reference's overflow guard (integral.py:66-72)
    assert lib.hog_integral16(1, 1, 300, 300, 300, 0, 8, 1, 301, 0, 0, None) == EINVAL
    assert b"65535" in lib.hog_last_error()
    # NMS threshold range (detector.py:291-292)
    assert lib.hog_nms(None, None, None, 3, 1.5, None, None, None, 0, None) == EINVAL
    assert lib.hog_nms(None, None, None, 3, float("nan"), None, None, None, 0, None) == EINVAL
    # resize and rectangles
    assert lib.hog_resize_bilinear(None, 1, 1, 8, 8, 8, 0, 0, 0, 4, 1.0, 1.0, None, 4, 0, 0,
                                   None) == EINVAL
    assert lib.hog_rect_histogram(None, 3, 8, 8, 8, None, 1, None, None) == EINVAL
    assert lib.hog_rect_histogram(None, 4, 8, 8, 8, None, 0, None, None) == 0  # empty batch
