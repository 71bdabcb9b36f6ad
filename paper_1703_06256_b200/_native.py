"""ctypes binding of libhogb200.so (the C ABI in include/hogb200.h).

There is deliberately no fallback: if the library or a CUDA device is
missing, every hot-path call raises ``NativeUnavailable``.
"""
from __future__ import annotations

import ctypes
import os

from .errors import FastHogError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HOGB200_LIB") or os.path.join(_HERE, "libhogb200.so")

HOG_OK, HOG_EINVAL, HOG_ECUDA, HOG_ERANGE = 0, 1, 2, 3
STAGE_BIN, STAGE_SCAN, STAGE_PLANES, STAGE_ALL, STAGE_GRID_U8 = 1, 2, 4, 7, 8

# (name, restype, argtypes) -- must match include/hogb200.h
_P, _I, _L, _D, _SZ = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_size_t
SIGNATURES = {
    "hog_version": (ctypes.c_char_p, []),
    "hog_last_error": (ctypes.c_char_p, []),
    "hog_last_pipeline_launches": (_I, []),
    "hog_plane_pitch": (_L, [_I]),
    "hog_lut_proof": (_I, [_P, _I, _P, _P]),
    "hog_lut_forget": (None, [_P]),
    "hog_grad_bin": (_I, [_P, _I, _I, _I, _I, _L, _L, _L, _P, _I, _P, _L, _L, _P]),
    "hog_scratch_bytes": (_SZ, [_I, _I, _I, _I, _I, _I]),
    "hog_set_band_rows": (None, [_I]),
    "hog_get_band_rows": (_I, [_I, _I, _I, _I, _I, _I]),
    "hog_integral": (_I, [_P, _I, _I, _I, _L, _L, _I, _P, _L, _L, _L, _P, _SZ, _P]),
    "hog_pipeline": (_I, [_P, _I, _I, _I, _I, _L, _L, _L, _P, _I, _P, _L, _L,
                          _P, _L, _L, _L, _I, _I, _I, _I, _P, _P, _SZ, _I, _P, _P]),
    "hog_pipeline_slab": (_I, [_P, _I, _I, _I, _I, _L, _L, _L, _P, _I, _P, _L, _L,
                               _P, _L, _L, _L, _I, _I, _I, _I, _P, _P, _SZ, _I, _I, _I, _P, _L, _P]),
    "hog_column_counts": (_I, [_P, _I, _I, _I, _L, _L, _I, _P, _P]),
    "hog_cell_grid": (_I, [_P, _I, _I, _I, _I, _L, _L, _L, _P, _I, _P, _I, _I, _P, _P]),
    "hog_cell_norm": (_I, [_P, _I, _I, _I, _I, _D, _P, _P]),
    "hog_window_features": (_I, [_P, _I, _I, _I, _I, _P, _I, _P, _I, _I, _I, _I, _I, _I, _D,
                                 _P, _D, _P, _P, _P]),
    "hog_scores_lattice": (_I, [_P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _I, _P, _D, _P, _P]),
    "hog_scores_lattice_u8": (_I, [_P, _I, _I, _I, _I, _I, _I, _I, _I, _I, _P, _D, _P, _P]),
    "hog_scores_i8_frag_bytes": (_SZ, [_I]),
    "hog_scores_i8_prepare": (_I, [_P, _I, _I, _I, _P, _P, _P]),
    "hog_scores_lattice_i8": (_I, [_P, _I, _I, _I, _I, _I, _I, _I, _I, _P, _I, _D, _D, _P, _P]),
    "hog_resize_bilinear": (_I, [_P, _I, _I, _I, _I, _L, _L, _L, _I, _I, _D, _D,
                                 _P, _L, _L, _L, _P]),
    "hog_integral16": (_I, [_P, _I, _I, _I, _L, _L, _I, _P, _L, _L, _L, _P]),
    "hog_rect_histogram": (_I, [_P, _I, _L, _L, _I, _P, _I, _P, _P]),
    "hog_detect_scratch_bytes": (_SZ, [_I, _L]),
    "hog_detect": (_I, [_P, _I, _I, _I, _D, _P, _P, _D, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P,
                        _SZ, _P]),
    "hog_nms_scratch_bytes": (_SZ, [_I]),
    "hog_nms": (_I, [_P, _P, _P, _I, _D, _P, _P, _P, _SZ, _P]),
    "hog_nms_f64": (_I, [_P, _P, _P, _I, _D, _P, _P, _P, _SZ, _P]),
    "hog_window_l2": (_I, [_P, _I, _I, _I, _I, _I, _P, _I, _P, _I, _I, _I, _I, _D, _P, _P, _P]),
}


class NativeUnavailable(RuntimeError):
    """libhogb200.so or a CUDA device is missing: there is no CPU fallback."""


class NativeError(FastHogError):
    """A libhogb200 call rejected its arguments or failed to launch."""


_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeUnavailable(
            f"{LIB_PATH} is missing; build it with `make` (or __graft_entry__.build()). "
            "The LUT-HOG path has no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def call(name: str, *args) -> None:
    rc = getattr(load(), name)(*args)
    if rc != HOG_OK:
        msg = load().hog_last_error().decode(errors="replace")
        raise NativeError(f"{name} failed ({rc}): {msg}")


def version() -> str:
    return load().hog_version().decode()
