"""Wire formats around the hot path: PNM ingestion and
the descriptor text dump, on native host code (libhogio.so, include/hogio.h).

* ``decode_pnm`` / ``read_image`` mirror image_io.py:90-158. They accept the same
  inputs and raise the same typed errors. ``read_batch`` decodes a list of
  same-shape files on all host threads straight into one pinned host buffer.
  That buffer is the source of the batch's H2D copy, so no intermediate
  numpy array is made.
* ``encode_*`` / ``write_image`` are the reference's byte layouts (image_io.py:125-158).
* ``format_descriptors`` / ``extract`` produce `fasthog extract`'s lines
  (cli.py:124-143): "x y v0 v1 ...". Integers are printed for unnormalised
  descriptors and ``format(v, ".9g")`` otherwise. The native formatter writes
  the whole scan's text in one call.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import MaxvalNot255, NonNumericToken, TruncatedData, UnsupportedMagic
from .image import Image

_HERE = os.path.dirname(os.path.abspath(__file__))
IO_LIB_PATH = os.environ.get("HOGIO_LIB") or os.path.join(_HERE, "libhogio.so")

_ERRORS = {1: UnsupportedMagic, 2: MaxvalNot255, 3: TruncatedData, 4: NonNumericToken,
           5: ValueError, 6: OSError, 7: ValueError}
_lib = None


def _io():
    global _lib
    if _lib is None:
        if not os.path.exists(IO_LIB_PATH):
            from ._native import NativeUnavailable

            raise NativeUnavailable(f"{IO_LIB_PATH} is missing; build it with `make`")
        lib = ctypes.CDLL(IO_LIB_PATH)
        P, I, L, SZ = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_size_t
        IP = ctypes.POINTER(ctypes.c_int)
        lib.hogio_last_error.restype = ctypes.c_char_p
        lib.hogio_pnm_header.argtypes = [ctypes.c_char_p, SZ, IP, IP, IP]
        lib.hogio_pnm_decode.argtypes = [ctypes.c_char_p, SZ, P, L, L]
        lib.hogio_decode_batch.argtypes = [ctypes.POINTER(ctypes.c_char_p), I, I, I, I, P, L, L, L,
                                           I, IP]
        lib.hogio_format_descriptors.argtypes = [P, P, P, L, I, I, P, L]
        lib.hogio_format_descriptors.restype = L
        _lib = lib
    return _lib


def _raise(rc: int):
    msg = _io().hogio_last_error().decode(errors="replace")
    raise _ERRORS.get(rc, ValueError)(msg)


def pnm_shape(data: bytes) -> tuple[int, int, int]:
    """(channels, height, width) from a PNM header."""
    c, h, w = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    rc = _io().hogio_pnm_header(data, len(data), ctypes.byref(c), ctypes.byref(h), ctypes.byref(w))
    if rc:
        _raise(rc)
    return c.value, h.value, w.value


def decode_pnm(data: bytes) -> Image:
    """image_io.py:90-122: P2/P3/P5/P6 with maxval 255 -> planar Image."""
    data = bytes(data)
    c, h, w = pnm_shape(data)
    out = np.empty((c, h, w), dtype=np.uint8)
    rc = _io().hogio_pnm_decode(data, len(data), out.ctypes.data, w, h * w)
    if rc:
        _raise(rc)
    return Image(out)


def read_image(path: str) -> Image:
    with open(path, "rb") as f:
        return decode_pnm(f.read())


def read_batch(paths, pinned: bool = True, threads: int | None = None):
    """Decode same-shape PNM files into one (N, C, H, W) uint8 host tensor
    (page-locked when `pinned`, ready for a non_blocking H2D copy), using all
    host threads.  Raises the first file's typed error."""
    import torch

    paths = [os.fspath(p) for p in paths]
    if not paths:
        raise ValueError("no files")
    with open(paths[0], "rb") as f:
        c, h, w = pnm_shape(f.read(4096))
    n = len(paths)
    out = torch.empty((n, c, h, w), dtype=torch.uint8)
    if pinned and torch.cuda.is_available():
        out = out.pin_memory()
    arr = (ctypes.c_char_p * n)(*[p.encode() for p in paths])
    status = (ctypes.c_int * n)()
    rc = _io().hogio_decode_batch(arr, n, c, h, w, out.data_ptr(), c * h * w, w, h * w,
                                  threads or os.cpu_count() or 1, status)
    if rc:
        _raise(rc)
    return out


def encode_pgm(plane: np.ndarray) -> bytes:
    """image_io.py:125-131."""
    plane = np.asarray(plane, dtype=np.uint8)
    if plane.ndim != 2 or plane.size == 0:
        raise ValueError("plane must be a nonempty 2-D array")
    h, w = plane.shape
    return b"P5\n%d %d\n255\n" % (w, h) + plane.tobytes()


def encode_ppm(planes: np.ndarray) -> bytes:
    """image_io.py:134-141."""
    planes = np.asarray(planes, dtype=np.uint8)
    if planes.ndim != 3 or planes.shape[0] != 3 or planes.size == 0:
        raise ValueError("planes must be a nonempty (3, height, width) array")
    _, h, w = planes.shape
    return b"P6\n%d %d\n255\n" % (w, h) + np.ascontiguousarray(planes.transpose(1, 2, 0)).tobytes()


def encode_image(image: Image) -> bytes:
    """image_io.py:144-148."""
    return encode_pgm(image.planes[0]) if image.channels == 1 else encode_ppm(image.planes)


def write_image(path: str, image: Image) -> None:
    with open(path, "wb") as f:
        f.write(encode_image(image))


def format_descriptors(xs, ys, values, normalization: str) -> bytes:
    """cli.py:124-143: the extract lines for rows of (x, y, descriptor)."""
    xs = np.ascontiguousarray(xs, dtype=np.int32)
    ys = np.ascontiguousarray(ys, dtype=np.int32)
    v = np.ascontiguousarray(values, dtype=np.float64)
    rows, dim = (v.shape[0], v.shape[1]) if v.ndim == 2 else (0, 0)
    lib = _io()
    as_int = 1 if normalization == "none" else 0
    need = lib.hogio_format_descriptors(xs.ctypes.data, ys.ctypes.data, v.ctypes.data, rows, dim,
                                        as_int, None, 0)
    buf = ctypes.create_string_buffer(max(int(need), 1))
    lib.hogio_format_descriptors(xs.ctypes.data, ys.ctypes.data, v.ctypes.data, rows, dim, as_int,
                                 buf, need)
    return buf.raw[:need]


def extract(image: Image, g, stride: int, out) -> int:
    """cli.py:130-143 (cmd_extract) on the device path: binning, planes and
    descriptors on the GPU, the text written a block of window rows at a time
    through the native formatter.  `out` is a binary file object; returns the
    number of lines."""
    from .descriptor import CellHistogramCache, window_origins
    from .errors import WindowOutOfBounds
    from .gradient import build_lut, gradient_map
    from .integral import build_integral_stack

    stack = build_integral_stack(gradient_map(image, build_lut(g.bins)))
    if g.window_w > stack.width or g.window_h > stack.height:
        raise WindowOutOfBounds(
            f"window {g.window_w}x{g.window_h} exceeds {stack.width}x{stack.height}")
    oxs, oys = window_origins(stack.width, stack.height, g, stride)
    cache = CellHistogramCache(stack, g, oxs, oys)
    lines = 0
    per_row = max(1, len(oxs) * g.bins * g.cells_x * g.cells_y)
    chunk = max(1, (1 << 22) // per_row)
    for r0 in range(0, len(oys), chunk):
        r1 = min(r0 + chunk, len(oys))
        block = cache.descriptors(slice(r0, r1))  # (rows, nox, D)
        xs = np.tile(oxs, r1 - r0)
        ys = np.repeat(oys[r0:r1], len(oxs))
        out.write(format_descriptors(xs, ys, block.reshape(len(xs), -1), g.normalization))
        lines += len(xs)
    return lines
