"""Orientation binning through the 511x511 lookup table (reference gradient.py).

The table is built on the host exactly as the reference builds it
(gradient.py:56-72: numpy arctan2 + scaled floor) -- the table IS the
definition of the binning -- and uploaded once per device.  The per-pixel
work (central differences, channel-max rule, LUT gather) runs in the
``hog_grad_bin`` CUDA kernel.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native, device as D
from .errors import BinCountOutOfRange, ImageTooSmall
from .image import Image

NO_BIN = -1
MIN_BINS = 2
MAX_BINS = 64

_TWO_PI = 2.0 * math.pi


def bin_of(dx: int, dy: int, bins: int) -> int:
    """gradient.py:29-42: bin of one gradient pair; (0,0) -> NO_BIN."""
    if dx == 0 and dy == 0:
        return NO_BIN
    phi = math.atan2(dy, dx)
    if phi < 0.0:
        phi += _TWO_PI
    return min(int(phi * bins / _TWO_PI), bins - 1)


@dataclass(frozen=True)
class OrientationLut:
    """511x511 table of bin indices, indexed by (dx+255, dy+255)."""

    bins: int
    table: np.ndarray

    def lookup(self, dx: int, dy: int) -> int:
        return int(self.table[dx + 255, dy + 255])


def build_lut(bins: int) -> OrientationLut:
    """gradient.py:56-72 (same numpy expression, so the same table)."""
    if not MIN_BINS <= bins <= MAX_BINS:
        raise BinCountOutOfRange(f"bins must be in [{MIN_BINS}, {MAX_BINS}], got {bins}")
    d = np.arange(-255, 256, dtype=np.float64)
    dx, dy = np.meshgrid(d, d, indexing="ij")
    phi = np.arctan2(dy, dx)
    phi[phi < 0.0] += _TWO_PI
    table = np.floor(phi * bins / _TWO_PI).astype(np.int16)
    np.minimum(table, bins - 1, out=table)
    table[255, 255] = NO_BIN
    table.setflags(write=False)
    return OrientationLut(bins=bins, table=table)


class BinMap:
    """Per-pixel bin indices (reference gradient.py:75-92).

    ``cells`` is the (height, width) int16 host array of the reference; when
    the map was produced on the GPU it is copied back lazily on first access,
    and ``device`` holds the int8 device bin map the next stage consumes.
    """

    def __init__(self, bins: int, cells: np.ndarray | None = None, device=None):
        if cells is None and device is None:
            raise ValueError("BinMap needs cells or a device map")
        self.bins = bins
        self._cells = None if cells is None else np.asarray(cells)
        self.device = device  # DevBinmap

    @property
    def cells(self) -> np.ndarray:
        if self._cells is None:
            c = self.device.view()[0].cpu().numpy().astype(np.int16)
            c.setflags(write=False)
            self._cells = c
        return self._cells

    @property
    def height(self) -> int:
        return self.device.h if self._cells is None else self._cells.shape[0]

    @property
    def width(self) -> int:
        return self.device.w if self._cells is None else self._cells.shape[1]

    def to_device(self):
        """int8 device copy (values outside [-1, bins) count nowhere, as in
        integral.py:76 where only cells == n contribute)."""
        if self.device is None:
            c = self._cells
            c8 = np.where((c >= 0) & (c < self.bins), c, NO_BIN).astype(np.int8)
            h, w = c8.shape
            dm = D.alloc_binmap(1, h, w)
            t = D.torch()
            pad = np.full((1, h, dm.pitch), NO_BIN, dtype=np.int8)
            pad[0, :, :w] = c8
            dm.data.copy_(t.from_numpy(pad))
            self.device = dm
        return self.device

    def __eq__(self, other):
        return (isinstance(other, BinMap) and self.bins == other.bins
                and np.array_equal(self.cells, other.cells))

    def __repr__(self):
        return f"BinMap(bins={self.bins}, {self.width}x{self.height})"


def gradient_map(image: Image, lut: OrientationLut) -> BinMap:
    """gradient.py:95-121 on the GPU (``hog_grad_bin``)."""
    if image.width < 3 or image.height < 3:
        raise ImageTooSmall(f"need at least 3x3, got {image.width}x{image.height}")
    frames = D.upload_frames(image.planes)
    return BinMap(lut.bins, device=grad_bin_device(frames, lut))


def grad_bin_device(frames: "D.DevFrames", lut: OrientationLut, out=None, stream=None):
    """Bin maps of device frames (N,C,H,W) -> DevBinmap."""
    lt = D.lut_device(lut.table)
    bm = out or D.alloc_binmap(frames.n, frames.h, frames.w)
    _native.call("hog_grad_bin", D.ptr(frames.data), frames.n, frames.c, frames.h, frames.w,
                 frames.pitch, frames.cstride, frames.fstride, D.ptr(lt), lut.bins,
                 D.ptr(bm.data), bm.pitch, bm.fstride, D.stream_handle(stream))
    return bm
