"""Device buffers for the LUT-HOG path (torch tensors used as plain HBM
allocations; the compute is libhogb200.so).

HBM layouts (include/hogb200.h):
  frames  uint8 (N, C, H, Wp)        Wp = round_up(W, 4)   (pitched rows)
  binmap  int8  (N, H, Wb)           Wb = round_up(W, 8); -1 = NO_BIN
  planes  int32 (N, H+1, bins, Pp)   Pp = round_up(W, 8) + 8 (row-major: the rows
                                     of all bins for one plane row are adjacent;
                                     HOGB200_PLANE_LAYOUT=bin gives (N, bins, H+1, Pp));
                                     the view is the logical (N, bins, H+1, W+1) and
                                     starts 7 elements into its allocation so
                                     plane column 1 of every row is 32-byte
                                     aligned: each lane's 8 columns are one
                                     256-bit store, and column 0 plus the
                                     previous row's padding form one sector.
  grid    int32 (N, ncy, ncx, bins)
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native


def torch():
    import torch as _t

    return _t


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise _native.NativeUnavailable(
            "no CUDA device: the LUT-HOG path runs only on the GPU (no CPU fallback)")
    _native.load()
    return t


def round_up(v: int, m: int) -> int:
    return (v + m - 1) // m * m


def stream_handle(stream=None) -> int:
    t = torch()
    s = stream if stream is not None else t.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(x) -> int:
    return int(x.data_ptr())


@dataclass
class DevFrames:
    """Pitched uint8 frames (N, C, H, pitch) on the device."""

    data: object
    n: int
    c: int
    h: int
    w: int

    @property
    def pitch(self) -> int:
        return self.data.shape[-1]

    @property
    def cstride(self) -> int:
        return self.h * self.pitch

    @property
    def fstride(self) -> int:
        return self.c * self.h * self.pitch


def alloc_frames(n, c, h, w, device=None) -> DevFrames:
    t = require_cuda()
    data = t.empty((n, c, h, round_up(w, 4)), dtype=t.uint8, device=device or "cuda")
    return DevFrames(data, n, c, h, w)


def upload_frames(frames: np.ndarray, device=None, out: DevFrames | None = None) -> DevFrames:
    """(N,C,H,W) or (C,H,W) uint8 host array -> pitched device frames."""
    t = require_cuda()
    a = np.asarray(frames, dtype=np.uint8)
    if a.ndim == 3:
        a = a[None]
    n, c, h, w = a.shape
    df = out or alloc_frames(n, c, h, w, device)
    if df.pitch == w:
        df.data.copy_(t.from_numpy(np.ascontiguousarray(a)), non_blocking=False)
    else:
        df.data[..., :w].copy_(t.from_numpy(np.ascontiguousarray(a)))
    return df


@dataclass
class DevBinmap:
    data: object  # int8 (N, H, pitch)
    n: int
    h: int
    w: int

    @property
    def pitch(self) -> int:
        return self.data.shape[-1]

    @property
    def fstride(self) -> int:
        return self.h * self.pitch

    def view(self):
        return self.data[..., : self.w]


def alloc_binmap(n, h, w, device=None) -> DevBinmap:
    t = require_cuda()
    return DevBinmap(t.empty((n, h, round_up(w, 8)), dtype=t.int8, device=device or "cuda"),
                     n, h, w)


@dataclass
class DevPlanes:
    """int32 planes of n frames: logical (n, bins, h+1, w+1), rows padded to
    `rowlen` = hog_plane_pitch(w) elements.  Two HBM layouts, both addressed by
    the C ABI through (pitch = row stride, nstride = bin stride, fstride =
    frame stride) in elements:
      bin-major   [n][bins][h+1][rowlen]   (the reference's (bins, H+1, W+1) order)
      row-major   [n][h+1][bins][rowlen]   (a plane row of every bin is contiguous)
    """

    base: object  # int32 allocation
    n: int
    bins: int
    h: int
    w: int
    rowlen: int
    offset: int = 7
    row_major: bool = False

    @property
    def pitch(self) -> int:  # elements between plane rows Y and Y+1 of one bin
        return self.bins * self.rowlen if self.row_major else self.rowlen

    @property
    def nstride(self) -> int:  # elements between bins
        return self.rowlen if self.row_major else (self.h + 1) * self.rowlen

    @property
    def fstride(self) -> int:
        return self.bins * (self.h + 1) * self.rowlen

    @property
    def ptr(self) -> int:
        return ptr(self.base) + 4 * self.offset

    def view(self):
        """(N, bins, H+1, W+1) int32 strided view of the logical planes."""
        flat = self.base[self.offset: self.offset + self.n * self.fstride]
        if self.row_major:
            v = flat.view(self.n, self.h + 1, self.bins, self.rowlen).permute(0, 2, 1, 3)
        else:
            v = flat.view(self.n, self.bins, self.h + 1, self.rowlen)
        return v[..., : self.w + 1]


def plane_layout_row_major() -> bool:
    """HBM layout of new plane buffers: row-major by default (a plane row of every
    bin is one contiguous run, so the plane kernel's row writes stay in fewer DRAM
    pages: measured on B200, c2 1.123 -> 1.110 ms, c4 2.149 -> 2.122 ms, the 64-frame
    shard 0.181 -> 0.177 ms, c1/c3/c5 unchanged; profiles/r2/plane_layout_ab.md).
    HOGB200_PLANE_LAYOUT=bin selects the reference's bin-major order."""
    import os

    return os.environ.get("HOGB200_PLANE_LAYOUT", "row") != "bin"


def alloc_planes(n, bins, h, w, device=None, row_major=None) -> DevPlanes:
    t = require_cuda()
    rowlen = int(_native.load().hog_plane_pitch(w))
    total = n * bins * (h + 1) * rowlen + 16
    base = t.empty(total, dtype=t.int32, device=device or "cuda")
    rm = plane_layout_row_major() if row_major is None else bool(row_major)
    return DevPlanes(base, n, bins, h, w, rowlen, row_major=rm)


@dataclass
class DevPlanes16:
    """uint16 planes (N, bins, H+1, pitch), pitch = round_up(W+1, 8) (acc_width=16)."""

    data: object
    n: int
    bins: int
    h: int
    w: int

    @property
    def pitch(self) -> int:
        return self.data.shape[-1]

    @property
    def nstride(self) -> int:
        return (self.h + 1) * self.pitch

    @property
    def fstride(self) -> int:
        return self.bins * self.nstride

    @property
    def ptr(self) -> int:
        return ptr(self.data)

    def view(self):
        return self.data[..., : self.w + 1]


def alloc_planes16(n, bins, h, w, device=None) -> DevPlanes16:
    t = require_cuda()
    data = t.empty((n, bins, h + 1, round_up(w + 1, 8)), dtype=t.uint16, device=device or "cuda")
    return DevPlanes16(data, n, bins, h, w)


def upload_planes(planes: np.ndarray, device=None):
    """A host (bins, H+1, W+1) uint32/uint16 stack -> device planes of the same width."""
    t = require_cuda()
    a = np.asarray(planes)
    bins, h1, w1 = a.shape
    if a.dtype == np.uint16:
        out = alloc_planes16(1, bins, h1 - 1, w1 - 1, device)
    else:
        out = alloc_planes(1, bins, h1 - 1, w1 - 1, device)
        a = a.astype(np.uint32).view(np.int32)
    out.view()[0].copy_(t.from_numpy(np.ascontiguousarray(a)))
    return out


def scratch(n, h, w, bins, stride=0, cell=0, device=None):
    t = require_cuda()
    nbytes = int(_native.load().hog_scratch_bytes(n, h, w, bins, stride, cell))
    return t.empty(max(nbytes, 256), dtype=t.uint8, device=device or "cuda"), nbytes


_LUT_CACHE: dict = {}


def lut_device(table: np.ndarray, device=None):
    """Upload a (511,511) int16 table as uint8 (NO_BIN -1 -> 0xFF), cached by content."""
    t = require_cuda()
    tab = np.asarray(table)
    dev = t.device(device or "cuda")
    if dev.index is None:
        dev = t.device("cuda", t.cuda.current_device())
    key = (dev.index, tab.shape, tab.tobytes()[:64], hash(tab.tobytes()))
    hit = _LUT_CACHE.get(key)
    if hit is None:
        if tab.shape != (511, 511):
            raise ValueError("orientation table must be 511x511")
        b = np.ascontiguousarray(tab.astype(np.int16)).astype(np.int8).view(np.uint8)
        hit = t.from_numpy(b.copy()).to(dev)
        _LUT_CACHE[key] = hit
    return hit
