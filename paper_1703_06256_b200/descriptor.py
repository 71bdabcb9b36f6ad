"""Window descriptors from cell histograms (reference descriptor.py).

Cell histograms are 4-corner reads of the integral planes (``hog_cell_grid``,
or fused into the plane kernel by ``hog_pipeline``); descriptor assembly,
per-block normalisation and scores run in ``hog_window_features``.  Index
bookkeeping (cell lattice, per-origin index maps) is host numpy, exactly the
reference's expressions (descriptor.py:162-188, 198-206).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native, device as D
from .errors import InvalidGeometry, WindowOutOfBounds
from .gradient import BinMap
from .integral import IntegralStack, Rect, check_rect

NORMALIZATIONS = ("none", "l1", "l2")
_NORM_CODE = {"none": 0, "l1": 1, "l2": 2}

_EPS = 1e-6


@dataclass(frozen=True)
class DescriptorGeometry:
    """Cell/block layout of a detection window (descriptor.py:26-70)."""

    window_w: int
    window_h: int
    cell: int
    block: int = 2
    block_stride: int = 1
    bins: int = 9
    normalization: str = "none"

    def __post_init__(self):
        if self.window_w < 1 or self.window_h < 1 or self.cell < 1:
            raise InvalidGeometry("window and cell sizes must be positive")
        if self.window_w % self.cell or self.window_h % self.cell:
            raise InvalidGeometry(
                f"cell {self.cell} does not divide window {self.window_w}x{self.window_h}")
        if not 1 <= self.block <= min(self.cells_x, self.cells_y):
            raise InvalidGeometry(
                f"block {self.block} does not fit {self.cells_x}x{self.cells_y} cells")
        if self.block_stride < 1:
            raise InvalidGeometry("block_stride must be >= 1")
        if self.bins < 1:
            raise InvalidGeometry("bins must be >= 1")
        if self.normalization not in NORMALIZATIONS:
            raise InvalidGeometry(f"unknown normalization {self.normalization!r}")

    @property
    def cells_x(self) -> int:
        return self.window_w // self.cell

    @property
    def cells_y(self) -> int:
        return self.window_h // self.cell

    @property
    def blocks_x(self) -> int:
        return (self.cells_x - self.block) // self.block_stride + 1

    @property
    def blocks_y(self) -> int:
        return (self.cells_y - self.block) // self.block_stride + 1


def descriptor_length(g: DescriptorGeometry) -> int:
    return g.blocks_x * g.blocks_y * g.block * g.block * g.bins


def eps_term(normalization: str) -> float:
    """descriptor.py:121,123: _EPS for l1, _EPS*_EPS for l2 (computed in Python)."""
    return _EPS if normalization == "l1" else _EPS * _EPS


def naive_histogram(binmap: BinMap, r: Rect) -> np.ndarray:
    """descriptor.py:77-91: the definitional per-pixel count (host reference
    helper of the API; not on the accelerated path)."""
    check_rect(r, binmap.width, binmap.height)
    sub = np.asarray(binmap.cells[r.y0:r.y1, r.x0:r.x1]).ravel()
    sub = sub[sub >= 0]
    if sub.size and int(sub.max()) >= binmap.bins:  # the reference's counts[v] += 1 raises here
        raise IndexError("list index out of range")
    return np.bincount(sub, minlength=binmap.bins).astype(np.int64)


def normalize(values: np.ndarray, scheme: str) -> np.ndarray:
    """descriptor.py:94-104 (single-vector helper of the API)."""
    if scheme == "none":
        return values
    v = np.asarray(values, dtype=np.float64)
    if scheme == "l1":
        return v / (np.abs(v).sum() + _EPS)
    if scheme == "l2":
        return v / np.sqrt((v * v).sum() + _EPS * _EPS)
    raise InvalidGeometry(f"unknown normalization {scheme!r}")


# --- device stages ---------------------------------------------------------

def cell_grid_device(planes: "D.DevPlanes", cell_xs, cell_ys, cell: int, stream=None):
    """descriptor.py:176-185: (N, ncy, ncx, bins) int32 on the device."""
    t = D.torch()
    if isinstance(planes, D.DevPlanes16):  # 16-bit stack: cells as a rectangle batch
        from .integral import rect_histograms_device

        xs, ys = np.asarray(cell_xs, dtype=np.int64), np.asarray(cell_ys, dtype=np.int64)
        X0, Y0 = np.meshgrid(xs, ys)
        rects = np.stack([X0, Y0, X0 + cell, Y0 + cell], -1).reshape(-1, 4)
        h = rect_histograms_device(planes, rects, stream)
        return h.to(t.int32).reshape(1, len(ys), len(xs), planes.bins)
    cx = t.as_tensor(np.asarray(cell_xs, dtype=np.int32), device=planes.base.device)
    cy = t.as_tensor(np.asarray(cell_ys, dtype=np.int32), device=planes.base.device)
    grid = t.empty((planes.n, len(cy), len(cx), planes.bins), dtype=t.int32,
                   device=planes.base.device)
    _native.call("hog_cell_grid", planes.ptr, planes.n, planes.h, planes.w, planes.bins,
                 planes.pitch, planes.nstride, planes.fstride, D.ptr(cx), len(cx), D.ptr(cy),
                 len(cy), cell, D.ptr(grid), D.stream_handle(stream))
    return grid


def window_features_device(grid, g: DescriptorGeometry, row_idx, col_idx, weights=None,
                           bias=0.0, want_scores=False, want_desc=False, stream=None):
    """descriptor.py:107-124 + detector.py:148-150 for every (iy, ix) pair of
    the index maps: returns (scores (N,noy,nox) f64 | None, desc (N,noy,nox,D) f64 | None)."""
    t = D.torch()
    dev = grid.device
    n, ncy, ncx, bins = grid.shape
    ri = t.as_tensor(np.ascontiguousarray(row_idx, dtype=np.int32), device=dev)
    ci = t.as_tensor(np.ascontiguousarray(col_idx, dtype=np.int32), device=dev)
    noy, nox = ri.shape[0], ci.shape[0]
    # the descriptor carries the GRID's bins (the stack's), as _assemble_blocks
    # does (descriptor.py:107-124); the kernel strides by them too
    Dn = g.blocks_x * g.blocks_y * g.block * g.block * bins
    scores = desc = wt = None
    if want_scores:
        wt = np.ascontiguousarray(weights, dtype=np.float64)
        if wt.ndim != 1 or len(wt) != Dn:  # np.dot(w, desc) raises here (detector.py:148-150)
            raise ValueError(f"shapes ({len(wt)},) and ({Dn},) not aligned: weights length "
                             f"{len(wt)} != descriptor length {Dn} ({bins} bins)")
        wt = t.as_tensor(wt, device=dev)
        scores = t.empty((n, noy, nox), dtype=t.float64, device=dev)
    if want_desc:
        desc = t.empty((n, noy, nox, Dn), dtype=t.float64, device=dev)
    if noy == 0 or nox == 0:
        return scores, desc
    _native.call("hog_window_features", D.ptr(grid), n, ncy, ncx, bins, D.ptr(ri), noy,
                 D.ptr(ci), nox, g.cells_x, g.cells_y, g.block, g.block_stride,
                 _NORM_CODE[g.normalization], eps_term(g.normalization),
                 D.ptr(wt) if wt is not None else None, float(bias),
                 D.ptr(scores) if scores is not None else None,
                 D.ptr(desc) if desc is not None else None, D.stream_handle(stream))
    return scores, desc


def _as_reference_dtype(desc_f64: np.ndarray, g: DescriptorGeometry) -> np.ndarray:
    # descriptor.py:115-118: unnormalised descriptors are the int64 counts
    return desc_f64.astype(np.int64) if g.normalization == "none" else desc_f64


# --- drop-in API -----------------------------------------------------------

def window_descriptor(stack: IntegralStack, origin, g: DescriptorGeometry) -> np.ndarray:
    """descriptor.py:127-150: descriptor of one window, straight from the planes."""
    ox, oy = origin
    if g.bins != stack.bins:
        raise InvalidGeometry(f"geometry bins {g.bins} != stack bins {stack.bins}")
    if not (0 <= ox and 0 <= oy and ox + g.window_w <= stack.width
            and oy + g.window_h <= stack.height):
        raise WindowOutOfBounds(
            f"window {g.window_w}x{g.window_h} at ({ox}, {oy}) exceeds "
            f"{stack.width}x{stack.height}")
    xs = ox + g.cell * np.arange(g.cells_x)
    ys = oy + g.cell * np.arange(g.cells_y)
    grid = cell_grid_device(_planes_of(stack), xs, ys, g.cell)
    _, desc = window_features_device(grid, g, np.arange(g.cells_y)[None],
                                     np.arange(g.cells_x)[None], want_desc=True)
    return _as_reference_dtype(desc[0, 0, 0].cpu().numpy(), g)


def _planes_of(stack: IntegralStack):
    return stack.device_planes()


def cell_lattice(origin_xs, origin_ys, g: DescriptorGeometry):
    """descriptor.py:162-188: cell origins and per-window-origin index maps."""
    offs_x = g.cell * np.arange(g.cells_x)
    offs_y = g.cell * np.arange(g.cells_y)
    cell_xs = np.unique(np.asarray(origin_xs)[:, None] + offs_x[None, :])
    cell_ys = np.unique(np.asarray(origin_ys)[:, None] + offs_y[None, :])
    col_idx = np.searchsorted(cell_xs, np.asarray(origin_xs)[:, None] + offs_x[None, :])
    row_idx = np.searchsorted(cell_ys, np.asarray(origin_ys)[:, None] + offs_y[None, :])
    return cell_xs, cell_ys, col_idx, row_idx


class CellHistogramCache:
    """Write-once table of cell histograms for a whole scan (descriptor.py:153-195).

    ``grid`` is computed on the device in one launch; ``device_grid`` keeps it
    resident for the window stage.
    """

    # descriptors are materialised on the device a block of window rows at a
    # time (about this many values per block) and kept on the host, so a
    # reference-style per-window loop (detector.py:140-154) costs one launch
    # and one copy per block, not per window
    BLOCK_VALUES = 1 << 22

    def __init__(self, stack: IntegralStack, g: DescriptorGeometry, origin_xs, origin_ys):
        self.geometry = g
        self.bins = stack.bins  # the grid's bins are the stack's (descriptor.py:176-185)
        cell_xs, cell_ys, self.col_idx, self.row_idx = cell_lattice(origin_xs, origin_ys, g)
        self.cell_xs, self.cell_ys = cell_xs, cell_ys
        if len(cell_xs) and len(cell_ys):
            self.device_grid = cell_grid_device(_planes_of(stack), cell_xs, cell_ys, g.cell)
        else:
            self.device_grid = None
        self._grid = None
        self._block = None  # (first window row, last + 1, descriptors (rows, nox, D))

    @property
    def grid(self) -> np.ndarray:
        if self._grid is None:
            if self.device_grid is None:
                gr = np.zeros((len(self.cell_ys), len(self.cell_xs), self.bins), np.int64)
            else:
                gr = self.device_grid[0].cpu().numpy().astype(np.int64)
            gr.setflags(write=False)
            self._grid = gr
        return self._grid

    def window_cells(self, origin_ix: int, origin_iy: int) -> np.ndarray:
        return self.grid[np.ix_(self.row_idx[origin_iy], self.col_idx[origin_ix])]

    def rows_per_block(self) -> int:
        g = self.geometry
        per_row = max(1, len(self.col_idx) * g.blocks_x * g.blocks_y * g.block * g.block * self.bins)
        return max(1, self.BLOCK_VALUES // per_row)

    def descriptor(self, origin_ix: int, origin_iy: int) -> np.ndarray:
        """descriptor.py:194-195.  The window row's block of descriptors is
        assembled on the device on first use and served from the host copy."""
        iy = range(len(self.row_idx))[origin_iy]  # IndexError / negative index as numpy
        ix = range(len(self.col_idx))[origin_ix]
        blk = self._block
        if blk is None or not blk[0] <= iy < blk[1]:
            r0 = iy - iy % self.rows_per_block()
            r1 = min(len(self.row_idx), r0 + self.rows_per_block())
            blk = self._block = (r0, r1, self.descriptors(slice(r0, r1)))
        return blk[2][iy - blk[0], ix].copy()

    def descriptors(self, iy_range=None):
        """All descriptors of window rows iy_range as (rows, nox, D), one launch."""
        rows = self.row_idx if iy_range is None else self.row_idx[iy_range]
        _, desc = window_features_device(self.device_grid, self.geometry, rows, self.col_idx,
                                         want_desc=True)
        return _as_reference_dtype(desc[0].cpu().numpy(), self.geometry)


def window_origins(width: int, height: int, g: DescriptorGeometry, stride: int):
    """descriptor.py:198-206: row-major grid of window origins."""
    if stride < 1:
        raise ValueError(f"stride must be >= 1, got {stride}")
    oxs = np.arange(0, width - g.window_w + 1, stride)
    oys = np.arange(0, height - g.window_h + 1, stride)
    return oxs, oys


def scan_descriptors(stack: IntegralStack, g: DescriptorGeometry, stride: int):
    """descriptor.py:209-223: (x, y, descriptor) for every window, row-major.
    Descriptors are materialised on the device a block of window rows at a time."""
    if g.window_w > stack.width or g.window_h > stack.height:
        raise WindowOutOfBounds(
            f"window {g.window_w}x{g.window_h} exceeds {stack.width}x{stack.height}")
    oxs, oys = window_origins(stack.width, stack.height, g, stride)
    cache = CellHistogramCache(stack, g, oxs, oys)
    chunk = cache.rows_per_block()
    for r0 in range(0, len(oys), chunk):
        block = cache.descriptors(slice(r0, min(r0 + chunk, len(oys))))
        for j in range(block.shape[0]):
            oy = int(oys[r0 + j])
            for ix, ox in enumerate(oxs):
                yield int(ox), oy, block[j, ix]
