"""CPU oracle for the LUT-HOG hot path -- TEST INFRASTRUCTURE ONLY.

Python face of ``hog_oracle.c`` (ctypes).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl
reference`` legs may import this module; the product package
(``paper_1703_06256_b200``) never does, and it fails loudly instead of
falling back here when its CUDA library is missing.

Every function restates one reference function (``/root/reference/pkg/src/
fasthog/<file>:<line>``).  The restatement is pinned against vectors the
reference itself produced (``tests/golden/``, made by
``tests/golden/make_golden.py``), so it is a checker, not a guess.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libhog_oracle.so")
_lib = None

NO_BIN = -1
EPS = 1e-6  # descriptor.py:23


def build() -> str:
    """Compile the C restatement (oracle/Makefile) if it is missing or stale."""
    src = os.path.join(_HERE, "hog_oracle.c")
    if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i, d = ctypes.c_int, ctypes.c_double
        L.oracle_build_lut.argtypes = [i, P]
        L.oracle_gradient_map.argtypes = [P, i, i, i, P, P]
        L.oracle_gradient_map.restype = i
        L.oracle_integral.argtypes = [P, i, i, i, P]
        L.oracle_cell_grid.argtypes = [P, i, i, i, P, i, P, i, i, P]
        L.oracle_window_descriptor.argtypes = [P, i, i, P, P, i, i, i, i, i, d, P]
        L.oracle_window_descriptor.restype = i
        L.oracle_dot_bias.argtypes = [P, P, i, d]
        L.oracle_dot_bias.restype = d
        L.oracle_resize_bilinear.argtypes = [P, i, i, i, i, i, P]
        L.oracle_run_batch.argtypes = [P, i, i, i, i, P, i, i, i, i, i, i, P, d, d, i, P, P]
        L.oracle_run_batch.restype = ctypes.c_uint64
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# --- gradient.py -----------------------------------------------------------

def build_lut(bins: int) -> np.ndarray:
    """gradient.py:56-72 -> (511, 511) int16 indexed [dx+255, dy+255]."""
    t = np.empty((511, 511), dtype=np.int16)
    lib().oracle_build_lut(bins, _p(t))
    return t


def gradient_map(planes: np.ndarray, lut: np.ndarray) -> np.ndarray:
    """gradient.py:95-121: (C,H,W) u8 -> (H,W) int16 bin map."""
    planes = np.ascontiguousarray(planes, dtype=np.uint8)
    C, H, W = planes.shape
    out = np.empty((H, W), dtype=np.int16)
    lut = np.ascontiguousarray(lut, dtype=np.int16)
    if lib().oracle_gradient_map(_p(planes), C, H, W, _p(lut), _p(out)) != 0:
        raise ValueError("image smaller than 3x3")
    return out


# --- integral.py -----------------------------------------------------------

def integral_stack(cells: np.ndarray, bins: int) -> np.ndarray:
    """integral.py:58-87 (32-bit): (H,W) int16 -> (bins, H+1, W+1) uint32."""
    cells = np.ascontiguousarray(cells, dtype=np.int16)
    H, W = cells.shape
    out = np.empty((bins, H + 1, W + 1), dtype=np.uint32)
    lib().oracle_integral(_p(cells), H, W, bins, _p(out))
    return out


# --- descriptor.py ---------------------------------------------------------

@dataclass(frozen=True)
class Geometry:
    """descriptor.py:26-70 (validation lives in the product; this is data)."""

    window_w: int
    window_h: int
    cell: int
    block: int = 2
    block_stride: int = 1
    bins: int = 9
    normalization: str = "none"

    @property
    def cells_x(self):
        return self.window_w // self.cell

    @property
    def cells_y(self):
        return self.window_h // self.cell

    @property
    def blocks_x(self):
        return (self.cells_x - self.block) // self.block_stride + 1

    @property
    def blocks_y(self):
        return (self.cells_y - self.block) // self.block_stride + 1

    @property
    def length(self):
        return self.blocks_x * self.blocks_y * self.block * self.block * self.bins


def window_origins(width, height, g, stride):
    """descriptor.py:198-206."""
    return (np.arange(0, width - g.window_w + 1, stride),
            np.arange(0, height - g.window_h + 1, stride))


def cell_index(origin_xs, origin_ys, g):
    """descriptor.py:162-188: cell lattice and per-origin index maps."""
    offs_x = g.cell * np.arange(g.cells_x)
    offs_y = g.cell * np.arange(g.cells_y)
    cell_xs = np.unique(np.asarray(origin_xs)[:, None] + offs_x[None, :])
    cell_ys = np.unique(np.asarray(origin_ys)[:, None] + offs_y[None, :])
    col_idx = np.searchsorted(cell_xs, np.asarray(origin_xs)[:, None] + offs_x[None, :])
    row_idx = np.searchsorted(cell_ys, np.asarray(origin_ys)[:, None] + offs_y[None, :])
    return cell_xs.astype(np.int64), cell_ys.astype(np.int64), col_idx, row_idx


def cell_grid(planes: np.ndarray, cell_xs, cell_ys, cell: int) -> np.ndarray:
    """descriptor.py:176-185 -> (ncy, ncx, bins) int64."""
    planes = np.ascontiguousarray(planes, dtype=np.uint32)
    bins, H1, W1 = planes.shape
    cx = np.ascontiguousarray(cell_xs, dtype=np.int64)
    cy = np.ascontiguousarray(cell_ys, dtype=np.int64)
    out = np.empty((len(cy), len(cx), bins), dtype=np.int64)
    lib().oracle_cell_grid(_p(planes), bins, H1 - 1, W1 - 1, _p(cx), len(cx), _p(cy), len(cy),
                           cell, _p(out))
    return out


def _eps_term(norm: str) -> float:
    return EPS if norm == "l1" else EPS * EPS  # descriptor.py:121,123


_NORM = {"none": 0, "l1": 1, "l2": 2}


def window_descriptor_from_grid(grid, rows, cols, g) -> np.ndarray:
    """descriptor.py:107-124 on grid[np.ix_(rows, cols)] (descriptor.py:190-195)."""
    grid = np.ascontiguousarray(grid, dtype=np.int64)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    out = np.empty(g.length, dtype=np.float64)
    lib().oracle_window_descriptor(_p(grid), grid.shape[1], grid.shape[2], _p(rows), _p(cols),
                                   g.cells_x, g.cells_y, g.block, g.block_stride,
                                   _NORM[g.normalization], _eps_term(g.normalization), _p(out))
    if g.normalization == "none":
        return out.astype(np.int64)
    return out


def window_descriptor(planes, origin, g) -> np.ndarray:
    """descriptor.py:127-150 (direct, uncached)."""
    ox, oy = origin
    xs = ox + g.cell * np.arange(g.cells_x)
    ys = oy + g.cell * np.arange(g.cells_y)
    grid = cell_grid(planes, xs, ys, g.cell)
    return window_descriptor_from_grid(grid, np.arange(g.cells_y), np.arange(g.cells_x), g)


def dot_bias(weights, desc, bias) -> float:
    """detector.py:131-137 (index-order summation)."""
    w = np.ascontiguousarray(weights, dtype=np.float64)
    d = np.ascontiguousarray(desc, dtype=np.float64)
    return float(lib().oracle_dot_bias(_p(w), _p(d), len(w), float(bias)))


def scan_scores(planes, g, stride, weights, bias) -> np.ndarray:
    """detector.py:157-199 with threshold=-inf: (noy, nox) float64 scores."""
    bins, H1, W1 = planes.shape
    oxs, oys = window_origins(W1 - 1, H1 - 1, g, stride)
    cell_xs, cell_ys, col_idx, row_idx = cell_index(oxs, oys, g)
    grid = cell_grid(planes, cell_xs, cell_ys, g.cell)
    out = np.empty((len(oys), len(oxs)), dtype=np.float64)
    for iy in range(len(oys)):
        for ix in range(len(oxs)):
            d = window_descriptor_from_grid(grid, row_idx[iy], col_idx[ix], g)
            out[iy, ix] = dot_bias(weights, d, bias)
    return out


# --- detector.py: pyramid --------------------------------------------------

def resize_bilinear(planes: np.ndarray, new_w: int, new_h: int) -> np.ndarray:
    """detector.py:202-221."""
    planes = np.ascontiguousarray(planes, dtype=np.uint8)
    C, H, W = planes.shape
    out = np.empty((C, new_h, new_w), dtype=np.uint8)
    lib().oracle_resize_bilinear(_p(planes), C, H, W, new_w, new_h, _p(out))
    return out


def pyramid_levels(width, height, g, scale_step):
    """detector.py:251-257: [(level, factor, w, h)] until the window no longer fits."""
    levels, level = [], 0
    while True:
        factor = scale_step ** level
        w = int(width / factor)
        h = int(height / factor)
        if w < g.window_w or h < g.window_h:
            break
        levels.append((level, factor, w, h))
        level += 1
    return levels


# --- detections (pure Python: small cases only) ------------------------------

def hits(scores, oxs, oys, threshold, scale, ww, wh, clamp=None):
    """detector.py:140-154 (strict >, row-major) + 194-199 (int(round(o*scale)))
    + 261-267 (pyramid clamp to clamp = (W, H)).  Returns (boxes, scores)."""
    boxes, out = [], []
    for iy in range(scores.shape[0]):
        for ix in range(scores.shape[1]):
            s = float(scores[iy, ix])
            if s > threshold:
                x, y, bw, bh = int(round(int(oxs[ix]) * scale)), int(round(int(oys[iy]) * scale)), ww, wh
                if clamp is not None:
                    x = min(max(x, 0), clamp[0] - 1)
                    y = min(max(y, 0), clamp[1] - 1)
                    bw = min(bw, clamp[0] - x)
                    bh = min(bh, clamp[1] - y)
                boxes.append((x, y, bw, bh))
                out.append(s)
    return np.array(boxes, dtype=np.int64).reshape(-1, 4), np.array(out, dtype=np.float64)


def iou(a, b) -> float:
    """detector.py:272-282."""
    ax, ay, aw, ah = a
    bx, by, bw, bh = b
    ix = max(0.0, min(ax + aw, bx + bw) - max(ax, bx))
    iy = max(0.0, min(ay + ah, by + bh) - max(ay, by))
    inter = ix * iy
    if inter <= 0.0:
        return 0.0
    return inter / (aw * ah + bw * bh - inter)


def nms(boxes, scores, scales, iou_threshold, float_boxes=False) -> np.ndarray:
    """detector.py:285-299: kept indices, in keep order.  sorted() is stable,
    so equal keys keep input order, as in the reference.  float_boxes: box
    coordinates stay Python floats (a caller's own Detections)."""
    conv = float if float_boxes else int
    boxes = [tuple(conv(v) for v in b) for b in np.asarray(boxes)]
    order = sorted(range(len(boxes)),
                   key=lambda i: (-float(scores[i]), boxes[i][1], boxes[i][0], float(scales[i])))
    kept = []
    for i in order:
        if all(iou(boxes[i], boxes[k]) <= iou_threshold for k in kept):
            kept.append(i)
    return np.array(kept, dtype=np.int64)


# --- whole-frame CPU baseline ---------------------------------------------

def run_batch(frames: np.ndarray, lut: np.ndarray, bins: int, cell: int, ww: int, wh: int,
              stride: int, mode: int, weights=None, bias=0.0, threads=1,
              want_outputs=False):
    """Per-frame pipeline (binmap -> planes -> grid -> scores/denominators) over
    a (N,C,H,W) batch on `threads` host threads.  mode 0: grid, 1: scores,
    2: per-cell l2.  Returns (checksum, grid or None, scores or None)."""
    frames = np.ascontiguousarray(frames, dtype=np.uint8)
    n, C, H, W = frames.shape
    lut = np.ascontiguousarray(lut, dtype=np.int16)
    w = np.ascontiguousarray(weights if weights is not None else np.zeros(1), dtype=np.float64)
    grid = scores = None
    gp = sp = None
    if want_outputs:
        g = Geometry(ww, wh, cell, 1, 1, bins)
        oxs, oys = window_origins(W, H, g, stride)
        cxs, cys, _, _ = cell_index(oxs, oys, g)
        grid = np.empty((n, len(cys), len(cxs), bins), dtype=np.int64)
        gp = _p(grid)
        if mode == 1:
            scores = np.empty((n, len(oys), len(oxs)), dtype=np.float64)
            sp = _p(scores)
    cs = lib().oracle_run_batch(_p(frames), n, C, H, W, _p(lut), bins, cell, ww, wh, stride, mode,
                                _p(w), float(bias), EPS * EPS, int(threads), gp, sp)
    return int(cs), grid, scores


def sha256(a: np.ndarray) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()

