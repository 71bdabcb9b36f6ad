"""Intra-frame split of one frame over several GPUs.

The reference processes a frame as a whole (integral.py:75-79: two cumsums per
bin).  Frame-level sharding (sharding.py) cannot help a single large frame,
e.g. one 8K frame with N_b = 18 and 2.4 GB of planes.  Here such a frame is cut into row
slabs, one per rank:

* Rank r owns the pixel rows [y0, y1), where y0 is a multiple of the lattice step.
  It bins the rows [y0, y1e) with y1e = min(y1 + cell, H). The extra rows let it finish
  the cells whose top row it owns. It reads one halo row above and one below for the
  vertical gradient (``hog_pipeline_slab`` halo flags), so its bin map equals
  rows [y0, y1e) of the whole frame's bin map.
* The only exchange is the column carry. Each rank counts the bins of its own rows per
  column (``hog_column_counts``, N_b x W int32). One all_gather then gives each rank the
  counts of every slab above it. Their sum is the carry that ``hog_pipeline_slab`` adds
  below plane row 0, so local plane row Y *is* global plane row y0 + Y. The exchange is
  N_b x W x 4 bytes per rank, 553 KB at 8K with N_b = 18.
* Grid rows whose cells start in [y0, y1) are computed locally from those plane rows.

With ``group=None`` the carry is supplied by the caller (``run(base=...)``).
That is how one process checks the decomposition on one GPU, and how the gloo tests
drive the host logic.
"""
from __future__ import annotations

import numpy as np

from . import _native, device as D
from .descriptor import DescriptorGeometry, cell_lattice, window_origins
from .gradient import build_lut


def slab_bounds(height: int, world: int, step: int) -> list[tuple[int, int]]:
    """Owned pixel rows [y0, y1) per rank: contiguous, covering [0, height), with every
    y0 a multiple of `step` (the scan lattice step) and sizes as even as that allows."""
    if world < 1:
        raise ValueError("world must be >= 1")
    units = -(-height // step)
    out, a = [], 0
    for r in range(world):
        b = a + units // world + (1 if r < units % world else 0)
        out.append((min(a * step, height), min(b * step, height)))
        a = b
    return out


def computed_rows(y0: int, y1: int, height: int, cell: int) -> tuple[int, int, int, int]:
    """(first, end, halo_top, halo_bot): the rows a slab bins, [y0, min(y1 + cell, H)), and
    whether the frame continues above / below them."""
    y1e = min(y1 + cell, height)
    return y0, y1e, int(y0 > 0), int(y1e < height)


def exclusive_carry(own_counts: list) -> list:
    """Column counts above each slab: exclusive prefix over ranks of their own
    per-column bin counts (the whole exchange of the split)."""
    out, run = [], None
    for c in own_counts:
        out.append(np.zeros_like(c) if run is None else run.copy())
        run = c.copy() if run is None else run + c
    return out


class SlabPipeline:
    """One rank's slab of an n-frame batch of H x W frames (fused pipeline,
    regular lattice: stride % 4 == 0, cell % stride == 0)."""

    def __init__(self, n: int, channels: int, height: int, width: int, bins: int, *,
                 stride: int, rank: int, world: int, cell: int = 8, window=(64, 128),
                 group=None, lut=None, device=None):
        t = D.require_cuda()
        self.n, self.c, self.H, self.w, self.bins = n, channels, height, width, bins
        self.stride, self.cell, self.rank, self.world, self.group = stride, cell, rank, world, group
        self.y0, self.y1 = slab_bounds(height, world, stride)[rank]
        _, self.y1e, self.ht, self.hb = computed_rows(self.y0, self.y1, height, cell)
        self.h = self.y1e - self.y0  # rows binned here
        self.empty = self.y1 <= self.y0  # more ranks than lattice rows: nothing to compute
        g = DescriptorGeometry(window[0], window[1], cell, block=1, block_stride=1, bins=bins)
        oxs, oys = window_origins(width, height, g, stride)
        cxs, cys, _, _ = cell_lattice(oxs, oys, g)
        self.ncx = len(cxs)
        own = cys[(cys >= self.y0) & (cys < self.y1)]  # global cell rows whose top is owned here
        self.cell_row0 = int(own[0]) // stride if len(own) else 0
        self.ncy = len(own)
        self.device = t.device(device or "cuda")
        dev = self.device
        self.lut = lut or build_lut(bins)
        self.lut_dev = D.lut_device(self.lut.table, dev)
        self.own = t.zeros((n, bins, width), dtype=t.int32, device=dev)
        self.base = t.zeros((n, bins, width), dtype=t.int32, device=dev)
        if self.empty:
            return
        # image rows [y0 - ht, y1e + hb): the halo rows are read, never binned
        self.frames = D.alloc_frames(n, channels, self.h + self.ht + self.hb, width, dev)
        self.binmap = D.alloc_binmap(n, self.h, width, dev)
        self.planes = D.alloc_planes(n, bins, self.h, width, dev)
        self.grid = t.empty((n, max(self.ncy, 1), self.ncx, bins), dtype=t.int32, device=dev)
        sb = int(_native.load().hog_scratch_bytes(n, self.h, width, bins, stride, cell))
        self.scratch = (t.empty(max(sb, 256), dtype=t.uint8, device=dev), sb)

    def upload(self, frames: np.ndarray):
        """frames: the FULL (n, C, H, W) batch; this rank copies its rows + halos."""
        if self.empty:
            return
        t = D.torch()
        a = np.ascontiguousarray(frames[:, :, self.y0 - self.ht: self.y1e + self.hb])
        dst = self.frames.data if self.frames.pitch == self.w else self.frames.data[..., : self.w]
        dst.copy_(t.from_numpy(a))

    def _call(self, stages: int, stream=None):
        fr, bm, pl = self.frames, self.binmap, self.planes
        scr, sb = self.scratch
        img = D.ptr(fr.data) + self.ht * fr.pitch
        _native.call("hog_pipeline_slab", img, self.n, self.c, self.h, self.w, fr.pitch,
                     fr.cstride, fr.fstride, D.ptr(self.lut_dev), self.bins, D.ptr(bm.data),
                     bm.pitch, bm.fstride, pl.ptr, pl.pitch, pl.nstride, pl.fstride, self.cell,
                     self.stride, self.ncx, max(self.ncy, 1) if self.ncy else 0,
                     D.ptr(self.grid) if self.ncy else None, D.ptr(scr), sb, stages, self.ht,
                     self.hb, D.ptr(self.base), self.bins * self.w, D.stream_handle(stream))

    def bin_and_count(self, stream=None):
        """Phase 1: bin map of the slab + this slab's own per-column counts."""
        if self.empty:
            return self.own
        self._call(_native.STAGE_BIN, stream)
        bm = self.binmap
        _native.call("hog_column_counts", D.ptr(bm.data), self.n, self.y1 - self.y0, self.w,
                     bm.pitch, bm.fstride, self.bins, D.ptr(self.own), D.stream_handle(stream))
        return self.own

    def exchange(self):
        """Phase 2: base = sum of the own counts of the ranks above (one all_gather:
        NCCL over NVLink on device buffers; a gloo group exchanges host copies)."""
        import torch.distributed as dist

        t = D.torch()
        on_dev = dist.get_backend(self.group) == "nccl"
        own = self.own if on_dev else self.own.cpu()
        parts = [t.empty_like(own) for _ in range(self.world)]
        dist.all_gather(parts, own, group=self.group)
        if self.rank == 0:
            self.base.zero_()
        else:
            above = t.stack(parts[: self.rank]).sum(0, dtype=t.int32)
            self.base.copy_(above, non_blocking=on_dev)

    def planes_and_grid(self, base=None, stream=None):
        """Phase 3: planes (global rows y0 .. y1e) and the owned grid rows."""
        if base is not None:
            self.base.copy_(base)
        if self.empty:
            return
        self._call(_native.STAGE_SCAN | _native.STAGE_PLANES, stream)

    def run(self, base=None):
        """All three phases; with a process group the carry comes from the
        exchange, otherwise from `base` (zeros for the top slab)."""
        self.bin_and_count()
        if self.group is not None:
            self.exchange()
            base = None
        self.planes_and_grid(base)

    def planes_view(self):
        """(n, bins, y1 - y0 + 1, W + 1): global plane rows y0 .. y1."""
        return self.planes.view()[:, :, : self.y1 - self.y0 + 1]

    def grid_view(self):
        """(n, ncy_own, ncx, bins): global cell rows cell_row0 .. cell_row0 + ncy - 1."""
        return self.grid[:, : self.ncy]
