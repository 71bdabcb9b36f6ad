"""Batched device pipeline: the path the benchmark configurations run.

One ``HogPipeline`` owns every HBM buffer for a frame batch of one shape and
runs LUT binning -> integral planes -> cell grid (fused into the plane
kernel when the scan lattice is regular) -> optional per-cell normalisation
and window scores on the GPU, with no host synchronisation.

By default the whole batch is one launch per stage.  ``chunks > 1`` splits
it into frame groups on two streams so that binning of group j+1 runs under
the plane kernel of group j.  On B200 that measured slower: both kernels are
issue/latency-bound, and the plane kernel loses more than the overlap saves
(profiles/r1_c2_ncu_summary.md).  Frames are independent, so multi-GPU runs
give each rank its own pipeline over its own frame shard, with no collective.
"""
from __future__ import annotations

import ctypes
import functools

import numpy as np

from . import _native, device as D
from .descriptor import (DescriptorGeometry, cell_lattice, descriptor_length, eps_term,
                         window_origins, _NORM_CODE)
from .gradient import build_lut


def on_device(fn):
    """Run a pipeline method with the pipeline's device current: the C ABI
    launches on the CUDA runtime's current device, and per-device state
    (shared-memory opt-in, streams) follows it.  One host thread can then
    drive pipelines on several GPUs."""
    @functools.wraps(fn)
    def wrap(self, *args, **kwargs):
        with D.torch().cuda.device(self.device):
            return fn(self, *args, **kwargs)
    return wrap


MAX_PIPELINE_BINS = 18  # hog_pipeline's fused limit; more bins run binning + hog_integral groups


def regular_lattice(cell_xs, cell_ys, stride: int, cell: int, bins: int) -> bool:
    """True when hog_pipeline can emit the grid from the plane kernel."""
    if stride % 4 or stride > 240 or cell % stride or cell // stride > 2 or cell % 4 or bins > 18:
        return False
    for cs in (cell_xs, cell_ys):
        if len(cs) == 0 or not np.array_equal(cs, np.arange(0, cs[-1] + 1, stride)):
            return False
    return True


def _tune_enabled() -> bool:
    import os

    return os.environ.get("HOGB200_TUNE", "1") != "0"


def default_chunks(n: int, pixels_per_frame: int) -> int:
    """Frame groups for the binning/plane overlap.  Measured on B200 (c2): the
    plane kernel loses more to a co-running binning kernel than the overlap
    saves, so the default is one chunk; HOGB200_CHUNKS overrides."""
    import os

    env = os.environ.get("HOGB200_CHUNKS")
    return max(1, min(n, int(env))) if env else 1


def _i8_enabled() -> bool:
    import os

    return os.environ.get("HOGB200_SCORES_I8", "1") != "0"


def i8_prepare(weights, cells_x: int, cells_y: int, bins: int):
    """Host side of the exact integer score path (hog_scores_i8_prepare):
    (fragment bytes, digits, scale) or None when the weights span more bits
    than the integer path holds (HOG_ERANGE) or the geometry is outside it."""
    import ctypes

    lib = _native.load()
    nbytes = lib.hog_scores_i8_frag_bytes(bins)
    if nbytes == 0 or cells_x != 8 or not 1 <= cells_y <= 16:
        return None
    w = np.ascontiguousarray(weights, dtype=np.float64)
    frag = np.zeros(nbytes, dtype=np.uint8)
    digits, scale = ctypes.c_int(0), ctypes.c_double(0.0)
    rc = lib.hog_scores_i8_prepare(w.ctypes.data, cells_x, cells_y, bins, frag.ctypes.data,
                                   ctypes.byref(digits), ctypes.byref(scale))
    if rc == _native.HOG_ERANGE:
        return None
    if rc != _native.HOG_OK:
        raise _native.NativeError(f"hog_scores_i8_prepare failed ({rc}): "
                                  f"{lib.hog_last_error().decode(errors='replace')}")
    return frag, digits.value, scale.value


def i8_weights(weights, cells_x: int, cells_y: int, bins: int, device):
    """i8_prepare with the fragments uploaded: (device tensor, digits, scale) or None."""
    r = i8_prepare(weights, cells_x, cells_y, bins)
    if r is None:
        return None
    t = D.torch()
    frag, digits, scale = r
    return t.as_tensor(frag, device=device), digits, scale


class HogPipeline:
    def __init__(self, n: int, channels: int, height: int, width: int, bins: int, *,
                 stride: int, cell: int = 8, window=(64, 128), normalization: str = "none",
                 weights=None, bias: float = 0.0, lut=None, device=None, chunks: int | None = None,
                 grid_dtype: str = "auto", band_rows: int | None = None,
                 window_norm: str | None = None):
        """window_norm="l2" (an EXTENSION, not a reference behaviour): per-window L2
        norms of the unnormalised window descriptors, for BASELINE configs[2]'s
        "per-window L2 normalisation" (the reference normalises per block);
        p.window_norms holds them and window_descriptors() divides by them."""
        t = D.require_cuda()
        if window_norm not in (None, "l2"):
            raise ValueError(f"window_norm must be None or 'l2', got {window_norm!r}")
        if window_norm is not None and normalization != "none":
            raise ValueError("window_norm applies to unnormalised cells (normalization='none')")
        self.window_norm = window_norm
        self.n, self.c, self.h, self.w, self.bins = n, channels, height, width, bins
        self.stride, self.cell = stride, cell
        self.geometry = DescriptorGeometry(window[0], window[1], cell, block=1, block_stride=1,
                                           bins=bins, normalization=normalization)
        g = self.geometry
        self.oxs, self.oys = window_origins(width, height, g, stride)
        self.cell_xs, self.cell_ys, self.col_idx, self.row_idx = cell_lattice(self.oxs, self.oys, g)
        self.ncx, self.ncy = len(self.cell_xs), len(self.cell_ys)
        self.fused = regular_lattice(self.cell_xs, self.cell_ys, stride, cell, bins)
        self.lut = lut or build_lut(bins)
        self.device = t.device(device or "cuda")
        dev = self.device
        self.frames = D.alloc_frames(n, channels, height, width, dev)
        self.binmap = D.alloc_binmap(n, height, width, dev)
        self.planes = D.alloc_planes(n, bins, height, width, dev)
        # the fused grid is stored as uint8 (cell counts <= cell^2 <= 255: exact,
        # 4x fewer grid bytes) unless a device consumer needs int32: per-cell
        # normalisation and the general window-feature path do; the lattice
        # score kernel (8 cells across) reads bytes
        u8_ok = (self.fused and cell * cell <= 255 and normalization == "none"
                 and (weights is None or g.cells_x == 8))
        if grid_dtype not in ("auto", "int32", "uint8"):
            raise ValueError("grid_dtype must be 'auto', 'int32' or 'uint8'")
        if grid_dtype == "uint8" and not u8_ok:
            raise ValueError("uint8 grid needs a fused lattice, cell*cell <= 255, no normalisation "
                             "and (if scored) 8 cells across")
        self.grid_u8 = grid_dtype == "uint8" or (grid_dtype == "auto" and u8_ok)
        self.grid = t.empty((n, self.ncy, self.ncx, bins),
                            dtype=t.uint8 if self.grid_u8 else t.int32, device=dev)
        self.lut_dev = D.lut_device(self.lut.table, dev)
        self.chunks = default_chunks(n, height * width) if chunks is None else max(1, min(chunks, n))
        # frame ranges of the chunks, each with its own scratch (stages of
        # different chunks run concurrently)
        base, rem = divmod(n, self.chunks)
        self.ranges, a = [], 0
        for j in range(self.chunks):
            b = a + base + (1 if j < rem else 0)
            self.ranges.append((a, b))
            a = b
        self.band_rows = 0 if band_rows is None else int(band_rows)  # 0: library's choice
        self.scratch = []
        self._alloc_scratch()
        self.side = t.cuda.Stream(device=dev) if self.chunks > 1 else None
        self.post = t.cuda.Stream(device=dev) if self.chunks > 1 else None
        self._post_done = None  # event: scores of the last pipelined run
        self.cx_dev = t.as_tensor(self.cell_xs.astype(np.int32), device=dev)
        self.cy_dev = t.as_tensor(self.cell_ys.astype(np.int32), device=dev)
        self.denom = None
        if normalization != "none":
            self.denom = t.empty((n, self.ncy, self.ncx), dtype=t.float64, device=dev)
        self.weights = None if weights is None else np.asarray(weights, dtype=np.float64)
        self.bias = float(bias)
        self.scores = None
        if self.weights is not None:
            if len(self.weights) != descriptor_length(g):
                raise ValueError("weights length does not match the geometry")
            self.scores = t.empty((n, len(self.oys), len(self.oxs)), dtype=t.float64, device=dev)
            self.w_dev = t.as_tensor(self.weights, device=dev)
        # exact integer-tensor-core scores (stride = cell, byte grid, 8 x <= 16
        # cells, <= 20 bins, weights within 47 bits); else the fp64 kernels
        self.i8 = None
        if (self.weights is not None and self.fused and self.grid_u8 and g.cells_x == 8
                and self.cell == self.stride and _i8_enabled()):
            self.i8 = i8_weights(self.weights, g.cells_x, g.cells_y, bins, dev)
        if self.weights is not None or window_norm is not None:
            self.ri_dev = t.as_tensor(self.row_idx.astype(np.int32), device=dev)
            self.ci_dev = t.as_tensor(self.col_idx.astype(np.int32), device=dev)
        self.window_norms = None
        if window_norm is not None:
            self.window_norms = t.empty((n, len(self.oys), len(self.oxs)), dtype=t.float64, device=dev)
            # per-cell sums of squares, then (regular lattice) per-row window sums
            self.cell_sq = t.empty(n * self.ncy * (self.ncx + len(self.oxs)), dtype=t.int32,
                                   device=dev)
        self.band_rows_timings = None
        if band_rows is None and self.chunks == 1 and _tune_enabled():
            self.band_rows = self._tune_band_rows()

    # -- plane-kernel band rows ---------------------------------------------
    def _scratch_bytes(self, a: int, b: int) -> int:
        lib = _native.load()
        lib.hog_set_band_rows(self.band_rows)
        try:
            return int(lib.hog_scratch_bytes(b - a, self.h, self.w, self.bins,
                                             self.stride if self.fused else 0,
                                             self.cell if self.fused else 0))
        finally:
            lib.hog_set_band_rows(0)

    def _alloc_scratch(self):
        t = D.torch()
        out = []
        for j, (a, b) in enumerate(self.ranges):
            sb = self._scratch_bytes(a, b)
            old = self.scratch[j][0] if j < len(self.scratch) else None
            buf = old if old is not None and old.numel() >= sb else \
                t.empty(max(sb, 256), dtype=t.uint8, device=self.device)
            out.append((buf, sb))
        self.scratch = out

    def auto_band_rows(self) -> int:
        """The library's own choice of band rows for this shape."""
        return int(_native.load().hog_get_band_rows(self.n, self.h, self.w, self.bins,
                                                    self.stride if self.fused else 0,
                                                    self.cell if self.fused else 0))

    @on_device
    def _tune_band_rows(self) -> int:
        """Time binning + carry scan + planes (+ grid) at a few band rows on this
        pipeline's own buffers and keep the fastest; the automatic choice stays
        unless another is > 0.5 % faster (c2: R = 64 beats the automatic 128 by
        0.9 % with the register-resident top row).  Measured on B200, the best R moves
        with the CTA-wave count of the shape (profiles/r1b_band_sweep.txt: c4
        best at 80, 8K pyramid level 1 at 40, c2/c3/level 0 at the automatic R).
        Any R gives bit-identical outputs; only the tiling changes."""
        t = D.torch()
        auto = self.auto_band_rows()
        cands = [auto] + [r for r in (32, 40, 48, 64, 80, 96, 128)
                          if r != auto and r <= max(D.round_up(self.h + 1, 8), 32)]
        # plus the two band heights whose plane-kernel grid (frames x bands CTAs, two
        # per SM) fills its last wave best: small batches lose most to the tail
        # (c2's 64-frame shard of an 8-GPU run)
        slots = 2 * 148
        def fill(r):
            ctas = self.n * (self.h // r + 1)
            return ctas / (-(-ctas // slots) * slots)
        extra = sorted((r for r in range(24, 161, 8) if r not in cands and r <= self.h + 1),
                       key=lambda r: (-fill(r), -r))[:2]
        cands += extra
        stream = t.cuda.current_stream(self.device)
        times = {}
        for r in cands:
            self.band_rows = r
            self._alloc_scratch()
            best = None
            for it in range(4):
                e0 = t.cuda.Event(enable_timing=True)
                e1 = t.cuda.Event(enable_timing=True)
                e0.record(stream)
                self._stage(0, _native.STAGE_ALL, stream)
                e1.record(stream)
                e1.synchronize()
                if it:
                    ms = e0.elapsed_time(e1)
                    best = ms if best is None else min(best, ms)
            times[r] = best
        pick = min(times, key=times.get)
        if times[pick] > 0.995 * times[auto]:  # min of 3 timed runs each: noise < 0.5 %
            pick = auto
        self.band_rows_timings = times
        self.band_rows = pick
        self.scratch = []  # exact size for the pick (the candidates' largest is not kept)
        self._alloc_scratch()
        return pick

    # -- data movement ------------------------------------------------------
    @on_device
    def upload(self, frames: np.ndarray, stream=None):
        t = D.torch()
        src = t.from_numpy(np.ascontiguousarray(frames))
        if self.frames.pitch == self.w:
            self.frames.data.copy_(src, non_blocking=True)
        else:
            self.frames.data[..., : self.w].copy_(src, non_blocking=True)

    # -- the hot path -------------------------------------------------------
    def _stage(self, j: int, stages: int, stream, events=None, frames_ptr=None):
        a, b = self.ranges[j]
        fr, bm, pl = self.frames, self.binmap, self.planes
        scr, sb = self.scratch[j]
        evs = None
        if events is not None:
            evs = (ctypes.c_void_p * 4)(*[e.cuda_event if e is not None else None for e in events])
        base = D.ptr(fr.data) if frames_ptr is None else frames_ptr
        lib = _native.load()
        lib.hog_set_band_rows(self.band_rows)
        try:
            self._pipeline_call(base, a, b, fr, bm, pl, scr, sb, stages, evs, stream)
        finally:
            lib.hog_set_band_rows(0)

    def _pipeline_call(self, base, a, b, fr, bm, pl, scr, sb, stages, evs, stream):
        if self.bins > MAX_PIPELINE_BINS:
            return self._grouped_call(base, a, b, fr, bm, pl, scr, sb, stages, evs, stream)
        _native.call("hog_pipeline", base + a * fr.fstride, b - a, self.c, self.h,
                     self.w, fr.pitch, fr.cstride, fr.fstride, D.ptr(self.lut_dev), self.bins,
                     D.ptr(bm.data) + a * bm.fstride, bm.pitch, bm.fstride,
                     pl.ptr + 4 * a * pl.fstride, pl.pitch, pl.nstride, pl.fstride,
                     self.cell, self.stride, self.ncx, self.ncy,
                     (D.ptr(self.grid) + self.grid.element_size() * a * self.ncy * self.ncx * self.bins)
                     if self.fused else None,
                     D.ptr(scr), sb, stages | (_native.STAGE_GRID_U8 if self.grid_u8 else 0), evs,
                     D.stream_handle(stream))
        # kernels this call launched (the library folds the carry scan into the plane
        # kernel for shapes with few bands)
        self._core_launches = getattr(self, "_core_launches", 0) + _native.load().hog_last_pipeline_launches()

    @on_device
    def _grouped_call(self, base, a, b, fr, bm, pl, scr, sb, stages, evs, stream):
        """N_b > 18 (hog_pipeline's fused limit): binning (hog_grad_bin), then the
        planes in bin groups (hog_integral); the cell grid comes from
        hog_cell_grid in _post (the lattice is not fused).  Stage events are not
        recorded on this path (no BASELINE configuration has N_b > 18)."""
        h = D.stream_handle(stream)
        bmp = D.ptr(bm.data) + a * bm.fstride
        if stages & _native.STAGE_BIN:
            _native.call("hog_grad_bin", base + a * fr.fstride, b - a, self.c, self.h, self.w,
                         fr.pitch, fr.cstride, fr.fstride, D.ptr(self.lut_dev), self.bins, bmp,
                         bm.pitch, bm.fstride, h)
        if stages & _native.STAGE_PLANES:
            _native.call("hog_integral", bmp, b - a, self.h, self.w, bm.pitch, bm.fstride,
                         self.bins, pl.ptr + 4 * a * pl.fstride, pl.pitch, pl.nstride, pl.fstride,
                         D.ptr(scr), sb, h)

    def run(self, stream=None, plane_events=None, frames_ptr=None, scores_ptr=None,
            pipelined: bool = False):
        """Enqueue the whole batch; results are ready in `stream` order (default:
        current stream).  plane_events: optional per-chunk (start, end) pairs of
        recorded torch.cuda.Events bracketing each plane-kernel launch on the
        stream it runs on.  frames_ptr / scores_ptr: read the frames from / write
        the scores to another device buffer of this pipeline's layout (the
        pyramid's level 0 reads the source frames in place and every level
        writes its slice of the pyramid's score maps directly)."""
        t = D.torch()
        main = stream if stream is not None else t.cuda.current_stream(self.device)
        self._core_launches = 0
        try:
            return self._run(main, plane_events, frames_ptr, scores_ptr, pipelined)
        finally:
            self._core_run = self._core_launches

    def _run(self, main, plane_events, frames_ptr, scores_ptr, pipelined):
        t = D.torch()
        if pipelined and self.chunks == 1 and self.scores is not None:
            # consecutive batches overlap: this batch's binning + carry scan run
            # while the previous batch's scores are still computing (on
            # self.post); its plane kernel waits for them (it rewrites the grid
            # they read).  Results are ready after join().
            if self.post is None:
                self.post = t.cuda.Stream(device=self.device)
            self._stage(0, _native.STAGE_BIN | _native.STAGE_SCAN, main, None, frames_ptr)
            if self._post_done is not None:
                main.wait_event(self._post_done)
            evs = None
            if plane_events is not None:
                e0, e1 = plane_events[0]
                evs = [None, None, e0, e1]
            self._stage(0, _native.STAGE_PLANES, main, evs, frames_ptr)
            planed = t.cuda.Event()
            planed.record(main)
            self.post.wait_event(planed)
            self._post(self.post, scores_ptr)
            self._post_done = t.cuda.Event()
            self._post_done.record(self.post)
            return
        self.join(main)
        if self.chunks == 1:
            evs = None
            if plane_events is not None:
                e0, e1 = plane_events[0]
                evs = [None, None, e0, e1]
            self._stage(0, _native.STAGE_ALL, main, evs, frames_ptr)
        else:
            # three streams: binning of group j+1 (main), planes of group j (side)
            # and the grid consumers (scores / normalisation) of group j-1 (post)
            side, post = self.side, self.post
            side.wait_stream(main)
            post.wait_stream(main)
            for j in range(self.chunks):
                self._stage(j, _native.STAGE_BIN | _native.STAGE_SCAN, main, None, frames_ptr)
                done = t.cuda.Event()
                done.record(main)
                side.wait_event(done)
                evs = None
                if plane_events is not None:
                    e0, e1 = plane_events[j]
                    evs = [None, None, e0, e1]
                self._stage(j, _native.STAGE_PLANES, side, evs, frames_ptr)
                planed = t.cuda.Event()
                planed.record(side)
                post.wait_event(planed)
                self._post(post, scores_ptr, *self.ranges[j])
            main.wait_stream(side)
            main.wait_stream(post)
            return
        self._post(main, scores_ptr)

    @on_device
    def join(self, stream=None):
        """Make `stream` wait for the scores of the last pipelined run."""
        if self._post_done is not None:
            t = D.torch()
            (stream if stream is not None else t.cuda.current_stream(self.device)).wait_event(
                self._post_done)
            self._post_done = None

    @on_device
    def run_staged(self, events, stream=None):
        """Diagnostic: the whole batch as one chunk with 4 recorded events
        bracketing binning, carry scan and planes (+ grid)."""
        t = D.torch()
        main = stream if stream is not None else t.cuda.current_stream(self.device)
        self.join(main)
        saved = self.ranges, self.scratch
        if self.chunks > 1:  # one chunk needs the whole-batch scratch
            sb = self._scratch_bytes(0, self.n)  # sized at this pipeline's band rows
            self.ranges = [(0, self.n)]
            self.scratch = [(t.empty(max(sb, 256), dtype=t.uint8, device=self.device), sb)]
        try:
            self._stage(0, _native.STAGE_ALL, main, events)
        finally:
            self.ranges, self.scratch = saved
        self._post(main)

    def _post(self, stream, scores_ptr=None, a: int = 0, b: int | None = None):
        """Grid consumers (cell grid if not fused, per-cell denominators,
        scores) for frames [a, b)."""
        s = D.stream_handle(stream)
        pl = self.planes
        b = self.n if b is None else b
        n = b - a
        cells = self.ncy * self.ncx
        nwin = len(self.oys) * len(self.oxs)
        gp = D.ptr(self.grid) + self.grid.element_size() * a * cells * self.bins
        dp = D.ptr(self.denom) + 8 * a * cells if self.denom is not None else None
        if self.scores is None:
            sp = None
        else:
            sp = (D.ptr(self.scores) if scores_ptr is None else scores_ptr) + 8 * a * nwin
        if not self.fused:
            _native.call("hog_cell_grid", pl.ptr + 4 * a * pl.fstride, n, self.h, self.w,
                         self.bins, pl.pitch, pl.nstride, pl.fstride, D.ptr(self.cx_dev), self.ncx,
                         D.ptr(self.cy_dev), self.ncy, self.cell, gp, s)
        g = self.geometry
        if self.denom is not None:
            _native.call("hog_cell_norm", gp, n, cells, self.bins, _NORM_CODE[g.normalization],
                         eps_term(g.normalization), dp, s)
        if self.window_norms is not None:
            _native.call("hog_window_l2", gp, self.grid.element_size(), n, self.ncy, self.ncx,
                         self.bins, D.ptr(self.ri_dev), len(self.oys), D.ptr(self.ci_dev),
                         len(self.oxs), g.cells_x, g.cells_y,
                         self.cell // self.stride if self.fused else 0, eps_term("l2"),
                         D.ptr(self.cell_sq) + 4 * a * self.ncy * (self.ncx + len(self.oxs)),
                         D.ptr(self.window_norms) + 8 * a * nwin, s)
        if self.scores is not None and self.i8 is not None:
            frag, digits, scale = self.i8
            _native.call("hog_scores_lattice_i8", gp, n, self.ncy, self.ncx, self.bins,
                         len(self.oys), len(self.oxs), g.cells_x, g.cells_y, D.ptr(frag), digits,
                         scale, self.bias, sp, s)
        elif self.scores is not None and self.fused and g.cells_x == 8 and self.grid_u8:
            _native.call("hog_scores_lattice_u8", gp, n, self.ncy, self.ncx,
                         self.bins, len(self.oys), len(self.oxs), g.cells_x, g.cells_y,
                         self.cell // self.stride, D.ptr(self.w_dev), self.bias, sp, s)
        elif self.scores is not None and self.fused and g.cells_x == 8:
            _native.call("hog_scores_lattice", gp, dp, n, self.ncy,
                         self.ncx, self.bins, len(self.oys), len(self.oxs), g.cells_x, g.cells_y,
                         self.cell // self.stride, D.ptr(self.w_dev), self.bias, sp, s)
        elif self.scores is not None:
            _native.call("hog_window_features", gp, n, self.ncy, self.ncx,
                         self.bins, D.ptr(self.ri_dev), len(self.oys), D.ptr(self.ci_dev),
                         len(self.oxs), g.cells_x, g.cells_y, 1, 1, _NORM_CODE[g.normalization],
                         eps_term(g.normalization), D.ptr(self.w_dev), self.bias,
                         sp, None, s)

    @on_device
    def detections(self, threshold: float, iou_threshold: float | None = None, scale: float = 1.0):
        """Per-frame detection lists of the last run (needs weights): windows with
        score > threshold in row-major order (detector.py:145-153, 194-199),
        greedy NMS when iou_threshold is given (detector.py:285-299) -- the
        threshold, box mapping and NMS all run on the device."""
        from . import detections as DT

        if self.scores is None:
            raise ValueError("detections need a pipeline built with weights")
        self.join()
        g = self.geometry
        ww, wh = DT.window_box_size(g.window_w, g.window_h, scale)
        boxes, sc, _, counts = DT.compact(self.scores, self.oxs, self.oys, threshold, scale, ww, wh)
        out = []
        for f in range(self.n):
            k = int(counts[f])
            b, s = boxes[f, :k], sc[f, :k]
            if iou_threshold is not None and k:
                t = D.torch()
                keep = DT.nms_indices(b, s, t.full((k,), float(scale), dtype=t.float64,
                                                   device=b.device), iou_threshold)
                kt = t.as_tensor(keep, device=b.device)
                b, s = b[kt], s[kt]
            out.append(DT.to_detections(b.cpu().numpy(), s.cpu().numpy(), scale))
        return out

    def launches_per_run(self) -> int:
        k = 3 * self.chunks  # grad_bin + carry scan + planes per chunk
        if getattr(self, "_core_run", 0):  # counted by the library during the last run()
            k = self._core_run
        if self.bins > MAX_PIPELINE_BINS:  # grad_bin + per bin group: offset, counts, scan, planes
            k = (1 + 4 * -(-self.bins // 16)) * self.chunks
        post = (0 if self.fused else 1) + (1 if self.denom is not None else 0) + \
            (1 if self.scores is not None else 0) + (2 if self.window_norms is not None else 0)
        return k + post * self.chunks  # grid consumers run per chunk

    # -- views ----------------------------------------------------------------
    def planes_view(self):
        return self.planes.view()

    def binmap_view(self):
        return self.binmap.view()

    def result(self):
        """The step's result tensor (what a caller reads back)."""
        if self.scores is not None:
            return self.scores
        if self.window_norms is not None:
            return self.window_norms
        if self.denom is not None:
            return self.denom
        return self.grid

    def window_descriptors(self, frame: int, rows=None):
        """EXTENSION (window_norm="l2"): per-window L2-normalised descriptors of window
        rows `rows` (a slice; default all) of one frame, (rows, nox, D) float64 on the
        device: the reference's unnormalised descriptor (descriptor.py:115-118) divided
        by the window's norm (IEEE division, so equal to d / np.sqrt((d*d).sum() + eps^2))."""
        if self.window_norms is None:
            raise ValueError("window_descriptors needs window_norm='l2'")
        from .descriptor import window_features_device

        t = D.torch()
        self.join()
        rows = slice(None) if rows is None else rows
        grid = self.grid[frame:frame + 1].to(t.int32)
        _, desc = window_features_device(grid, self.geometry, self.row_idx[rows], self.col_idx,
                                         want_desc=True)
        return desc[0] / self.window_norms[frame, rows][..., None]

    def normalized_grid(self):
        """Per-cell normalised histograms (descriptor.py:119-124 with block=1)."""
        return self.grid.to(D.torch().float64) / self.denom[..., None]

    def bytes_alg_per_frame(self) -> int:
        """SURVEY §8d compulsory bytes per frame."""
        H, W, C, nb = self.h, self.w, self.c, self.bins
        b = C * H * W + H * W + 4 * nb * (H + 1) * (W + 1)
        b += self.grid.element_size() * nb * self.ncx * self.ncy
        if self.scores is not None:
            b += 8 * len(self.oxs) * len(self.oys)
        if self.denom is not None:
            b += 8 * self.ncx * self.ncy
        if self.window_norms is not None:
            b += 8 * len(self.oxs) * len(self.oys)
        return b

    def plane_kernel_bytes_per_frame(self) -> int:
        """Algorithmic bytes of k_planes per frame: bin map read + planes + grid written."""
        H, W, nb = self.h, self.w, self.bins
        b = H * W + 4 * nb * (H + 1) * (W + 1)
        if self.fused:
            b += self.grid.element_size() * nb * self.ncx * self.ncy
        return b


def pyramid_levels(width: int, height: int, window_w: int, window_h: int, scale_step: float):
    """detector.py:251-257: [(level, factor, w, h)] while the window fits."""
    out, level = [], 0
    while True:
        factor = scale_step ** level
        w = int(width / factor)
        h = int(height / factor)
        if w < window_w or h < window_h:
            break
        out.append((level, factor, w, h))
        level += 1
    return out


class PyramidPipeline:
    """Multi-scale scan of a frame batch (detector.py:224-269), on the device.

    Every level is resized from the ORIGINAL frame (detector.py:258) by
    ``hog_resize_bilinear`` and then runs a level ``HogPipeline`` (binning,
    planes, cell grid, scores).  Frames go through in chunks of ``chunk``
    so the per-level buffers (planes: 4*N_b B/px) are reused; every level's
    score map of every frame is kept (``scores[level]``: (N, noy, nox) f64).
    """

    def __init__(self, n: int, channels: int, height: int, width: int, bins: int, *,
                 stride: int, scale_step: float, weights, bias: float = 0.0, cell: int = 8,
                 window=(64, 128), chunk: int = 4, device=None, lut=None,
                 streams: int | None = None):
        t = D.require_cuda()
        if scale_step <= 1.0:
            raise ValueError(f"scale_step must be > 1, got {scale_step}")
        self.n, self.c, self.h, self.w, self.bins = n, channels, height, width, bins
        self.chunk = max(1, min(chunk, n))
        self.device = t.device(device or "cuda")
        self.lut = lut or build_lut(bins)
        self.levels = pyramid_levels(width, height, window[0], window[1], scale_step)
        if not self.levels:
            from .errors import WindowLargerThanImage

            raise WindowLargerThanImage(
                f"window {window[0]}x{window[1]} exceeds image {width}x{height}")
        self.src = D.alloc_frames(n, channels, height, width, self.device)
        self.pipes = [HogPipeline(self.chunk, channels, h, w, bins, stride=stride, cell=cell,
                                  window=window, weights=weights, bias=bias, lut=self.lut,
                                  device=self.device)
                      for (_, _, w, h) in self.levels]
        self.scores = [t.empty((n,) + tuple(p.scores.shape[1:]), dtype=t.float64,
                               device=self.device) for p in self.pipes]
        if streams is None:
            import os

            # measured on B200 (c5, 32 x 8K): 1 stream 85.1 ms, 2: 76.6, 3: 75.7; with
            # the byte-grid scores, 2: 68.9, 3: 68.3, 4: 67.9, 6: 67.7
            # (profiles/r1b_c5_schedule_sweep.txt)
            streams = int(os.environ.get("HOGB200_PYR_STREAMS", "4"))
        self.streams = max(1, min(int(streams), len(self.levels)))
        self._side = [t.cuda.Stream(device=self.device) for _ in range(self.streams - 1)]
        import os

        # level -> stream (a level's chunks stay on one stream: its buffers are reused in
        # order) and the order levels are issued in within a chunk
        #   HOGB200_PYR_ASSIGN  rr: level i on stream i mod S; lpt: largest level first onto
        #                       the stream with the least pixels so far
        #   HOGB200_PYR_ORDER   asc: level 0 first; desc: smallest level first; asc-desc:
        #                       descending in the last chunk only (the step ends on big kernels)
        assign = os.environ.get("HOGB200_PYR_ASSIGN", "rr")
        self.order_mode = os.environ.get("HOGB200_PYR_ORDER", "asc")
        nl = len(self.levels)
        if assign == "lpt":
            load = [0] * self.streams
            self.level_stream = [0] * nl
            for i, (_, _, w, h) in enumerate(self.levels):  # levels come largest first
                k = min(range(self.streams), key=lambda j: (load[j], j))
                self.level_stream[i] = k
                load[k] += w * h
        else:
            self.level_stream = [i % self.streams for i in range(nl)]

    @on_device
    def upload(self, frames: np.ndarray):
        t = D.torch()
        src = t.from_numpy(np.ascontiguousarray(frames))
        if self.src.pitch == self.w:
            self.src.data.copy_(src, non_blocking=True)
        else:
            self.src.data[..., : self.w].copy_(src, non_blocking=True)

    @on_device
    def run(self, stream=None, plane_events=None, chunk_ready=None, level_done=None):
        """plane_events: optional list; (start, end, algorithmic bytes) of every
        plane-kernel launch is appended (events recorded on the launch stream).
        chunk_ready(a, m, stream): called before `stream` first reads frames
        [a, a+m) (e.g. to wait for their H2D copy); level_done(level, a, m,
        stream): called once scores[level][a:a+m] are enqueued on `stream`
        (e.g. to start their D2H).

        Level 0 reads the source frames in place and every level writes its
        score maps straight into ``scores[level]`` (no device copies).  Levels
        are spread over ``self.streams`` streams (level i on stream i mod S),
        so the launch-bound small levels and the FP64 score kernels run beside
        the plane writes of other levels; one level's chunks stay in order on
        its stream, which is what makes reusing its buffers safe."""
        t = D.torch()
        main = stream if stream is not None else t.cuda.current_stream(self.device)
        sts = [main] + self._side[: self.streams - 1]
        for st in sts[1:]:
            st.wait_stream(main)
        src = self.src
        for a in range(0, self.n, self.chunk):
            m = min(self.chunk, self.n - a)
            if chunk_ready is not None:
                for st in sts:
                    chunk_ready(a, m, st)
            # a partial last chunk runs through the level pipelines' own buffers
            # (they process p.n frames: direct pointers would run past the batch)
            whole = m == self.chunk
            last = a + self.chunk >= self.n
            idx = list(range(len(self.levels)))
            if self.order_mode == "desc" or (self.order_mode == "asc-desc" and last):
                idx.reverse()
            for i in idx:
                (level, factor, w, h), p = self.levels[i], self.pipes[i]
                st = sts[self.level_stream[i] % len(sts)]
                dst = p.frames
                with t.cuda.stream(st):
                    if level == 0 and not whole:
                        dst.data[:m].copy_(src.data[a:a + m])
                    elif level != 0:
                        _native.call("hog_resize_bilinear", D.ptr(src.data) + a * src.fstride, m,
                                     self.c, self.h, self.w, src.pitch, src.cstride, src.fstride,
                                     h, w, self.h / h, self.w / w, D.ptr(dst.data), dst.pitch,
                                     dst.cstride, dst.fstride, D.stream_handle(st))
                    pev = None
                    if plane_events is not None:
                        pev = []
                        for _ in range(p.chunks):
                            e0 = t.cuda.Event(enable_timing=True)
                            e1 = t.cuda.Event(enable_timing=True)
                            e0.record(st)
                            e1.record(st)
                            pev.append((e0, e1))
                            plane_events.append(
                                (e0, e1, p.plane_kernel_bytes_per_frame() * p.n // p.chunks))
                    if whole:
                        p.run(st, plane_events=pev,
                              frames_ptr=D.ptr(src.data) + a * src.fstride if level == 0 else None,
                              scores_ptr=D.ptr(self.scores[level][a]))
                    else:
                        p.run(st, plane_events=pev)
                        self.scores[level][a:a + m].copy_(p.scores[:m])
                if level_done is not None:
                    level_done(level, a, m, st)
        for st in sts[1:]:
            main.wait_stream(st)

    def pixels_per_frame(self) -> int:
        """Pixels of every pyramid level of one frame."""
        return sum(w * h for (_, _, w, h) in self.levels)

    def bytes_alg_per_frame(self) -> int:
        """SURVEY §8d for c5: per level bytes_alg, plus the resize (w*h written,
        min(H, 2h)*W source rows read) for levels >= 1."""
        b = 0
        for (level, _, w, h), p in zip(self.levels, self.pipes):
            b += p.bytes_alg_per_frame()
            if level:
                b += self.c * (w * h + min(self.h, 2 * h) * self.w)
        return b

    def launches_per_run(self) -> int:
        per_chunk = sum(p.launches_per_run() + (1 if lv else 0)
                        for (lv, _, _, _), p in zip(self.levels, self.pipes))
        return per_chunk * ((self.n + self.chunk - 1) // self.chunk)

    @on_device
    def detections(self, frame: int, threshold: float, iou_threshold: float | None = None,
                   window=(64, 128)):
        """One frame's boxes as pyramid_scan returns them (detector.py:252-268),
        optionally followed by greedy NMS (detector.py:285-299).  Per level the
        hits are compacted on the device with the level's scale and clamped to
        the original frame; NMS sorts and suppresses the concatenation there."""
        from . import detections as DT

        t = D.torch()
        bl, sl, cl = [], [], []
        for (level, factor, w, h), p in zip(self.levels, self.pipes):
            ww, wh = DT.window_box_size(window[0], window[1], factor)
            boxes, sc, _, counts = DT.compact(self.scores[level][frame:frame + 1], p.oxs, p.oys,
                                              threshold, factor, ww, wh, clamp=(self.w, self.h))
            k = int(counts[0])
            bl.append(boxes[0, :k])
            sl.append(sc[0, :k])
            cl.append(t.full((k,), float(factor), dtype=t.float64, device=boxes.device))
        b, s, c = t.cat(bl), t.cat(sl), t.cat(cl)
        if iou_threshold is not None and len(s):
            kt = t.as_tensor(DT.nms_indices(b, s, c, iou_threshold), device=b.device)
            b, s, c = b[kt], s[kt], c[kt]
        return DT.to_detections(b.cpu().numpy(), s.cpu().numpy(), c.cpu().numpy())
