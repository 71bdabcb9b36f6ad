"""Detections on the device: threshold compaction of a
score map into boxes, and greedy NMS.

The reference builds its detection list on the host, window by window
(detector.py:145-153, 194-199, 261-267) and runs greedy NMS over Python
objects (detector.py:272-299).  Here the score map never leaves the GPU:
``hog_detect`` writes only the hits (row-major, the reference's list order)
and ``hog_nms`` sorts and suppresses them on the device; the host receives
the surviving boxes.
"""
from __future__ import annotations

import numpy as np

from . import _native, device as D


def window_box_size(window_w: int, window_h: int, scale: float) -> tuple[int, int]:
    """detector.py:143-144: int(round(window * scale)) (Python round, half to even)."""
    return int(round(window_w * scale)), int(round(window_h * scale))


def compact(scores, oxs, oys, threshold: float, scale: float, ww: int, wh: int,
            clamp: tuple[int, int] = (0, 0), cap: int | None = None, stream=None):
    """Hits of a (n, noy, nox) float64 device score map with score > threshold.

    Returns (boxes, scores, windows, counts): device tensors boxes (n, cap, 4)
    int32 (x, y, w, h), scores (n, cap) float64, windows (n, cap) int64
    (iy * nox + ix), and the host array counts (n,) -- frame f's hits are
    rows [0, counts[f]) in row-major window order (detector.py:145-153)."""
    t = D.require_cuda()
    lib = _native.load()
    n, noy, nox = (int(v) for v in scores.shape)
    dev = scores.device
    oxs_d = t.as_tensor(np.asarray(oxs, dtype=np.int32), device=dev)
    oys_d = t.as_tensor(np.asarray(oys, dtype=np.int32), device=dev)
    sb = int(lib.hog_detect_scratch_bytes(n, noy * nox))
    scratch = t.empty(max(sb, 256), dtype=t.uint8, device=dev)
    count = t.zeros(n, dtype=t.int32, device=dev)
    cap = int(cap if cap is not None else min(noy * nox, 4096))
    while True:
        boxes = t.empty((n, max(cap, 1), 4), dtype=t.int32, device=dev)
        out_s = t.empty((n, max(cap, 1)), dtype=t.float64, device=dev)
        out_w = t.empty((n, max(cap, 1)), dtype=t.int64, device=dev)
        _native.call("hog_detect", D.ptr(scores), n, noy, nox, float(threshold), D.ptr(oxs_d),
                     D.ptr(oys_d), float(scale), int(ww), int(wh), int(clamp[0]), int(clamp[1]),
                     cap, D.ptr(boxes), D.ptr(out_s), D.ptr(out_w), D.ptr(count), D.ptr(scratch),
                     sb, D.stream_handle(stream))
        counts = count.cpu().numpy()
        need = int(counts.max()) if n else 0
        if need <= cap:
            return boxes, out_s, out_w, counts
        cap = need  # rerun with room for every hit


def nms_indices(boxes, scores, scales, iou_threshold: float, stream=None) -> np.ndarray:
    """detector.py:285-299 on the device: kept indices into the (N, 4) int32
    or float64 boxes / (N,) float64 scores / scales device tensors, in keep
    order (int32 boxes: hog_nms; float64 boxes: hog_nms_f64)."""
    t = D.require_cuda()
    n = int(boxes.shape[0])
    if n == 0:
        return np.zeros(0, dtype=np.int64)
    lib = _native.load()
    dev = boxes.device
    sb = int(lib.hog_nms_scratch_bytes(n))
    scratch = t.empty(max(sb, 256), dtype=t.uint8, device=dev)
    keep = t.empty(n, dtype=t.int32, device=dev)
    kc = t.zeros(1, dtype=t.int32, device=dev)
    boxes, scores, scales = boxes.contiguous(), scores.contiguous(), scales.contiguous()
    fn = "hog_nms_f64" if boxes.dtype == t.float64 else "hog_nms"
    if fn == "hog_nms" and boxes.dtype != t.int32:
        raise TypeError(f"boxes must be int32 or float64, got {boxes.dtype}")
    _native.call(fn, D.ptr(boxes), D.ptr(scores), D.ptr(scales), n, float(iou_threshold),
                 D.ptr(keep), D.ptr(kc), D.ptr(scratch), sb, D.stream_handle(stream))
    k = int(kc.item())
    return keep[:k].cpu().numpy().astype(np.int64)


def to_detections(boxes_h: np.ndarray, scores_h: np.ndarray, scales_h):
    """Host Detection objects from (k, 4) boxes, (k,) scores and scales."""
    from .detector import Detection

    sc = np.broadcast_to(np.asarray(scales_h, dtype=np.float64), scores_h.shape)
    return [Detection(x=int(b[0]), y=int(b[1]), w=int(b[2]), h=int(b[3]), score=float(s),
                      scale=float(c))
            for b, s, c in zip(boxes_h.tolist(), scores_h.tolist(), sc.tolist())]
