#!/usr/bin/env python
"""hog_integral throughput vs N_b (the drop-in build_integral_stack path):
<= 18 bins run the single-write plane kernel directly, more bins run it in
groups of <= 16 bins over a bin-offset copy of the bin map.  Prints achieved
GB/s of plane bytes (4*N_b*(H+1)*(W+1) per frame) against the copy peak.
usage: python tools/integral_bins_probe.py [frames] [h] [w]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1703_06256_b200 import _native, device as D, synth  # noqa: E402
from paper_1703_06256_b200.gradient import build_lut, grad_bin_device  # noqa: E402
from paper_1703_06256_b200.integral import integral_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
h = int(sys.argv[2]) if len(sys.argv) > 2 else 480
w = int(sys.argv[3]) if len(sys.argv) > 3 else 640
cfg = synth.CONFIGS["c2"]
frames = np.ascontiguousarray(synth.make_batch(cfg, 0, n)[:, :, :h, :w])
fr = D.upload_frames(frames)
try:
    peak = float(json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"])
except Exception:
    peak = 6650.0
for bins in (8, 16, 18, 20, 32, 48, 64):
    bm = grad_bin_device(fr, build_lut(bins))
    pl = integral_device(bm, bins)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        integral_device(bm, bins, out=pl)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts[1:])
    gb = 4 * bins * (h + 1) * (w + 1) * n / 1e9
    print(json.dumps({"bins": bins, "frames": n, "ms": round(ms, 4), "plane_gb": round(gb, 3),
                      "gbs": round(gb / (ms / 1e3), 1), "frac": round(gb / (ms / 1e3) / peak, 3),
                      "lib": os.path.basename(_native.LIB_PATH)}))
