"""Plane-kernel time vs band rows R (HOGB200_BAND_ROWS) per frame shape.

    python tools/band_sweep.py [--shapes c2,c4,c5l0,c5l3] [--rows 16,32,64,...]

For each shape a fresh HogPipeline per R (scratch depends on R); the plane
kernel is timed with the stage events of run_staged (median of 7), and the
CTA-wave count the launch implies is printed beside it.
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1703_06256_b200 as H  # noqa: E402
from paper_1703_06256_b200 import synth  # noqa: E402
from paper_1703_06256_b200.pipeline import pyramid_levels  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="c2,c4,c3,c5l0,c5l1,c5l3,c5l6")
ap.add_argument("--rows", default="0,16,24,32,40,48,64,80,96,128,160,192,240")
a = ap.parse_args()


def shape(key):
    if key.startswith("c5l"):
        cfg = synth.CONFIGS["c5"]
        lv = int(key[3:])
        _, _, w, h = pyramid_levels(cfg.width, cfg.height, 64, 128, 1.2)[lv]
        return cfg, 16, h, w
    cfg = synth.CONFIGS[key]
    return cfg, cfg.frames, cfg.height, cfg.width


for key in a.shapes.split(","):
    cfg, n, h, w = shape(key)
    rng = np.random.default_rng(1)
    base = synth.make_frame(cfg, 0)
    frames = np.empty((n, cfg.channels, h, w), np.uint8)
    for i in range(n):  # cheap distinct frames: shifted crops of one blurred frame
        y = int(rng.integers(0, base.shape[1] - h + 1))
        x = int(rng.integers(0, base.shape[2] - w + 1))
        frames[i] = base[:, y:y + h, x:x + w]
    for R in [int(r) for r in a.rows.split(",")]:
        if R:
            os.environ["HOGB200_BAND_ROWS"] = str(R)
        else:
            os.environ.pop("HOGB200_BAND_ROWS", None)
        p = H.HogPipeline(n, cfg.channels, h, w, cfg.bins, stride=cfg.stride)
        p.upload(frames)
        ts = []
        for it in range(10):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            for e in ev:
                e.record()
            p.run_staged(ev)
            torch.cuda.synchronize()
            if it >= 3:
                ts.append(ev[2].elapsed_time(ev[3]))
        ms = statistics.median(ts)
        gb = p.plane_kernel_bytes_per_frame() * n / ms / 1e6
        print(f"{key:6s} n={n:3d} {w}x{h} R={R or 'auto':>4}  planes {ms:8.3f} ms  {gb:7.0f} GB/s",
              flush=True)
        del p
        torch.cuda.empty_cache()
