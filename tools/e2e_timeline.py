"""Per-job timeline of bench.py's c2 e2e step (no nsys in the image): CUDA
events around each chunk's H2D copy, kernels and D2H copy, printed as
start/end offsets from the step start.  Eager launches (the bench replays the
same work as one CUDA graph).

    python tools/e2e_timeline.py [--chunk 64] [--slots 4] [--tail 4]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1703_06256_b200 as H  # noqa: E402
from paper_1703_06256_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--chunk", type=int, default=64)
ap.add_argument("--slots", type=int, default=4)
ap.add_argument("--tail", type=int, default=4)
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
nf = cfg.frames
frames = synth.make_batch(cfg, 0, nf)
sizes = [a.chunk] * (nf // a.chunk) + ([nf % a.chunk] if nf % a.chunk else [])
if a.tail > 1 and sizes[-1] >= a.tail:
    last = sizes.pop()
    sizes += [last // a.tail] * (a.tail - 1) + [last - (last // a.tail) * (a.tail - 1)]
w, b = synth.make_weights(cfg) if cfg.scored else (None, 0.0)
streams = [torch.cuda.Stream() for _ in range(min(a.slots, len(sizes)))]
pipes = {}
jobs, s0 = [], 0
for j, sz in enumerate(sizes):
    si = j % len(streams)
    if (si, sz) not in pipes:
        pipes[(si, sz)] = H.HogPipeline(sz, cfg.channels, cfg.height, cfg.width, cfg.bins,
                                        stride=cfg.stride, normalization=cfg.normalization,
                                        weights=w, bias=b)
    jobs.append((si, s0, s0 + sz, pipes[(si, sz)]))
    s0 += sz
host_in = torch.from_numpy(frames).pin_memory()
res = jobs[0][3].result()
host_out = torch.empty((nf,) + tuple(res.shape[1:]), dtype=res.dtype).pin_memory()


def ev():
    return torch.cuda.Event(enable_timing=True)


def step(record):
    cur = torch.cuda.current_stream()
    t0 = ev()
    t0.record(cur)
    for st in streams:
        st.wait_stream(cur)
    marks = []
    for si, x0, x1, q in jobs:
        st = streams[si]
        with torch.cuda.stream(st):
            e = [ev() for _ in range(4)]
            e[0].record(st)
            q.frames.data[..., : cfg.width].copy_(host_in[x0:x1], non_blocking=True)
            e[1].record(st)
            q.run(stream=st)
            e[2].record(st)
            host_out[x0:x1].copy_(q.result(), non_blocking=True)
            e[3].record(st)
            marks.append((si, x1 - x0, e))
    for st in streams:
        cur.wait_stream(st)
    t1 = ev()
    t1.record(cur)
    torch.cuda.synchronize()
    if record:
        print(f"step {t0.elapsed_time(t1):.3f} ms  ({len(jobs)} jobs, {len(streams)} streams)")
        for si, n, e in marks:
            t = [t0.elapsed_time(x) for x in e]
            print(f"  s{si} {n:3d} fr  h2d {t[0]:6.3f}-{t[1]:6.3f} ({t[1]-t[0]:.3f})  "
                  f"kern -{t[2]:6.3f} ({t[2]-t[1]:.3f})  d2h -{t[3]:6.3f} ({t[3]-t[2]:.3f})")


for i in range(4):
    step(i == 3)
