"""Per-job timeline of bench.py's c2 e2e step (no nsys in the image): CUDA
events around each chunk's H2D copy, kernels and D2H copy, printed as
start/end offsets from the step start.  Eager launches (the bench replays the
same work as one CUDA graph).

    python tools/e2e_timeline.py [--chunk 64] [--slots 4] [--tail 4] [--multi]

Default: bench.py's schedule (one H2D stream, one compute stream, one D2H
stream, `slots` buffer sets).  --multi: the earlier schedule, every job's
copy-compute-copy on one of `slots` streams (profiles/r1b_e2e_timeline_multistream.txt:
the H2D copies of different streams share the link and all land late).
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
ap.add_argument("--multi", action="store_true")
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
nf = cfg.frames
frames = synth.make_batch(cfg, 0, nf)
sizes = [a.chunk] * (nf // a.chunk) + ([nf % a.chunk] if nf % a.chunk else [])
if a.tail > 1 and sizes[-1] >= a.tail:
    last = sizes.pop()
    sizes += [last // a.tail] * (a.tail - 1) + [last - (last // a.tail) * (a.tail - 1)]
w, b = synth.make_weights(cfg) if cfg.scored else (None, 0.0)
streams_slots = list(range(min(a.slots, len(sizes))))
streams = [torch.cuda.Stream() for _ in (streams_slots if a.multi else [0])]
copy = [] if a.multi else [torch.cuda.Stream(), torch.cuda.Stream()]
pipes = {}
jobs, s0 = [], 0
for j, sz in enumerate(sizes):
    si = j % len(streams_slots)
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
    for st in streams + copy:
        st.wait_stream(cur)
    marks, done = [], []
    for j, (si, x0, x1, q) in enumerate(jobs):
        e = [ev() for _ in range(4)]
        if a.multi:
            st_in = st_c = st_out = streams[si]
        else:
            st_in, st_c, st_out = copy[0], streams[0], copy[1]
            if j >= len(streams_slots):
                st_in.wait_event(done[j - len(streams_slots)][0])
        with torch.cuda.stream(st_in):
            e[0].record(st_in)
            q.frames.data[..., : cfg.width].copy_(host_in[x0:x1], non_blocking=True)
            e[1].record(st_in)
        st_c.wait_event(e[1])
        if not a.multi and j >= len(streams_slots):
            st_c.wait_event(done[j - len(streams_slots)][1])
        q.run(stream=st_c)
        e[2].record(st_c)
        st_out.wait_event(e[2])
        with torch.cuda.stream(st_out):
            host_out[x0:x1].copy_(q.result(), non_blocking=True)
            e[3].record(st_out)
        done.append((e[2], e[3]))
        marks.append((si, x1 - x0, e))
    for st in streams + copy:
        cur.wait_stream(st)
    t1 = ev()
    t1.record(cur)
    torch.cuda.synchronize()
    if record:
        print(f"step {t0.elapsed_time(t1):.3f} ms  ({len(jobs)} jobs, "
              f"{'multi-stream' if a.multi else 'in-order copy streams'}, {a.slots} slots)")
        for si, n, e in marks:
            t = [t0.elapsed_time(x) for x in e]
            print(f"  s{si} {n:3d} fr  h2d {t[0]:6.3f}-{t[1]:6.3f} ({t[1]-t[0]:.3f})  "
                  f"kern -{t[2]:6.3f} ({t[2]-t[1]:.3f})  d2h -{t[3]:6.3f} ({t[3]-t[2]:.3f})")


for i in range(4):
    step(i == 3)
