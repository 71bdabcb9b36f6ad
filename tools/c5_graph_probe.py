"""c5 pyramid step launched eagerly (ctypes launches from Python, ~240 per step) against the
same K steps captured as one CUDA graph."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1703_06256_b200 as H  # noqa: E402
from paper_1703_06256_b200 import synth  # noqa: E402

cfg = synth.CONFIGS["c5"]
nf, K = 32, 5
frames = synth.make_batch(cfg, 0, nf)
w, b = synth.make_weights(cfg)
p = H.PyramidPipeline(nf, 1, cfg.height, cfg.width, cfg.bins, stride=cfg.stride,
                      scale_step=cfg.pyramid_step, weights=w, bias=b, chunk=16)
p.upload(frames)
for _ in range(3):
    p.run()
torch.cuda.synchronize()
ref = [s.clone() for s in p.scores]


def timed(fn):
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a.record()
    fn()
    z.record()
    host = time.perf_counter() - t0
    torch.cuda.synchronize()
    return a.elapsed_time(z) / K, host * 1e3 / K


def eager():
    for _ in range(K):
        p.run()


for rep in range(2):
    ms, host = timed(eager)
    print(f"eager: {ms:.3f} ms per step (host enqueue {host:.2f} ms per step)")
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    eager()
torch.cuda.synchronize()
for rep in range(3):
    ms, host = timed(g.replay)
    print(f"graph: {ms:.3f} ms per step (host {host:.3f} ms per step)")
print("scores equal:", all(torch.equal(a, b_) for a, b_ in zip(ref, p.scores)))
