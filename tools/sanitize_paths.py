"""Every device entry point once, at small sizes, for compute-sanitizer
(memcheck / racecheck / synccheck stand in for the reference's
determinism tests).  Run it bare first (it checks the outputs against the
oracle, so the sanitizer sees the real code paths), then e.g.

    compute-sanitizer --tool memcheck  python tools/sanitize_paths.py
    compute-sanitizer --tool racecheck python tools/sanitize_paths.py
    compute-sanitizer --tool synccheck python tools/sanitize_paths.py

Band-row tuning is off (HOGB200_TUNE=0): it times kernels on unwritten frames.

On this round's GPU pool compute-sanitizer is closed by the operators (it left
GPUs needing a reset; profiles/r1b_compute_sanitizer_unavailable.txt), so the
bare run -- every entry point at small, misaligned and ragged sizes against
the oracle (profiles/r1b_all_paths_small_vs_oracle.txt) -- is the check.
"""
import os
import sys

os.environ.setdefault("HOGB200_TUNE", "0")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1703_06256_b200 as H  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1703_06256_b200 import synth  # noqa: E402


def check(name, ok):
    print(f"{name:48s} {'ok' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        raise SystemExit(1)


def crop(key, n, h, w, first=3):
    cfg = synth.CONFIGS[key]
    return cfg, np.ascontiguousarray(synth.make_batch(cfg, first, n)[:, :, :h, :w])


# 1. fused pipeline (bin map, planes, byte grid), gray stride 4 and RGB, + scores
for key, (h, w) in (("c2", (150, 300)), ("c4", (140, 330)), ("c3", (130, 270))):
    cfg, fr = crop(key, 2, h, w)
    wts, b = (synth.make_weights(cfg) if cfg.scored else (None, 0.0))
    p = H.HogPipeline(2, cfg.channels, h, w, cfg.bins, stride=cfg.stride,
                      normalization=cfg.normalization, weights=wts, bias=b)
    p.upload(fr)
    p.run()
    torch.cuda.synchronize()
    lut = O.build_lut(cfg.bins)
    cells = O.gradient_map(fr[1], lut)
    planes = O.integral_stack(cells, cfg.bins)
    check(f"{key} bin map / planes", np.array_equal(p.binmap_view()[1].cpu().numpy(), cells)
          and np.array_equal(p.planes_view()[1].cpu().numpy().view(np.uint32), planes))
    if p.scores is not None:
        g = O.Geometry(64, 128, 8, 1, 1, cfg.bins, cfg.normalization)
        ref = O.scan_scores(planes, g, cfg.stride, wts, b)
        check(f"{key} scores", np.allclose(p.scores[1].cpu().numpy(), ref, rtol=1e-9, atol=1e-9))

# 2. chunked three-stream pipeline and pipelined batches
cfg, fr = crop("c4", 3, 140, 330)
wts, b = synth.make_weights(cfg)
p = H.HogPipeline(3, 3, 140, 330, cfg.bins, stride=8, weights=wts, bias=b, chunks=3)
p.upload(fr)
p.run()
q = H.HogPipeline(3, 3, 140, 330, cfg.bins, stride=8, weights=wts, bias=b)
q.upload(fr)
q.run(pipelined=True)
q.run(pipelined=True)
q.join()
torch.cuda.synchronize()
check("chunked / pipelined scores", torch.equal(p.scores, q.scores))

# 3. general path: planes -> cell grid -> block-2 L2 window descriptor
cfg, fr = crop("c3", 1, 140, 200)
img = H.Image(fr[0])
lut = H.build_lut(9)
st = H.build_integral_stack(H.gradient_map(img, lut))
geo = H.DescriptorGeometry(64, 128, 8, block=2, block_stride=1, bins=9, normalization="l2")
d = H.window_descriptor(st, (8, 4), geo)
ref = O.window_descriptor(O.integral_stack(O.gradient_map(fr[0], O.build_lut(9)), 9), (8, 4),
                          O.Geometry(64, 128, 8, 2, 1, 9, "l2"))
check("window_descriptor block 2 / l2", np.allclose(d, ref, rtol=0, atol=1e-12))

# 4. pyramid (resize + levels on 3 streams), detections + NMS
cfg = synth.CONFIGS["c5"]
fr = np.ascontiguousarray(synth.make_batch(cfg, 1, 1)[:, :, :300, :420])
wts, b = synth.make_weights(cfg)
pp = H.PyramidPipeline(1, 1, 300, 420, 18, stride=8, scale_step=1.2, weights=wts, bias=b, chunk=1)
pp.upload(fr)
pp.run()
dets = pp.detections(0, 0.0, iou_threshold=0.5)
torch.cuda.synchronize()
model = H.LinearModel(H.DescriptorGeometry(64, 128, 8, 1, 1, 18), wts, b)
ref = H.nms(H.pyramid_scan(H.Image(fr[0]), model, 1.2, 8, 0.0), 0.5)
check("pyramid detections + NMS", [(x.x, x.y, x.w, x.h) for x in dets] == [(x.x, x.y, x.w, x.h) for x in ref])

# 5. 16-bit planes and batched rectangle queries
small = np.ascontiguousarray(fr[0, :, :120, :150])
st16 = H.build_integral_stack(H.gradient_map(H.Image(small), H.build_lut(8)), acc_width=16)
ref16 = O.integral_stack(O.gradient_map(small, O.build_lut(8)), 8).astype(np.uint16)
check("integral16", np.array_equal(np.asarray(st16.planes), ref16))
r = H.Rect(5, 7, 60, 90)
check("rect_histogram", np.array_equal(np.asarray(H.rect_histogram(st16, r)),
                                       ref16[:, 90, 60].astype(np.int64) - ref16[:, 7, 60]
                                       - ref16[:, 90, 5] + ref16[:, 7, 5]))
print("all paths ok")
