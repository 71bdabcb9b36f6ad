"""Device threshold compaction + greedy NMS against the
reference's own outputs (golden vectors) and the pinned oracle.  Boxes and
keep lists are exact; scores within the score tolerance of test_gpu_parity."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1703_06256_b200 as H  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1703_06256_b200 import detections as DT  # noqa: E402
from paper_1703_06256_b200 import synth  # noqa: E402


def dev(a, dtype):
    return torch.as_tensor(np.asarray(a, dtype=dtype), device="cuda")


@pytest.mark.parametrize("case,thrs", [("random", (0.0, 0.2, 0.45, 0.8, 1.0)),
                                       ("pyramid", (0.0, 0.3, 0.5, 1.0))])
def test_device_nms_golden(golden, case, thrs):
    key = "nms/random" if case == "random" else "pyramid"
    boxes, scores, scales = golden[f"{key}/boxes"], golden[f"{key}/score"], golden[f"{key}/scale"]
    for t in thrs:
        keep = DT.nms_indices(dev(boxes, np.int32), dev(scores, np.float64),
                              dev(scales, np.float64), t)
        assert np.array_equal(keep, golden[f"nms/{case}/{t}"]), t


def test_nms_api_matches_reference_on_pyramid(golden):
    img, w = golden["pyramid/image"], golden["pyramid/weights"]
    g = H.DescriptorGeometry(16, 16, 8, block=2, block_stride=1, bins=9)
    model = H.LinearModel(g, w, -0.5)
    dets = H.pyramid_scan(H.Image(img), model, 1.3, 4, float("-inf"))
    assert np.array_equal(np.array([d.box for d in dets]), golden["pyramid/boxes"])
    for t in (0.0, 0.3, 0.5, 1.0):
        kept = H.nms(dets, t)
        ref = [dets[i] for i in golden[f"nms/pyramid/{t}"]]
        assert [(d.box, d.scale) for d in kept] == [(d.box, d.scale) for d in ref]


@pytest.mark.parametrize("thr", [0.0, 1.5])
def test_pyramid_scan_threshold_golden(golden, thr):
    img, w = golden["pyramid/image"], golden["pyramid/weights"]
    g = H.DescriptorGeometry(16, 16, 8, block=2, block_stride=1, bins=9)
    dets = H.pyramid_scan(H.Image(img), H.LinearModel(g, w, -0.5), 1.3, 4, thr)
    ref_b, ref_s = golden[f"pyramid_thr{thr}/boxes"], golden[f"pyramid_thr{thr}/score"]
    assert np.array_equal(np.array([d.box for d in dets]).reshape(-1, 4), ref_b)
    np.testing.assert_allclose([d.score for d in dets], ref_s, rtol=1e-9, atol=1e-12)
    assert np.array_equal([d.scale for d in dets], golden[f"pyramid_thr{thr}/scale"])


def test_random_nms_vs_oracle():
    rng = np.random.default_rng(99)
    k = 3000
    boxes = np.stack([rng.integers(0, 900, k), rng.integers(0, 600, k),
                      rng.integers(4, 200, k), rng.integers(4, 200, k)], 1)
    scores = np.round(rng.normal(0, 1, k), 2)
    scales = rng.choice([1.0, 1.2], k)
    for t in (0.1, 0.5):
        keep = DT.nms_indices(dev(boxes, np.int32), dev(scores, np.float64), dev(scales, np.float64), t)
        assert np.array_equal(keep, O.nms(boxes, scores, scales, t))


def test_pipeline_detections_vs_oracle():
    # c1 geometry (one 800x600 frame, scored): threshold, then NMS, all on the device
    cfg = synth.CONFIGS["c1"]
    frames = synth.make_batch(cfg, 0, 1)
    w, b = synth.make_weights(cfg)
    p = H.HogPipeline(1, 1, cfg.height, cfg.width, cfg.bins, stride=cfg.stride, weights=w, bias=b)
    p.upload(frames)
    p.run()
    torch.cuda.synchronize()
    sc = p.scores[0].cpu().numpy()
    thr = float(np.quantile(sc, 0.9))
    rb, rs = O.hits(sc, p.oxs, p.oys, thr, 1.0, 64, 128)
    got = p.detections(thr)[0]
    assert np.array_equal(np.array([d.box for d in got]).reshape(-1, 4), rb)
    assert np.array_equal([d.score for d in got], rs)
    kept = p.detections(thr, iou_threshold=0.3)[0]
    ref = O.nms(rb, rs, np.ones(len(rs)), 0.3)
    assert [d.box for d in kept] == [tuple(int(v) for v in rb[i]) for i in ref]


def test_compaction_capacity_rerun_and_empty():
    s = torch.as_tensor(np.random.default_rng(3).normal(size=(2, 40, 50)), device="cuda")
    oxs, oys = np.arange(50) * 4, np.arange(40) * 4
    boxes, sc, win, counts = DT.compact(s, oxs, oys, 0.0, 1.0, 64, 128, cap=7)
    ref = (s > 0).sum(dim=(1, 2)).cpu().numpy()
    assert np.array_equal(counts, ref) and boxes.shape[1] >= ref.max()
    for f in range(2):
        idx = np.flatnonzero(s[f].cpu().numpy().ravel() > 0)
        assert np.array_equal(win[f, :counts[f]].cpu().numpy(), idx)
    _, _, _, none = DT.compact(s, oxs, oys, 1e9, 1.0, 64, 128)
    assert none.sum() == 0
    assert DT.nms_indices(torch.zeros((0, 4), dtype=torch.int32, device="cuda"),
                          torch.zeros(0, dtype=torch.float64, device="cuda"),
                          torch.zeros(0, dtype=torch.float64, device="cuda"), 0.5).size == 0


def test_pyramid_pipeline_detections_nms():
    # batched pyramid (c5 geometry on a crop) -> per-level device compaction ->
    # device NMS == oracle restatement of pyramid_scan + nms
    cfg = synth.CONFIGS["c5"]
    img = synth.make_batch(cfg, 1, 1)[:, :, :300, :420].copy()
    rng = np.random.default_rng(8)
    w = rng.normal(0, 0.01, 128 * cfg.bins)
    p = H.PyramidPipeline(1, 1, 300, 420, cfg.bins, stride=8, scale_step=1.2, weights=w, bias=0.0)
    p.upload(img)
    p.run()
    torch.cuda.synchronize()
    g = O.Geometry(64, 128, 8, 1, 1, cfg.bins)
    lut = O.build_lut(cfg.bins)
    allsc = np.concatenate([p.scores[lv][0].cpu().numpy().ravel() for lv, *_ in p.levels])
    thr = float(np.quantile(allsc, 0.7))
    bl, sl, cl = [], [], []
    for (level, factor, lw, lh), q in zip(p.levels, p.pipes):
        lim = img[0] if level == 0 else O.resize_bilinear(img[0], lw, lh)
        sc = p.scores[level][0].cpu().numpy()
        ref_sc = O.scan_scores(O.integral_stack(O.gradient_map(lim, lut), cfg.bins), g, 8, w, 0.0)
        np.testing.assert_allclose(sc, ref_sc, rtol=1e-9, atol=1e-12)
        b, s = O.hits(sc, q.oxs, q.oys, thr, factor, int(round(64 * factor)),
                      int(round(128 * factor)), clamp=(420, 300))
        bl.append(b)
        sl.append(s)
        cl.append(np.full(len(s), factor))
    rb, rs, rc = np.concatenate(bl), np.concatenate(sl), np.concatenate(cl)
    got = p.detections(0, thr)
    assert np.array_equal(np.array([d.box for d in got]).reshape(-1, 4), rb)
    kept = p.detections(0, thr, iou_threshold=0.4)
    ref = O.nms(rb, rs, rc, 0.4)
    assert [(d.box, d.scale) for d in kept] == [(tuple(int(v) for v in rb[i]), rc[i]) for i in ref]


def test_nms_api_greedy_definition():
    rng = np.random.default_rng(3)
    for _ in range(30):
        dets = [H.Detection(int(rng.integers(0, 40)), int(rng.integers(0, 40)),
                            int(rng.integers(4, 20)), int(rng.integers(4, 20)),
                            float(rng.normal())) for _ in range(int(rng.integers(0, 20)))]
        thr = float(rng.uniform(0, 1))
        kept = H.nms(dets, thr)
        for i, a in enumerate(kept):
            for b in kept[i + 1:]:
                assert H.iou(a.box, b.box) <= thr
        assert [k.score for k in kept] == sorted([k.score for k in kept], reverse=True)
        ref = O.nms([d.box for d in dets], [d.score for d in dets], [d.scale for d in dets], thr)
        assert [id(k) for k in kept] == [id(dets[i]) for i in ref]


def test_random_nms_float_boxes_vs_oracle():
    """Non-integer boxes (a caller's own Detections) take hog_nms_f64: same
    keep list as the reference's Python-float IoU, including y/x ties."""
    rng = np.random.default_rng(7)
    k = 2500
    boxes = np.stack([rng.integers(0, 300, k) / 3.0, rng.integers(0, 200, k) * 0.1,
                      rng.integers(12, 600, k) / 3.0, rng.integers(40, 2000, k) * 0.1], 1)
    scores = np.round(rng.normal(0, 1, k), 1)  # many score ties -> (y, x, scale) order
    scales = rng.choice([1.0, 1.2, 1.44], k)
    for t in (0.0, 0.3, 0.5, 1.0):
        keep = DT.nms_indices(dev(boxes, np.float64), dev(scores, np.float64),
                              dev(scales, np.float64), t)
        assert np.array_equal(keep, O.nms(boxes, scores, scales, t, float_boxes=True))


def test_nms_api_float_detections():
    rng = np.random.default_rng(11)
    for _ in range(20):
        dets = [H.Detection(float(rng.integers(0, 80)) / 4, float(rng.integers(0, 80)) / 4,
                            float(rng.integers(8, 80)) / 4, float(rng.integers(8, 80)) / 4,
                            float(np.round(rng.normal(), 1)), float(rng.choice([1.0, 1.2])))
                for _ in range(int(rng.integers(1, 40)))]
        thr = float(rng.uniform(0, 1))
        kept = H.nms(dets, thr)
        ref = O.nms([d.box for d in dets], [d.score for d in dets], [d.scale for d in dets], thr,
                    float_boxes=True)
        assert [id(k) for k in kept] == [id(dets[i]) for i in ref]
