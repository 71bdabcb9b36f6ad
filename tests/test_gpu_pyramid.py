"""Config c5 (8K, N_b = 18, 20-level pyramid, stride 8) on the GPU.

Full-size checks use properties that do not need the whole 2.4 GB plane
stack on the host: plane values in columns < X depend only on pixels in
columns < X, so the oracle's planes of a full-height, 512-column crop must
equal the GPU planes exactly there; the bin map and every level's resize are
compared whole; cells and windows inside the crop are compared exactly (grid)
and within the score tolerance.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1703_06256_b200 as H  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1703_06256_b200 import synth  # noqa: E402


def score_tol(w):
    return 1e-12 * float(np.abs(w).sum()) * 64 + 1e-12


@pytest.mark.parametrize("n,chunk,streams", [(2, 2, 1), (3, 2, 3)])
def test_pyramid_pipeline_small_vs_oracle(n, chunk, streams):
    """Whole chunks read the source frames in place and write the pyramid's
    score maps directly; a partial last chunk goes through the level buffers;
    levels spread over several streams give the same maps."""
    cfg = synth.CONFIGS["c5"]
    frames = np.stack([synth.make_frame(cfg, i)[:, :300, :520] for i in range(n)])
    w, bias = synth.make_weights(cfg)
    p = H.PyramidPipeline(n, 1, 300, 520, 18, stride=8, scale_step=1.2, weights=w, bias=bias,
                          chunk=chunk, streams=streams)
    p.upload(frames)
    p.run()
    torch.cuda.synchronize()
    g = O.Geometry(64, 128, 8, 1, 1, 18)
    lut = O.build_lut(18)
    levels = O.pyramid_levels(520, 300, g, 1.2)
    assert [(lv, f, ww, hh) for lv, f, ww, hh in p.levels] == levels
    for i in range(n):
        for (level, factor, lw, lh) in levels:
            img = frames[i] if level == 0 else O.resize_bilinear(frames[i], lw, lh)
            planes = O.integral_stack(O.gradient_map(img, lut), 18)
            ref = O.scan_scores(planes, g, 8, w, bias)
            np.testing.assert_allclose(p.scores[level][i].cpu().numpy(), ref, rtol=0,
                                       atol=score_tol(w))
    # boxes exactly as pyramid_scan maps them (detector.py:252-268)
    dets = p.detections(0, float("-inf"))
    ref = H.pyramid_scan(H.Image(frames[0]), H.LinearModel(
        H.DescriptorGeometry(64, 128, 8, 1, 1, 18), w, bias), 1.2, 8, float("-inf"))
    assert [(d.x, d.y, d.w, d.h, d.scale) for d in dets] == \
        [(d.x, d.y, d.w, d.h, d.scale) for d in ref]
    np.testing.assert_allclose([d.score for d in dets], [d.score for d in ref], rtol=0,
                               atol=score_tol(w))


def test_c5_full_size_level0_and_resizes():
    cfg = synth.CONFIGS["c5"]
    frame = synth.make_frame(cfg, 0)  # (1, 4320, 7680)
    w, bias = synth.make_weights(cfg)
    p = H.HogPipeline(1, 1, cfg.height, cfg.width, 18, stride=8, weights=w, bias=bias)
    assert p.fused
    p.upload(frame[None])
    p.run()
    torch.cuda.synchronize()
    lut = O.build_lut(18)
    cells = O.gradient_map(frame, lut)
    assert np.array_equal(p.binmap_view()[0].cpu().numpy().astype(np.int16), cells)
    X = 512
    planes_crop = O.integral_stack(np.ascontiguousarray(cells[:, : X]), 18)  # (18, 4321, 513)
    gpu = p.planes_view()[0, :, :, : X + 1].cpu().numpy().view(np.uint32)
    assert np.array_equal(gpu, planes_crop)
    # last-column totals of the whole stack: every interior non-sentinel pixel counted once
    tot = p.planes_view()[0, :, -1, -1].cpu().numpy().astype(np.int64)
    assert tot.sum() == int((cells >= 0).sum())
    # cells and windows entirely inside the crop
    g = O.Geometry(64, 128, 8, 1, 1, 18)
    ncx_crop = (X - 8) // 8 + 1
    cxs = np.arange(ncx_crop) * 8
    cys = np.arange(p.ncy) * 8
    grid_ref = O.cell_grid(planes_crop, cxs, cys, 8)
    assert np.array_equal(p.grid[0, :, :ncx_crop].cpu().numpy().astype(np.int64), grid_ref)
    ref_scores = O.scan_scores(planes_crop[:, :, :], g, 8, w, bias)  # windows with ox+64 <= X
    got = p.scores[0, :, : ref_scores.shape[1]].cpu().numpy()
    np.testing.assert_allclose(got, ref_scores, rtol=0, atol=score_tol(w))
    # every pyramid level's resize of the full frame, bit-exact
    for (level, factor, lw, lh) in H.pyramid_levels(cfg.width, cfg.height, H.DescriptorGeometry(
            64, 128, 8, 1, 1, 18), 1.2)[1:4]:
        out = H.resize_bilinear(H.Image(frame), lw, lh)
        assert O.sha256(out.planes) == O.sha256(O.resize_bilinear(frame, lw, lh))
