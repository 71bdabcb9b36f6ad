"""Config c5 at full size: one 7680x4320 frame through PyramidPipeline, every
one of its 20 pyramid levels checked against the oracle (detector.py:224-269).

Per level: the resized image (bit-exact, detector.py:202-221), the bin map
(bit-exact, gradient.py:95-121), the cell grid (bit-exact,
descriptor.py:176-185) and the window scores (fp64, within the score
tolerance; the north star allows 1e-5 relative).  Level 0's whole plane
stack (18 x 4321 x 7681 uint32, 2.4 GB) is compared bin by bin against the
oracle's integral_stack (integral.py:58-87).  The oracle levels run on all
host threads (one level per thread; ctypes drops the GIL).
"""
import os
from concurrent.futures import ThreadPoolExecutor

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


@pytest.fixture(scope="module")
def c5_run():
    cfg = synth.CONFIGS["c5"]
    frame = synth.make_frame(cfg, 0)  # (1, 4320, 7680)
    w, bias = synth.make_weights(cfg)
    p = H.PyramidPipeline(1, 1, cfg.height, cfg.width, cfg.bins, stride=cfg.stride,
                          scale_step=cfg.pyramid_step, weights=w, bias=bias, chunk=1)
    p.upload(frame[None])
    p.run()
    torch.cuda.synchronize()
    return cfg, frame, w, bias, p


def _oracle_level(frame, level, lw, lh, lut, cfg, w, bias):
    img = frame if level == 0 else O.resize_bilinear(frame, lw, lh)
    cells = O.gradient_map(img, lut)
    _, grid, scores = O.run_batch(img[None], lut, cfg.bins, 8, 64, 128, cfg.stride, 1, w, bias,
                                  threads=1, want_outputs=True)
    return img, cells, grid[0], scores[0]


def test_c5_every_level_vs_oracle(c5_run):
    cfg, frame, w, bias, p = c5_run
    g = O.Geometry(64, 128, 8, 1, 1, cfg.bins)
    levels = O.pyramid_levels(cfg.width, cfg.height, g, cfg.pyramid_step)
    assert len(levels) == 20
    assert [tuple(lv) for lv in p.levels] == [tuple(lv) for lv in levels]
    lut = O.build_lut(cfg.bins)
    # biggest levels first so the pool's tail is short
    order = sorted(levels, key=lambda t: -t[2] * t[3])
    with ThreadPoolExecutor(max_workers=max(2, os.cpu_count() or 2)) as pool:
        futs = {lv[0]: pool.submit(_oracle_level, frame, lv[0], lv[2], lv[3], lut, cfg, w, bias)
                for lv in order}
        tol = score_tol(w)
        windows = 0
        for (level, factor, lw, lh), q in zip(levels, p.pipes):
            img, cells, grid, scores = futs[level].result()
            if level:  # the level image the pipeline binned (resized on the device)
                dev_img = q.frames.data[0, :, :, :lw].cpu().numpy()
                assert np.array_equal(dev_img, img), f"level {level}: resize differs"
            assert np.array_equal(q.binmap_view()[0].cpu().numpy().astype(np.int16), cells), \
                f"level {level}: bin map differs"
            assert q.fused
            assert np.array_equal(q.grid[0].cpu().numpy().astype(np.int64), grid), \
                f"level {level}: cell grid differs"
            got = p.scores[level][0].cpu().numpy()
            assert got.shape == scores.shape
            err = np.abs(got - scores)
            assert err.max() <= tol, f"level {level}: max score error {err.max():.3g} > {tol:.3g}"
            rel = err / np.maximum(np.abs(scores), 1e-300)
            assert rel.max() < 1e-5, f"level {level}: max relative error {rel.max():.3g}"
            windows += scores.size
    assert windows == 1_588_705  # windows over the 8K pyramid


def test_c5_level0_whole_planes(c5_run):
    """Level 0's whole 2.4 GB plane stack, bin by bin, bit-exact."""
    cfg, frame, w, bias, p = c5_run
    q = p.pipes[0]
    # level 0 reads the source frame in place; re-run it through its own
    # buffers' planes (the pyramid run already wrote them for this frame)
    lut = O.build_lut(cfg.bins)
    cells = O.gradient_map(frame, lut)
    ref = O.integral_stack(cells, cfg.bins)  # (18, 4321, 7681) uint32
    gpu = q.planes_view()[0]
    for b in range(cfg.bins):
        got = gpu[b].cpu().numpy().view(np.uint32)
        assert np.array_equal(got, ref[b]), f"level-0 plane of bin {b} differs"
    # every interior non-sentinel pixel counted once
    assert int(ref[:, -1, -1].astype(np.int64).sum()) == int((cells >= 0).sum())
