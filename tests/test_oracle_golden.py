"""Pin the CPU oracle (oracle/) against vectors the reference itself produced.

The golden vectors come from ``tests/golden/make_golden.py`` run against the
reference package.  Once these pass, the oracle is a trusted checker for the
CUDA path at sizes where the reference is too slow to call directly.
CPU only.
"""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1703_06256_b200 import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
CASES = ["gray45x37", "rgb48x40", "gray133x77", "rgb3x3", "gray300x200_b18",
         "rgbtie70x50", "c2frame0_crop"]


def test_lut_matches_reference_for_every_bin_count():
    # gradient.py:56-72 for N = 2..64; 261,121 entries each, via SHA-256
    ref = json.load(open(os.path.join(GOLDEN, "lut_sha256.json")))
    bad = [n for n in range(2, 65) if O.sha256(O.build_lut(n).astype("<i2")) != ref[str(n)]]
    assert bad == []


def test_lut_known_answers():
    # test_gradient.py:19-31 (reference known angles at N=8)
    t = O.build_lut(8)
    look = lambda dx, dy: int(t[dx + 255, dy + 255])  # noqa: E731
    assert [look(1, 0), look(0, 1), look(-1, 0), look(0, -1), look(0, 0), look(255, 255)] == \
        [0, 2, 4, 6, -1, 1]


def test_lut_full_tables(golden):
    for n in (8, 9):
        assert np.array_equal(O.build_lut(n).astype(np.int8), golden[f"lut{n}"])


@pytest.mark.parametrize("name", CASES)
def test_binmap_and_planes(golden, name):
    img, bins = golden[f"{name}/image"], int(golden[f"{name}/bins"])
    cells = O.gradient_map(img, O.build_lut(bins))
    assert np.array_equal(cells, golden[f"{name}/binmap"])
    planes = O.integral_stack(cells, bins)
    assert O.sha256(planes) == str(golden[f"{name}/planes_sha"])
    if f"{name}/planes" in golden.files:
        assert np.array_equal(planes, golden[f"{name}/planes"])


def _geom(gname, bins, norm):
    if gname == "g16b2":
        return O.Geometry(16, 16, 8, 2, 1, bins, norm)
    return O.Geometry(16, 24, 8, 2, 1, bins, norm)


@pytest.mark.parametrize("name", CASES)
def test_grids_and_descriptors(golden, name):
    img, bins = golden[f"{name}/image"], int(golden[f"{name}/bins"])
    planes = O.integral_stack(O.gradient_map(img, O.build_lut(bins)), bins)
    H, W = img.shape[1:]
    checked = 0
    for gname in ("g16b2", "g16x24"):
        for norm in ("none", "l1", "l2"):
            for stride in (1, 3, 8):
                key = f"{name}/{gname}/{norm}/s{stride}"
                if f"{key}/descs_sha" not in golden.files:
                    continue
                g = _geom(gname, bins, norm)
                oxs, oys = O.window_origins(W, H, g, stride)
                cxs, cys, col_idx, row_idx = O.cell_index(oxs, oys, g)
                grid = O.cell_grid(planes, cxs, cys, g.cell)
                if norm == "none":
                    assert np.array_equal(grid, golden[f"{key}/grid"])
                descs = np.stack([O.window_descriptor_from_grid(grid, row_idx[iy], col_idx[ix], g)
                                  for iy in range(len(oys)) for ix in range(len(oxs))])
                # normalised values are bit-exact too: integer sums, IEEE sqrt/div
                assert O.sha256(descs) == str(golden[f"{key}/descs_sha"])
                checked += 1
    if bins == 9 and H >= 24:
        assert checked > 0


def _score_tol(weights, grid_max):
    return 1e-12 * float(np.abs(weights).sum()) * max(1.0, grid_max) + 1e-12


@pytest.mark.parametrize("name", CASES)
def test_scan_scores(golden, name):
    img, bins = golden[f"{name}/image"], int(golden[f"{name}/bins"])
    planes = O.integral_stack(O.gradient_map(img, O.build_lut(bins)), bins)
    H, W = img.shape[1:]
    for gname in ("g16b2", "g16x24"):
        if f"{name}/{gname}/weights" not in golden.files:
            continue
        w = golden[f"{name}/{gname}/weights"]
        g = _geom(gname, bins, "none")
        for stride in (2, 4):
            s = O.scan_scores(planes, g, stride, w, 0.125)
            ref = golden[f"{name}/{gname}/scan_s{stride}/score"]
            np.testing.assert_allclose(s.ravel(), ref, rtol=0, atol=_score_tol(w, 64))
            oxs, oys = O.window_origins(W, H, g, stride)
            xy = np.array([(x, y) for y in oys for x in oxs])
            assert np.array_equal(xy, golden[f"{name}/{gname}/scan_s{stride}/xy"])
    for norm in ("none", "l2"):
        for stride in (4, 8):
            key = f"{name}/b1_{norm}/s{stride}"
            if f"{key}/score" not in golden.files:
                continue
            g = O.Geometry(16, 32, 8, 1, 1, bins, norm)
            w = golden[f"{key}/weights"]
            s = O.scan_scores(planes, g, stride, w, 0.0)
            np.testing.assert_allclose(s.ravel(), golden[f"{key}/score"], rtol=0,
                                       atol=_score_tol(w, 64))
            if norm == "none":
                oxs, oys = O.window_origins(W, H, g, stride)
                cxs, cys, _, _ = O.cell_index(oxs, oys, g)
                assert np.array_equal(O.cell_grid(planes, cxs, cys, 8), golden[f"{key}/grid"])


def test_config1_every_stage(golden):
    cfg = synth.CONFIGS["c1"]
    frame = synth.make_frame(cfg, 0)
    assert O.sha256(frame) == str(golden["c1/frame_sha"])
    cells = O.gradient_map(frame, O.build_lut(cfg.bins))
    assert O.sha256(cells) == str(golden["c1/binmap_sha"])
    planes = O.integral_stack(cells, cfg.bins)
    assert O.sha256(planes) == str(golden["c1/planes_sha"])
    g = O.Geometry(64, 128, 8, 1, 1, cfg.bins)
    oxs, oys = O.window_origins(cfg.width, cfg.height, g, cfg.stride)
    cxs, cys, _, _ = O.cell_index(oxs, oys, g)
    assert O.sha256(O.cell_grid(planes, cxs, cys, 8)) == str(golden["c1/grid_sha"])
    w, bias = synth.make_weights(cfg)
    _, grid, scores = O.run_batch(frame[None], O.build_lut(cfg.bins), cfg.bins, 8, 64, 128,
                                  cfg.stride, 1, w, bias, threads=2, want_outputs=True)
    ref = golden["c1/scores"]
    rel = np.abs(scores[0] - ref) / np.abs(ref)
    assert rel.max() < 1e-12


def test_resize_bit_exact(golden):
    src = golden["resize/src"]
    for (nw, nh) in ((80, 69), (40, 33), (97, 83), (13, 7), (96, 82)):
        assert np.array_equal(O.resize_bilinear(src, nw, nh), golden[f"resize/{nw}x{nh}"])


def test_resize_large_bit_exact(golden):
    big = synth.make_frame(synth.CONFIGS["c5"], 0)[:, :540, :960].copy()
    assert O.sha256(big) == str(golden["resize_big/src_sha"])
    for (nw, nh) in ((800, 450), (666, 375), (555, 312)):
        assert O.sha256(O.resize_bilinear(big, nw, nh)) == str(golden[f"resize_big/{nw}x{nh}_sha"])


def test_pyramid_level_loop(golden):
    # detector.py:224-269 restated with the oracle stages
    img = golden["pyramid/image"]
    w = golden["pyramid/weights"]
    g = O.Geometry(16, 16, 8, 2, 1, 9)
    H, W = img.shape[1:]
    lut = O.build_lut(9)
    boxes, scores, scales = [], [], []
    for level, factor, lw, lh in O.pyramid_levels(W, H, g, 1.3):
        scaled = img if level == 0 else O.resize_bilinear(img, lw, lh)
        planes = O.integral_stack(O.gradient_map(scaled, lut), 9)
        s = O.scan_scores(planes, g, 4, w, -0.5)
        oxs, oys = O.window_origins(lw, lh, g, 4)
        ww, wh = int(round(16 * factor)), int(round(16 * factor))
        for iy, oy in enumerate(oys):
            for ix, ox in enumerate(oxs):
                x = min(max(int(round(ox * factor)), 0), W - 1)
                y = min(max(int(round(oy * factor)), 0), H - 1)
                boxes.append((x, y, min(ww, W - x), min(wh, H - y)))
                scores.append(s[iy, ix])
                scales.append(factor)
    assert np.array_equal(np.array(boxes), golden["pyramid/boxes"])
    assert np.array_equal(np.array(scales), golden["pyramid/scale"])
    np.testing.assert_allclose(scores, golden["pyramid/score"], rtol=0, atol=_score_tol(w, 64))


@pytest.mark.parametrize("case", ["pyramid", "random"])
def test_oracle_nms_golden(golden, case):
    # pins the oracle's NMS restatement to the reference's own nms() output
    if case == "random":
        boxes, scores, scales = (golden["nms/random/boxes"], golden["nms/random/score"],
                                 golden["nms/random/scale"])
        thrs = (0.0, 0.2, 0.45, 0.8, 1.0)
    else:
        boxes, scores, scales = (golden["pyramid/boxes"], golden["pyramid/score"],
                                 golden["pyramid/scale"])
        thrs = (0.0, 0.3, 0.5, 1.0)
    for t in thrs:
        assert np.array_equal(O.nms(boxes, scores, scales, t), golden[f"nms/{case}/{t}"])


def test_oracle_threshold_hits_golden(golden):
    # threshold + box mapping + clamping of every pyramid level == the
    # reference's pyramid_scan at a finite threshold
    img, w = golden["pyramid/image"], golden["pyramid/weights"]
    g = O.Geometry(16, 16, 8, 2, 1, 9)
    lut = O.build_lut(9)
    for thr in (0.0, 1.5):
        bl, sl, cl = [], [], []
        for (level, factor, lw, lh) in O.pyramid_levels(img.shape[2], img.shape[1], g, 1.3):
            lim = img if level == 0 else O.resize_bilinear(img, lw, lh)
            sc = O.scan_scores(O.integral_stack(O.gradient_map(lim, lut), 9), g, 4, w, -0.5)
            oxs, oys = O.window_origins(lw, lh, g, 4)
            b, s = O.hits(sc, oxs, oys, thr, factor, int(round(16 * factor)), int(round(16 * factor)),
                          clamp=(img.shape[2], img.shape[1]))
            bl.append(b)
            sl.append(s)
            cl.append(np.full(len(s), factor))
        assert np.array_equal(np.concatenate(bl), golden[f"pyramid_thr{thr}/boxes"])
        np.testing.assert_allclose(np.concatenate(sl), golden[f"pyramid_thr{thr}/score"], rtol=1e-12)
        assert np.array_equal(np.concatenate(cl), golden[f"pyramid_thr{thr}/scale"])
