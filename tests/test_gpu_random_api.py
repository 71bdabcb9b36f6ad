"""Seeded random sweep of the drop-in API (the reference's own function names,
each body a C-ABI call) against the pinned CPU oracle, over geometries the
golden vectors do not hold: random window / cell / block / block-stride /
normalisation combinations and scan strides for scan_descriptors and scan
(descriptor.py:94-124, 209-223; detector.py:140-199), random rectangles
(integral.py:90-115), direct window descriptors (descriptor.py:127-150), and
pyramid scans with random scale steps (detector.py:224-269).

Bit-exact for integer descriptors, L1/L2-normalised descriptors (same IEEE
operations in the same order), rectangle histograms and boxes; scores within
1e-12 * sum|w| * max|d| (the north star allows 1e-5 relative)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1703_06256_b200 as H  # noqa: E402
from oracle import oracle as O  # noqa: E402


def image(rng, c, h, w):
    img = rng.integers(0, 256, (c, h, w), dtype=np.uint8)
    if rng.integers(0, 2):  # smooth half of the cases: small gradients, ties, flat runs
        g = img.astype(np.float64)
        for ax in (1, 2):
            g = (g + np.roll(g, 1, ax) + np.roll(g, -1, ax)) / 3
        img = np.rint(g / 8).astype(np.uint8) * 8
    return img


def geometry(rng, bins):
    cell = int(rng.choice([4, 6, 8]))
    cx, cy = int(rng.integers(2, 6)), int(rng.integers(2, 7))
    block = int(rng.choice([1, 2, 2, 3]))
    block = min(block, cx, cy)
    bs = int(rng.integers(1, block + 1))
    # (cells - block) must be a multiple of the block stride (descriptor.py:50-58)
    cx = block + (cx - block) // bs * bs
    cy = block + (cy - block) // bs * bs
    norm = str(rng.choice(["none", "l1", "l2"]))
    return (cx * cell, cy * cell, cell, block, bs, bins, norm)


@pytest.mark.parametrize("i", range(24))
def test_random_descriptors_and_scan(i):
    rng = np.random.default_rng((1703, 6256, i))
    c, bins = int(rng.choice([1, 3])), int(rng.choice([4, 6, 8, 9, 12, 18]))
    ga = geometry(rng, bins)
    h, w = int(ga[1] + rng.integers(0, 60)), int(ga[0] + rng.integers(0, 90))
    stride = int(rng.integers(1, 12))
    img = image(rng, c, h, w)
    g, go = H.DescriptorGeometry(*ga), O.Geometry(*ga)
    st = H.build_integral_stack(H.gradient_map(H.Image(img), H.build_lut(bins)))
    planes = O.integral_stack(O.gradient_map(img, O.build_lut(bins)), bins)
    assert np.array_equal(st.planes, planes)

    # scan_descriptors: every window, row-major, against the oracle's cached-grid path
    oxs, oys = O.window_origins(w, h, go, stride)
    cxs, cys, col_idx, row_idx = O.cell_index(oxs, oys, go)
    grid = O.cell_grid(planes, cxs, cys, go.cell)
    got = list(H.scan_descriptors(st, g, stride))
    assert len(got) == len(oxs) * len(oys)
    k = 0
    for iy, oy in enumerate(oys):
        for ix, ox in enumerate(oxs):
            x, y, d = got[k]
            k += 1
            ref = O.window_descriptor_from_grid(grid, row_idx[iy], col_idx[ix], go)
            assert (x, y) == (int(ox), int(oy))
            assert d.dtype == ref.dtype
            assert np.array_equal(d, ref), f"descriptor ({ox},{oy}) differs: {ga} stride {stride}"

    # a direct (uncached) window descriptor at a random origin
    ox, oy = int(rng.integers(0, w - ga[0] + 1)), int(rng.integers(0, h - ga[1] + 1))
    assert np.array_equal(H.window_descriptor(st, (ox, oy), g), O.window_descriptor(planes, (ox, oy), go))

    # scan: scores of every window and the (x, y) list in the reference's order
    wts = rng.standard_normal(go.length).astype(np.float32).astype(np.float64)
    bias = float(np.float32(rng.standard_normal()))
    dets = H.scan(st, H.LinearModel(g, wts, bias), stride, float("-inf"))
    ref = O.scan_scores(planes, go, stride, wts, bias)
    assert [(d.x, d.y) for d in dets] == [(int(x), int(y)) for y in oys for x in oxs]
    dmax = float(ga[2] * ga[2]) if ga[6] == "none" else 1.0
    np.testing.assert_allclose(np.array([d.score for d in dets]).reshape(ref.shape), ref, rtol=0,
                               atol=1e-12 * float(np.abs(wts).sum()) * dmax + 1e-12)

    # rectangle histograms at random rectangles (integral.py:90-115) against a pixel recount
    cells = O.gradient_map(img, O.build_lut(bins))
    for _ in range(6):
        x0, y0 = int(rng.integers(0, w)), int(rng.integers(0, h))
        x1, y1 = int(rng.integers(x0 + 1, w + 1)), int(rng.integers(y0 + 1, h + 1))
        patch = cells[y0:y1, x0:x1]
        want = np.array([(patch == n).sum() for n in range(bins)], dtype=np.int64)
        assert np.array_equal(H.rect_histogram(st, H.Rect(x0, y0, x1, y1)), want)


@pytest.mark.parametrize("i", range(6))
def test_random_pyramid_scan(i):
    rng = np.random.default_rng((1703, 6256, 100 + i))
    bins = int(rng.choice([8, 9, 18]))
    cell = 8
    ww, wh = 8 * int(rng.integers(2, 5)), 8 * int(rng.integers(2, 6))
    h, w = int(wh * rng.uniform(1.5, 3.5)), int(ww * rng.uniform(1.5, 4.0))
    step = float(rng.choice([1.1, 1.2, 1.25, 1.5, 2.0]))
    stride = int(rng.choice([4, 8, 6]))
    img = image(rng, int(rng.choice([1, 3])), h, w)
    ga = (ww, wh, cell, 1, 1, bins, "none")
    g, go = H.DescriptorGeometry(*ga), O.Geometry(*ga)
    wts = rng.standard_normal(go.length).astype(np.float32).astype(np.float64)
    bias = float(np.float32(rng.standard_normal()))
    thr = float(np.float32(rng.uniform(-2.0, 2.0)))
    dets = H.pyramid_scan(H.Image(img), H.LinearModel(g, wts, bias), step, stride, thr)
    lut = O.build_lut(bins)
    tol = 1e-12 * float(np.abs(wts).sum()) * 64 + 1e-12
    boxes, scores, scales = [], [], []
    for (level, factor, lw, lh) in O.pyramid_levels(w, h, go, step):
        lv = img if level == 0 else O.resize_bilinear(img, lw, lh)
        planes = O.integral_stack(O.gradient_map(lv, lut), bins)
        sc = O.scan_scores(planes, go, stride, wts, bias)
        oxs, oys = O.window_origins(lw, lh, go, stride)
        # a score within the tolerance of the threshold may fall on either side
        assert not np.any(np.abs(sc - thr) <= tol), "pick another seed: score on the threshold"
        b, s = O.hits(sc, oxs, oys, thr, factor, int(round(ww * factor)), int(round(wh * factor)),
                      clamp=(w, h))
        boxes += [tuple(r) for r in b.tolist()]
        scores += s.tolist()
        scales += [factor] * len(s)
    assert [(d.x, d.y, d.w, d.h) for d in dets] == boxes
    assert [d.scale for d in dets] == scales
    np.testing.assert_allclose([d.score for d in dets], scores, rtol=0, atol=tol)
