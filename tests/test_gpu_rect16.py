"""16-bit accumulator planes (hog_integral16) and device rectangle queries
(hog_rect_histogram) -- SURVEY §8f rank 4 -- against the pinned oracle and
the reference's golden bin maps.  Bit-exact."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1703_06256_b200 as H  # noqa: E402
from oracle import oracle as O  # noqa: E402

SMALL = ["gray45x37", "rgb48x40", "gray133x77", "rgb3x3", "rgbtie70x50"]


@pytest.mark.parametrize("name", SMALL)
def test_integral16_golden(golden, name):
    img, bins = golden[f"{name}/image"], int(golden[f"{name}/bins"])
    bm = H.gradient_map(H.Image(img), H.build_lut(bins))
    st16 = H.build_integral_stack(bm, acc_width=16)
    assert st16.planes.dtype == np.uint16
    ref = O.integral_stack(golden[f"{name}/binmap"], bins)
    assert O.sha256(ref) == str(golden[f"{name}/planes_sha"])
    assert np.array_equal(st16.planes, ref.astype(np.uint16))


@pytest.mark.parametrize("shape,bins", [((255, 257), 8), ((3, 21845), 9), ((200, 300), 18),
                                        ((64, 1000), 4)])
def test_integral16_limits_and_shapes(shape, bins):
    h, w = shape
    assert h * w <= 65535
    rng = np.random.default_rng(h * 7 + w)
    cells = rng.integers(-1, bins, (h, w)).astype(np.int16)
    cells[rng.random((h, w)) < 0.2] = bins + 3  # out-of-range user values count nowhere
    st = H.build_integral_stack(H.BinMap(bins, cells), acc_width=16)
    ref = O.integral_stack(np.where(cells >= bins, -1, cells).astype(np.int16), bins)
    assert np.array_equal(st.planes, ref.astype(np.uint16))
    if h * w == 65535:  # the worst case fits exactly: one bin everywhere
        one = H.build_integral_stack(H.BinMap(bins, np.zeros((h, w), np.int16)), acc_width=16)
        assert int(one.planes[0, -1, -1]) == 65535
    with pytest.raises(H.AccumulatorOverflowRisk):  # one pixel over the guard
        H.build_integral_stack(H.BinMap(bins, np.zeros((h, 65535 // h + 1), np.int16)),
                               acc_width=16)


@pytest.mark.parametrize("acc", [32, 16])
def test_rect_queries_vs_oracle(golden, acc):
    img, bins = golden["gray300x200_b18/image"], int(golden["gray300x200_b18/bins"])
    bm = H.gradient_map(H.Image(img), H.build_lut(bins))
    st = H.build_integral_stack(bm, acc_width=acc)
    cells = golden["gray300x200_b18/binmap"]
    rng = np.random.default_rng(acc)
    rects = []
    for _ in range(300):
        x0, x1 = sorted(rng.choice(bm.width + 1, 2, replace=False))
        y0, y1 = sorted(rng.choice(bm.height + 1, 2, replace=False))
        rects.append(H.Rect(int(x0), int(y0), int(x1), int(y1)))
    got = H.rect_histograms(st, rects)
    assert got.dtype == np.int64
    for r, row in zip(rects, got):
        sub = cells[r.y0:r.y1, r.x0:r.x1]
        ref = np.array([(sub == b).sum() for b in range(bins)])
        assert np.array_equal(row, ref)
    r = rects[0]
    assert np.array_equal(H.rect_histogram(st, r), got[0])
    assert H.rect_count(st, 3, r) == int(got[0, 3])
    with pytest.raises(H.BinOutOfRange):
        H.rect_count(st, bins, r)
    with pytest.raises(H.RectOutOfBounds):
        H.rect_histogram(st, H.Rect(0, 0, bm.width + 1, 2))


def test_window_stage_on_16bit_stack(golden):
    # CellHistogramCache / window descriptors read 16-bit planes through the
    # rectangle kernel: identical to the 32-bit stack
    img, bins = golden["gray133x77/image"], int(golden["gray133x77/bins"])
    bm = H.gradient_map(H.Image(img), H.build_lut(bins))
    g = H.DescriptorGeometry(16, 24, 8, 2, 1, bins, "l2")
    oxs, oys = H.window_origins(bm.width, bm.height, g, 3)
    c32 = H.CellHistogramCache(H.build_integral_stack(bm), g, oxs, oys)
    c16 = H.CellHistogramCache(H.build_integral_stack(bm, acc_width=16), g, oxs, oys)
    assert np.array_equal(c32.grid, c16.grid)
    assert np.array_equal(c32.descriptor(2, 1), c16.descriptor(2, 1))


def test_host_built_stack_is_uploaded():
    # an IntegralStack made from a host array (reference constructor) works too
    rng = np.random.default_rng(5)
    cells = rng.integers(-1, 8, (40, 50)).astype(np.int16)
    planes = O.integral_stack(cells, 8)
    st = H.IntegralStack(8, 50, 40, 32, planes=planes)
    assert H.rect_count(st, 2, H.Rect(3, 4, 30, 33)) == int((cells[4:33, 3:30] == 2).sum())
