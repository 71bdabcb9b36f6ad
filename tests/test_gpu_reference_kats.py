"""Known-answer and property tests of the reference's own test strategy
(test_gradient.py, test_integral.py, test_descriptor.py,
test_detector.py, test_acceptance.py), restated against the CUDA path.
Each test cites the reference test it mirrors; values are bit-exact."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1703_06256_b200 as H  # noqa: E402
from oracle import oracle as O  # noqa: E402


def test_ramp_interior_is_bin_zero():
    # test_gradient.py:95-102: a left-to-right ramp has dx = 2, dy = 0 inside
    img = np.tile(np.arange(0, 40, dtype=np.uint8) * 3, (20, 1))[None]
    cells = H.gradient_map(H.Image(img), H.build_lut(8)).cells
    assert (cells[1:-1, 1:-1] == 0).all()
    assert (cells[0] == H.NO_BIN).all() and (cells[-1] == H.NO_BIN).all()
    assert (cells[:, 0] == H.NO_BIN).all() and (cells[:, -1] == H.NO_BIN).all()


def test_channel_tie_goes_to_first_channel():
    # test_gradient.py:117-122 / conftest.py:32-47: equal dx^2+dy^2 in two
    # channels -> the lower channel index wins (strict >)
    img = np.zeros((3, 5, 5), np.uint8)
    img[0, :, :] = np.arange(5)[None, :] * 10     # channel 0: horizontal gradient
    img[1, :, :] = np.arange(5)[:, None] * 10     # channel 1: vertical, same magnitude
    cells = H.gradient_map(H.Image(img), H.build_lut(8)).cells
    ref = O.gradient_map(img, O.build_lut(8))
    assert np.array_equal(cells, ref)
    assert (cells[1:-1, 1:-1] == H.bin_of(20, 0, 8)).all()  # channel 0's direction
    img2 = img[[1, 0, 2]].copy()                   # swap: now the vertical one is first
    cells2 = H.gradient_map(H.Image(img2), H.build_lut(8)).cells
    assert (cells2[1:-1, 1:-1] == H.bin_of(0, 20, 8)).all()


@pytest.mark.parametrize("acc", [32, 16])
def test_uniform_interior_corner_total(acc):
    # test_integral.py:41-46: a 5x5 map whose 3x3 interior is bin 2 -> total 9
    cells = np.full((5, 5), H.NO_BIN, np.int16)
    cells[1:4, 1:4] = 2
    st = H.build_integral_stack(H.BinMap(8, cells), acc_width=acc)
    assert int(st.planes[2, -1, -1]) == 9 and int(st.planes.sum(axis=(1, 2))[[0, 1, 3]].sum()) == 0
    assert H.rect_count(st, 2, H.Rect(0, 0, 5, 5)) == 9
    # monotone and zero-padded (test_integral.py:60-78)
    p = st.planes.astype(np.int64)
    assert (p[:, 0, :] == 0).all() and (p[:, :, 0] == 0).all()
    assert (np.diff(p, axis=1) >= 0).all() and (np.diff(p, axis=2) >= 0).all()


def test_uniform_field_gives_full_cells():
    # test_descriptor.py:111-119: every interior pixel in one bin -> each cell
    # histogram fully in that bin (cell 8 -> 64)
    cells = np.full((34, 42), 5, np.int16)
    st = H.build_integral_stack(H.BinMap(9, cells))
    g = H.DescriptorGeometry(16, 16, 8, block=1, block_stride=1, bins=9)
    d = H.window_descriptor(st, (8, 8), g)
    assert d.dtype == np.int64 and len(d) == 36
    assert (d.reshape(4, 9)[:, 5] == 64).all() and d.reshape(4, 9)[:, [0, 1, 2, 3, 4, 6, 7, 8]].sum() == 0


def test_l2_block_norm_3_4_5():
    # test_descriptor.py:188-193: a block holding counts 3 and 4 normalises to
    # 3/sqrt(25+eps^2), 4/sqrt(25+eps^2)
    cells = np.full((16, 16), H.NO_BIN, np.int16)
    cells[0, 0:3] = 1          # cell (0, 0): three pixels of bin 1
    cells[0, 8:12] = 2         # cell (0, 1): four pixels of bin 2
    st = H.build_integral_stack(H.BinMap(4, cells))
    with pytest.raises(H.InvalidGeometry):  # a 3x3 block does not fit 2x2 cells
        H.DescriptorGeometry(16, 16, 8, block=3, block_stride=1, bins=4, normalization="l2")
    g = H.DescriptorGeometry(16, 16, 8, block=2, block_stride=1, bins=4, normalization="l2")
    d = H.window_descriptor(st, (0, 0), g)
    assert len(d) == 16 and d[1] == 3 / math.sqrt(25 + 1e-6 * 1e-6)
    assert d[4 + 2] == 4 / math.sqrt(25 + 1e-6 * 1e-6) and np.count_nonzero(d) == 2
    g = H.DescriptorGeometry(16, 16, 8, block=2, block_stride=1, bins=4, normalization="none")
    assert np.flatnonzero(H.window_descriptor(st, (0, 0), g)).tolist() == [1, 6]
    n = H.normalize(np.array([3.0, 4.0]), "l2")
    assert n[0] == 3 / math.sqrt(25 + 1e-12) and n[1] == 4 / math.sqrt(25 + 1e-12)


def test_translation_reuse():
    # test_descriptor.py:218-225: shifting the image by the stride shifts the
    # descriptor grid by one origin
    rng = np.random.default_rng(5)
    img = rng.integers(0, 256, (1, 60, 80), dtype=np.uint8)
    g = H.DescriptorGeometry(16, 24, 8, block=2, block_stride=1, bins=9)
    lut = H.build_lut(9)
    a = H.build_integral_stack(H.gradient_map(H.Image(img), lut))
    b = H.build_integral_stack(H.gradient_map(H.Image(img[:, 4:, 4:].copy()), lut))
    for (x, y) in ((4, 4), (12, 8), (20, 20)):
        assert np.array_equal(H.window_descriptor(a, (x + 4, y + 4), g),
                              H.window_descriptor(b, (x, y), g))


def test_scan_threads_and_order():
    # test_detector.py:151-157 (threaded == sequential) and row-major order
    rng = np.random.default_rng(8)
    img = rng.integers(0, 256, (1, 70, 90), dtype=np.uint8)
    g = H.DescriptorGeometry(16, 24, 8, block=2, block_stride=1, bins=9)
    model = H.LinearModel(g, rng.normal(size=H.descriptor_length(g)), 0.1)
    st = H.build_integral_stack(H.gradient_map(H.Image(img), H.build_lut(9)))
    one = H.scan(st, model, 6, -1.0)
    four = H.scan(st, model, 6, -1.0, threads=4)
    assert [(d.x, d.y, d.score) for d in one] == [(d.x, d.y, d.score) for d in four]
    assert [(d.y, d.x) for d in one] == sorted((d.y, d.x) for d in one)
    # every score == dot(weights, descriptor) + bias (test_detector.py:139-148)
    for d in one[:: max(1, len(one) // 25)]:
        ref = float(np.dot(model.weights, H.window_descriptor(st, (d.x, d.y), g)) + model.bias)
        assert abs(d.score - ref) <= 1e-9 * max(1.0, abs(ref))


def test_planted_high_gradient_patch_is_detected():
    # test_acceptance.py (criterion 7): a striped patch in flat noise, a model
    # that rewards its orientation -> the best detection sits on the patch
    rng = np.random.default_rng(12)
    img = (rng.integers(100, 104, (1, 96, 128))).astype(np.uint8)
    img[0, 40:72, 64:96] = np.where((np.arange(32) // 2) % 2 == 0, 30, 220)[None, :].repeat(32, 0)
    g = H.DescriptorGeometry(32, 32, 8, block=1, block_stride=1, bins=8)
    w = np.zeros(H.descriptor_length(g))
    w.reshape(-1, 8)[:, [0, 4]] = 1.0      # vertical stripes: horizontal gradients
    st = H.build_integral_stack(H.gradient_map(H.Image(img), H.build_lut(8)))
    dets = H.scan(st, H.LinearModel(g, w, 0.0), 8, 100.0)
    best = max(dets, key=lambda d: d.score)
    assert (best.x, best.y) == (64, 40)
    kept = H.nms(dets, 0.3)
    assert (kept[0].x, kept[0].y) == (64, 40)
