"""Host-side logic of the drop-in surface (CPU only): geometry validation,
typed errors, model I/O, NMS, lattice/pyramid bookkeeping -- restatements of
the reference's host code, checked against the oracle and reference KATs."""
import math

import numpy as np
import pytest

import paper_1703_06256_b200 as H
from oracle import oracle as O
from paper_1703_06256_b200.pipeline import regular_lattice


def test_bin_of_known_angles():
    # reference test_gradient.py:19-31
    assert [H.bin_of(1, 0, 8), H.bin_of(0, 1, 8), H.bin_of(-1, 0, 8), H.bin_of(0, -1, 8),
            H.bin_of(0, 0, 8), H.bin_of(255, 255, 8)] == [0, 2, 4, 6, H.NO_BIN, 1]


@pytest.mark.parametrize("bins", [2, 4, 8, 9, 18, 64])
def test_build_lut_equals_oracle(bins):
    assert np.array_equal(H.build_lut(bins).table, O.build_lut(bins))


@pytest.mark.parametrize("bins", [1, 0, -3, 65, 1000])
def test_build_lut_rejects_bad_bins(bins):
    with pytest.raises(H.BinCountOutOfRange):
        H.build_lut(bins)


def test_descriptor_lengths():
    assert H.descriptor_length(H.DescriptorGeometry(64, 128, 8, 2, 1, 9)) == 3780
    assert H.descriptor_length(H.DescriptorGeometry(16, 16, 8, 2, 1, 9)) == 36
    assert H.descriptor_length(H.DescriptorGeometry(64, 128, 8, 1, 1, 8)) == 1024
    assert H.descriptor_length(H.DescriptorGeometry(64, 128, 8, 1, 1, 18)) == 2304


@pytest.mark.parametrize("kw", [dict(window_w=17, window_h=16, cell=8),
                                dict(window_w=16, window_h=16, cell=8, block=3),
                                dict(window_w=16, window_h=16, cell=8, normalization="l3"),
                                dict(window_w=16, window_h=16, cell=8, block_stride=0)])
def test_geometry_validation(kw):
    with pytest.raises(H.InvalidGeometry):
        H.DescriptorGeometry(**kw)


def test_normalize_kats():
    v = np.zeros(9)
    v[0], v[1] = 3.0, 4.0
    out = H.normalize(v, "l2")
    assert abs(out[0] - 0.6) < 1e-6 and abs(out[1] - 0.8) < 1e-6
    assert not H.normalize(np.zeros(5), "l1").any()


def test_model_round_trip_and_errors():
    g = H.DescriptorGeometry(16, 16, 8, 2, 1, 9)
    m = H.LinearModel(g, np.random.default_rng(1).normal(size=36), 0.25)
    back = H.load_model(H.save_model(m))
    assert back.geometry == g and back.bias == 0.25 and np.array_equal(back.weights, m.weights)
    with pytest.raises(H.BadHeader):
        H.load_model("SVMMODEL 1\n16 16 8 2 1 9 none\n0\n")
    with pytest.raises(H.LengthMismatch):
        H.load_model("HOGMODEL 1\n16 16 8 2 1 9 none\n0\n" + "0.0\n" * 35)
    with pytest.raises(H.NonFiniteWeight):
        H.load_model("HOGMODEL 1\n16 16 8 2 1 9 none\nnan\n" + "0.0\n" * 36)


def test_iou_and_nms_argument_checks():
    # nms itself runs on the device (tests/test_gpu_detections.py); the argument
    # check happens on the host before any device work, as in detector.py:291-292
    assert H.iou((0, 0, 10, 10), (5, 0, 10, 10)) == pytest.approx(1 / 3)
    assert H.iou((0, 0, 10, 10), (10, 0, 10, 10)) == 0.0
    with pytest.raises(ValueError):
        H.nms([], 1.5)
    with pytest.raises(ValueError):
        H.nms([H.Detection(0, 0, 4, 4, 1.0)], -0.1)
    assert H.nms([], 0.5) == []


def test_pyramid_levels_match_oracle():
    g = H.DescriptorGeometry(64, 128, 8, 1, 1, 18)
    lv = H.pyramid_levels(7680, 4320, g, 1.2)
    assert lv == O.pyramid_levels(7680, 4320, O.Geometry(64, 128, 8, 1, 1, 18), 1.2)
    assert len(lv) == 20 and lv[1][2:] == (6400, 3600)


def test_regular_lattice_detection():
    for stride, cell, W, regular in ((8, 8, 800, True), (4, 8, 640, True), (3, 8, 45, False),
                                     (1, 8, 45, False), (16, 8, 400, False)):
        g = H.DescriptorGeometry(64, 128, cell, 1, 1, 8)
        oxs, oys = H.window_origins(W, 480, g, stride)
        from paper_1703_06256_b200.descriptor import cell_lattice
        cx, cy, _, _ = cell_lattice(oxs, oys, g)
        assert regular_lattice(cx, cy, stride, cell, 8) == regular


def test_window_origins_and_errors():
    g = H.DescriptorGeometry(16, 16, 8, 2, 1, 9)
    oxs, oys = H.window_origins(50, 34, g, 6)
    assert len(oxs) == (50 - 16) // 6 + 1 and len(oys) == (34 - 16) // 6 + 1
    with pytest.raises(ValueError):
        H.window_origins(50, 34, g, 0)


def test_rect_and_naive_histogram_host_helpers():
    cells = np.full((10, 10), H.NO_BIN, dtype=np.int16)
    cells[1:-1, 1:-1] = 2
    bm = H.BinMap(8, cells)
    assert H.naive_histogram(bm, H.Rect(0, 0, 10, 8))[2] == 8 * 7
    with pytest.raises(H.RectOutOfBounds):
        H.naive_histogram(bm, H.Rect(0, 0, 11, 5))
    assert math.isclose(H.Rect(1, 2, 4, 6).area, 12)
    # out-of-range bin values: the reference's list indexing raises IndexError
    bad = cells.copy()
    bad[3, 3] = 9
    with pytest.raises(IndexError):
        H.naive_histogram(H.BinMap(8, bad), H.Rect(0, 0, 10, 10))
