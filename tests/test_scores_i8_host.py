"""Host side of the exact integer-tensor-core score path (CPU, no GPU):
hog_scores_i8_prepare's digit decomposition and fragment layout, and the
integer arithmetic of k_scores_i8 restated in numpy, checked against the
oracle's float64 window scores (detector.py:140-154)."""
import ctypes
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1703_06256_b200 import _native, synth
from paper_1703_06256_b200.pipeline import i8_prepare

LIB = _native.LIB_PATH
pytestmark = pytest.mark.skipif(not os.path.exists(LIB), reason="libhogb200.so not built")


def ks_of(bins):
    return 2 if bins <= 8 else (bins + 3) // 4


def decode(frag, digits, cells_y, bins):
    """Fragments back to W[cy][cx][n] = sum_s d_s 256^s (int64); also checks
    that pad rows / pad bins are zero."""
    KS = ks_of(bins)
    P = 4 * KS
    words = np.frombuffer(frag.tobytes(), dtype=np.uint32)
    d = np.zeros((digits, 16, 8 * P), dtype=np.int64)
    for s in range(digits):
        for ks in range(KS):
            for lane in range(32):
                for r in range(4):
                    row = (lane >> 2) + 8 * (r & 1)
                    k0 = 32 * ks + 4 * (lane & 3) + 16 * (r >> 1)
                    word = int(words[((s * KS + ks) * 32 + lane) * 4 + r])
                    for q in range(4):
                        b = (word >> (8 * q)) & 0xFF
                        d[s, row, k0 + q] = b - 256 if b >= 128 else b
    d = d.reshape(digits, 16, 8, P)
    assert not d[:, cells_y:].any() and not d[..., bins:].any()
    W = np.zeros((16, 8, P), dtype=np.int64)
    for s in reversed(range(digits)):
        W = W * 256 + d[s]
    return W[:cells_y, :, :bins]


@pytest.mark.parametrize("key", ["c1", "c4", "c5"])
def test_config_weights_are_exact(key):
    cfg = synth.CONFIGS[key]
    w, _ = synth.make_weights(cfg)
    cells_y, bins = 16, cfg.bins
    frag, digits, scale = i8_prepare(w, 8, cells_y, bins)
    assert digits == 5  # float32 N(0, 0.01) weights span ~37 bits
    W = decode(frag, digits, cells_y, bins)
    assert np.array_equal(W.astype(np.float64) * scale, w.reshape(cells_y, 8, bins))


@pytest.mark.parametrize("bins,cells_y", [(4, 16), (9, 8), (12, 3), (16, 16), (20, 1)])
def test_float64_weights_rounded_to_47_bits(bins, cells_y):
    rng = np.random.default_rng(bins * 7 + cells_y)
    w = rng.normal(0, 0.05, cells_y * 8 * bins)  # 53-bit mantissas: not exact
    w[3] = 0.0
    frag, digits, scale = i8_prepare(w, 8, cells_y, bins)
    assert digits == 6
    W = decode(frag, digits, cells_y, bins)
    top = np.frexp(np.abs(w).max())[1]
    err = np.abs(W.astype(np.float64) * scale - w.reshape(cells_y, 8, bins))
    assert err.max() <= 2.0 ** (top - 47)
    assert np.abs(W).max() < 2 ** 47


def test_prepare_rejects():
    lib = _native.load()
    assert lib.hog_scores_i8_frag_bytes(21) == 0 and lib.hog_scores_i8_frag_bytes(0) == 0
    frag = np.zeros(lib.hog_scores_i8_frag_bytes(8), dtype=np.uint8)
    dg, sc = ctypes.c_int(0), ctypes.c_double(0)
    w = np.zeros(16 * 8 * 8)
    assert lib.hog_scores_i8_prepare(w.ctypes.data, 7, 16, 8, frag.ctypes.data,
                                     ctypes.byref(dg), ctypes.byref(sc)) == _native.HOG_EINVAL
    assert lib.hog_scores_i8_prepare(w.ctypes.data, 8, 17, 8, frag.ctypes.data,
                                     ctypes.byref(dg), ctypes.byref(sc)) == _native.HOG_EINVAL
    w[5] = np.nan
    assert lib.hog_scores_i8_prepare(w.ctypes.data, 8, 16, 8, frag.ctypes.data,
                                     ctypes.byref(dg), ctypes.byref(sc)) == _native.HOG_ERANGE
    w[5] = 1e-300  # 2^-997 and below: the power-of-two scale would leave float64
    assert i8_prepare(w, 8, 16, 8) is None
    w[:] = 0.0  # all-zero weights: every digit zero
    frag2, digits, scale = i8_prepare(w, 8, 16, 8)
    assert not frag2.any() and digits == 4 and scale == 1.0


def kernel_restated(grid, frag, digits, scale, bias, cells_y, bins):
    """k_scores_i8's arithmetic in numpy: per grid row the (digit, cell row)
    partial dots of 8-cell window rows, digits combined exactly, the cell rows
    of each window summed (int64), one rounding to float64, plus the bias."""
    W = decode(frag, digits, cells_y, bins)
    ncy, ncx, _ = grid.shape
    noy, nox = ncy - cells_y + 1, ncx - 7
    g = grid.astype(np.int64)
    tot = np.zeros((noy, nox), dtype=np.int64)
    for cy in range(cells_y):
        for cx in range(8):
            tot += g[cy:cy + noy, cx:cx + nox, :] @ W[cy, cx]
    return tot.astype(np.float64) * scale + bias


@pytest.mark.parametrize("key,h,w", [("c1", 600, 800), ("c5", 300, 520)])
def test_integer_scores_match_oracle(key, h, w):
    cfg = synth.CONFIGS[key]
    frame = synth.make_batch(cfg, 0, 1)[0][:, :h, :w]
    wts, _ = synth.make_weights(cfg)
    bias = -0.375
    lut = O.build_lut(cfg.bins)
    planes = O.integral_stack(O.gradient_map(frame, lut), cfg.bins)
    g = O.Geometry(64, 128, 8, 1, 1, cfg.bins)
    ref = O.scan_scores(planes, g, 8, wts, bias)
    cxs = np.arange(0, w - 8 + 1, 8)
    cys = np.arange(0, h - 8 + 1, 8)
    grid = O.cell_grid(planes, cxs, cys, 8)
    frag, digits, scale = i8_prepare(wts, 8, 16, cfg.bins)
    got = kernel_restated(grid, frag, digits, scale, bias, 16, cfg.bins)
    assert got.shape == ref.shape
    # exact integer dot + one rounding vs OpenBLAS-order float64: ~1 ulp apart
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)
