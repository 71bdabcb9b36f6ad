"""Exact integer-tensor-core window scores (k_scores_i8 through
hog_scores_lattice_i8), detector.py:140-154.

For float32-valued weights the kernel computes the window dot EXACTLY and
rounds it once, so its scores must equal, bit for bit, the exact integer dot
of the device cell grid with the integer weights (numpy int64) rounded the
same way; against the oracle's float64 scores (the reference's arithmetic)
they agree to ~1 ulp (tolerance below: 1e-12 relative, far inside the north
star's 1e-5).  Float64-valued weights are rounded to 47 bits (an error of the
size of float64 rounding) and are checked against the oracle and the fp64
score kernel."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1703_06256_b200 as H  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1703_06256_b200 import _native, synth  # noqa: E402
from paper_1703_06256_b200 import device as D  # noqa: E402
from paper_1703_06256_b200.pipeline import i8_prepare  # noqa: E402


def score_tol(w):
    return 1e-12 * float(np.abs(w).sum()) * 64 + 1e-12


def exact_scores(grid, w, cells_y, bins, bias):
    """Exact dot (int64) of every window with float32-valued weights, then
    float64(dot) * 2^-F + bias -- the kernel's single rounding."""
    _, digits, scale = i8_prepare(w, 8, cells_y, bins)
    W = np.rint(w / scale).astype(np.int64).reshape(cells_y, 8, bins)
    assert np.array_equal(W * scale, w.reshape(cells_y, 8, bins))
    n, ncy, ncx, _ = grid.shape
    noy, nox = ncy - cells_y + 1, ncx - 7
    g = grid.astype(np.int64)
    tot = np.zeros((n, noy, nox), dtype=np.int64)
    for cy in range(cells_y):
        for cx in range(8):
            tot += g[:, cy:cy + noy, cx:cx + nox, :] @ W[cy, cx]
    return tot.astype(np.float64) * scale + bias


def run(frames, bins, window=(64, 128), weights=None, bias=0.0, monkeypatch=None, i8=True):
    n, c, h, w = frames.shape
    if monkeypatch is not None:
        monkeypatch.setenv("HOGB200_SCORES_I8", "1" if i8 else "0")
    p = H.HogPipeline(n, c, h, w, bins, stride=8, window=window, weights=weights, bias=bias)
    assert (p.i8 is not None) == i8
    p.upload(frames)
    p.run()
    torch.cuda.synchronize()
    return p


CASES = [  # (bins, channels, h, w, window, n): KS 2..5, u32 / u16 / byte staging,
    (8, 1, 600, 800, (64, 128), 1),      # c1
    (8, 3, 300, 1280, (64, 128), 3),     # c4 rows (RGB), 153 window columns: partial CTA tile
    (18, 1, 300, 1000, (64, 128), 2),    # c5 bins: u16 staging, 20-byte cells
    (9, 1, 257, 611, (64, 128), 2),      # odd bins: byte staging, 12-byte cells
    (4, 1, 200, 333, (64, 128), 1),      # 4 bins in 8-byte cells
    (12, 1, 180, 700, (64, 64), 2),      # 8 cell rows
    (16, 3, 150, 520, (64, 32), 1),      # 4 cell rows
    (20, 1, 140, 300, (64, 136), 1),     # 17 cell rows: > 16 -> fp64 kernel (checked below)
    (18, 1, 1400, 150, (64, 128), 1),    # one column tile, many bands (T < noy)
]


@pytest.mark.parametrize("bins,c,h,w,window,n", CASES)
def test_i8_scores_exact(monkeypatch, bins, c, h, w, window, n):
    rng = np.random.default_rng(bins * 100 + h)
    frames = rng.integers(0, 256, (n, c, h, w), dtype=np.uint8)
    if n > 1:  # one blurred frame (realistic gradients) beside the noise
        frames[0] = synth.make_batch(synth.CONFIGS["c5"], 0, 1)[0, :1, :h, :w].repeat(c, 0)
    cells_y = window[1] // 8
    wts = rng.normal(0, 0.01, 8 * cells_y * bins).astype(np.float32).astype(np.float64)
    bias = -0.3125
    i8 = cells_y <= 16 and bins <= 20
    p = run(frames, bins, window, wts, bias, monkeypatch, i8=i8)
    got = p.scores.cpu().numpy()
    g = O.Geometry(window[0], window[1], 8, 1, 1, bins)
    lut = O.build_lut(bins)
    for i in range(n):
        ref = O.scan_scores(O.integral_stack(O.gradient_map(frames[i], lut), bins), g, 8, wts, bias)
        np.testing.assert_allclose(got[i], ref, rtol=1e-12, atol=1e-12)
    if i8:
        exact = exact_scores(p.grid.cpu().numpy(), wts, cells_y, bins, bias)
        assert np.array_equal(got, exact)  # bit for bit: one rounding of the exact dot


@pytest.mark.parametrize("bins", [8, 18])
def test_i8_float64_weights_vs_fp64_kernel(monkeypatch, bins):
    rng = np.random.default_rng(bins)
    frames = rng.integers(0, 256, (2, 1, 300, 700), dtype=np.uint8)
    wts = rng.normal(0, 0.01, 128 * bins)  # float64 mantissas: rounded to 47 bits
    p8 = run(frames, bins, weights=wts, bias=0.25, monkeypatch=monkeypatch, i8=True)
    pf = run(frames, bins, weights=wts, bias=0.25, monkeypatch=monkeypatch, i8=False)
    a, b = p8.scores.cpu().numpy(), pf.scores.cpu().numpy()
    np.testing.assert_allclose(a, b, rtol=1e-12, atol=score_tol(wts))
    g = O.Geometry(64, 128, 8, 1, 1, bins)
    lut = O.build_lut(bins)
    for i in range(2):
        ref = O.scan_scores(O.integral_stack(O.gradient_map(frames[i], lut), bins), g, 8, wts, 0.25)
        np.testing.assert_allclose(a[i], ref, rtol=1e-9, atol=score_tol(wts))


def test_i8_config_batches_vs_oracle():
    # c4's geometry (RGB, 8 bins) and c5's (18 bins) at full width
    for key, n, crop in (("c4", 4, None), ("c5", 1, (520, 7680))):
        cfg = synth.CONFIGS[key]
        frames = synth.make_batch(cfg, 0, n)
        if crop:
            frames = frames[:, :, :crop[0], :crop[1]].copy()
        _, c, h, w = frames.shape
        wts, bias = synth.make_weights(cfg)
        p = H.HogPipeline(n, c, h, w, cfg.bins, stride=8, weights=wts, bias=bias)
        assert p.i8 is not None
        p.upload(frames)
        p.run()
        torch.cuda.synchronize()
        got = p.scores.cpu().numpy()
        assert np.array_equal(got, exact_scores(p.grid.cpu().numpy(), wts, 16, cfg.bins, bias))
        _, _, ref = O.run_batch(frames, O.build_lut(cfg.bins), cfg.bins, 8, 64, 128, 8, 1, wts, bias,
                                threads=8, want_outputs=True)
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)


def test_i8_abi_rejects():
    lib = _native.load()
    g = torch.zeros((1, 20, 20, 8), dtype=torch.uint8, device="cuda")
    s = torch.zeros((1, 5, 13), dtype=torch.float64, device="cuda")
    f = torch.zeros(lib.hog_scores_i8_frag_bytes(8), dtype=torch.uint8, device="cuda")
    call, ptr = _native.call, D.ptr
    with pytest.raises(_native.NativeError, match="window grid exceeds"):
        call("hog_scores_lattice_i8", ptr(g), 1, 20, 20, 8, 6, 13, 8, 16, ptr(f), 5, 1.0, 0.0, ptr(s), None)
    with pytest.raises(_native.NativeError, match="digits"):
        call("hog_scores_lattice_i8", ptr(g), 1, 20, 20, 8, 5, 13, 8, 16, ptr(f), 7, 1.0, 0.0, ptr(s), None)
    with pytest.raises(_native.NativeError, match="8 cells across"):
        call("hog_scores_lattice_i8", ptr(g), 1, 20, 20, 8, 5, 13, 7, 16, ptr(f), 5, 1.0, 0.0, ptr(s), None)
