"""Seeded random sweep of the batched pipeline (HogPipeline -> hog_pipeline and the
score kernels, through the C ABI) against the pinned CPU oracle: random
channel counts, frame shapes (ragged widths, widths that are not multiples of
the strip or chunk sizes, heights that leave partial bands), bin counts 2..20
and 32, scan strides that do and do not divide the cell, batch sizes, band
heights, scored and unscored.  gradient.py:95-121, integral.py:58-87,
descriptor.py:153-195, detector.py:140-154.

Bit-exact for bin maps, planes and cell grids; scores within the tolerance of
tests/test_gpu_parity.py (1e-12 * sum|w| * 64, far inside the north star's
1e-5 relative)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1703_06256_b200 as H  # noqa: E402
from oracle import oracle as O  # noqa: E402

N_CASES = 36


def case(i):
    rng = np.random.default_rng((20170306, i))
    c = int(rng.choice([1, 1, 3]))
    bins = int(rng.choice([2, 3, 4, 5, 6, 7, 8, 8, 9, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 18, 19, 20, 32]))
    stride = int(rng.choice([4, 8, 8, 2, 16, 12, 5]))
    h = int(rng.integers(128, 300))
    w = int(rng.integers(64, 1400 if i % 3 else 300))
    n = int(rng.integers(1, 5))
    scored = bool(rng.integers(0, 2))
    band = int(rng.choice([0, 0, 16, 24, 40, 56, 104]))
    smooth = bool(rng.integers(0, 2))
    return rng, c, bins, stride, h, w, n, scored, band, smooth


def frames_of(rng, n, c, h, w, smooth):
    f = rng.integers(0, 256, (n, c, h, w), dtype=np.uint8)
    if smooth:  # neighbour-correlated values: small gradients, ties and zero-gradient runs
        g = f.astype(np.float64)
        for ax in (2, 3):
            g = (g + np.roll(g, 1, ax) + np.roll(g, -1, ax) + np.roll(g, 2, ax)) / 4
        f = np.rint(g / 4).astype(np.uint8) * 4
    return f


@pytest.mark.parametrize("i", range(N_CASES))
def test_random_case_vs_oracle(i):
    rng, c, bins, stride, h, w, n, scored, band, smooth = case(i)
    frames = frames_of(rng, n, c, h, w, smooth)
    weights, bias = None, 0.0
    if scored:  # float32-valued weights, as a LinearModel read from text holds
        weights = rng.standard_normal(8 * 16 * bins).astype(np.float32).astype(np.float64)
        bias = float(np.float32(rng.standard_normal()))
    if band and band % stride and 8 % stride == 0:
        band = band // stride * stride or stride
    p = H.HogPipeline(n, c, h, w, bins, stride=stride, weights=weights, bias=bias,
                      band_rows=band or None)
    p.upload(frames)
    p.run()
    torch.cuda.synchronize()
    lut = O.build_lut(bins)
    _, grid, scores = O.run_batch(frames, lut, bins, 8, 64, 128, stride, 1 if scored else 0,
                                  weights, bias, threads=4, want_outputs=True)
    got = p.grid.cpu().numpy().astype(np.int64)
    assert got.shape == grid.shape
    assert np.array_equal(got, grid), f"cell grid differs (case {i}: c={c} bins={bins} stride={stride} {h}x{w} n={n})"
    k = int(rng.integers(0, n))
    cells = O.gradient_map(frames[k], lut)
    assert np.array_equal(p.binmap_view()[k].cpu().numpy().astype(np.int16), cells)
    assert np.array_equal(p.planes_view()[k].cpu().numpy().view(np.uint32),
                          O.integral_stack(cells, bins))
    if scored:
        tol = 1e-12 * float(np.abs(weights).sum()) * 64 + 1e-12
        np.testing.assert_allclose(p.scores.cpu().numpy(), scores, rtol=1e-5, atol=tol)
