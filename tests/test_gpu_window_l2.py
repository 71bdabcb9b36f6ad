"""EXTENSION, not a reference behaviour: per-window L2 normalisation for
BASELINE configs[2] ("64x128 windows at stride 8 with per-window L2
normalisation of the cell histograms").  The reference normalises per block
(descriptor.py:107-124), which tests/test_gpu_parity.py checks per cell; this
labelled extension has no reference oracle, so it is checked against a numpy
restatement over the reference's unnormalised descriptor with the reference's
epsilon convention (descriptor.py:123): norm = np.sqrt((d*d).sum() + _EPS*_EPS),
bit-exact (integer sums, IEEE sqrt and division)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1703_06256_b200 as H  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1703_06256_b200 import synth  # noqa: E402

EPS = 1e-6


def restated_norms(grid, row_idx, col_idx):
    """(noy, nox) norms of every window's unnormalised descriptor."""
    q = (grid.astype(np.int64) ** 2).sum(-1)  # per-cell sum of squares
    S = q[row_idx[:, None, :, None], col_idx[None, :, None, :]].sum((2, 3))
    return np.sqrt(S.astype(np.float64) + EPS * EPS)


@pytest.mark.parametrize("key,crop,n", [("c3", (400, 700), 2), ("c2", (300, 500), 3),
                                        ("c3", None, 1)])
def test_window_l2_vs_numpy_restatement(key, crop, n):
    cfg = synth.CONFIGS[key]
    h, w = crop or (cfg.height, cfg.width)
    frames = np.ascontiguousarray(synth.make_batch(cfg, 3, n)[:, :, :h, :w])
    p = H.HogPipeline(n, cfg.channels, h, w, cfg.bins, stride=cfg.stride, window_norm="l2")
    p.upload(frames)
    p.run()
    torch.cuda.synchronize()
    _, grid, _ = O.run_batch(frames, O.build_lut(cfg.bins), cfg.bins, 8, 64, 128, cfg.stride, 0,
                             threads=2, want_outputs=True)
    assert np.array_equal(p.grid.cpu().numpy().astype(np.int64), grid)
    got = p.window_norms.cpu().numpy()
    for f in range(n):
        ref = restated_norms(grid[f], p.row_idx, p.col_idx)
        assert np.array_equal(got[f], ref)
    # normalised descriptors of a few window rows == d / norm, d the unnormalised descriptor
    g = O.Geometry(64, 128, 8, 1, 1, cfg.bins)
    rows = slice(0, 2)
    desc = p.window_descriptors(n - 1, rows).cpu().numpy()
    for iy in range(2):
        for ix in (0, len(p.oxs) // 2, len(p.oxs) - 1):
            d = O.window_descriptor_from_grid(grid[n - 1], p.row_idx[iy], p.col_idx[ix], g)
            d = np.asarray(d, dtype=np.float64)
            assert np.array_equal(desc[iy, ix], d / np.sqrt((d * d).sum() + EPS * EPS))
    assert p.result() is p.window_norms
