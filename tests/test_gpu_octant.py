"""Octant binning (N_b in {4, 8}): the table folded into sign tests of four
linear forms (k_bin_oct.cu), checked three ways.

1. The device proof (hog_lut_proof) runs the kernel's classifier on all
   261,121 (dx, dy) pairs against the reference's own table
   (gradient.py:55-72): zero mismatching entries for N_b = 4 and 8.
2. An image holding every (dx, dy) pair at the centre of its own 3x3 block
   goes through hog_grad_bin (the octant kernel, which the profiler must see)
   and matches the oracle's gradient_map bit for bit, so the byte spreads and
   the lane / half-warp halos are covered as well as the classifier.
3. A table that differs from the reference in one entry fails the proof by
   exactly that entry, and hog_grad_bin then honours the table as given (the
   table-gather kernel), matching the oracle run with the same table.
"""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1703_06256_b200 as H  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1703_06256_b200 import _native, device as D  # noqa: E402
from paper_1703_06256_b200.gradient import OrientationLut, grad_bin_device  # noqa: E402


def proof(table, bins):
    lt = D.lut_device(table)
    out = ctypes.c_longlong(-99)
    _native.call("hog_lut_proof", D.ptr(lt), bins, ctypes.addressof(out), None)
    return out.value


@pytest.mark.parametrize("bins", [2, 3, 4, 5, 8, 9, 16, 18, 64])
def test_proof_against_reference_table(bins):
    got = proof(H.build_lut(bins).table, bins)
    assert got == (0 if bins in (4, 8) else -1)


def all_pairs_image(seed=0):
    """Every (dx, dy) in [-255, 255]^2 at the centre of one 3x3 block."""
    rng = np.random.default_rng(seed)
    d = np.arange(-255, 256)
    dx, dy = np.meshgrid(d, d, indexing="ij")
    n = 511
    img = rng.integers(0, 256, size=(3 * n, 3 * n), dtype=np.int64)
    left = np.maximum(0, -dx)
    top = np.maximum(0, -dy)
    # block (i, j): centre row 3i+1, centre column 3j+1; dx along columns
    blk = img.reshape(n, 3, n, 3)
    blk[:, 1, :, 0] = left
    blk[:, 1, :, 2] = left + dx
    blk[:, 0, :, 1] = top
    blk[:, 2, :, 1] = top + dy
    return blk.reshape(3 * n, 3 * n).astype(np.uint8), dx, dy


def ran_octant_kernel(fn):
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    names = [e.name for e in prof.events() if e.device_type.name == "CUDA"]
    return any("k_grad_bin_oct" in nm for nm in names), names


@pytest.mark.parametrize("bins", [4, 8])
def test_every_pair_through_the_kernel(bins):
    img, dx, dy = all_pairs_image()
    lut = H.build_lut(bins)
    frames = D.upload_frames(img[None])
    box = {}

    def run():
        box["bm"] = grad_bin_device(frames, lut)

    used, names = ran_octant_kernel(run)
    assert used, f"octant kernel not launched: {sorted(set(names))}"
    got = box["bm"].data[0, :, : img.shape[1]].cpu().numpy().astype(np.int16)
    want = O.gradient_map(img[None], O.build_lut(bins))
    assert np.array_equal(got, want)
    # the centres hold exactly the table, pair by pair
    centres = got[1::3, 1::3]
    assert np.array_equal(centres, lut.table)


def test_altered_table_is_honoured():
    base = H.build_lut(8).table
    t = base.copy()
    t[255 + 3, 255 + 5] = (t[255 + 3, 255 + 5] + 3) % 8  # (dx, dy) = (3, 5)
    assert proof(t, 8) == 1
    img, _, _ = all_pairs_image(1)
    frames = D.upload_frames(img[None])
    lut = OrientationLut(bins=8, table=t)
    box = {}

    def run():
        box["bm"] = grad_bin_device(frames, lut)

    used, _ = ran_octant_kernel(run)
    assert not used
    got = box["bm"].data[0, :, : img.shape[1]].cpu().numpy().astype(np.int16)
    want = O.gradient_map(img[None], t.astype(np.int16))
    assert np.array_equal(got, want)
    assert got[1 + 3 * (255 + 3), 1 + 3 * (255 + 5)] == t[258, 260]


@pytest.mark.parametrize("shape", [(1, 7, 9), (3, 31, 40), (2, 130, 264), (1, 600, 800)])
def test_octant_odd_shapes_match_oracle(shape):
    """Widths not a multiple of 8 or 128, heights not a multiple of the
    sub-band: ragged half-warps, partial 8-byte groups, padded row blocks."""
    n, h, w = shape
    rng = np.random.default_rng(h * 1000 + w)
    frames = rng.integers(0, 256, size=(n, 1, h, w), dtype=np.uint8)
    lut = H.build_lut(8)
    bm = grad_bin_device(D.upload_frames(frames), lut)
    got = bm.data[:, :, :w].cpu().numpy().astype(np.int16)
    for i in range(n):
        assert np.array_equal(got[i], O.gradient_map(frames[i], O.build_lut(8)))


@pytest.mark.parametrize("shape", [(2, 130, 264), (1, 72, 640)])
def test_octant_rgb_channel_rule(shape):
    """RGB: per-channel gradients, largest dx^2 + dy^2 wins, first channel on ties
    (gradient.py:113-117), then the octant tests.  Channel 1 is the negative of
    channel 0 (equal magnitudes, opposite gradients) and channel 2 repeats channel 0
    on half the rows, so ties are everywhere; the rest is random."""
    n, h, w = shape
    rng = np.random.default_rng(w)
    f = rng.integers(0, 256, size=(n, 3, h, w), dtype=np.uint8)
    f[:, 1] = 255 - f[:, 0]
    f[:, 2, : h // 2] = f[:, 0, : h // 2]
    lut = H.build_lut(8)
    frames = D.upload_frames(f)
    box = {}

    def run():
        box["bm"] = grad_bin_device(frames, lut)

    used, names = ran_octant_kernel(run)
    assert used, sorted(set(names))
    got = box["bm"].data[:, :, :w].cpu().numpy().astype(np.int16)
    for i in range(n):
        assert np.array_equal(got[i], O.gradient_map(f[i], O.build_lut(8)))
