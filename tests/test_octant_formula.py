"""CPU check of the octant binning formula (k_bin_oct.cu) against the
reference's own table (gradient.py:55-72, pinned by tests/golden/lut_sha256.json
through the oracle): for N_b = 8 and 4, over all 261,121 (dx, dy) pairs, the
bin from the sign bits of the four perturbed linear forms equals the table,
and rounding each form once to fp16 (what one fp16 FMA does to an exact
integer) keeps every sign, overflow included.  The device proof
(hog_lut_proof, tests/test_gpu_octant.py) checks the kernel's own code."""
import numpy as np
import pytest

from oracle import oracle as O


def forms():
    d = np.arange(-255, 256, dtype=np.int64)
    dx, dy = np.meshgrid(d, d, indexing="ij")  # table index [dx + 255, dy + 255]
    d1, d2 = dy - dx, dy + dx
    f1 = 512 * dy + dx          # y' of the point rotated by ~1/512 rad
    g2 = dy - 512 * dx          # -x'
    f3 = 512 * d1 + d2          # y' - x'
    g4 = d1 - 512 * d2          # -(y' + x')
    return f1, g2, f3, g4


def octant_bins(bins):
    f1, g2, f3, g4 = forms()
    s1, t2, s3, t4 = f1 < 0, g2 < 0, f3 < 0, g4 < 0
    if bins == 8:
        b2 = s1
        b1 = ~(s1 ^ t2)             # s1 ^ s2 with s2 = ~t2
        b0 = ~(s1 ^ t2 ^ s3 ^ t4)   # two flipped signs cancel
        out = 4 * b2.astype(np.int16) + 2 * b1 + b0
    else:
        out = 2 * s1.astype(np.int16) + ~(s1 ^ t2)
    out[255, 255] = -1  # (0, 0): NO_BIN
    return out


@pytest.mark.parametrize("bins", [4, 8])
def test_octant_formula_equals_reference_table(bins):
    assert np.array_equal(octant_bins(bins), O.build_lut(bins))


def test_fp16_rounding_keeps_signs():
    with np.errstate(over="ignore"):
        for f in forms():
            h = f.astype(np.float16)
            assert np.array_equal(h < 0, f < 0)
            assert np.array_equal(h == 0, f == 0)
            assert not np.isnan(h).any()


def test_zero_only_at_origin():
    f1 = forms()[0]
    assert np.count_nonzero(f1 == 0) == 1 and f1[255, 255] == 0
