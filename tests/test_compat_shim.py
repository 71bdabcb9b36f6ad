"""The `fasthog` shim (compat/): a reference user's imports resolve to this
package's names (CPU: import surface only; GPU: one call through it)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _import_shim():
    sys.path.insert(0, os.path.join(ROOT, "compat"))
    try:
        import fasthog
        return fasthog
    finally:
        sys.path.pop(0)


def test_shim_exposes_the_reference_surface():
    fh = _import_shim()
    import paper_1703_06256_b200 as H

    assert "compat" in fh.__file__
    for name in ("build_lut", "gradient_map", "build_integral_stack", "CellHistogramCache",
                 "window_descriptor", "scan_descriptors", "scan", "pyramid_scan", "nms",
                 "decode_pnm", "Image", "DescriptorGeometry", "LinearModel", "FastHogError"):
        assert getattr(fh, name) is getattr(H, name)
    from fasthog.gradient import NO_BIN, bin_of
    from fasthog.integral import rect_count
    from fasthog.errors import AccumulatorOverflowRisk
    assert NO_BIN == -1 and bin_of(1, 0, 8) == 0 and rect_count is H.rect_count
    assert AccumulatorOverflowRisk is H.AccumulatorOverflowRisk
    assert fh.image_io.decode_pnm(b"P5 2 1 255 ab").planes.tolist() == [[[97, 98]]]


@pytest.mark.gpu
def test_shim_runs_on_the_device():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    fh = _import_shim()
    img = np.random.default_rng(0).integers(0, 256, (1, 40, 50), dtype=np.uint8)
    st = fh.build_integral_stack(fh.gradient_map(fh.Image(img), fh.build_lut(9)))
    assert st.planes.shape == (9, 41, 51) and st.planes.dtype == np.uint32
