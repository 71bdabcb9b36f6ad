"""hog_resize_bilinear (detector.py:202-221) against the pinned oracle over
downscale ratios on both sides of 2x (the limit of the experiment builds' row-shared
k_resize_rows; the product library runs k_resize everywhere), widths that leave partial
256-column tiles, RGB, and frame batches.  Bit-exact."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import oracle as O  # noqa: E402
from paper_1703_06256_b200 import _native, synth  # noqa: E402
from paper_1703_06256_b200 import device as D  # noqa: E402


def resize_dev(frames, nw, nh):
    n, c, h, w = frames.shape
    src = torch.as_tensor(frames, device="cuda")
    dst = torch.full((n, c, nh, nw), 7, dtype=torch.uint8, device="cuda")
    _native.call("hog_resize_bilinear", D.ptr(src), n, c, h, w, w, h * w, c * h * w, nh, nw,
                 h / nh, w / nw, D.ptr(dst), nw, nh * nw, c * nh * nw, None)
    torch.cuda.synchronize()
    return dst.cpu().numpy()


@pytest.mark.parametrize("c,h,w,nw,nh", [
    (1, 540, 960, 800, 450),   # 1.2
    (1, 540, 960, 480, 270),   # exactly 2
    (1, 540, 961, 480, 270),   # just above 2: per-pixel kernel
    (3, 300, 700, 583, 250),   # RGB, partial last tile
    (1, 97, 300, 299, 96),     # ~1.0
    (1, 400, 1000, 257, 100),  # 3.9
    (1, 130, 70, 64, 128),     # window-sized level, < 1 tile
])
def test_resize_vs_oracle(c, h, w, nw, nh):
    rng = np.random.default_rng(h * w + nw)
    frames = rng.integers(0, 256, (2, c, h, w), dtype=np.uint8)
    frames[1] = synth.make_frame(synth.CONFIGS["c5"], 1)[:1, :h, :w].repeat(c, 0)
    got = resize_dev(frames, nw, nh)
    for i in range(2):
        assert np.array_equal(got[i], O.resize_bilinear(frames[i], nw, nh))
