"""PNM ingestion and the descriptor text dump on the
native host library libhogio.so, against the reference's own decode results,
error classes and formatter output (tests/golden, made by make_golden.py)."""
import io

import numpy as np
import pytest

import paper_1703_06256_b200 as H
from paper_1703_06256_b200 import image_io

PNM = ["p5", "p6", "p2_comments", "p3", "p5_trailing", "p5_hash_after_maxval", "p2_underscore_plus",
       "p2_leading_zeros", "bad_magic", "maxval_16bit", "maxval_zero", "truncated_raw",
       "truncated_ascii", "nonnumeric", "sample_range", "negative_width", "empty", "header_only"]


@pytest.mark.parametrize("name", PNM)
def test_decode_pnm_golden(golden, name):
    blob = bytes(golden[f"pnm/{name}/bytes"])
    err = str(golden[f"pnm/{name}/error"])
    if err:
        with pytest.raises(getattr(H, err)):
            H.decode_pnm(blob)
    else:
        img = H.decode_pnm(blob)
        assert img.planes.dtype == np.uint8
        assert np.array_equal(img.planes, golden[f"pnm/{name}/planes"])


def test_encode_roundtrip_and_batch(tmp_path):
    rng = np.random.default_rng(4)
    gray = [rng.integers(0, 256, (1, 37, 53), dtype=np.uint8) for _ in range(5)]
    paths = []
    for i, g in enumerate(gray):
        p = tmp_path / f"f{i}.pgm"
        H.write_image(str(p), H.Image(g))
        paths.append(p)
        assert np.array_equal(H.read_image(str(p)).planes, g)
    batch = H.read_batch(paths, pinned=False, threads=3)
    assert tuple(batch.shape) == (5, 1, 37, 53)
    assert np.array_equal(batch.numpy(), np.stack(gray))
    rgb = rng.integers(0, 256, (3, 9, 11), dtype=np.uint8)
    assert np.array_equal(H.decode_pnm(image_io.encode_image(H.Image(rgb))).planes, rgb)
    # a bad file in a batch raises its typed error; a different shape is rejected
    (tmp_path / "bad.pgm").write_bytes(b"P5 53 37 255 " + bytes(10))
    with pytest.raises(H.TruncatedData):
        H.read_batch(paths + [tmp_path / "bad.pgm"], pinned=False)
    H.write_image(str(tmp_path / "small.pgm"), H.Image(gray[0][:, :10, :10].copy()))
    with pytest.raises(ValueError):
        H.read_batch(paths + [tmp_path / "small.pgm"], pinned=False)
    with pytest.raises(OSError):
        H.read_batch(paths + [tmp_path / "missing.pgm"], pinned=False)


def test_format_descriptors_golden(golden):
    v = golden["fmt/values"]
    txt = image_io.format_descriptors([3], [5], v[None], "l2").decode()
    assert txt == "3 5 " + str(golden["fmt/l2"]) + "\n"
    i = golden["fmt/ints"]
    txt = image_io.format_descriptors([0, 7], [1, 2], np.stack([i, i]), "none").decode()
    assert txt == "".join(f"{x} {y} " + str(golden["fmt/none"]) + "\n" for x, y in ((0, 1), (7, 2)))
    assert image_io.format_descriptors([], [], np.zeros((0, 4)), "none") == b""


def test_format_matches_python_on_random_values():
    rng = np.random.default_rng(11)
    v = np.concatenate([rng.random(300), rng.normal(0, 1e-5, 300), rng.normal(0, 1e9, 100)])
    txt = image_io.format_descriptors([1], [2], v[None], "l1").decode().split()
    assert txt[2:] == [format(float(x), ".9g") for x in v]


@pytest.mark.gpu
@pytest.mark.parametrize("norm", ["none", "l2"])
def test_extract_text_golden(golden, norm):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    g = H.DescriptorGeometry(16, 24, 8, block=2, block_stride=1, bins=9, normalization=norm)
    buf = io.BytesIO()
    n = image_io.extract(H.Image(golden["extract/image"]), g, 6, buf)
    assert buf.getvalue() == bytes(golden[f"extract/{norm}"])
    assert n == buf.getvalue().count(b"\n")
