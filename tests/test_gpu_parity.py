"""Parity of the CUDA path (through the C ABI) with the reference's golden
vectors and with the pinned CPU oracle.  Bit-exact for bin maps, planes,
cell grids and normalised descriptors; scores within a stated tolerance.

Score tolerance: |gpu - ref| <= 1e-12 * sum|w| * 64 + 1e-12 (absolute), far
inside the north-star's 1e-5 relative bound; fp64 accumulation in a
different order than OpenBLAS's ddot is the only source of difference.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1703_06256_b200 as H  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1703_06256_b200 import synth  # noqa: E402

CASES = ["gray45x37", "rgb48x40", "gray133x77", "rgb3x3", "gray300x200_b18",
         "rgbtie70x50", "c2frame0_crop"]


def score_tol(w):
    return 1e-12 * float(np.abs(w).sum()) * 64 + 1e-12


def geom(gname, bins, norm="none"):
    if gname == "g16b2":
        return H.DescriptorGeometry(16, 16, 8, 2, 1, bins, norm)
    return H.DescriptorGeometry(16, 24, 8, 2, 1, bins, norm)


@pytest.mark.parametrize("name", CASES)
def test_binmap_and_planes_golden(golden, name):
    img, bins = golden[f"{name}/image"], int(golden[f"{name}/bins"])
    bm = H.gradient_map(H.Image(img), H.build_lut(bins))
    assert bm.cells.dtype == np.int16
    assert np.array_equal(bm.cells, golden[f"{name}/binmap"])
    st = H.build_integral_stack(bm)
    assert st.planes.dtype == np.uint32
    assert O.sha256(st.planes) == str(golden[f"{name}/planes_sha"])


@pytest.mark.parametrize("name", CASES)
def test_grids_and_descriptors_golden(golden, name):
    img, bins = golden[f"{name}/image"], int(golden[f"{name}/bins"])
    st = H.build_integral_stack(H.gradient_map(H.Image(img), H.build_lut(bins)))
    for gname in ("g16b2", "g16x24"):
        for norm in ("none", "l1", "l2"):
            for stride in (1, 3, 8):
                key = f"{name}/{gname}/{norm}/s{stride}"
                if f"{key}/descs_sha" not in golden.files:
                    continue
                g = geom(gname, bins, norm)
                oxs, oys = H.window_origins(st.width, st.height, g, stride)
                if norm == "none":
                    cache = H.CellHistogramCache(st, g, oxs, oys)
                    assert np.array_equal(cache.grid, golden[f"{key}/grid"])
                descs = np.stack([d for _, _, d in H.scan_descriptors(st, g, stride)])
                assert descs.dtype == (np.int64 if norm == "none" else np.float64)
                assert O.sha256(descs) == str(golden[f"{key}/descs_sha"]), key


@pytest.mark.parametrize("name", CASES)
def test_scan_scores_golden(golden, name):
    img, bins = golden[f"{name}/image"], int(golden[f"{name}/bins"])
    st = H.build_integral_stack(H.gradient_map(H.Image(img), H.build_lut(bins)))
    for gname in ("g16b2", "g16x24"):
        if f"{name}/{gname}/weights" not in golden.files:
            continue
        w = golden[f"{name}/{gname}/weights"]
        model = H.LinearModel(geom(gname, bins), w, 0.125)
        for stride in (2, 4):
            dets = H.scan(st, model, stride, float("-inf"))
            xy = np.array([(d.x, d.y) for d in dets])
            assert np.array_equal(xy, golden[f"{name}/{gname}/scan_s{stride}/xy"])
            np.testing.assert_allclose([d.score for d in dets],
                                       golden[f"{name}/{gname}/scan_s{stride}/score"],
                                       rtol=0, atol=score_tol(w))
    for norm in ("none", "l2"):
        for stride in (4, 8):
            key = f"{name}/b1_{norm}/s{stride}"
            if f"{key}/score" not in golden.files:
                continue
            g = H.DescriptorGeometry(16, 32, 8, 1, 1, bins, norm)
            w = golden[f"{key}/weights"]
            dets = H.scan(st, H.LinearModel(g, w, 0.0), stride, float("-inf"))
            np.testing.assert_allclose([d.score for d in dets], golden[f"{key}/score"],
                                       rtol=0, atol=score_tol(w))


def test_config1_full_pipeline_golden(golden):
    cfg = synth.CONFIGS["c1"]
    frame = synth.make_frame(cfg, 0)
    w, bias = synth.make_weights(cfg)
    p = H.HogPipeline(1, 1, cfg.height, cfg.width, cfg.bins, stride=cfg.stride, weights=w,
                      bias=bias)
    assert p.fused
    p.upload(frame[None])
    p.run()
    torch.cuda.synchronize()
    assert O.sha256(p.binmap_view()[0].cpu().numpy().astype(np.int16)) == str(golden["c1/binmap_sha"])
    planes = p.planes_view()[0].cpu().numpy().view(np.uint32)
    assert O.sha256(planes) == str(golden["c1/planes_sha"])
    grid = p.grid[0].cpu().numpy().astype(np.int64)
    assert O.sha256(grid) == str(golden["c1/grid_sha"])
    ref = golden["c1/scores"]
    s = p.scores[0].cpu().numpy()
    assert s.shape == ref.shape
    assert (np.abs(s - ref) / np.abs(ref)).max() < 1e-10  # north star: 1e-5


@pytest.mark.parametrize("key,count", [("c2", 3), ("c3", 2), ("c4", 2)])
def test_config_batches_vs_oracle(key, count):
    cfg = synth.CONFIGS[key]
    frames = synth.make_batch(cfg, 0, count)
    weights, bias = synth.make_weights(cfg) if cfg.scored else (None, 0.0)
    p = H.HogPipeline(count, cfg.channels, cfg.height, cfg.width, cfg.bins, stride=cfg.stride,
                      normalization=cfg.normalization, weights=weights, bias=bias)
    assert p.fused
    p.upload(frames)
    p.run()
    torch.cuda.synchronize()
    lut = O.build_lut(cfg.bins)
    mode = 1 if cfg.scored else (2 if cfg.normalization == "l2" else 0)
    _, grid, scores = O.run_batch(frames, lut, cfg.bins, 8, 64, 128, cfg.stride, mode,
                                  weights, bias, threads=4, want_outputs=True)
    assert np.array_equal(p.grid.cpu().numpy().astype(np.int64), grid)
    # planes and bin map of the first frame, bit-exact
    cells = O.gradient_map(frames[0], lut)
    assert np.array_equal(p.binmap_view()[0].cpu().numpy().astype(np.int16), cells)
    assert np.array_equal(p.planes_view()[0].cpu().numpy().view(np.uint32),
                          O.integral_stack(cells, cfg.bins))
    if cfg.scored:
        np.testing.assert_allclose(p.scores.cpu().numpy(), scores, rtol=1e-5,
                                   atol=score_tol(weights))
        rel = np.abs(p.scores.cpu().numpy() - scores) / np.maximum(np.abs(scores), 1e-300)
        assert np.median(rel) < 1e-12
    if cfg.normalization == "l2":
        g = grid.astype(np.float64)
        den = np.sqrt((g * g).sum(axis=-1) + 1e-6 * 1e-6)
        assert np.array_equal(p.denom.cpu().numpy(), den)
        assert np.array_equal(p.normalized_grid().cpu().numpy(), g / den[..., None])


def test_fused_grid_equals_generic_corner_reads():
    # the fused-grid kernel and the generic 4-corner kernel on the same planes
    cfg = synth.CONFIGS["c2"]
    frames = synth.make_batch(cfg, 5, 4)
    p = H.HogPipeline(4, 1, cfg.height, cfg.width, cfg.bins, stride=cfg.stride)
    p.upload(frames)
    p.run()
    from paper_1703_06256_b200.descriptor import cell_grid_device

    generic = cell_grid_device(p.planes, p.cell_xs, p.cell_ys, 8)
    assert p.grid.dtype == torch.uint8  # unscored c2: exact uint8 cell counts
    assert torch.equal(generic, p.grid.to(torch.int32))
    q = H.HogPipeline(4, 1, cfg.height, cfg.width, cfg.bins, stride=cfg.stride, grid_dtype="int32")
    q.upload(frames)
    q.run()
    assert torch.equal(generic, q.grid)


@pytest.mark.parametrize("w,h,c,bins", [(3, 3, 1, 8), (5, 4, 3, 9), (37, 29, 1, 8),
                                        (129, 65, 1, 18), (255, 7, 3, 4), (641, 13, 1, 2),
                                        (70, 66, 1, 30), (33, 31, 3, 64)])
def test_odd_shapes_and_bin_counts_vs_oracle(w, h, c, bins):
    rng = np.random.default_rng(w * 1000 + h * 10 + bins)
    img = rng.integers(0, 256, (c, h, w), dtype=np.uint8)
    lut = H.build_lut(bins)
    bm = H.gradient_map(H.Image(img), lut)
    ref = O.gradient_map(img, O.build_lut(bins))
    assert np.array_equal(bm.cells, ref)
    st = H.build_integral_stack(bm)
    assert np.array_equal(st.planes, O.integral_stack(ref, bins))


def test_user_binmap_with_out_of_range_values():
    # integral.py:76: only cells == n count; other values (incl. -1) count nowhere
    rng = np.random.default_rng(9)
    cells = rng.integers(-3, 12, size=(40, 53)).astype(np.int16)
    st = H.build_integral_stack(H.BinMap(9, cells))
    ref = np.zeros((9, 41, 54), np.uint32)
    for n in range(9):
        ref[n, 1:, 1:] = np.cumsum(np.cumsum(cells == n, axis=0), axis=1)
    assert np.array_equal(st.planes, ref)


def test_acc_width_16():
    cells = np.full((255, 255), -1, np.int16)
    cells[1:-1, 1:-1] = 1
    st = H.build_integral_stack(H.BinMap(4, cells), acc_width=16)
    assert st.planes.dtype == np.uint16 and st.planes[1, 255, 255] == 253 * 253
    with pytest.raises(H.AccumulatorOverflowRisk):
        big = np.full((300, 300), 1, np.int16)
        H.build_integral_stack(H.BinMap(4, big), acc_width=16)


def test_constant_image_all_sentinel_and_zero_planes():
    img = np.full((1, 17, 23), 128, np.uint8)
    bm = H.gradient_map(H.Image(img), H.build_lut(8))
    assert (bm.cells == H.NO_BIN).all()
    assert not H.build_integral_stack(bm).planes.any()


def test_errors_match_reference():
    with pytest.raises(H.ImageTooSmall):
        H.gradient_map(H.Image(np.zeros((1, 2, 5), np.uint8)), H.build_lut(8))
    st = H.build_integral_stack(H.gradient_map(H.Image(np.zeros((1, 20, 20), np.uint8) + 5),
                                               H.build_lut(8)))
    g = H.DescriptorGeometry(16, 16, 8, 2, 1, 8)
    with pytest.raises(H.WindowOutOfBounds):
        H.window_descriptor(st, (5, 5), g)
    with pytest.raises(H.InvalidGeometry):
        H.window_descriptor(st, (0, 0), H.DescriptorGeometry(16, 16, 8, 2, 1, 9))
    small = H.build_integral_stack(H.gradient_map(H.Image(np.zeros((1, 12, 12), np.uint8)),
                                                  H.build_lut(9)))
    with pytest.raises(H.WindowLargerThanImage):
        H.scan(small, H.LinearModel(H.DescriptorGeometry(16, 16, 8, 2, 1, 9), np.zeros(36), 0),
               1, 0.0)


def test_window_descriptor_equals_cached_scan(golden):
    img = golden["rgb48x40/image"]
    st = H.build_integral_stack(H.gradient_map(H.Image(img), H.build_lut(9)))
    for norm in ("none", "l2"):
        g = H.DescriptorGeometry(16, 24, 8, 2, 1, 9, norm)
        for x, y, d in H.scan_descriptors(st, g, 5):
            assert np.array_equal(d, H.window_descriptor(st, (x, y), g))


def test_resize_golden(golden):
    src = golden["resize/src"]
    for (nw, nh) in ((80, 69), (40, 33), (97, 83), (13, 7), (96, 82)):
        out = H.resize_bilinear(H.Image(src), nw, nh)
        assert np.array_equal(out.planes, golden[f"resize/{nw}x{nh}"])


def test_resize_large_golden(golden):
    big = synth.make_frame(synth.CONFIGS["c5"], 0)[:, :540, :960].copy()
    for (nw, nh) in ((800, 450), (666, 375), (555, 312)):
        out = H.resize_bilinear(H.Image(big), nw, nh)
        assert O.sha256(out.planes) == str(golden[f"resize_big/{nw}x{nh}_sha"])


def test_pyramid_scan_golden(golden):
    img = golden["pyramid/image"]
    g = H.DescriptorGeometry(16, 16, 8, 2, 1, 9)
    model = H.LinearModel(g, golden["pyramid/weights"], -0.5)
    dets = H.pyramid_scan(H.Image(img), model, 1.3, 4, float("-inf"))
    assert np.array_equal(np.array([d.box for d in dets]), golden["pyramid/boxes"])
    assert np.array_equal(np.array([d.scale for d in dets]), golden["pyramid/scale"])
    np.testing.assert_allclose([d.score for d in dets], golden["pyramid/score"], rtol=0,
                               atol=score_tol(golden["pyramid/weights"]))


def test_native_library_is_the_one_loaded():
    from paper_1703_06256_b200 import _native

    lib = _native.load()
    assert os.path.samefile(lib._name, _native.LIB_PATH)


@pytest.mark.parametrize("stride,norm", [(8, "none"), (4, "none"), (8, "l2"), (4, "l1")])
def test_lattice_scores_vs_oracle(stride, norm):
    # hog_scores_lattice (fused lattice path) against the oracle's per-window
    # descriptor + dot (descriptor.py:107-124, detector.py:148-150)
    cfg = synth.CONFIGS["c2"]
    frames = synth.make_batch(cfg, 11, 2)[:, :, :200, :300].copy()
    w = np.random.default_rng(stride * 10 + len(norm)).normal(0, 0.01, 1024)
    p = H.HogPipeline(2, 1, 200, 300, 8, stride=stride, normalization=norm, weights=w, bias=0.25)
    assert p.fused
    p.upload(frames)
    p.run()
    torch.cuda.synchronize()
    g = O.Geometry(64, 128, 8, 1, 1, 8, norm)
    lut = O.build_lut(8)
    for i in range(2):
        planes = O.integral_stack(O.gradient_map(frames[i], lut), 8)
        ref = O.scan_scores(planes, g, stride, w, 0.25)
        np.testing.assert_allclose(p.scores[i].cpu().numpy(), ref, rtol=1e-9, atol=score_tol(w))


@pytest.mark.parametrize("key", ["c2", "c4", "c3"])
def test_fused_lookback_variant_matches(monkeypatch, key):
    # opt-in fused kernel (binning + decoupled look-back inside k_planes) is
    # bit-identical to the three-kernel path
    cfg = synth.CONFIGS[key]
    frames = synth.make_batch(cfg, 3, 3)
    outs = []
    for fused in ("0", "1"):
        monkeypatch.setenv("HOGB200_FUSED", fused)
        p = H.HogPipeline(3, cfg.channels, cfg.height, cfg.width, cfg.bins, stride=cfg.stride)
        p.upload(frames)
        p.run()
        torch.cuda.synchronize()
        outs.append((p.binmap_view().clone(), p.planes_view().clone(), p.grid.clone()))
    for a, b in zip(*outs):
        assert torch.equal(a, b)


@pytest.mark.parametrize("shape", [("c2", None), ("c4", None), ("c3", None), ("c5", (600, 2100))])
def test_tma_store_variant_matches(monkeypatch, shape):
    # opt-in TMA store path (plane rows staged in shared memory, written by
    # cp.async.bulk from a store warp): bit-identical to the default path and
    # to the oracle; the c5 crop (N_b = 18, 2100 wide) runs several super-strips
    key, crop = shape
    cfg = synth.CONFIGS[key]
    h, w = crop or (cfg.height, cfg.width)
    frames = synth.make_batch(cfg, 5, 2) if crop is None else \
        np.ascontiguousarray(synth.make_batch(cfg, 5, 1)[:, :, :h, :w])
    n = frames.shape[0]
    outs = []
    for tma in ("0", "1"):
        monkeypatch.setenv("HOGB200_TMA", tma)
        p = H.HogPipeline(n, cfg.channels, h, w, cfg.bins, stride=cfg.stride)
        p.upload(frames)
        p.run()
        torch.cuda.synchronize()
        outs.append((p.binmap_view().clone(), p.planes_view().clone(), p.grid.clone()))
    for a, b in zip(*outs):
        assert torch.equal(a, b)
    lut = O.build_lut(cfg.bins)
    ref = O.integral_stack(O.gradient_map(frames[n - 1], lut), cfg.bins)
    assert np.array_equal(outs[1][1][n - 1].cpu().numpy().view(np.uint32), ref)


@pytest.mark.parametrize("bins,stride,h,w", [(18, 8, 300, 1000), (8, 4, 203, 611), (9, 8, 129, 64)])
def test_scores_rows_kernel(monkeypatch, bins, stride, h, w):
    # k_scores_rows over the byte grid (default: 16-byte cp.async of misaligned
    # grid rows -- every case here has rows that are not 16-byte multiples --
    # zero-fill past the end of the grid) and over the int32 grid, against the
    # oracle's per-window dot products and against the first lattice kernel
    rng = np.random.default_rng(bins * 1000 + h)
    frames = synth.make_batch(synth.CONFIGS["c5"], 2, 1)[:, :, :h, :w].copy()
    frames = np.concatenate([frames, rng.integers(0, 256, frames.shape, dtype=np.uint8)])
    wts = rng.normal(0, 0.01, 128 * bins)
    got = []
    for gd, v1 in (("auto", None), ("int32", None), ("int32", "1")):
        if v1:
            monkeypatch.setenv("HOGB200_SCORES_V1", v1)
        p = H.HogPipeline(2, 1, h, w, bins, stride=stride, weights=wts, bias=-0.125, grid_dtype=gd)
        assert p.grid_u8 == (gd == "auto")
        p.upload(frames)
        p.run()
        torch.cuda.synchronize()
        got.append(p.scores.cpu().numpy())
    np.testing.assert_allclose(got[0], got[1], rtol=1e-12, atol=score_tol(wts))
    np.testing.assert_allclose(got[0], got[2], rtol=1e-12, atol=score_tol(wts))
    g = O.Geometry(64, 128, 8, 1, 1, bins)
    lut = O.build_lut(bins)
    for i in range(2):
        ref = O.scan_scores(O.integral_stack(O.gradient_map(frames[i], lut), bins), g, stride, wts, -0.125)
        np.testing.assert_allclose(got[0][i], ref, rtol=1e-9, atol=score_tol(wts))


@pytest.mark.parametrize("chunks,h,w", [(2, 200, 320), (3, 200, 320), (3, 140, 330)])
def test_chunked_two_stream_pipeline_matches(chunks, h, w):
    # frame groups on two streams (binning of group j+1 under the planes of
    # group j) give the same bin maps, planes, grid and scores as one launch;
    # at 140 x 330 a frame's byte grid is 5,576 bytes, so the groups' grid
    # slices start off 16-byte boundaries (the score kernel's staging copies)
    cfg = synth.CONFIGS["c4"]
    frames = np.ascontiguousarray(synth.make_batch(cfg, 7, 5)[:, :, :h, :w])
    w_, b = synth.make_weights(cfg)
    outs = []
    for ch in (1, chunks):
        p = H.HogPipeline(5, 3, h, w, cfg.bins, stride=cfg.stride, weights=w_, bias=b, chunks=ch)
        assert p.chunks == ch
        p.upload(frames)
        p.run()
        torch.cuda.synchronize()
        outs.append((p.binmap_view().clone(), p.planes_view().clone(), p.grid.clone(),
                     p.scores.clone()))
    for a, c in zip(*outs):
        assert torch.equal(a, c)


@pytest.mark.parametrize("stride,norm", [(8, "l2"), (12, "none"), (12, "l1")])
def test_chunked_pipeline_grid_consumers(stride, norm):
    # per-group grid consumers on the third stream: per-cell denominators +
    # int32 lattice scores (fused, normalised), and the general cell-grid +
    # window-feature path (stride 12: no regular lattice), equal to one launch
    cfg = synth.CONFIGS["c3"]
    frames = np.ascontiguousarray(synth.make_batch(cfg, 9, 5)[:, :, :260, :330])
    w = np.random.default_rng(stride).normal(0, 0.01, 128 * cfg.bins)
    outs = []
    for ch in (1, 3):
        p = H.HogPipeline(5, 1, 260, 330, cfg.bins, stride=stride, normalization=norm, weights=w,
                          bias=0.1, chunks=ch)
        assert p.fused == (stride == 8)
        p.upload(frames)
        p.run()
        torch.cuda.synchronize()
        outs.append([p.grid.clone(), p.scores.clone()] +
                    ([p.denom.clone()] if p.denom is not None else []))
    for a, c in zip(*outs):
        assert torch.equal(a, c)
    g = O.Geometry(64, 128, 8, 1, 1, cfg.bins, norm)
    lut = O.build_lut(cfg.bins)
    ref = O.scan_scores(O.integral_stack(O.gradient_map(frames[4], lut), cfg.bins), g, stride, w, 0.1)
    np.testing.assert_allclose(outs[1][1][4].cpu().numpy(), ref, rtol=1e-9, atol=score_tol(w))


@pytest.mark.parametrize("wh,stride", [(16, 8), (24, 8), (16, 4), (40, 4)])
def test_scores_rows_short_windows(wh, stride):
    # windows 1-5 cells tall: the score kernel's active-row masks include the
    # short runs (cells_y < 4) and, at stride 4, the one-parity runs
    rng = np.random.default_rng(wh * 10 + stride)
    frames = rng.integers(0, 256, (2, 1, 90, 260), dtype=np.uint8)
    bins = 9
    cells_y = wh // 8
    wts = rng.normal(0, 0.01, 8 * cells_y * bins)
    p = H.HogPipeline(2, 1, 90, 260, bins, stride=stride, window=(64, wh), weights=wts, bias=0.5)
    assert p.fused and p.grid_u8
    p.upload(frames)
    p.run()
    torch.cuda.synchronize()
    g = O.Geometry(64, wh, 8, 1, 1, bins)
    lut = O.build_lut(bins)
    for i in range(2):
        ref = O.scan_scores(O.integral_stack(O.gradient_map(frames[i], lut), bins), g, stride, wts, 0.5)
        np.testing.assert_allclose(p.scores[i].cpu().numpy(), ref, rtol=1e-9, atol=score_tol(wts))


@pytest.mark.parametrize("key,crop", [("c4", (300, 1280)), ("c3", (400, 1000)), ("c5", (260, 2100)),
                                      ("c2", None)])
def test_band_rows_invariance(key, crop):
    # the plane kernel's band rows only change the tiling: every R gives the
    # same bin map, planes and grid (and the oracle's planes); c5's crop is
    # 2100 wide with N_b = 18 (several super-strips per CTA), c4 is RGB
    # with 8 columns per lane
    cfg = synth.CONFIGS[key]
    h, w = crop or (cfg.height, cfg.width)
    frames = np.ascontiguousarray(synth.make_batch(cfg, 13, 2)[:, :, :h, :w])
    outs = []
    for rows in (16, 40, 96, 240, None):
        p = H.HogPipeline(2, cfg.channels, h, w, cfg.bins, stride=cfg.stride, band_rows=rows)
        if rows is None:
            assert p.band_rows in p.band_rows_timings  # tuned among the measured candidates
        p.upload(frames)
        p.run()
        torch.cuda.synchronize()
        outs.append((p.binmap_view().clone(), p.planes_view().clone(), p.grid.clone()))
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            assert torch.equal(a, b)
    lut = O.build_lut(cfg.bins)
    ref = O.integral_stack(O.gradient_map(frames[1], lut), cfg.bins)
    assert np.array_equal(outs[0][1][1].cpu().numpy().view(np.uint32), ref)


def test_pipelined_batches_scores():
    # consecutive pipelined runs: batch k's scores (post stream) overlap batch
    # k+1's binning; batch k+1's plane kernel must wait for them (it rewrites
    # the grid they read).  Alternate two batches with separate score buffers.
    cfg = synth.CONFIGS["c4"]
    n = 16
    fa = synth.make_batch(cfg, 20, n)
    fb = synth.make_batch(cfg, 40, n)
    w, b = synth.make_weights(cfg)
    p = H.HogPipeline(n, 3, cfg.height, cfg.width, cfg.bins, stride=cfg.stride, weights=w, bias=b)
    outs = [torch.empty_like(p.scores) for _ in range(4)]
    for i, fr in enumerate((fa, fb, fa, fb)):
        p.upload(fr)
        p.run(pipelined=True, scores_ptr=outs[i].data_ptr())
    p.join()
    torch.cuda.synchronize()
    q = H.HogPipeline(n, 3, cfg.height, cfg.width, cfg.bins, stride=cfg.stride, weights=w, bias=b)
    refs = []
    for fr in (fa, fb):
        q.upload(fr)
        q.run()
        torch.cuda.synchronize()
        refs.append(q.scores.clone())
    for i in range(4):
        assert torch.equal(outs[i], refs[i % 2])


@pytest.mark.parametrize("bins,h,w,wh", [(8, 300, 700, 128), (18, 250, 1000, 128), (9, 180, 400, 40)])
def test_scores_rows_five_rows_per_warp(monkeypatch, bins, h, w, wh):
    # 5 window rows per warp (chosen when it saves a CTA wave, c4) against 4
    # and the oracle; window-row counts that are not multiples of 5 or 20
    rng = np.random.default_rng(bins + h)
    frames = rng.integers(0, 256, (3, 1, h, w), dtype=np.uint8)
    cells_y = wh // 8
    wts = rng.normal(0, 0.01, 8 * cells_y * bins)
    got = []
    for ty in ("4", "5"):
        monkeypatch.setenv("HOGB200_SCORES_TY", ty)
        p = H.HogPipeline(3, 1, h, w, bins, stride=8, window=(64, wh), weights=wts, bias=0.3)
        p.upload(frames)
        p.run()
        torch.cuda.synchronize()
        got.append(p.scores.cpu().numpy())
    np.testing.assert_allclose(got[0], got[1], rtol=1e-12, atol=score_tol(wts))
    g = O.Geometry(64, wh, 8, 1, 1, bins)
    lut = O.build_lut(bins)
    for i in (0, 2):
        ref = O.scan_scores(O.integral_stack(O.gradient_map(frames[i], lut), bins), g, 8, wts, 0.3)
        np.testing.assert_allclose(got[1][i], ref, rtol=1e-9, atol=score_tol(wts))


@pytest.mark.parametrize("key,count", [("c4", 80), ("c2", 256)])
def test_big_batch_paths_vs_oracle(key, count):
    # the variants only big batches select (>= 64 Mpx: 8 plane columns per
    # lane with 256-bit stores for c4; band rows / sub-bands sized for many
    # CTAs): first and last frame against the oracle, scores of both
    cfg = synth.CONFIGS[key]
    frames = synth.make_batch(cfg, 100, count)
    weights, bias = synth.make_weights(cfg) if cfg.scored else (None, 0.0)
    p = H.HogPipeline(count, cfg.channels, cfg.height, cfg.width, cfg.bins, stride=cfg.stride,
                      weights=weights, bias=bias)
    p.upload(frames)
    p.run()
    torch.cuda.synchronize()
    lut = O.build_lut(cfg.bins)
    ends = [0, count - 1]
    mode = 1 if cfg.scored else 0
    _, grid, scores = O.run_batch(frames[ends], lut, cfg.bins, 8, 64, 128, cfg.stride, mode,
                                  weights, bias, threads=4, want_outputs=True)
    assert np.array_equal(p.grid[ends].cpu().numpy().astype(np.int64), grid)
    for i in ends:
        cells = O.gradient_map(frames[i], lut)
        assert np.array_equal(p.binmap_view()[i].cpu().numpy().astype(np.int16), cells)
        assert np.array_equal(p.planes_view()[i].cpu().numpy().view(np.uint32),
                              O.integral_stack(cells, cfg.bins))
    if cfg.scored:
        np.testing.assert_allclose(p.scores[ends].cpu().numpy(), scores, rtol=1e-9,
                                   atol=score_tol(weights))


@pytest.mark.parametrize("bins,stride,norm", [(20, 8, "none"), (32, 4, "l2"), (64, 8, "none")])
def test_pipeline_more_than_18_bins_vs_oracle(bins, stride, norm):
    """N_b > 18: HogPipeline bins, then builds the planes in bin groups through the
    single-write plane kernel (hog_integral) and the grid with hog_cell_grid."""
    cfg = synth.CONFIGS["c2"]
    frames = np.ascontiguousarray(synth.make_batch(cfg, 5, 3)[:, :, :200, :330])
    rng = np.random.default_rng(bins)
    w = rng.normal(0, 0.01, 128 * bins)
    scored = norm == "none"
    p = H.HogPipeline(3, 1, 200, 330, bins, stride=stride, normalization=norm,
                      weights=w if scored else None, bias=0.25)
    assert not p.fused
    p.upload(frames)
    p.run()
    torch.cuda.synchronize()
    lut = O.build_lut(bins)
    for i in range(3):
        cells = O.gradient_map(frames[i], lut)
        assert np.array_equal(p.binmap_view()[i].cpu().numpy().astype(np.int16), cells)
        assert np.array_equal(p.planes_view()[i].cpu().numpy().view(np.uint32),
                              O.integral_stack(cells, bins))
    mode = 1 if scored else 2
    _, grid, scores = O.run_batch(frames, lut, bins, 8, 64, 128, stride, mode,
                                  w if scored else None, 0.25, threads=2, want_outputs=True)
    assert np.array_equal(p.grid.cpu().numpy().astype(np.int64), grid)
    if scored:
        np.testing.assert_allclose(p.scores.cpu().numpy(), scores, rtol=0, atol=score_tol(w))
