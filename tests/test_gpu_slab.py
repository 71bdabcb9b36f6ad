"""Intra-frame split on the device: every slab of a frame
run through hog_pipeline_slab (halo rows + column carry) reproduces the
single-GPU bin map, planes and cell grid bit-exactly.  The slabs run one
after another in this process, each with the carry the exchange would deliver
(exclusive prefix of the slabs' hog_column_counts), so no kernel waits on
another rank."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1703_06256_b200 as H  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1703_06256_b200 import slab, synth  # noqa: E402


@pytest.mark.parametrize("key,crop,world", [("c2", None, 2), ("c2", None, 5), ("c4", (300, 400), 3),
                                            ("c5", (1080, 1920), 8), ("c3", None, 4)])
def test_slabs_reproduce_whole_frame(key, crop, world):
    cfg = synth.CONFIGS[key]
    h, w = crop or (cfg.height, cfg.width)
    frames = np.ascontiguousarray(synth.make_batch(cfg, 2, 2)[:, :, :h, :w])
    whole = H.HogPipeline(2, cfg.channels, h, w, cfg.bins, stride=cfg.stride, grid_dtype="int32")
    whole.upload(frames)
    whole.run()
    parts = [slab.SlabPipeline(2, cfg.channels, h, w, cfg.bins, stride=cfg.stride, rank=r,
                               world=world) for r in range(world)]
    own = []
    for p in parts:
        p.upload(frames)
        own.append(p.bin_and_count().clone())
    run = torch.zeros_like(own[0])
    for p, o in zip(parts, own):  # the exclusive prefix the all_gather provides
        p.planes_and_grid(base=run)
        run = run + o
    torch.cuda.synchronize()
    wp, wb, wg = whole.planes_view(), whole.binmap_view(), whole.grid
    covered = 0
    for p in parts:
        if p.empty:
            continue
        assert torch.equal(p.binmap.view(), wb[:, p.y0:p.y1e]), (p.rank, "binmap")
        assert torch.equal(p.planes_view(), wp[:, :, p.y0:p.y1 + 1]), (p.rank, "planes")
        assert torch.equal(p.planes.view(), wp[:, :, p.y0:p.y1e + 1]), (p.rank, "ext planes")
        if p.ncy:
            assert torch.equal(p.grid_view(), wg[:, p.cell_row0:p.cell_row0 + p.ncy]), p.rank
        covered += p.ncy
    assert covered == wg.shape[1]
    # and the whole-frame path itself against the oracle (last frame)
    lut = O.build_lut(cfg.bins)
    ref = O.integral_stack(O.gradient_map(frames[1], lut), cfg.bins)
    assert np.array_equal(wp[1].cpu().numpy().view(np.uint32), ref)
