"""Intra-frame split run live: two processes, each a rank
of a gloo group on cuda:0, run SlabPipeline.run(group=...) so the real
all_gather of per-slab column counts delivers the carry
(integral.py:75-79 across ranks).  Each rank's plane rows and cell-grid rows
must equal the whole-frame run's, bit for bit.  No kernel waits on the other
rank: the exchange is a host-side collective between the two launches.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, key, crop, out):
    import torch.distributed as dist

    import paper_1703_06256_b200 as H
    from oracle import oracle as O
    from paper_1703_06256_b200 import slab, synth

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synth.CONFIGS[key]
        h, w = crop or (cfg.height, cfg.width)
        frames = np.ascontiguousarray(synth.make_batch(cfg, 1, 2)[:, :, :h, :w])
        sp = slab.SlabPipeline(2, cfg.channels, h, w, cfg.bins, stride=cfg.stride, rank=rank,
                               world=world, group=dist.group.WORLD)
        sp.upload(frames)
        sp.run()  # bin + own counts -> all_gather -> planes + grid
        torch.cuda.synchronize()
        whole = H.HogPipeline(2, cfg.channels, h, w, cfg.bins, stride=cfg.stride,
                              grid_dtype="int32")
        whole.upload(frames)
        whole.run()
        torch.cuda.synchronize()
        ok_planes = torch.equal(sp.planes_view(), whole.planes_view()[:, :, sp.y0: sp.y1 + 1])
        ok_grid = torch.equal(sp.grid_view(),
                              whole.grid[:, sp.cell_row0: sp.cell_row0 + sp.ncy])
        # and the oracle, for frame 0 of this slab's rows
        lut = O.build_lut(cfg.bins)
        ref = O.integral_stack(O.gradient_map(frames[0], lut), cfg.bins)[:, sp.y0: sp.y1 + 1]
        ok_oracle = np.array_equal(sp.planes_view()[0].cpu().numpy().view(np.uint32), ref)
        out[rank] = (bool(ok_planes), bool(ok_grid), bool(ok_oracle), sp.y0, sp.y1,
                     int(sp.base.sum().item()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("key,crop,world", [("c2", None, 2), ("c5", (1100, 1600), 2),
                                            ("c4", (360, 640), 3)])
def test_slab_split_live_exchange(key, crop, world):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_rank, args=(world, _port(), key, crop, out), nprocs=world, join=True)
    for r in range(world):
        ok_planes, ok_grid, ok_oracle, y0, y1, carry = out[r]
        assert ok_planes and ok_grid and ok_oracle, (r, out[r])
    assert out[0][5] == 0 and all(out[r][5] > 0 for r in range(1, world))
    assert [out[r][4] for r in range(world - 1)] == [out[r][3] for r in range(1, world)]
