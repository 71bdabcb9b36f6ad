"""Intra-frame multi-GPU split, host logic on CPU:
slab bounds, the exclusive column carry, and a world_size-2 gloo run of the
one exchange (all_gather of per-slab column counts) checked against the
oracle's whole-frame planes.  The CUDA side is tests/test_gpu_slab.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_1703_06256_b200 import slab, synth


@pytest.mark.parametrize("h,world,step", [(480, 2, 4), (4320, 8, 8), (600, 3, 8), (131, 4, 4),
                                          (20, 8, 8)])
def test_slab_bounds_partition(h, world, step):
    b = slab.slab_bounds(h, world, step)
    assert len(b) == world and b[0][0] == 0 and b[-1][1] == h
    for (a0, a1), (c0, c1) in zip(b, b[1:]):
        assert a1 == c0
    for y0, y1 in b:
        assert (y0 % step == 0 or y0 == h) and y0 <= y1  # trailing ranks may get no rows
    sizes = [y1 - y0 for y0, y1 in b if y1 < h]
    if sizes:
        assert max(sizes) - min(sizes) <= step
    f, e, ht, hb = slab.computed_rows(b[0][0], b[0][1], h, 8)
    assert f == 0 and ht == 0 and e == min(b[0][1] + 8, h) and hb == int(e < h)


def _global(cfg, bins):
    frame = synth.make_batch(cfg, 0, 1)[0][:, :200, :300].copy()
    cells = O.gradient_map(frame, O.build_lut(bins))
    return cells, O.integral_stack(cells, bins)


def _local_planes(cells, y0, y1e, base, bins):
    """Slab planes: local SAT of rows [y0, y1e) plus the carry row sum_{x'<X} base."""
    loc = O.integral_stack(cells[y0:y1e].copy(), bins).astype(np.int64)
    carry = np.zeros((bins, cells.shape[1] + 1), np.int64)
    carry[:, 1:] = np.cumsum(base, axis=1)
    return loc + carry[:, None, :]


def test_exclusive_carry_reproduces_whole_frame_planes():
    bins = 8
    cells, full = _global(synth.CONFIGS["c2"], bins)
    H = cells.shape[0]
    bounds = slab.slab_bounds(H, 3, 4)
    own = [np.stack([(cells[y0:y1] == b).sum(0) for b in range(bins)]) for y0, y1 in bounds]
    bases = slab.exclusive_carry(own)
    for (y0, y1), base in zip(bounds, bases):
        _, y1e, _, _ = slab.computed_rows(y0, y1, H, 8)
        assert np.array_equal(_local_planes(cells, y0, y1e, base, bins), full[:, y0:y1e + 1])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        bins = 18
        cells, full = _global(synth.CONFIGS["c5"], bins)
        H = cells.shape[0]
        y0, y1 = slab.slab_bounds(H, world, 8)[rank]
        _, y1e, _, _ = slab.computed_rows(y0, y1, H, 8)
        own = torch.as_tensor(np.stack([(cells[y0:y1] == b).sum(0) for b in range(bins)])
                              .astype(np.int32))
        parts = [torch.empty_like(own) for _ in range(world)]
        dist.all_gather(parts, own)  # the split's only exchange
        base = sum((parts[r] for r in range(rank)), torch.zeros_like(own)).numpy()
        ok = np.array_equal(_local_planes(cells, y0, y1e, base, bins), full[:, y0:y1e + 1])
        out[rank] = (ok, y0, y1, int(base.sum()))
    finally:
        dist.destroy_process_group()


def test_gloo_two_rank_carry_exchange():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    assert out[0][0] and out[1][0]
    assert out[0][2] == out[1][1]  # contiguous slabs
    assert out[0][3] == 0 and out[1][3] > 0  # the top slab has no carry
