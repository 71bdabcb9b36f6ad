"""Multi-rank host logic on CPU: world_size-2 gloo over 127.0.0.1 (frame
sharding + the max-over-ranks timing reduction bench.py uses)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1703_06256_b200 import sharding, synth


def test_shards_partition_the_batch():
    n, world = 513, 4
    got = [list(sharding.split(n, r, world)) for r in range(world)]
    assert sum(got, []) == list(range(n))
    assert max(map(len, got)) - min(map(len, got)) <= 1
    assert list(sharding.shard(1, 2, 512)) == list(range(512, 1024))
    with pytest.raises(ValueError):
        sharding.shard(2, 2, 8)


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
        cfg = synth.CONFIGS["c2"]
        frames = sharding.shard(rank, world, 2)
        # each rank regenerates exactly its own frames from the per-frame seeds
        batch = synth.make_batch(cfg, frames.start, len(frames))
        local = synth.batch_sha256(batch)
        # slowest-rank timing: rank-dependent fake times
        t = sharding.max_over_ranks([1.0 + rank, 5.0 - rank])
        out[rank] = (local, t, list(frames))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_shard_and_max():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    assert out[0][2] == [0, 1] and out[1][2] == [2, 3]
    # both ranks agree on the max over ranks
    assert out[0][1] == out[1][1] == [2.0, 5.0]
    # shards are distinct frames, equal to the single-process generation
    cfg = synth.CONFIGS["c2"]
    full = synth.make_batch(cfg, 0, 4)
    assert out[0][0] == synth.batch_sha256(full[:2])
    assert out[1][0] == synth.batch_sha256(full[2:])
    assert not np.array_equal(full[0], full[2])


def _gather_worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 7
        mine = sharding.split(n, rank, world)
        g = sharding.HostGather(f"test_{port}", (n, 3, 2), np.float64, mine, rank, dist.barrier,
                                pin=False)
        # each rank writes only its own contiguous slice
        loc = g.local()
        assert loc.shape[0] == len(mine)
        for j, f in enumerate(mine):
            loc[j] = float(f) + 0.25
        dist.barrier()
        if rank == 0:
            out["gathered"] = g.array.copy()
        g.close()
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_host_gather_in_frame_order():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_gather_worker, args=(world, port, out), nprocs=world, join=True)
    want = np.broadcast_to((np.arange(7) + 0.25)[:, None, None], (7, 3, 2))
    assert np.array_equal(out["gathered"], want)
    assert not os.path.exists(f"/dev/shm/hogb200_test_{port}")  # rank 0 removed the buffer
