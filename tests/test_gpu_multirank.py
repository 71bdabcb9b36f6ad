"""Strong frame split through bench.py itself: the config's batch
is cut into contiguous shards, one per rank, and every rank's results land in
its slice of one host buffer shared by the node's ranks.  The gathered batch
of a 2-rank run must equal the 1-rank run's bit for bit.

Both ranks run on cuda:0 (HOGB200_BENCH_SAME_GPU=1) with gloo for the
barrier / max-over-ranks plumbing: there is no data-path collective, so no
kernel of one rank waits on the other's.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bench(world, args, dump):
    env = dict(os.environ, HOGB200_BENCH_SAME_GPU="1", HOGB200_BENCH_BACKEND="gloo",
               HOGB200_TUNE="0")
    common = ["bench.py", "--gpus", str(world), "--steps", "2", "--warmup", "3",
              "--no-cpu-baseline", "--dump-result", dump] + args
    if world == 1:
        cmd = [sys.executable] + common
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={world}", "--master-addr", "127.0.0.1",
               "--master-port", str(_port())] + common
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    return line, np.load(dump)


@pytest.mark.parametrize("config,frames,world", [("c2", 8, 2), ("c4", 6, 2), ("c2", 5, 3)])
def test_strong_split_gather_equals_one_rank(tmp_path, config, frames, world):
    args = ["--config", config, "--frames", str(frames)]
    one, res1 = _bench(1, args, str(tmp_path / "one.npy"))
    many, resn = _bench(world, args, str(tmp_path / "many.npy"))
    assert one["scaling"] == many["scaling"] == "strong"
    assert one["config"]["global_frames"] == many["config"]["global_frames"] == frames
    assert many["config"]["frames_per_gpu"] == -(-frames // world)  # rank 0's shard
    assert many["n_gpus"] == world
    assert res1.shape[0] == resn.shape[0] == frames
    assert res1.dtype == resn.dtype
    assert np.array_equal(res1, resn)  # ordered host gather, bit for bit
    assert many["e2e"]["matches_device_run"] and one["e2e"]["matches_device_run"]
