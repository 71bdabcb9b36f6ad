#!/usr/bin/env python
"""Benchmark of the LUT-HOG hot path on B200 (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

A step is one pass of the hot path (LUT binning -> N_b int32 integral planes
-> cell-histogram grid [-> per-cell L2 / window scores]) over one batch of a
BASELINE configuration (default c2 = BASELINE.json configs[1]: 512 blurred
640x480 frames, N_b=8, 64x128 windows at stride 4).  Frames are independent:
under torchrun the config's batch is split into contiguous frame shards, one
per rank (strong scaling, BASELINE "sharded across 1/2/4/8 GPUs"; no
collective on the data path), and every rank's results land, in frame
order, in one host buffer shared by the node's ranks (the e2e leg's
gather); timings are max over ranks.  --scaling weak gives every rank a
whole batch of its own instead.

--impl reference times the reference algorithm's CPU implementation (the
oracle port in oracle/, all host threads) on a bounded sample of the same
workload; only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

NVML_REASONS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
    0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
    0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--frames", type=int, default=0,
                    help="override the batch size (strong: frames split over the ranks; "
                         "weak: frames per rank)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the config's batch split over the ranks (default); "
                         "weak: every rank runs a whole batch of distinct frames")
    ap.add_argument("--dump-result", default="",
                    help="rank 0 saves the gathered e2e result (whole batch, frame order) "
                         "to this .npy path")
    ap.add_argument("--window-l2", action="store_true",
                    help="EXTENSION for c3's wording: per-window L2 norms of the unnormalised "
                         "window descriptors instead of the reference's per-cell (block=1) L2")
    ap.add_argument("--split-frame", action="store_true",
                    help="one frame of the config (c5: one 8K frame) cut into row slabs, one "
                         "per rank, with the column-carry all_gather (SURVEY 8f-2); reports "
                         "per-frame latency")
    ap.add_argument("--shard-of", type=int, default=0,
                    help="diagnostic: run only rank 0's shard of a W-way strong split "
                         "(the per-GPU regime of a W-GPU run, measured on one GPU)")
    ap.add_argument("--chunks", type=int, default=0, help="override binning/plane overlap chunks")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--e2e-chunk", type=int, default=0,
                    help="frames per H2D/compute/D2H chunk (0: a quarter of the step's frames, so "
                         "every chunk has its own buffer set; measured best, profiles/r2/e2e_chunking_ab.txt)")
    ap.add_argument("--e2e-slots", type=int, default=4, help="pipelines/streams in flight (e2e)")
    ap.add_argument("--e2e-tail", type=int, default=1,
                    help="split the step's last chunk in this many pieces (1: no split; steps overlap, "
                         "so a short last chunk buys nothing)")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch the timed steps (and the e2e step) eagerly, no CUDA graph")
    ap.add_argument("--e2e-overlap", type=int, default=1,
                    help="e2e: step k+1's first copies start while step k's last chunks drain")
    ap.add_argument("--pipelined", type=int, default=1,
                    help="scored configs: batch k's scores run beside batch k+1's binning")
    ap.add_argument("--pyr-streams", type=int, default=0,
                    help="c5: streams the pyramid levels are spread over (0: library default)")
    ap.add_argument("--pyr-chunk", type=int, default=16,
                    help="c5: frames per pyramid chunk (level buffers: ~7.8 GB of planes per frame)")
    return ap.parse_args()


def workload_name(cfg, window_l2: bool = False) -> str:
    kind = "i.i.d. uniform noise" if cfg.sigma is None else f"blurred noise sigma={cfg.sigma}"
    extra = f" + {cfg.rects} rects" if cfg.rects else ""
    tail = ", linear score" if cfg.scored else ""
    norm = f", per-cell {cfg.normalization}" if cfg.normalization != "none" else ""
    if window_l2:
        norm = (", per-window l2 (EXTENSION: the reference normalises per block; checked against "
                "a numpy restatement)")
    return (f"{cfg.key}: {cfg.frames}x {cfg.channels}x{cfg.height}x{cfg.width} u8 ({kind}{extra}), "
            f"N_b={cfg.bins}, cell 8, 64x128 windows stride {cfg.stride}{norm}{tail}")


def bench_config(cfg, nf_global: int, world: int, scaling: str, per_rank: int) -> dict:
    """The workload description both arms print (identical keys and values:
    the driver compares the arms' configs)."""
    H, W = cfg.height, cfg.width
    return {"workload": workload_name(cfg), "global_frames": nf_global,
            "frames_per_gpu": per_rank, "scaling": scaling,
            "parallelism": (f"{scaling} frame split over {world} GPU(s), contiguous shards, "
                            "no collective on the data path, results gathered in one host buffer"),
            "l2": f"inputs larger than L2 ({nf_global * cfg.channels * H * W / 1e6:.0f} MB of frames "
                  f"per step in, > 4 B/px of planes out, vs 126 MB L2)"}


def shard_frames(nf_global: int, rank: int, world: int, scaling: str) -> range:
    from paper_1703_06256_b200 import sharding

    if scaling == "weak":
        return sharding.shard(rank, world, nf_global // world)
    return sharding.split(nf_global, rank, world)


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(config_key, key="k_planes_bytes_per_launch"):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        return json.load(open(p)).get(config_key, {}).get(key)
    except Exception:
        return None


class ClockSampler:
    """NVML poller for SM clock + throttle reasons during the timed region."""

    def __init__(self, dev_index: int):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        self._h = None
        try:
            import pynvml

            pynvml.nvmlInit()
            import torch

            h = None
            try:
                uuid = str(torch.cuda.get_device_properties(dev_index).uuid)
                h = pynvml.nvmlDeviceGetHandleByUUID(("GPU-" + uuid).encode())
            except Exception:
                h = None
            if h is None:
                vis = os.environ.get("CUDA_VISIBLE_DEVICES")
                idx = int(vis.split(",")[dev_index]) if vis and vis.split(",")[0].isdigit() else dev_index
                h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self._nv, self._h = pynvml, h
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._h = None

    def _poll(self):
        nv = self._nv
        while not self._stop.is_set():
            self.sample()
            time.sleep(0.002)

    def sample(self):
        if self._h is None:
            return
        nv = self._nv
        try:
            self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
            self.reasons |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(self._h))
        except Exception:
            pass

    def start(self):
        if self._h is None:
            return
        self._t = threading.Thread(target=self._poll, daemon=True)
        self._t.start()

    def stop(self):
        if self._h is None:
            return None
        self._stop.set()
        self._t.join()
        self.sample()
        names = [n for b, n in NVML_REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


def gen_frames(cfg, first, count):
    from paper_1703_06256_b200 import synth

    return synth.make_batch(cfg, first, count)


# --------------------------------------------------------------------------
# CPU legs (oracle port): cpu_baseline and --impl reference

def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_run(cfg, frames, threads):
    from oracle import oracle as O
    from paper_1703_06256_b200 import synth

    lut = O.build_lut(cfg.bins)
    mode = 1 if cfg.scored else (2 if cfg.normalization == "l2" else 0)
    w, b = synth.make_weights(cfg) if cfg.scored else (None, 0.0)
    t0 = time.perf_counter()
    if not cfg.pyramid_step:
        O.run_batch(frames, lut, cfg.bins, 8, 64, 128, cfg.stride, mode, w, b, threads=threads)
        return time.perf_counter() - t0
    # pyramid (detector.py:224-269): every level resized from the original frame
    # (resizes on a host thread pool; ctypes drops the GIL), then each level of
    # all frames as one batch on `threads` threads
    from concurrent.futures import ThreadPoolExecutor

    n, C, H, W = frames.shape
    g = O.Geometry(64, 128, 8, 1, 1, cfg.bins)
    with ThreadPoolExecutor(max_workers=threads) as pool:
        for (level, factor, lw, lh) in O.pyramid_levels(W, H, g, cfg.pyramid_step):
            if level == 0:
                batch = frames
            else:
                batch = np.stack(list(pool.map(lambda f: O.resize_bilinear(f, lw, lh), frames)))
            O.run_batch(batch, lut, cfg.bins, 8, 64, 128, cfg.stride, mode, w, b, threads=threads)
    return time.perf_counter() - t0


def cpu_sample_size(cfg, frames1, threads, seconds):
    t1 = cpu_run(cfg, frames1[:1], 1)
    return max(threads, min(cfg.frames, int(seconds * threads / max(t1, 1e-3)))), t1


def host_info() -> dict:
    """CPU model, numpy and BLAS of the host the CPU legs ran on."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    blas = None
    try:
        b = np.show_config(mode="dicts")["Build Dependencies"]["blas"]
        blas = f"{b.get('name')} {b.get('version')}"
    except Exception:
        pass
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(), "affinity_cores": host_threads(),
            "numpy": np.__version__, "blas": blas}


def _ref_frame(args):
    """One frame through the vendored reference (fasthog, baseline/_ref) by
    its public API, the way SURVEY §8d maps the config: gradient_map ->
    build_integral_stack -> scan (threshold -inf) | scan_descriptors drained."""
    frame, key, bins, stride, norm, scored, w, b = args
    import fasthog as F

    lut = _REF_LUT.setdefault(bins, F.build_lut(bins))
    t0 = time.perf_counter()
    stack = F.build_integral_stack(F.gradient_map(F.Image(frame), lut))
    g = F.DescriptorGeometry(64, 128, 8, block=1, block_stride=1, bins=bins, normalization=norm)
    if scored:
        F.scan(stack, F.LinearModel(g, np.asarray(w, dtype=np.float64), float(b)), stride,
               float("-inf"))
    else:
        for _ in F.scan_descriptors(stack, g, stride):
            pass
    return time.perf_counter() - t0


_REF_LUT: dict = {}


def python_reference_sample(cfg, frames, seconds=6.0):
    """The real Python reference (baseline/_ref, vendored by pip from
    /root/reference) timed on a few frames: one process, then one frame per
    host core in a process pool (OPENBLAS_NUM_THREADS=1).  Absent on the box
    -> reported as unavailable."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "fasthog")):
        return {"unavailable": "baseline/_ref not installed (pip install --target baseline/_ref)"}
    if cfg.pyramid_step:
        return {"unavailable": "one 8K frame's 20-level pyramid takes ~130 s in the Python "
                               "reference (SURVEY 8a-13); not sampled"}
    if ref not in sys.path:
        sys.path.insert(0, ref)
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from paper_1703_06256_b200 import synth

    w, b = synth.make_weights(cfg) if cfg.scored else (None, 0.0)
    job = lambda f: (f, cfg.key, cfg.bins, cfg.stride, cfg.normalization, cfg.scored, w, b)  # noqa: E731
    t, k = 0.0, 0
    while k == 0 or (t < seconds / 2 and k < len(frames)):
        t += _ref_frame(job(frames[k % len(frames)]))
        k += 1
    one = k * cfg.height * cfg.width / t / 1e6
    out = {"one_process_mpx_s": one, "one_process_frames": k, "one_process_s": t}
    try:
        import multiprocessing as mp

        procs = host_threads()
        jobs = [job(frames[i % len(frames)]) for i in range(procs)]
        ctx = mp.get_context("fork")
        with ctx.Pool(procs) as pool:
            pool.map(_ref_frame, jobs[:procs])  # warm: imports + LUT per worker
            t0 = time.perf_counter()
            pool.map(_ref_frame, jobs)
            wall = time.perf_counter() - t0
        out.update({"pool_mpx_s": procs * cfg.height * cfg.width / wall / 1e6,
                    "pool_processes": procs, "pool_frames": procs, "pool_s": wall})
    except Exception as exc:  # pragma: no cover - pool failures only lose the sample
        out["pool_error"] = str(exc)[:200]
    out["api"] = ("fasthog gradient_map -> build_integral_stack -> "
                  + ("scan(threshold=-inf)" if cfg.scored else "scan_descriptors drained"))
    return out


def cpu_baseline(cfg, seconds, frames=None):
    """The oracle port on the host cores over a bounded sample of the workload
    (`frames`, if given, are the benchmark's own frames: no regeneration)."""
    threads = host_threads()
    probe = frames[:1] if frames is not None else gen_frames(cfg, 0, 1)
    count, t1 = cpu_sample_size(cfg, probe, threads, seconds)
    if frames is not None and len(frames) >= count:
        frames = frames[:count]
    else:
        frames = gen_frames(cfg, 0, count)
    # whole passes over the sample until at least a quarter of the time budget
    # is spent (a whole c2 batch takes ~0.1 s on 16 threads: one pass is noisy)
    dt, passes = 0.0, 0
    while passes == 0 or (dt < seconds / 4 and passes < 1000):
        dt += cpu_run(cfg, frames, threads)
        passes += 1
    px = passes * count * cfg.height * cfg.width
    return {"value": px / dt / 1e6, "unit": "Mpixel/s", "cores": threads, "kind": "port",
            "sample": f"{passes} pass(es) over {count} {cfg.key} frames ({cfg.frames} per step) "
                      f"(oracle/hog_oracle.c, {threads} threads, {dt:.1f} s; 1 frame on 1 thread: "
                      f"{t1 * 1e3:.0f} ms)",
            "single_thread_mpx_s": cfg.height * cfg.width / t1 / 1e6,
            "host": host_info(),
            "python_reference": python_reference_sample(cfg, frames if frames is not None else probe)}


def global_frames(args, cfg, world: int) -> tuple[int, str]:
    """(frames in the whole job's batch, scaling).  Strong scaling needs a
    frame per rank; a batch smaller than the world (c1: one frame) runs weak."""
    scaling = args.scaling
    if scaling == "strong" and (args.frames or cfg.frames) < world:
        scaling = "weak"
    if scaling == "weak":
        return world * (args.frames or cfg.frames), scaling
    return args.frames or cfg.frames, scaling


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    nf_global, scaling = global_frames(args, cfg, world)
    threads = host_threads()
    probe = gen_frames(cfg, 0, 1)
    # each step: a bounded sample sized for ~3 s of all-core CPU work
    per_step, t1 = cpu_sample_size(cfg, probe, threads, 3.0)
    frames = gen_frames(cfg, 0, per_step)
    for _ in range(args.warmup):
        cpu_run(cfg, frames, threads)
    times = [cpu_run(cfg, frames, threads) for _ in range(args.steps)]
    ms = statistics.mean(times) * 1e3
    px = per_step * cfg.height * cfg.width
    value = px / (ms / 1e3) / 1e6
    line = {
        "impl": "reference", "metric": "Mpixel/s (LUT binning + per-bin integral planes + window HOG)",
        "value": value, "unit": "Mpixel/s (source pixels)" if cfg.pyramid_step else "Mpixel/s",
        "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None,
        "dtype": "int32" if not cfg.scored else "int32+f64", "data": "synthetic",
        "config": bench_config(cfg, nf_global, world, scaling,
                               len(shard_frames(nf_global, 0, world, scaling))),
        "reference": {"frames_per_step": per_step,
                      "implementation": "reference algorithm restated in C (oracle/, pinned to "
                                        "the reference's golden vectors), all host threads; "
                                        "rank 0 only"},
        "cpu_baseline": {"value": value, "unit": "Mpixel/s", "cores": threads, "kind": "port",
                         "sample": f"{per_step} of {cfg.frames} {cfg.key} frames per step"},
        "e2e": {"value": value, "unit": "Mpixel/s (source pixels)" if cfg.pyramid_step else "Mpixel/s",
                "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------
# GPU leg

def main():
    args = parse_args()
    from paper_1703_06256_b200 import synth

    cfg = synth.CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist

    import paper_1703_06256_b200 as H
    from paper_1703_06256_b200 import sharding
    from paper_1703_06256_b200.errors import PathMismatch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # HOGB200_BENCH_SAME_GPU=1 + HOGB200_BENCH_BACKEND=gloo: plumbing check of the
    # multi-rank path on a one-GPU box (ranks share cuda:0; nothing waits on
    # another rank's kernels).  Real runs: one GPU per rank, NCCL.
    if os.environ.get("HOGB200_BENCH_SAME_GPU") == "1":
        local = 0
    backend = os.environ.get("HOGB200_BENCH_BACKEND", "nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    red_dev = dev if backend == "nccl" else torch.device("cpu")

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(vals):
        t = torch.tensor(vals, dtype=torch.float64, device=red_dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    if args.split_frame:
        return bench_split_frame(args, cfg, dev, world, rank, local, barrier, max_over_ranks,
                                 backend)
    nf_global, scaling = global_frames(args, cfg, world)
    if args.shard_of > 1:  # diagnostic: one rank's shard of a W-way split, on this GPU
        if world > 1:
            raise SystemExit("--shard-of is a one-process diagnostic")
        mine = sharding.split(nf_global, 0, args.shard_of)
    else:
        mine = shard_frames(nf_global, rank, world, scaling)
    nf, first = len(mine), mine.start  # this rank's contiguous shard of the batch
    frames = gen_frames(cfg, first, nf)  # frame i always comes from seed (config, i)
    weights, bias = synth.make_weights(cfg) if cfg.scored else (None, 0.0)
    job = {"nf_global": nf_global if args.shard_of <= 1 else nf, "scaling": scaling,
           "mine": mine, "config": bench_config(cfg, nf_global, world, scaling, nf)}
    if args.window_l2:
        job["config"]["workload"] = workload_name(cfg, window_l2=True)
    if args.shard_of > 1:
        job["config"]["shard_of"] = (f"diagnostic: rank 0's {nf}-frame shard of a {args.shard_of}-way "
                                     f"split of {nf_global} frames, run alone on one GPU; value "
                                     f"counts the shard's pixels only")
    if cfg.pyramid_step:
        return bench_pyramid(args, cfg, frames, nf, weights, bias, dev, world, rank, local,
                             barrier, max_over_ranks, job)
    p = H.HogPipeline(nf, cfg.channels, cfg.height, cfg.width, cfg.bins, stride=cfg.stride,
                      normalization="none" if args.window_l2 else cfg.normalization,
                      weights=weights, bias=bias, device=dev, chunks=args.chunks or None,
                      window_norm="l2" if args.window_l2 else None)
    p.upload(frames)
    p.run()
    torch.cuda.synchronize()

    # parity gate before any timing (reference bench.py:147-166 pattern)
    from oracle import oracle as O

    check = [0, nf - 1] if nf > 1 else [0]
    mode = 1 if cfg.scored else (2 if cfg.normalization == "l2" and not args.window_l2 else 0)
    _, g_ref, s_ref = O.run_batch(frames[check], O.build_lut(cfg.bins), cfg.bins, 8, 64, 128,
                                  cfg.stride, mode, weights, bias, threads=2, want_outputs=True)
    if not np.array_equal(p.grid[check].cpu().numpy().astype(np.int64), g_ref):
        raise PathMismatch("GPU cell grid differs from the oracle; refusing to time")
    if cfg.scored:
        s = p.scores[check].cpu().numpy()
        if (np.abs(s - s_ref) > 1e-5 * np.abs(s_ref) + 1e-12).any():
            raise PathMismatch("GPU scores differ from the oracle beyond 1e-5; refusing to time")
    if args.window_l2:  # numpy restatement of the extension over the oracle's grid
        for j, f in enumerate(check):
            q = (g_ref[j] ** 2).sum(-1)
            S = q[p.row_idx[:, None, :, None], p.col_idx[None, :, None, :]].sum((2, 3))
            if not np.array_equal(p.window_norms[f].cpu().numpy(),
                                  np.sqrt(S.astype(np.float64) + 1e-6 * 1e-6)):
                raise PathMismatch("per-window L2 norms differ from the restatement")

    K, W = args.steps, args.warmup
    for _ in range(W):
        p.run()
    torch.cuda.synchronize()
    nch = p.chunks
    pev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in range(nch)] for _ in range(K)]
    for step_ev in pev:  # materialise the CUDA events before handing them to the library
        for e0, e1 in step_ev:
            e0.record()
            e1.record()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    pipelined = bool(args.pipelined and p.scores is not None and p.chunks == 1)

    def timed_steps():
        p.join()
        for i in range(K):
            p.run(plane_events=pev[i], pipelined=pipelined)
        p.join()

    launch = timed_steps
    if not args.no_graph:
        # the K timed steps as one CUDA graph (kernel launches and the plane
        # kernel's events are graph nodes): no host launch gaps between steps
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            timed_steps()
        graph.replay()  # warm replay
        launch = graph.replay
    sampler = ClockSampler(local)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    sampler.start()
    torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include "timed/": the timed kernels only
    start.record()
    launch()
    end.record()
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    barrier()
    total_ms = start.elapsed_time(end)
    # k_planes: summed launch durations per step (chunks run back to back on one stream)
    plane_ms = sum(e0.elapsed_time(e1) for step_ev in pev for e0, e1 in step_ev) / K
    total_ms, plane_ms = max_over_ranks([total_ms, plane_ms])
    ms_per_step = total_ms / K
    px_step = job["nf_global"] * cfg.height * cfg.width  # the whole job's batch
    value = px_step / (ms_per_step / 1e3) / 1e6

    # diagnostic (outside the timed region): one more batch with per-stage events
    sev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for e in sev:
        e.record()
    p.run_staged(sev)
    torch.cuda.synchronize()
    stages_ms = {"grad_bin": sev[0].elapsed_time(sev[1]), "carry_scan": sev[1].elapsed_time(sev[2]),
                 "planes_grid": sev[2].elapsed_time(sev[3])}

    peak, peak_src = measured_peak()
    plane_bytes = p.plane_kernel_bytes_per_frame() * nf
    achieved = plane_bytes / (plane_ms / 1e3) / 1e9
    traffic = ncu_traffic(cfg.key)
    step_bytes = p.bytes_alg_per_frame() * nf
    step_gbs = step_bytes / (ms_per_step / 1e3) / 1e9

    # end to end through the public API: pinned host frames in, result out, per step
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(p, H, cfg, frames, nf, K, W, dev, world, max_over_ranks, barrier,
                      args.e2e_chunk, args.e2e_slots, not args.no_graph, args.e2e_tail,
                      bool(args.e2e_overlap), job=job, rank=rank, dump=args.dump_result)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, args.cpu_seconds, frames)

    if rank == 0:
        line = {
            "metric": "Mpixel/s (LUT binning + per-bin integral planes + window HOG)",
            "value": value, "unit": "Mpixel/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "int32" if not cfg.scored else "int32+f64",
            "data": "synthetic",
            "config": job["config"],
            "diagnostics": {"shard_frames": [mine.start, mine.stop],
                       "compulsory_gb_per_gpu_step": step_bytes / 1e9,
                       "k_planes_ms_per_step": plane_ms,
                       "stages_ms_diagnostic": stages_ms,
                       "chunks": nch, "cuda_graph": not args.no_graph,
                       "overlap": ("binning of frame group j+1 on a second stream under the "
                                   "plane kernel of group j" if nch > 1 else "none (one launch per stage)"),
                       "fused_grid": bool(p.fused),
                       "pipelined_batches": pipelined,
                       "band_rows": {"used": p.band_rows, "library_default": p.auto_band_rows(),
                                     "tuned_ms": p.band_rows_timings}},
            "roofline": {"bound": "hbm", "kernel": "k_planes", "achieved": achieved,
                         "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "peak_source": peak_src,
                         # the kernel is ~97 % stores: also against the write-only ceiling
                         # (cudaMemset of the same bytes, 7,349 GB/s: profiles/r1_tma_store_ab.md)
                         "write_only_ceiling": {"peak": 7349.0, "frac": achieved / 7349.0,
                                                "source": "builder-measured cudaMemset rate, round 1"},
                         "alg_bytes_per_launch": plane_bytes / nch, "launches_per_step": nch,
                         "alg_bytes_def": "bin map read (1 B/px) + int32 planes written "
                                          "(4*N_b*(H+1)*(W+1)) + cell grid written "
                                          f"({p.grid.dtype}, {p.grid.element_size()} B/bin)"},
            "pipeline_roofline": {"achieved": step_gbs, "peak": peak, "unit": "GB/s",
                                  "frac": step_gbs / peak,
                                  "alg_bytes_per_step": step_bytes,
                                  "alg_bytes_def": "SURVEY 8d bytes_alg per frame x frames "
                                                   f"(cell grid {p.grid.dtype})"},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": p.launches_per_run() * K,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def bench_split_frame(args, cfg, dev, world, rank, local, barrier, max_over_ranks, backend):
    """One frame over `world` ranks: rank r bins its row slab
    (+ halo rows), counts its rows' bins per column, one all_gather of those
    counts (N_b x W int32 per rank, NCCL over NVLink) gives the carry from the
    slabs above, then planes + cell-grid rows.  Per-frame latency = slowest
    rank, every step bracketed by the exchange."""
    import torch
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_1703_06256_b200 import slab, synth
    from paper_1703_06256_b200.errors import PathMismatch

    frame = synth.make_batch(cfg, 0, 1)
    group = dist.group.WORLD if world > 1 else None
    sp = slab.SlabPipeline(1, cfg.channels, cfg.height, cfg.width, cfg.bins, stride=cfg.stride,
                           rank=rank, world=world, group=group, device=dev)
    sp.upload(frame)
    sp.run()
    torch.cuda.synchronize()
    # parity gate: this rank's cell-grid rows against the oracle's whole-frame grid
    _, g_ref, _ = O.run_batch(frame, O.build_lut(cfg.bins), cfg.bins, 8, 64, 128, cfg.stride, 0,
                              threads=host_threads(), want_outputs=True)
    got = sp.grid_view()[0].cpu().numpy().astype(np.int64)
    ok = np.array_equal(got, g_ref[0, sp.cell_row0: sp.cell_row0 + sp.ncy])
    if max_over_ranks([0.0 if ok else 1.0])[0] != 0.0:
        raise PathMismatch("slab cell grid differs from the oracle; refusing to time")
    K, W = args.steps, args.warmup
    for _ in range(W):
        sp.run()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(K):
        sp.run()
    t1.record()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    ms = max_over_ranks([t0.elapsed_time(t1) / K])[0]
    barrier()
    if rank == 0:
        px = cfg.height * cfg.width
        line = {
            "metric": "Mpixel/s (LUT binning + per-bin integral planes + window HOG)",
            "value": px / (ms / 1e3) / 1e6, "unit": "Mpixel/s", "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": f"split-frame: 1 frame of {workload_name(cfg)}",
                       "global_frames": 1, "frames_per_gpu": 1, "scaling": "strong",
                       "parallelism": f"one frame in {world} row slab(s); one all_gather of "
                                      f"{cfg.bins}x{cfg.width} int32 column counts per rank "
                                      f"({'nccl' if backend == 'nccl' else backend})",
                       "l2": "frame planes larger than L2"},
            "diagnostics": {"slab_rows": [sp.y0, sp.y1], "exchange_bytes_per_rank":
                            4 * cfg.bins * cfg.width, "latency_ms_per_frame": ms},
            "e2e": None, "cpu_baseline": None, "gpu_launches": 4 * K, "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def bench_pyramid(args, cfg, frames, nf, weights, bias, dev, world, rank, local, barrier,
                  max_over_ranks, job):
    """Config c5: every frame scanned over its 20-level pyramid (detector.py:224-269).
    Mpixel/s counts source pixels; pyramid-level pixels are reported beside."""
    import torch

    import paper_1703_06256_b200 as H
    from oracle import oracle as O
    from paper_1703_06256_b200.errors import PathMismatch

    p = H.PyramidPipeline(nf, cfg.channels, cfg.height, cfg.width, cfg.bins, stride=cfg.stride,
                          scale_step=cfg.pyramid_step, weights=weights, bias=bias,
                          chunk=min(args.pyr_chunk, nf), device=dev,
                          streams=args.pyr_streams or None)
    p.upload(frames)
    p.run()
    torch.cuda.synchronize()
    # parity gate: every pyramid level of frame 0 against the oracle (one
    # level per host thread; ctypes drops the GIL)
    from concurrent.futures import ThreadPoolExecutor

    lut = O.build_lut(cfg.bins)

    def ref_level(lv):
        level, _, lw, lh = lv
        img = frames[0] if level == 0 else O.resize_bilinear(frames[0], lw, lh)
        return O.run_batch(img[None], lut, cfg.bins, 8, 64, 128, cfg.stride, 1, weights, bias,
                           threads=1, want_outputs=True)[2][0]

    with ThreadPoolExecutor(max_workers=host_threads()) as pool:
        refs = list(pool.map(ref_level, p.levels))
    for (level, _, _, _), ref in zip(p.levels, refs):
        got = p.scores[level][0].cpu().numpy()
        if got.shape != ref.shape or (np.abs(got - ref) > 1e-5 * np.abs(ref) + 1e-12).any():
            raise PathMismatch(f"pyramid level {level} scores differ from the oracle")
    K, W = args.steps, args.warmup
    for _ in range(W):
        p.run()
    torch.cuda.synchronize()
    pev = []
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    sampler.start()
    torch.cuda.nvtx.range_push("timed")
    start.record()
    for _ in range(K):
        p.run(plane_events=pev)
    end.record()
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    barrier()
    total_ms = start.elapsed_time(end)
    plane_ms = sum(e0.elapsed_time(e1) for e0, e1, _ in pev)
    plane_bytes = sum(b for _, _, b in pev)
    total_ms, plane_ms = max_over_ranks([total_ms, plane_ms])
    ms = total_ms / K
    # diagnostic (outside the timed region): one pass with the levels on one
    # stream, so the plane kernels' event durations are not shared with the
    # concurrent levels' kernels
    serial = None
    if p.streams > 1:
        saved, p.streams = p.streams, 1
        sev = []
        torch.cuda.synchronize()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record()
        p.run(plane_events=sev)
        s1.record()
        torch.cuda.synchronize()
        p.streams = saved
        sp_ms = sum(e0.elapsed_time(e1) for e0, e1, _ in sev)
        sp_gbs = sum(b for _, _, b in sev) / (sp_ms / 1e3) / 1e9
        serial = {"step_ms": s0.elapsed_time(s1), "k_planes_ms": sp_ms, "k_planes_gbs": sp_gbs,
                  "k_planes_frac": sp_gbs / measured_peak()[0]}
    src_px = job["nf_global"] * cfg.height * cfg.width
    lvl_px = job["nf_global"] * p.pixels_per_frame()
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e_pyramid(p, cfg, frames, nf, K, W, dev, world, max_over_ranks, barrier,
                              job=job, rank=rank, dump=args.dump_result)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, args.cpu_seconds, frames)
    peak, peak_src = measured_peak()
    achieved = plane_bytes / (plane_ms / 1e3) / 1e9
    step_bytes = p.bytes_alg_per_frame() * nf
    if rank == 0:
        line = {
            "metric": "Mpixel/s (LUT binning + per-bin integral planes + window HOG)",
            "value": src_px / (ms / 1e3) / 1e6, "unit": "Mpixel/s (source pixels)",
            "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": ms,
            "higher_is_better": True, "scaling": job["scaling"], "vs_baseline": None,
            "dtype": "int32+f64", "data": "synthetic",
            "config": job["config"],
            "diagnostics": {"shard_frames": [job["mine"].start, job["mine"].stop],
                       "levels": len(p.levels), "level_mpixel_per_s": lvl_px / (ms / 1e3) / 1e6,
                       "frames_per_chunk": p.chunk, "level_streams": p.streams,
                       "band_rows_per_level": [q.band_rows for q in p.pipes],
                       "one_stream_diagnostic": serial,
                       "compulsory_gb_per_gpu_step": step_bytes / 1e9},
            # the plane kernels of different levels overlap on the level streams
            # inside the timed region, so their event durations there are not
            # per-kernel times: the roofline uses the one-stream pass (same
            # launches, events not shared with other kernels), measured right
            # after the timed steps; the overlapped rate is kept as a diagnostic
            "roofline": {"bound": "hbm", "kernel": "k_planes",
                         "achieved": serial["k_planes_gbs"] if serial else achieved, "peak": peak,
                         "unit": "GB/s",
                         "frac": (serial["k_planes_gbs"] if serial else achieved) / peak,
                         "traffic": None,
                         "traffic_level0": {
                             "bytes": ncu_traffic(cfg.key, "level0_k_planes_bytes_per_launch"),
                             "alg_bytes": ncu_traffic(cfg.key, "level0_alg_bytes_per_launch"),
                             "launch": "pyramid level 0 of a 16-frame chunk (ncu)"},
                         "timing": ("one-stream pass of the same step (every level's plane kernel "
                                    "timed alone on its stream)" if serial else
                                    "plane-kernel events inside the timed region"),
                         "overlapped_events_gbs": achieved,
                         "peak_source": peak_src, "launches_per_step": len(pev) // K,
                         "alg_bytes_per_step": plane_bytes / K},
            "pipeline_roofline": {"achieved": step_bytes / (ms / 1e3) / 1e9, "peak": peak,
                                  "unit": "GB/s", "frac": step_bytes / (ms / 1e3) / 1e9 / peak,
                                  "alg_bytes_per_step": step_bytes},
            "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": p.launches_per_run() * K, "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    return 0


def run_e2e_pyramid(p, cfg, frames, nf, K, W, dev, world, max_over_ranks, barrier, job=None,
                    rank=0, dump=""):
    """c5 end to end through PyramidPipeline: per step, H2D of every source
    frame from pinned host memory (one copy per frame chunk on a copy stream;
    chunk j's levels start when its frames have landed) and D2H of every
    level's score maps (each level's slice leaves on a second copy stream as
    soon as it is scored).  Consecutive steps overlap: a chunk's copy waits
    only for the previous step's levels of that chunk."""
    import torch

    host_in = torch.from_numpy(frames).pin_memory()
    # every level's score maps of the whole batch, one node-wide host buffer per level
    gathers = [open_gather(job, s.shape[1:], s.dtype, rank, barrier, tag=f"lvl{i}")
               for i, s in enumerate(p.scores)]
    host_out = [gth.local() for gth in gathers]
    cin, cout = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    src = p.src.data

    done_prev = {}  # chunk start -> events after the previous step's levels of that chunk
    out_prev = {}   # chunk start -> events after the previous step's score copies of that chunk

    def step():
        """One e2e step.  A chunk's H2D copy waits only until the previous
        step's levels of that chunk have read the source frames, so step k+1's
        first chunk crosses PCIe while step k's last chunk is computing."""
        nonlocal done_prev, out_prev
        cur = torch.cuda.current_stream()
        cout.wait_stream(cur)
        ready, done, out = {}, {}, {}
        with torch.cuda.stream(cin):
            for a in range(0, nf, p.chunk):
                m = min(p.chunk, nf - a)
                for ev in done_prev.get(a, []):
                    cin.wait_event(ev)
                src[a:a + m].copy_(host_in[a:a + m], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(cin)
                ready[a] = ev

        def chunk_ready(a, m, st):
            st.wait_event(ready[a])
            # this step's scores of the chunk overwrite what the previous step is still
            # copying out: wait for that chunk's copies only (not for the whole step's)
            for ev in out_prev.get(a, []):
                st.wait_event(ev)

        def level_done(level, a, m, st):
            ev = torch.cuda.Event()
            ev.record(st)
            done.setdefault(a, []).append(ev)
            cout.wait_event(ev)
            with torch.cuda.stream(cout):
                host_out[level][a:a + m].copy_(p.scores[level][a:a + m], non_blocking=True)
                left = torch.cuda.Event()
                left.record(cout)
            out.setdefault(a, []).append(left)

        p.run(cur, chunk_ready=chunk_ready, level_done=level_done)
        done_prev, out_prev = done, out

    cin.wait_stream(torch.cuda.current_stream())
    for _ in range(max(1, W)):
        step()
    torch.cuda.synchronize()
    barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(K):
        step()
    torch.cuda.current_stream().wait_stream(cout)  # the last step's score maps have left
    t1.record()
    torch.cuda.current_stream().wait_stream(cin)
    torch.cuda.synchronize()
    ms = max_over_ranks([t0.elapsed_time(t1) / K])[0]
    ok = all(torch.equal(h, s.cpu()) for h, s in zip(host_out, p.scores))
    ok = max_over_ranks([0.0 if ok else 1.0])[0] == 0.0
    barrier()  # every shard's score maps are in the shared buffers
    if dump and rank == 0:
        np.savez(dump, *[gth.array for gth in gathers])
    d2h = int(sum(h.numel() * h.element_size() for h in host_out))
    for gth in gathers:
        gth.close()
    return {"value": job["nf_global"] * cfg.height * cfg.width / (ms / 1e3) / 1e6,
            "unit": "Mpixel/s (source pixels)", "ms_per_step": ms,
            "h2d_bytes_per_step": int(host_in.numel() * host_in.element_size()),
            "d2h_bytes_per_step": d2h,
            "gather": "each rank's score maps land in its slices of node-wide page-locked host "
                      "buffers (/dev/shm, cudaHostRegister), one per level, in frame order",
            "result": "window scores of every pyramid level", "chunk_frames": p.chunk,
            "streams": "1 H2D + 4 level streams + 1 D2H", "cuda_graph": False,
            "steps_overlap": True, "matches_device_run": ok}


def open_gather(job, res_shape, dtype, rank, barrier, tag=""):
    """The job's result buffer: one host array for the whole batch (frame
    order) shared by the node's ranks; this rank writes its shard's slice."""
    import torch

    from paper_1703_06256_b200 import sharding

    np_dtype = torch.empty((), dtype=dtype).numpy().dtype
    run = os.environ.get("MASTER_PORT") if int(os.environ.get("WORLD_SIZE", "1")) > 1 else os.getpid()
    return sharding.HostGather(f"{run}_{tag}", (job["nf_global"],) + tuple(res_shape), np_dtype,
                               job["mine"], rank, barrier,
                               single_process=int(os.environ.get("WORLD_SIZE", "1")) == 1)


def run_e2e(p, H, cfg, frames, nf, K, W, dev, world, max_over_ranks, barrier, chunk=64, nslots=2,
            use_graph=True, tail=1, overlap=True, job=None, rank=0, dump=""):
    """Per step: H2D of every frame from pinned host memory, the pipeline, and
    D2H of the step's result, in frame chunks.  Each direction has ONE copy
    stream, so chunks cross PCIe in order at full bandwidth (copies issued on
    several streams share the link and all land late: measured with
    tools/e2e_timeline.py); one compute stream runs each chunk as soon as it
    has landed.  `nslots` buffer sets rotate, guarded by events (a chunk's H2D
    waits until the chunk nslots back has been computed, its kernels until
    that chunk's result has left)."""
    import torch

    from paper_1703_06256_b200 import synth

    if chunk <= 0:  # four chunks per step, each with its own buffer set (nslots = 4)
        chunk = (nf + 3) // 4
    chunk = max(1, min(nf, chunk))
    # job schedule: full chunks, with the last chunk split in `tail` pieces so
    # the work left after the final H2D (its compute + D2H) is short
    sizes = [chunk] * (nf // chunk) + ([nf % chunk] if nf % chunk else [])
    if tail > 1 and sizes and sizes[-1] >= tail:
        last = sizes.pop()
        sizes += [last // tail] * (tail - 1) + [last - (last // tail) * (tail - 1)]
    weights, bias = synth.make_weights(cfg) if cfg.scored else (None, 0.0)
    h2d, comp, d2h = (torch.cuda.Stream(device=dev) for _ in range(3))
    pipes = {}  # (slot, size) -> pipeline

    def pipe(si, sz):
        if (si, sz) not in pipes:
            pipes[(si, sz)] = H.HogPipeline(sz, cfg.channels, cfg.height, cfg.width, cfg.bins,
                                            stride=cfg.stride, normalization=cfg.normalization,
                                            weights=weights, bias=bias, device=dev)
        return pipes[(si, sz)]

    # buffer sets: chunk j of a step runs on set j % nslots; with fewer chunks than sets
    # (c1: one frame, one chunk) consecutive steps rotate over nslots // chunks groups of
    # sets, so step k+1's copy and compute still overlap step k's result leaving
    nslots_arg = max(1, nslots)
    nslots = max(1, min(nslots_arg, len(sizes)))
    reps = max(1, nslots_arg // len(sizes)) if overlap else 1
    jobs, a = [], 0
    for j, sz in enumerate(sizes):
        jobs.append((a, a + sz, [pipe(r * nslots + j % nslots, sz) for r in range(reps)]))
        a += sz
    host_in = torch.from_numpy(frames).pin_memory()
    res = jobs[0][2][0].result()
    gather = open_gather(job, res.shape[1:], res.dtype, rank, barrier)
    host_out = gather.local()  # this shard's slice of the node-wide result buffer

    def steps(nsteps):
        """nsteps e2e steps.  Buffer reuse is guarded per pipeline (frames buffer
        free once its last chunk is computed, result buffer free once that
        result has left), so with overlap=True step k+1's first H2D copies
        start while step k's last chunks are still computing / leaving; the
        streams join the caller's stream only around the whole run."""
        cur = torch.cuda.current_stream()
        for st in (h2d, comp, d2h):
            st.wait_stream(cur)
        last = {}  # pipeline -> (computed, left) events of its latest chunk
        for step in range(nsteps):
            for a, b, qs in jobs:
                q = qs[step % len(qs)]
                prev = last.get(id(q))
                if prev is not None:
                    h2d.wait_event(prev[0])  # frames buffer free
                with torch.cuda.stream(h2d):
                    dst = q.frames.data if q.frames.pitch == cfg.width else q.frames.data[..., : cfg.width]
                    dst.copy_(host_in[a:b], non_blocking=True)
                    landed = torch.cuda.Event()
                    landed.record(h2d)
                comp.wait_event(landed)
                if prev is not None:
                    comp.wait_event(prev[1])  # result buffer free
                q.run(stream=comp)
                computed = torch.cuda.Event()
                computed.record(comp)
                d2h.wait_event(computed)
                with torch.cuda.stream(d2h):
                    host_out[a:b].copy_(q.result(), non_blocking=True)
                    left = torch.cuda.Event()
                    left.record(d2h)
                last[id(q)] = (computed, left)
            if not overlap:
                for st in (h2d, comp, d2h):
                    cur.wait_stream(st)
                for st in (h2d, comp, d2h):
                    st.wait_stream(cur)
                last.clear()
        for st in (h2d, comp, d2h):
            cur.wait_stream(st)

    steps(W)
    torch.cuda.synchronize()
    replay = lambda: steps(K)  # noqa: E731
    if use_graph:
        # the K timed steps (H2D copies, kernels, D2H copies on their streams)
        # as one CUDA graph: no per-chunk host launch cost inside the timed loop
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            steps(K)
        torch.cuda.synchronize()
        replay = g.replay
        replay()
        torch.cuda.synchronize()
    barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    replay()
    t1.record()
    torch.cuda.synchronize()
    ms = max_over_ranks([t0.elapsed_time(t1) / K])[0]
    # the D2H result must equal the device-resident run's result
    ok = bool(torch.equal(host_out.to(dev), p.result().to(host_out.dtype)))
    ok = max_over_ranks([0.0 if ok else 1.0])[0] == 0.0
    barrier()  # every shard has landed in the shared buffer: rank 0 holds the whole batch
    if dump and rank == 0:
        np.save(dump, gather.array)
    gather.close()
    return {"value": job["nf_global"] * cfg.height * cfg.width / (ms / 1e3) / 1e6,
            "unit": "Mpixel/s",
            "ms_per_step": ms, "h2d_bytes_per_step": int(host_in.numel() * host_in.element_size()),
            "d2h_bytes_per_step": int(host_out.numel() * host_out.element_size()),
            "gather": (f"each rank's D2H lands in its slice of one {gather.nbytes / 1e6:.1f} MB "
                       "page-locked host buffer shared by the node's ranks (/dev/shm, "
                       "cudaHostRegister): the batch's results in frame order on the host"),
            "bytes_per_gpu": "h2d/d2h bytes are this rank's shard",
            "result": "cell grid" if not cfg.scored else "window scores",
            "chunk_frames": sizes, "buffer_sets": nslots * reps,
            "streams": "1 H2D + 1 compute + 1 D2H (in-order copies)", "cuda_graph": bool(use_graph),
            "steps_overlap": bool(overlap),
            "matches_device_run": ok}


if __name__ == "__main__":
    sys.exit(main())
