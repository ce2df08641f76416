"""N>1 host path on CPU (gloo, world size 2): stream sharding, shard invariance
and the end-of-run counter reduction.  The per-stream compute is
the fp64 oracle standing in for the GPU kernels (the CUDA path itself is
covered by the -m gpu tests); what is tested here is the multi-process logic
bench.py runs under torchrun: contiguous stream shards, per-stream data that do
not depend on the number of ranks, no data exchange, and SUM/MAX counters.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2204_03418_b200 import shard as sh
from paper_2204_03418_b200 import synth

PER_RANK = 2
TICKS = 6


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run_streams(lo, hi, n_global):
    """Oracle step outputs of global streams [lo, hi) of a small C2-shaped layer."""
    cfg = synth.config(2, n_streams=n_global, in_spatial=(6, 5))
    cfg.layers[0].cin = cfg.layers[0].cout = 8
    (W, b), L = synth.params(cfg)[0], cfg.layers[0]
    d = O.Desc(2, L.cin, L.cout, L.kernel, L.stride, L.padding, L.dilation, L.groups, cfg.in_spatial)
    sm = O.StepMachine(d, W.double().numpy(), b.double().numpy(), hi - lo)
    outs = []
    for t in range(TICKS):
        x = synth.frame(cfg, t, lo, hi, device="cpu", n_global=n_global).float().numpy()
        y = sm.forward_step(x)
        if y is not None:
            outs.append(y)
    return np.stack(outs)


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r, w, _ = sh.env_rank_world()
        sd = sh.shard(r, w, PER_RANK, scaling="weak")
        assert (sd.lo, sd.hi, sd.n_global) == (rank * PER_RANK, (rank + 1) * PER_RANK, world * PER_RANK)
        ys = _run_streams(sd.lo, sd.hi, sd.n_global)
        sh.barrier()
        red = sh.reduce_counters(stream_steps=PER_RANK * TICKS, elapsed_ms=10.0 * (rank + 1),
                                 parity_fails=rank, max_rel_err=1e-6 * (rank + 1))
        gathered = [None] * world
        dist.all_gather_object(gathered, ys)      # test-only: compare against a 1-process run
        if rank == 0:
            np.save(os.path.join(out_dir, "y.npy"), np.concatenate(gathered, axis=1))
            np.save(os.path.join(out_dir, "red.npy"),
                    np.array([red["stream_steps"], red["parity_fails"], red["elapsed_ms"], red["max_rel_err"],
                              red["throughput"]]))
    finally:
        dist.destroy_process_group()


def test_shard_ranges():
    # weak: B streams per rank
    shards = [sh.shard(r, 4, 3, scaling="weak") for r in range(4)]
    assert [(s.lo, s.hi) for s in shards] == [(0, 3), (3, 6), (6, 9), (9, 12)]
    assert all(s.n_global == 12 for s in shards)
    with pytest.raises(ValueError):
        sh.shard(4, 4, 3)
    # strong (default): the config's global count fixed, contiguous near-equal blocks
    for n, g in [(1024, 8), (256, 8), (16384, 8), (10, 4), (7, 3), (512, 2)]:
        s = [sh.shard(r, g, n) for r in range(g)]
        assert s[0].lo == 0 and s[-1].hi == n and all(a.hi == b.lo for a, b in zip(s, s[1:]))
        assert max(x.per_rank for x in s) - min(x.per_rank for x in s) <= 1
        assert all(x.n_global == n and x.scaling == "strong" for x in s)
    assert [(x.lo, x.hi) for x in (sh.shard(r, 4, 10) for r in range(4))] == [(0, 2), (2, 5), (5, 7), (7, 10)]
    # fewer streams than ranks (C1): replicas of the whole set
    assert all((x.lo, x.hi, x.scaling) == (0, 1, "replicas") for x in (sh.shard(r, 8, 1) for r in range(8)))


def test_single_process_counters_are_identity():
    red = sh.reduce_counters(stream_steps=100, elapsed_ms=50.0)
    assert red["stream_steps"] == 100 and red["elapsed_ms"] == 50.0
    assert red["throughput"] == pytest.approx(2000.0)


def _worker_strong(rank, world, port, out_dir, n_global):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r, w, _ = sh.env_rank_world()
        sd = sh.shard(r, w, n_global)                # strong: the job's global stream count is fixed
        ys = _run_streams(sd.lo, sd.hi, n_global)
        sh.barrier()
        red = sh.reduce_counters(stream_steps=sd.per_rank * TICKS, elapsed_ms=5.0 + rank)
        gathered = [None] * world
        dist.all_gather_object(gathered, (sd.lo, sd.hi, ys))
        if rank == 0:
            np.save(os.path.join(out_dir, "y.npy"), np.concatenate([g[2] for g in gathered], axis=1))
            np.save(os.path.join(out_dir, "ranges.npy"), np.array([(g[0], g[1]) for g in gathered]))
            np.save(os.path.join(out_dir, "red.npy"), np.array([red["stream_steps"], red["elapsed_ms"],
                                                                red["throughput"]]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_global", [5, 4])
def test_gloo_world2_strong_uneven_shards(tmp_path, n_global):
    """Strong scaling over 2 ranks with an uneven (5 = 2 + 3) and an even split:
    the shards tile [0, B), every stream's outputs are bitwise those of a
    1-process run over all B streams, and the counters sum the job's
    stream-steps over the slowest rank's time."""
    world = 2
    mp.spawn(_worker_strong, args=(world, _free_port(), str(tmp_path), n_global), nprocs=world, join=True)
    ranges = np.load(tmp_path / "ranges.npy")
    assert ranges.tolist() == [[0, n_global // 2], [n_global // 2, n_global]]
    y2 = np.load(tmp_path / "y.npy")
    y1 = _run_streams(0, n_global, n_global)
    assert y2.shape == y1.shape and np.array_equal(y2, y1)
    ss, ms, thr = np.load(tmp_path / "red.npy")
    assert ss == n_global * TICKS and ms == 6.0 and thr == pytest.approx(ss / 0.006)


def test_gloo_world2_shard_invariance_and_counters(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    y2 = np.load(tmp_path / "y.npy")
    y1 = _run_streams(0, world * PER_RANK, world * PER_RANK)
    # per-stream outputs are bitwise identical whether the streams ran on 1 or 2 ranks
    assert y2.shape == y1.shape and np.array_equal(y2, y1)
    ss, fails, ms, err, thr = np.load(tmp_path / "red.npy")
    assert ss == world * PER_RANK * TICKS            # SUM of stream-steps
    assert fails == 1                                 # SUM of parity fails (0 + 1)
    assert ms == 20.0 and err == pytest.approx(2e-6)  # MAX over ranks
    assert thr == pytest.approx(ss / 0.020)           # whole-job throughput = SUM / MAX time


def test_bench_host_path_under_torchrun_gloo():
    """bench.py's multi-rank code path (torchrun launch, rank/world from the
    environment, strong shards of every config, barrier, SUM/MAX counters, the
    one JSON line from rank 0) on CPU with gloo and world size 2 (--dry-run:
    stand-in timings of 1 + rank ms per step, no GPU work)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if not k.startswith("CO_")}
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus",
                          "2", "--steps", "4", "--warmup", "3", "--dry-run"], cwd=root, env=env,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1                          # rank 0 alone prints
    j = json.loads(lines[0])
    assert j["n_gpus"] == 2 and j["scaling"] == "strong" and j["steps"] == 4
    c = j["configs"]
    # strong shards: rank 1's block of each config, global count fixed
    assert c["C2"]["global_streams"] == 256 and c["C4"]["global_streams"] == 1024
    # whole-job throughput = all ranks' stream-steps / the slowest rank's time (2 ms per step)
    assert c["C2"]["stream_steps"] == 256 * 4 and c["C2"]["value"] == pytest.approx(256 * 4 / 8e-3)
    assert c["C5"]["value"] == pytest.approx(16384 * 4 / 8e-3)
    assert c["C1"]["scaling"] == "replicas" and c["C1"]["stream_steps"] == 2 * 4   # one stream on each rank
    assert j["value"] == c["C2"]["value"]
