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
        sd = sh.shard(r, w, PER_RANK)
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
    shards = [sh.shard(r, 4, 3) for r in range(4)]
    assert [(s.lo, s.hi) for s in shards] == [(0, 3), (3, 6), (6, 9), (9, 12)]
    assert all(s.n_global == 12 for s in shards)
    with pytest.raises(ValueError):
        sh.shard(4, 4, 3)


def test_single_process_counters_are_identity():
    red = sh.reduce_counters(stream_steps=100, elapsed_ms=50.0)
    assert red["stream_steps"] == 100 and red["elapsed_ms"] == 50.0
    assert red["throughput"] == pytest.approx(2000.0)


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
