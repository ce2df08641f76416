"""Multi-GPU plumbing for the continual-conv step.

Streams are independent (one handle's streams share only the clock and the
read-only weights, "the same global clock"), so the path partitions
without any data exchange.  Strong scaling (the default, BASELINE.json configs
"1024 streams sharded over 1/2/4/8 GPUs"): the config's global
stream count B is fixed and rank r of g owns the contiguous global streams
[floor(r B / g), floor((r+1) B / g)) -- shards differ by at most one stream
when g does not divide B.  Weak scaling (an option): every rank runs B streams,
rank r owning [r B, (r+1) B).  A config with fewer streams than ranks (C1's
single stream) runs as independent replicas.  Each rank builds its own handles
on its own GPU; weights are regenerated bitwise identically from the seed.

There is no collective on the hot path; torch.distributed (NCCL on GPUs, gloo
in the CPU tests) only carries the barrier before timing and the end-of-run
counters:

* SUM over ranks of [stream_steps, parity_fails]
* MAX over ranks of [elapsed_ms, max_rel_err]

Whole-job throughput = SUM(stream_steps) / MAX(elapsed).
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Tuple


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    lo: int                # first global stream of this rank
    hi: int                # one past the last
    n_global: int          # streams of the whole job
    scaling: str = "strong"

    @property
    def per_rank(self) -> int:
        return self.hi - self.lo


def env_rank_world() -> Tuple[int, int, int]:
    """(rank, world, local_rank) from the torchrun environment (1 process if unset)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(rank: int, world: int, n: int, scaling: str = "strong") -> Shard:
    """This rank's streams.  strong: n global streams split into contiguous,
    near-equal blocks (replicas of all n when n < world); weak: n per rank."""
    if world < 1 or not (0 <= rank < world) or n < 1:
        raise ValueError(f"bad shard rank={rank} world={world} n={n}")
    if scaling == "weak":
        return Shard(rank, world, rank * n, (rank + 1) * n, world * n, "weak")
    if scaling != "strong":
        raise ValueError(f"scaling must be 'strong' or 'weak', not {scaling!r}")
    if n < world:                                  # e.g. C1's one stream: independent replicas
        return Shard(rank, world, 0, n, n, "replicas")
    return Shard(rank, world, rank * n // world, (rank + 1) * n // world, n, "strong")


def _dist():
    import torch.distributed as dist
    return dist if (dist.is_available() and dist.is_initialized()) else None


def _device():
    import torch
    dist = _dist()
    if dist is not None and dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def barrier() -> None:
    dist = _dist()
    if dist is not None:
        dist.barrier()


def reduce_counters(stream_steps: float, elapsed_ms: float, parity_fails: float = 0.0,
                    max_rel_err: float = 0.0) -> dict:
    """End-of-run counters over all ranks (no-op in a single process)."""
    import torch
    dist = _dist()
    s = torch.tensor([float(stream_steps), float(parity_fails)], dtype=torch.float64, device=_device())
    m = torch.tensor([float(elapsed_ms), float(max_rel_err)], dtype=torch.float64, device=_device())
    if dist is not None:
        dist.all_reduce(s, op=dist.ReduceOp.SUM)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
    stream_steps, parity_fails = s.tolist()
    elapsed_ms, max_rel_err = m.tolist()
    return {"stream_steps": stream_steps, "parity_fails": parity_fails, "elapsed_ms": elapsed_ms,
            "max_rel_err": max_rel_err,
            "throughput": stream_steps / (elapsed_ms / 1e3) if elapsed_ms > 0 else 0.0}
