"""Multi-GPU plumbing for the continual-conv step.

Streams are independent (one handle's streams share only the clock and the
read-only weights), so the path partitions without any data exchange:
rank r of a world of g processes owns the contiguous global streams
[r*B, (r+1)*B) and runs its own handles on its own GPU.  There is no collective
on the hot path; torch.distributed (NCCL on GPUs, gloo in the CPU tests) only
carries the barrier before timing and the end-of-run counters:

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
    per_rank: int          # streams per rank (weak scaling: fixed per GPU)

    @property
    def lo(self) -> int:
        return self.rank * self.per_rank

    @property
    def hi(self) -> int:
        return (self.rank + 1) * self.per_rank

    @property
    def n_global(self) -> int:
        return self.world * self.per_rank


def env_rank_world() -> Tuple[int, int, int]:
    """(rank, world, local_rank) from the torchrun environment (1 process if unset)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(rank: int, world: int, per_rank: int) -> Shard:
    if world < 1 or not (0 <= rank < world) or per_rank < 1:
        raise ValueError(f"bad shard rank={rank} world={world} per_rank={per_rank}")
    return Shard(rank, world, per_rank)


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
