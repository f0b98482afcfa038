"""Multi-GPU = replicas: every rank owns one GPU, one host
scheduler loop and one independent tenant set; no data-path collective exists
on this path. torch.distributed (gloo) only moves the scalar results:
throughput counters are summed, device time is the max over ranks, latency
samples are pooled on rank 0.

Rendezvous follows torchrun's environment (RANK, WORLD_SIZE, LOCAL_RANK,
MASTER_ADDR=127.0.0.1, MASTER_PORT)."""
from __future__ import annotations

import os
from dataclasses import dataclass


@dataclass
class Rank:
    rank: int = 0
    world: int = 1
    local: int = 0


def init_from_env(backend: str = "gloo") -> Rank:
    world = int(os.environ.get("WORLD_SIZE", "1"))
    r = Rank(int(os.environ.get("RANK", "0")), world, int(os.environ.get("LOCAL_RANK", "0")))
    if world > 1:
        import torch.distributed as dist

        if not dist.is_initialized():
            dist.init_process_group(backend)
    return r


def _dist():
    import torch.distributed as dist

    return dist if dist.is_available() and dist.is_initialized() else None


def barrier() -> None:
    d = _dist()
    if d is not None:
        d.barrier()


def reduce(values: list[float], op: str) -> list[float]:
    """Elementwise sum or max over ranks (every rank gets the result)."""
    d = _dist()
    if d is None:
        return list(values)
    import torch

    t = torch.tensor(values, dtype=torch.float64)
    d.all_reduce(t, op=d.ReduceOp.MAX if op == "max" else d.ReduceOp.SUM)
    return t.tolist()


def gather_samples(samples: list[float]) -> list[float]:
    """All ranks' samples, concatenated (for pooled percentiles)."""
    d = _dist()
    if d is None:
        return list(samples)
    out: list = [None] * d.get_world_size()
    d.all_gather_object(out, list(samples))
    return [x for part in out for x in part]
