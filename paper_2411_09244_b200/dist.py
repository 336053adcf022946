"""Multi-GPU plumbing for the ensemble path.

The hot path shards with no data-path exchange along the ensemble dimension: every
member is an independent parareal problem (BASELINE config 4), so ranks own disjoint
member ranges and only the timing is reduced (max over ranks).  One process per GPU,
`torch.distributed` for the plumbing (NCCL on the GPU box, gloo in the CPU tests).
Interval sharding of one problem (one all-gather of the F endpoints per iteration) is
in `sharded.py`.
"""

from __future__ import annotations

import os


def world():
    """(rank, world_size, local_rank) from the torchrun environment (1 process if unset)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_members(n_members: int, rank: int, world_size: int) -> range:
    """Contiguous, balanced member range of `rank` (sizes differ by at most one)."""
    if n_members < 0 or world_size < 1 or not 0 <= rank < world_size:
        raise ValueError("need n_members >= 0, world_size >= 1, 0 <= rank < world_size")
    base, extra = divmod(n_members, world_size)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (the device-timed step duration) across the job."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_member_results(local: dict, device=None) -> dict:
    """All-gather {member_index: iterations} dictionaries (report per-member counts)."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return dict(local)
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, local)
    merged = {}
    for d in out:
        merged.update(d)
    return merged
