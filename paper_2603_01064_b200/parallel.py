"""RHS-batch sharding across processes (one process per GPU).

The batched configs (BASELINE configs 1-3) shard the right-hand sides: every rank
owns a contiguous RHS range and a full replica of the hierarchy and weights.  The
NMGF cycle is per-RHS independent (norms, convergence tests and freezing are per
RHS; Alg 3/4 act on one right-hand side at a time), so there is no
collective on the data path; torch.distributed is used only for the barrier around
the timed region, the max-over-ranks of the measured time and the gather of reports.
"""
from __future__ import annotations

from typing import List, Tuple


def shard_range(total: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous split of `total` RHS over `world` ranks: (start, count) of `rank`.
    The first total % world ranks get one extra RHS."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def weak_shard(per_rank: int, rank: int) -> Tuple[int, int]:
    """Weak scaling: rank r solves RHS [r * per_rank, (r + 1) * per_rank) of the global stream."""
    return rank * per_rank, per_rank


def max_over_ranks(value: float, group=None) -> float:
    """Max of a host float over all ranks (timing: the job ends when the slowest rank ends)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def gather_reports(report, group=None) -> List:
    """All ranks' report objects in rank order (outside any timed region)."""
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return [report]
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, report, group=group)
    return out
