"""RHS-batch sharding and slab sharding across processes (one process per GPU).

The batched configs (BASELINE configs 1-3) shard the right-hand sides: every rank
owns a contiguous RHS range and a full replica of the hierarchy and weights.  The
NMGF cycle is per-RHS independent (norms, convergence tests and freezing are per
RHS; Alg 3/4 act on one right-hand side at a time), so there is no
collective on the data path; torch.distributed is used only for the barrier around
the timed region, the max-over-ranks of the measured time and the gather of reports.

The single-system config (BASELINE config 4) instead row-shards the 2D operator
(nmg_create_hierarchy_slab): rank r owns rows i2 in [r R, r R + R),
R = n / world, of every right-hand side's row-major [i2][i1] image.  slab_rows /
split_slabs / join_slabs are the host-side partition logic of that layout.
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


def slab_rows(n: int, world: int, rank: int) -> Tuple[int, int]:
    """(first global row, rows) of `rank`'s slab of an n x n image split over `world` ranks."""
    if world < 1 or not (0 <= rank < world) or n % world:
        raise ValueError(f"cannot split {n} rows over {world} ranks")
    R = n // world
    return rank * R, R


def split_slabs(y, n: int, world: int):
    """[nrhs][n*n] (or [nrhs][n][n]) -> list of contiguous per-rank slabs [nrhs][R][n]."""
    y3 = y.reshape(y.shape[0], n, n)
    out = []
    for r in range(world):
        r0, R = slab_rows(n, world, r)
        s = y3[:, r0:r0 + R, :]
        out.append(s.copy() if hasattr(s, "copy") and not hasattr(s, "contiguous") else s.contiguous())
    return out


def join_slabs(slabs, n: int):
    """Inverse of split_slabs: per-rank [nrhs][R][n] slabs -> [nrhs][n*n]."""
    try:
        import numpy as np
        if isinstance(slabs[0], np.ndarray):
            return np.concatenate(slabs, axis=1).reshape(slabs[0].shape[0], n * n)
    except ImportError:
        pass
    import torch
    return torch.cat(list(slabs), dim=1).reshape(slabs[0].shape[0], n * n)
