"""Multi-GPU plumbing: one process per GPU, torch.distributed
for rendezvous; the data path is the engine's own ncclAllReduce.

Two ways the path shards:
  * K sweep   -- K values are independent fixpoints on a replicated graph:
                 split_k_values() hands each rank a share, no collective;
  * one big fixpoint -- the support tasks are split t % world == rank; each
                 round every rank all-reduces its partial supports (exact u32
                 sums) and runs the same deterministic prune (engine_join()).
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import torch
import torch.distributed as dist

from .truss import Engine, nccl_unique_id


def world_rank() -> tuple:
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(), dist.get_rank()
    return 1, 0


def split_k_values(ks: Sequence[int], rank: int, world: int) -> List[int]:
    """Snake (boustrophedon) assignment of the sorted K list: costs fall
    monotonically-ish with K, so snake order balances better than round robin.
    Every K lands on exactly one rank."""
    out = []
    for i, k in enumerate(sorted(ks)):
        lap, pos = divmod(i, world)
        owner = pos if lap % 2 == 0 else world - 1 - pos
        if owner == rank:
            out.append(k)
    return out


def broadcast_nccl_id(group: Optional[dist.ProcessGroup] = None) -> bytes:
    """Rank 0 draws an NCCL unique id; every rank receives it."""
    world, rank = world_rank()
    obj = [nccl_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def engine_join(engine: Engine, group: Optional[dist.ProcessGroup] = None) -> None:
    """Make `engine` run its fixpoints edge-partitioned over all ranks
    (collective)."""
    world, rank = world_rank()
    engine.set_nccl(rank, world, broadcast_nccl_id(group))


def max_over_ranks(x: float, device: Optional[torch.device] = None) -> float:
    world, _ = world_rank()
    if world == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, device: Optional[torch.device] = None) -> float:
    world, _ = world_rank()
    if world == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
