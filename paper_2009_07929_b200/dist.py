"""Multi-GPU plumbing: one process per GPU, torch.distributed
for rendezvous; the data path is the engine's own ncclAllReduce.

Three ways the path shards:
  * K sweep   -- K values are independent fixpoints on a replicated graph:
                 split_k_values() hands each rank a share, no collective;
  * one big fixpoint -- every full support pass covers this rank's share
                 of the tasks (A22 tasks split by their exact work in carried runs, work-
                 balanced chunk ranges in recompute runs); the partial
                 supports are all-reduced (engine_join(): ncclAllReduce,
                 exact u32 sums) or, fused (engine_join_fused(), recompute
                 runs), every increment goes straight to the owner rank's
                 buffer over NVLink peer memory during the support pass and
                 only the owned spans are all-gathered; then every rank runs
                 the same deterministic prune / carried rounds;
  * device-resident group (engine_join_group(), the default for bench.py
                 --gpus N) -- the same split of full passes with the
                 all-reduce done by kernels over NVLink peer memory inside
                 the fixpoint's CUDA graph, and the carried rounds' removals
                 sharded across ranks with their decrements exchanged the
                 same way: one graph launch per fixpoint, no host round trip.
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import torch
import torch.distributed as dist

import ctypes

from .truss import Engine, device_copy, ipc_close, ipc_handle, ipc_open, nccl_unique_id


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


def engine_join_group(engine: Engine, group: Optional[dist.ProcessGroup] = None) -> list:
    """Device-resident partitioned fixpoint (ktg_engine_set_group): shares
    this rank's exchange area and support buffers as CUDA IPC handles over
    torch.distributed (collective), maps every peer's, installs the group and
    meets the peers in a barrier. Every fixpoint then runs as one CUDA-graph
    launch per rank: full passes split by work, S all-reduced by kernels over
    NVLink peer memory; carried rounds' removals sharded, decrements
    exchanged the same way. Call after engine.load(); returns the mapped peer
    pointers (ipc_close them once the engine is done)."""
    world, rank = world_rank()
    area, _ = engine.group_area()
    s0, s1, _ = engine.support_buffers()
    mine = (ipc_handle(area), ipc_handle(s0), ipc_handle(s1))
    allh = [None] * world
    dist.all_gather_object(allh, mine, group=group)
    mapped = []

    def table(i, own):
        out = []
        for q in range(world):
            if q == rank:
                out.append(own)
            else:
                p = ipc_open(allh[q][i])
                mapped.append(p)
                out.append(p)
        return out

    engine.set_group(rank, world, table(0, area), table(1, s0), table(2, s1))
    dist.barrier(group=group)
    return mapped


def _reduce_device(device):
    return device if dist.get_backend() == "nccl" else "cpu"


def max_over_ranks(x: float, device: Optional[torch.device] = None) -> float:
    world, _ = world_rank()
    if world == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_reduce_device(device))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, device: Optional[torch.device] = None) -> float:
    world, _ = world_rank()
    if world == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_reduce_device(device))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def engine_join_fused(engine: Engine, group: Optional[dist.ProcessGroup] = None) -> list:
    """Fused reduce-scatter (ktg_engine_set_peers): exchanges the support
    buffers' CUDA IPC handles (collective), maps every peer's buffers, and
    installs the per-round exchange (barrier; all-gather of the owned spans
    by peer copies; sum of the round's triangle count). Call after
    engine.load(). Returns the mapped peer pointers (ipc_close them after the
    engine is done)."""
    world, rank = world_rank()
    s0, s1, _ = engine.support_buffers()
    mine = (ipc_handle(s0), ipc_handle(s1))
    allh = [None] * world
    dist.all_gather_object(allh, mine, group=group)
    p0 = [s0 if q == rank else ipc_open(allh[q][0]) for q in range(world)]
    p1 = [s1 if q == rank else ipc_open(allh[q][1]) for q in range(world)]
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"

    def exchange(phase, d_s, slots, span, d_tri, stream):
        v = ctypes.c_uint64()
        device_copy(ctypes.addressof(v), ctypes.addressof(v), 0, stream)  # wait for this rank's stream
        dist.barrier(group=group)
        if phase == 0:  # every rank's previous prune (buffer zeroing) is done
            return
        device_copy(ctypes.addressof(v), d_tri, 8, stream)
        t = torch.tensor([v.value], dtype=torch.int64, device=dev)
        dist.all_reduce(t, group=group)
        v.value = int(t.item())
        device_copy(d_tri, ctypes.addressof(v), 8, stream)
        src = p0 if d_s == s0 else p1
        for q in range(world):
            lo = q * span
            cnt = min(span, slots - lo)
            if q != rank and cnt > 0:
                device_copy(d_s + 4 * lo, src[q] + 4 * lo, 4 * cnt, stream)
        dist.barrier(group=group)  # no rank zeroes or adds again before all copies

    engine.set_peers(rank, world, p0, p1, exchange)
    return [p for q, p in enumerate(p0 + p1) if q % world != rank]
