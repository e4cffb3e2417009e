"""Multi-GPU plumbing over torch.distributed (one process per GPU).

* ``attach(ctx)`` — rank 0 creates the NCCL unique id of the planner's own
  communicator, torch.distributed broadcasts it, every rank attaches it to its
  planner context; plans on that context are then row-sharded across ranks
  (include/parplan_c.h: pp_context_attach_comm).
* ``shard`` / ``global_best`` — the multi-graph sweep: each rank plans its
  contiguous share of the instances; the global argmin is an all-gather of
  (cost, sweep index) pairs and a lexicographic min (lowest index on ties).
* ``max_over_ranks`` — the benchmark's max-over-ranks device time.
"""
from __future__ import annotations

import os
from typing import Sequence

import torch
import torch.distributed as dist


def world() -> tuple:
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))


def attach(ctx) -> None:
    from .capi import comm_unique_id

    rank, size = dist.get_rank(), dist.get_world_size()
    obj = [comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx.attach_comm(size, rank, obj[0])


def shard(items: Sequence, rank: int, size: int) -> list:
    """Contiguous block of ``items`` for ``rank`` (sizes differ by at most one)."""
    n = len(items)
    lo = rank * n // size
    hi = (rank + 1) * n // size
    return [(i, items[i]) for i in range(lo, hi)]


def global_best(local: Sequence[tuple]) -> tuple:
    """local: [(cost, sweep_index, payload)] -> the global (cost, index, payload) minimum."""
    gathered = [None] * dist.get_world_size()
    dist.all_gather_object(gathered, list(local))
    flat = [x for part in gathered for x in part]
    return min(flat, key=lambda x: (x[0], x[1]))


def max_over_ranks(value: float, device=None) -> float:
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
