"""Per-round best-cost exchange across ranks (K4 of DESIGN.md) and the
Metropolis acceptance rule of the search.

Candidates and MCMC chains are sharded over ranks with no data-path
collective; once per round every rank contributes its best
(makespan, candidate index) and all ranks agree on the global argmin with
two MIN all-reduces over NCCL (CPU tensors under gloo in the tests):

1. MIN of the makespans (int64: ns makespans of 10^12 fit; no packing);
2. MIN of (rank << 32 | index) over the ranks that hold that makespan, so
   ties go to the lowest rank, then the lowest index -- any world size
   below 2^31 and any batch below 2^32.

The owner then broadcasts the winning strategy (a picklable object).
The reference has no multi-rank search; its per-candidate gate accepts
the first improvement in walk order (optimize.cpp:1382-1392).
"""
from __future__ import annotations

import math
from typing import Any

I64_MAX = (1 << 63) - 1


def exchange_best(dist, makespan: int, index: int, rank: int, device="cpu") -> tuple[int, int, int]:
    """-> (global best makespan, owner rank, owner's candidate index)."""
    import torch
    if not 0 <= index < (1 << 32):
        raise ValueError(f"candidate index {index} outside [0, 2^32)")
    if not 0 <= rank < (1 << 31):
        raise ValueError(f"rank {rank} outside [0, 2^31)")
    m = torch.tensor([int(makespan)], dtype=torch.int64, device=device)
    dist.all_reduce(m, op=dist.ReduceOp.MIN)
    best = int(m.item())
    k = torch.tensor([(rank << 32) | index if int(makespan) == best else I64_MAX],
                     dtype=torch.int64, device=device)
    dist.all_reduce(k, op=dist.ReduceOp.MIN)
    key = int(k.item())
    return best, key >> 32, key & 0xFFFFFFFF


def broadcast_from(dist, obj: Any, owner: int, rank: int) -> Any:
    """The owner's object on every rank (broadcast_object_list)."""
    box = [obj if rank == owner else None]
    dist.broadcast_object_list(box, src=owner)
    return box[0]


def metropolis_accept(beta: float, current: int, proposal: int, u: float) -> bool:
    """P = min(1, exp(beta (T - T'))) (memory term 0), without
    evaluating exp of a large positive argument: improvements are accepted
    outright, otherwise u < exp(d) with d <= 0 (underflows to 0, never
    overflows)."""
    d = beta * (float(current) - float(proposal))
    if d >= 0.0:
        return True
    return u < math.exp(d)
