"""Multi-rank host logic on CPU (gloo, world_size 2): the per-round
best-cost exchange of bench.py -- a packed int64 (makespan, rank, id) MIN
all-reduce -- picks the global argmin with the lowest (rank, id) on ties."""
import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def pack_key(makespan: torch.Tensor, rank: int) -> torch.Tensor:
    best = torch.min(makespan, dim=0)
    return (best.values << 24) | (rank << 20) | best.indices


def _worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = torch.Generator().manual_seed(rank)
    ms = torch.randint(1000, 2000, (64,), generator=g, dtype=torch.int64)
    if rank == 1:
        ms[17] = 900  # global best lives on rank 1, candidate 17
    key = pack_key(ms, rank)
    dist.all_reduce(key, op=dist.ReduceOp.MIN)
    results[rank] = (int(key) >> 24, (int(key) >> 20) & 0xF, int(key) & 0xFFFFF)
    dist.destroy_process_group()


def test_best_cost_exchange_gloo():
    mgr = mp.Manager()
    results = mgr.dict()
    port = 29500 + os.getpid() % 1000
    mp.spawn(_worker, args=(2, port, results), nprocs=2, join=True)
    assert results[0] == results[1] == (900, 1, 17)


def test_bench_key_packing_matches():
    import bench  # noqa: F401  (bench uses the same packing)
    ms = torch.tensor([5, 3, 3, 9], dtype=torch.int64)
    k = pack_key(ms, 2)
    assert (int(k) >> 24, (int(k) >> 20) & 0xF, int(k) & 0xFFFFF) == (3, 2, 1)
