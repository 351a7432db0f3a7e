"""Multi-rank host logic on CPU (gloo, world_size 2): the per-round
best-cost exchange the search and bench.py use (paper_2205_02473_b200.exchange)
and SyncSearch._exchange itself, run as product code over gloo."""
import os
import types

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2205_02473_b200.exchange import (broadcast_from, exchange_best,
                                            metropolis_accept)

NS_BIG = 980_573_000_000  # a config-4 makespan in ns: > 2^39, broke the packed key


def _init(rank, world, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _worker(rank, world, port, results):
    _init(rank, world, port)
    g = torch.Generator().manual_seed(rank)
    ms = torch.randint(NS_BIG, NS_BIG + 10**6, (64,), generator=g, dtype=torch.int64)
    if rank == 1:
        ms[17] = NS_BIG - 5  # global best lives on rank 1, candidate 17
    best = torch.min(ms, dim=0)
    out = exchange_best(dist, int(best.values), int(best.indices), rank)
    # ties: both ranks hold the same makespan -> lowest rank, then index
    tie = exchange_best(dist, 1234, 3 if rank == 0 else 1, rank)
    # index beyond the old 20-bit field
    wide = exchange_best(dist, 7 + rank, (1 << 31) + rank, rank)
    obj = broadcast_from(dist, {"strategy": f"from-rank-{rank}"}, out[1], rank)
    results[rank] = (out, tie, wide, obj)
    dist.destroy_process_group()


def test_exchange_best_gloo():
    mgr = mp.Manager()
    results = mgr.dict()
    port = 29500 + os.getpid() % 1000
    mp.spawn(_worker, args=(2, port, results), nprocs=2, join=True)
    assert results[0] == results[1]
    out, tie, wide, obj = results[0]
    assert out == (NS_BIG - 5, 1, 17)
    assert tie == (1234, 0, 3)
    assert wide == (7, 0, 1 << 31)
    assert obj == {"strategy": "from-rank-1"}


def _search_worker(rank, world, port, results):
    """SyncSearch._exchange (product code) with a stub engine: the round's
    global best proposal and its makespan reach every rank."""
    _init(rank, world, port)
    from paper_2205_02473_b200.search import SyncSearch, SyncState
    s = SyncSearch.__new__(SyncSearch)
    s.dist, s.rank, s.engine = dist, rank, types.SimpleNamespace(device=0)
    cand = SyncState([[0], [1, 2]], [1 + rank, 2], -1)
    ms = NS_BIG + 100 - rank * 50
    got = s._exchange(ms, 5 + rank, cand)
    results[rank] = (got.groups, got.ks, got.makespan)
    dist.destroy_process_group()


def test_syncsearch_exchange_gloo():
    mgr = mp.Manager()
    results = mgr.dict()
    port = 30600 + os.getpid() % 1000
    mp.spawn(_search_worker, args=(2, port, results), nprocs=2, join=True)
    assert results[0] == results[1] == ([[0], [1, 2]], [2, 2], NS_BIG + 50)


def test_metropolis_no_overflow():
    # beta * improvement = 0.01 * 10^6: exp() of it would overflow
    assert metropolis_accept(0.01, 10**6 + 1000, 1000, 0.999)
    assert metropolis_accept(0.01, 100, 100, 0.999)
    assert not metropolis_accept(0.01, 1000, 10**6, 1e-300)
    assert metropolis_accept(0.01, 1000, 1100, 0.3)       # exp(-1) = 0.37
    assert not metropolis_accept(0.01, 1000, 1100, 0.4)


def test_exchange_rejects_out_of_range():
    with pytest.raises(ValueError):
        exchange_best(None, 1, 1 << 32, 0)
