"""Reference-shaped Replayer API (proj/include/dpro/replay.hpp:27-91) on top
of the CUDA engine. Same names, argument meaning, results and exceptions as
the reference; every call goes through libdpro_cuda.so (no CPU fallback).

    replay(g)                      replay.cpp:37-134   -> K1 (one batch of 1)
    replay_many(graphs)            -- batched form the search uses
    execution_graph(g, r)          replay.cpp:136-144
    critical_path(exec_graph, r)   replay.cpp:146-226  -> K3
    sync_makespan(cluster, b, k)   replay.cpp:228-246  -> t_sync grid
    partial_replay(g, tensor, k)   replay.cpp:248-258
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _native as N
from .engine import Batch, Csr, default_engine
from .errors import CycleError, EngineError, Error, LookupError_, MissingProfileError
from .graph import (ClusterSpec, DeviceId, GlobalDFG, GraphBuilder, is_communication,
                    is_virtual)


@dataclass
class ScheduleEntry:
    start: int = 0
    end: int = 0
    device: DeviceId = field(default_factory=DeviceId)


@dataclass
class ReplayResult:
    iteration_time_us: int = 0
    schedule: dict[str, ScheduleEntry] = field(default_factory=dict)
    device_timelines: dict[DeviceId, list[str]] = field(default_factory=dict)
    utilization: dict[DeviceId, float] = field(default_factory=dict)
    # engine state kept for critical_path (K3 runs on the replayed batch)
    _batch: Batch | None = field(default=None, repr=False, compare=False)
    _cand: int = field(default=0, repr=False, compare=False)
    _graph: GlobalDFG | None = field(default=None, repr=False, compare=False)


@dataclass
class PathEntry:
    op: str
    dur: int = 0
    communication: bool = False


@dataclass
class PathRun:
    communication: bool = False
    ops: list[str] = field(default_factory=list)
    dur_us: int = 0


@dataclass
class CriticalPath:
    ops: list[PathEntry] = field(default_factory=list)
    runs: list[PathRun] = field(default_factory=list)
    conforming: bool = False
    total_us: int = 0


def _raise_status(g: GlobalDFG, batch: Batch, cand: int, status: int, err: int) -> None:
    if status == N.DPRO_MISSING_PROFILE:
        raise MissingProfileError(f"op {g.op_at(int(err)).id} has no duration")
    if status == N.DPRO_CYCLE:
        mask = batch.scheduled(cand)
        stuck = [g.op_at(i).id for i in np.flatnonzero(mask == 0)]
        raise CycleError(
            f"replay requires an acyclic graph; {len(stuck)} ops never became ready", stuck)
    if status != N.DPRO_OK:
        raise EngineError(f"replay failed with engine status {status}")


def _result(g: GlobalDFG, batch: Batch, cand: int, T: int, start: np.ndarray,
            end: np.ndarray) -> ReplayResult:
    csr = g.to_csr()
    devs = csr["devices"]
    r = ReplayResult(iteration_time_us=int(T), _batch=batch, _cand=cand, _graph=g)
    ops = g.ops()
    r.schedule = {op.id: ScheduleEntry(int(start[i]), int(end[i]), op.device)
                  for i, op in enumerate(ops)}
    order, dev_off, busy = batch.timelines(cand)
    for d, dv in enumerate(devs):
        a, b = int(dev_off[d]), int(dev_off[d + 1])
        if b > a:  # the reference only creates timelines on dispatch
            r.device_timelines[dv] = [ops[i].id for i in order[a:b]]
            r.utilization[dv] = (float(busy[d]) / float(T)) if T > 0 else 0.0
    return r


def replay_many(graphs: Sequence[GlobalDFG], engine=None) -> list[ReplayResult]:
    """Replays several graphs in ONE batched launch; raises on the first
    failing graph exactly as replay() would."""
    eng = engine or default_engine()
    batch = eng.batch([Csr.from_dict(g.to_csr()) for g in graphs])
    batch.replay(want_schedule=True)
    ms, st, er, start, end = batch.results(schedule=True)
    out = []
    for i, g in enumerate(graphs):
        _raise_status(g, batch, i, int(st[i]), int(er[i]))
        a, b = int(batch.op_off[i]), int(batch.op_off[i + 1])
        out.append(_result(g, batch, i, int(ms[i]), start[a:b], end[a:b]))
    return out


def replay_times(graphs: Sequence[GlobalDFG], engine=None) -> list[int | None]:
    """Iteration times of several graphs from ONE makespan-only batched
    launch. A graph whose replay fails gives None: replay(g) on it raises the
    reference's error, so callers that must fail in order re-run it there."""
    if not graphs:
        return []
    eng = engine or default_engine()
    batch = eng.batch([Csr.from_dict(g.to_csr()) for g in graphs])
    batch.replay(want_schedule=False)
    ms, st, _, _, _ = batch.results(schedule=False)
    return [int(ms[i]) if int(st[i]) == N.DPRO_OK else None for i in range(len(graphs))]


def replay(g: GlobalDFG) -> ReplayResult:
    """dpro::replay (replay.hpp:40-48)."""
    return replay_many([g])[0]


def execution_graph(g: GlobalDFG, result: ReplayResult) -> GlobalDFG:
    """replay.cpp:136-144: original edges plus consecutive timeline pairs."""
    b = GraphBuilder(g)
    for tl in result.device_timelines.values():
        for i in range(1, len(tl)):
            b.add_edge(tl[i - 1], tl[i])
    eg = b.build()
    eg._exec_of = result  # noqa: SLF001 - marks the graph K3 may stand in for
    return eg


def critical_path(exec_graph: GlobalDFG, result: ReplayResult, engine=None) -> CriticalPath:
    """replay.cpp:146-226 on the GPU (K3). When exec_graph is
    execution_graph(g, result) of a replay() result, K3 runs on the replayed
    batch (timeline edges read from the engine's queues); otherwise on
    exec_graph itself with result's schedule (dpro_cuda_critical_path)."""
    path = CriticalPath(total_us=result.iteration_time_us)
    if exec_graph.size() == 0:
        path.conforming = True
        return path
    if getattr(exec_graph, "_exec_of", None) is result and result._batch is not None:
        g = result._graph
        idx = [exec_graph.index_of(g.op_at(int(i)).id)
               for i in result._batch.critical_paths()[result._cand]]
    else:
        eng = engine or default_engine()
        csr = Csr.from_dict(exec_graph.to_csr())
        n = exec_graph.size()
        start = np.array([result.schedule[o.id].start for o in exec_graph.ops()], np.int64)
        end = np.array([result.schedule[o.id].end for o in exec_graph.ops()], np.int64)
        out = np.zeros(n, np.uint32)
        ln = np.zeros(1, np.int64)
        s = csr.as_struct()
        rc = N.lib.dpro_cuda_critical_path(eng.ctx, s, N.ptr(start), N.ptr(end),
                                           int(result.iteration_time_us), N.ptr(out), N.ptr(ln))
        if rc != N.DPRO_OK:
            raise EngineError(f"critical_path failed ({rc})")
        idx = out[: int(ln[0])].tolist()
    for i in idx:
        op = exec_graph.op_at(int(i))
        path.ops.append(PathEntry(op.id, op.dur, is_communication(op.kind)))
    for e in path.ops:
        op = exec_graph.op(e.op)
        if is_virtual(op.kind):
            continue
        comm = is_communication(op.kind)
        if not path.runs or path.runs[-1].communication != comm:
            path.runs.append(PathRun(comm, [], 0))
        path.runs[-1].ops.append(e.op)
        path.runs[-1].dur_us += e.dur
    path.conforming = len(path.runs) <= 2 and (
        len(path.runs) < 2 or (not path.runs[0].communication and path.runs[1].communication))
    return path


def sync_makespan_grid(cluster: ClusterSpec, bytes_: Sequence[int], ks: Sequence[int],
                       engine=None) -> list[int]:
    """Batched t_sync(bytes, k) (the memoized grid of optimize.cpp:562-576)."""
    for k in ks:
        if k < 1:
            raise Error(f"sync_makespan: partition count must be >= 1, got {k}")
    out, st = (engine or default_engine()).tsync_grid(cluster, bytes_, ks)
    if np.any(st != N.DPRO_OK):
        raise EngineError(f"t_sync grid failed: statuses {st.tolist()}")
    return [int(x) for x in out]


def sync_makespan(cluster: ClusterSpec, bytes_: int, k: int) -> int:
    """replay.cpp:228-246."""
    return sync_makespan_grid(cluster, [bytes_], [k])[0]


def partial_replay(g: GlobalDFG, tensor: str, k: int = 1) -> int:
    """replay.cpp:248-258."""
    if g.has_base(tensor):
        b = g.base_bytes(tensor)
    elif g.has_tensor_unit(tensor):
        b = g.tensor_unit(tensor).bytes
    else:
        raise LookupError_(f"unknown tensor: {tensor}")
    return sync_makespan(g.cluster(), b, k)
