"""Memory rewrites and the memory pass (proj/src/optimize.cpp:815-1021),
evaluated on the GPU: every candidate is replayed in one batched launch and
its peak memory estimated by K5 on the schedule already in HBM.

    validate(g)                     graph.cpp:332-425 (validity only)
    recompute_candidate(g)          optimize.cpp:819-877 (sqrt(N) checkpoints)
    grad_accum_candidate(g, meta)   optimize.cpp:879-959 (2 micro-batches)
    apply_recompute / apply_grad_accum   apply_strategy, optimize.cpp:515-531
    memory_pass(g, budget, meta)    optimize.cpp:972-1021

Rewrites are string-keyed graph surgery on the host (same op names, so the
same index order and tie-breaks as the reference); the measurement of each
candidate (replay + peak memory) is the GPU's.
"""
from __future__ import annotations

import copy
import enum
import math
from collections import deque
from dataclasses import dataclass

from .errors import Error, TransformError
from .graph import (GlobalDFG, GraphBuilder, OpKind, is_communication, is_virtual, round_us)
from .memory import ModelMeta, estimate_peak_memory_many
from .replay import replay_many


class BudgetError(Error):
    """dpro::BudgetError (errors.hpp:110-115)."""

    def __init__(self, what: str, best_peak_bytes: int):
        super().__init__(what)
        self.best_peak_bytes = best_peak_bytes


class StrategyKind(enum.IntEnum):
    """optimize.hpp:48-54."""
    OP_FUSION = 0
    TENSOR_FUSION = 1
    PARTITION = 2
    RECOMPUTE = 3
    GRAD_ACCUM = 4

    def __str__(self) -> str:  # optimize.cpp:150-164
        return ["op-fusion", "tensor-fusion", "partition", "recompute", "grad-accum"][self]


@dataclass
class Strategy:
    """optimize.hpp:58-67."""
    kind: StrategyKind = StrategyKind.OP_FUSION
    a: str = ""
    b: str = ""
    k: int = 1
    dur_us: int = -1


def local_part(op_id: str) -> str:
    """optimize.cpp:41-44."""
    arrow = op_id.find("->")
    return op_id if arrow < 0 else op_id[arrow + 2:]


def topo_order(g: GlobalDFG) -> list[int] | None:
    """GlobalDFG::topo_order (graph.cpp:145-162): Kahn with a FIFO seeded in
    index order; None on a cycle."""
    indeg = [len(g.pred_indices(i)) for i in range(g.size())]
    ready = deque(i for i in range(g.size()) if indeg[i] == 0)
    order = []
    while ready:
        i = ready.popleft()
        order.append(i)
        for s in g.succ_indices(i):
            indeg[s] -= 1
            if indeg[s] == 0:
                ready.append(s)
    return order if len(order) == g.size() else None


def validate(g: GlobalDFG) -> bool:
    """The validity verdict of graph.cpp:332-425 (the rewrites only read
    `valid`)."""
    if topo_order(g) is None:
        return False
    sends: dict[str, list] = {}
    recvs: dict[str, list] = {}
    for o in g.ops():
        if o.dur < 0 or (is_virtual(o.kind) and o.dur != 0):
            return False
        if is_communication(o.kind):
            if not o.tensor or o.bytes <= 0 or not o.transaction:
                return False
            (sends if o.kind == OpKind.SEND else recvs).setdefault(o.transaction, []).append(o)
    for txn, ops in sends.items():
        if len(ops) > 1 or txn not in recvs:
            return False
        r = recvs[txn][0]
        if ops[0].tensor != r.tensor or ops[0].bytes != r.bytes:
            return False
    for txn, ops in recvs.items():
        if len(ops) > 1 or txn not in sends:
            return False
    referenced = set()
    for unit in g.tensor_units().values():
        for want, table in ((OpKind.VIRTUAL_IN, unit.vin), (OpKind.VIRTUAL_OUT, unit.vout)):
            for vid in table.values():
                referenced.add(vid)
                if not g.has_op(vid) or g.op(vid).kind != want:
                    return False
        if any(not g.has_op(c) for c in unit.comm_ops):
            return False
    return not any(is_virtual(o.kind) and o.id not in referenced for o in g.ops())


def recompute_candidate(g: GlobalDFG) -> tuple[GlobalDFG, Strategy] | None:
    """optimize.cpp:819-877: per node, the FW chain (topological order) is cut
    into c = ceil(sqrt(n)) segments; every non-checkpoint FW of a segment is
    re-run as RFW.<x> feeding the backward ops, gated on the backward of the
    segment's checkpoint and chained from the previous checkpoint."""
    order = topo_order(g)
    if order is None:
        return None
    chains: dict[str, list[str]] = {}
    for idx in order:
        op = g.op_at(idx)
        if op.kind != OpKind.FW:
            continue
        if not local_part(op.id).startswith("FW."):
            return None
        chains.setdefault(op.node, []).append(op.id)
    b = GraphBuilder(g)
    any_ = False
    checkpoints = 0
    for node in sorted(chains):
        chain = chains[node]
        n = len(chain)
        if n < 2:
            continue
        if any(not g.has_edge(chain[i], chain[i + 1]) for i in range(n - 1)):
            return None
        c = int(math.ceil(math.sqrt(n)))
        seg_base, seg_rem = divmod(n, c)
        lo, prev_cp = 0, -1
        for s in range(c):
            ln = seg_base + (1 if s < seg_rem else 0)
            cp = lo + ln - 1
            gate = f"{node}->BW.{local_part(chain[cp])[3:]}"
            prev_rfw = ""
            for i in range(lo, cp):
                fw = g.op(chain[i])
                rfw = copy.copy(fw)
                rfw.id = f"{node}->RFW.{local_part(fw.id)[3:]}"
                rfw.produces = []
                b.add_op(rfw)
                for succ in g.succs(fw.id):
                    if g.op(succ).kind != OpKind.BW:
                        continue
                    b.remove_edge(fw.id, succ)
                    b.add_edge(rfw.id, succ)
                if not prev_rfw:
                    if prev_cp >= 0:
                        b.add_edge(chain[prev_cp], rfw.id)
                    if g.has_op(gate):
                        b.add_edge(gate, rfw.id)
                else:
                    b.add_edge(prev_rfw, rfw.id)
                prev_rfw = rfw.id
            prev_cp = cp
            lo += ln
        checkpoints = c
        any_ = True
    if not any_:
        return None
    out = b.build()
    if not validate(out):
        return None
    return out, Strategy(StrategyKind.RECOMPUTE, "", "", checkpoints, -1)


def grad_accum_candidate(g: GlobalDFG, meta: ModelMeta) -> tuple[GlobalDFG, Strategy] | None:
    """optimize.cpp:879-959: every FW/BW op becomes two micro-batch copies
    <id>@mb0/@mb1 with round_us(dur * microbatch_scale); a node's @mb1
    sources wait for its @mb0 backward sinks."""
    dup = [op.kind in (OpKind.FW, OpKind.BW) for op in g.ops()]
    if not any(dup):
        return None
    b = GraphBuilder()
    b.set_cluster(g.cluster())
    for unit in g.tensor_units().values():
        b.add_tensor_unit(unit)
    ops = g.ops()
    for i, op in enumerate(ops):  # kept ops (GraphBuilder(g) minus remove_op)
        if not dup[i]:
            b.add_op(copy.copy(op))
    for i, op in enumerate(ops):
        if not dup[i]:
            continue
        for mb in range(2):
            c = copy.copy(op)
            c.id = f"{op.id}@mb{mb}"
            c.dur = round_us(float(op.dur) * meta.microbatch_scale)
            c.produces = [] if mb == 0 else list(op.produces)
            b.add_op(c)
    for i, op in enumerate(ops):
        for s in g.succ_indices(i):
            sid = ops[s].id
            if dup[i] and dup[s]:
                b.add_edge(op.id + "@mb0", sid + "@mb0")
                b.add_edge(op.id + "@mb1", sid + "@mb1")
            elif dup[i]:
                b.add_edge(op.id + "@mb1", sid)
            elif dup[s]:
                b.add_edge(op.id, sid + "@mb0")
            else:
                b.add_edge(op.id, sid)
    sinks: dict[str, list[str]] = {}
    sources: dict[str, list[str]] = {}
    for i, op in enumerate(ops):
        if op.kind == OpKind.BW and not any(dup[s] for s in g.succ_indices(i)):
            sinks.setdefault(op.node, []).append(op.id)
        if op.kind == OpKind.FW and not any(dup[p] for p in g.pred_indices(i)):
            sources.setdefault(op.node, []).append(op.id)
    for node in sorted(sinks):
        for e in sinks[node]:
            for s in sources.get(node, []):
                b.add_edge(e + "@mb0", s + "@mb1")
    out = b.build()
    if not validate(out):
        return None
    return out, Strategy(StrategyKind.GRAD_ACCUM, "", "", 2, -1)


def apply_recompute(g: GlobalDFG) -> GlobalDFG:
    """apply_strategy(kRecompute), optimize.cpp:515-522."""
    r = recompute_candidate(g)
    if r is None:
        raise TransformError("re-computation does not apply to this graph")
    return r[0]


def apply_grad_accum(g: GlobalDFG, meta: ModelMeta) -> GlobalDFG:
    """apply_strategy(kGradAccum), optimize.cpp:523-531."""
    r = grad_accum_candidate(g, meta)
    if r is None:
        raise TransformError("gradient accumulation does not apply to this graph")
    return r[0]


def max_peaks(graphs: list[GlobalDFG], meta: ModelMeta) -> tuple[list[int], list[int]]:
    """(max-over-nodes peak, iteration time) of each graph: ONE batched
    replay and ONE K5 launch (optimize.cpp:961-968 per graph)."""
    results = replay_many(graphs)
    peaks = estimate_peak_memory_many(graphs, results, meta)
    return ([max(p.values(), default=0) for p in peaks],
            [r.iteration_time_us for r in results])


def memory_pass(g: GlobalDFG, budget_bytes: int, meta: ModelMeta,
                applied: list[Strategy] | None = None) -> GlobalDFG:
    """optimize.cpp:972-1021: if the peak exceeds the budget, take the
    fastest of {recompute, grad-accum} that fits, else raise BudgetError
    with the smallest peak reached."""
    if budget_bytes <= 0:
        return g
    (base_peak,), _ = max_peaks([g], meta)
    if base_peak <= budget_bytes:
        return g
    cands = [c for c in (recompute_candidate(g), grad_accum_candidate(g, meta)) if c]
    peaks, times = max_peaks([c[0] for c in cands], meta) if cands else ([], [])
    best = None
    for i in range(len(cands)):
        if peaks[i] > budget_bytes:
            continue
        if best is None or times[i] < times[best]:
            best = i
    if best is None:
        reached = min([base_peak] + peaks)
        raise BudgetError(f"peak memory {base_peak} bytes exceeds budget {budget_bytes} "
                          "bytes and no rewrite closes the gap", reached)
    if applied is not None:
        applied.append(cands[best][1])
    return cands[best][0]
