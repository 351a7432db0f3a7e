"""Graph rewrites of the reference's optimizer (proj/src/optimize.cpp) on a
GlobalDFG, and the memory pass evaluated on the GPU: every candidate is
replayed in one batched launch and its peak memory estimated by K5 on the
schedule already in HBM.

    CostModel                       optimize.cpp:82-145 (fused-op table)
    apply_op_fusion(g, a, b, ...)   optimize.cpp:245-317
    apply_tensor_fusion(g, t1, t2)  optimize.cpp:366-455
    apply_tensor_partition(g, t, k) optimize.cpp:459-492
    apply_strategy / _set           optimize.cpp:506-541
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
import re
from collections import deque
from dataclasses import dataclass, field

import numpy as np

from .errors import (CycleError, Error, IoError, LookupError_, SchemaError, SpliceError,
                     TransformError)
from .graph import (DeviceId, GlobalDFG, GraphBuilder, Op, OpKind, TensorUnit, is_communication,
                    is_computation, is_virtual, round_us)
from .ingest import CommTopology, expand_tensor
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


_STOD = re.compile(r"^[+-]?((\d+\.?\d*|\.\d+)([eE][+-]?\d+)?|inf(inity)?|nan)$", re.I)


@dataclass
class CostModel:
    """optimize.hpp:35-46: fused durations by (op a, op b), with a ratio
    fallback."""
    fused_us: dict[tuple[str, str], float] = field(default_factory=dict)
    fallback_ratio: float = 0.8

    def fused_dur_us(self, a, b) -> float:
        """optimize.cpp:84-103: table entry (full ids, then local parts) if
        it does not exceed a.dur + b.dur, else fallback_ratio * (a + b)."""
        cap = float(a.dur) + float(b.dur)

        def lookup(ka: str, kb: str) -> float:
            v = self.fused_us.get((ka, kb))
            return -1.0 if v is None or v > cap else v

        v = lookup(a.id, b.id)
        if v >= 0:
            return v
        v = lookup(local_part(a.id), local_part(b.id))
        if v >= 0:
            return v
        return self.fallback_ratio * cap

    @staticmethod
    def from_csv(text: str) -> "CostModel":
        """optimize.cpp:105-137: rows "op_a, op_b, fused_dur_us"."""
        m = CostModel()
        for line in text.splitlines():
            row = line.strip(" \t\r\n")
            if not row or row[0] == "#":
                continue
            fields = row.split(",")
            if len(fields) != 3:
                raise SchemaError(f"cost model row needs op_a, op_b, fused_dur_us: {row}",
                                  "fused_dur_us")
            a, b, val = (f.strip(" \t\r\n") for f in fields)
            if val == "fused_dur_us":
                continue  # header row
            if not _STOD.match(val):  # what std::stod consumes whole
                raise SchemaError(f"cost model duration is not a number: {row}", "fused_dur_us")
            dur = float(val)
            m.fused_us[(a, b)] = dur
        return m

    @staticmethod
    def load(path: str) -> "CostModel":
        try:
            with open(path) as f:
                return CostModel.from_csv(f.read())
        except OSError as e:
            raise IoError(f"cannot open cost model: {path}") from e


def fused_op_id(a: str, b: str) -> str:
    """optimize.cpp:76-78."""
    return a + "+" + local_part(b)


def apply_op_fusion(g: GlobalDFG, a: str, b: str, cost: CostModel | None = None,
                    dur_us_override: int = -1) -> GlobalDFG:
    """optimize.cpp:245-317: a and b (computation ops on one device joined
    by an edge, with no second path a -> ... -> b) become one op."""
    cost = cost or CostModel()
    oa, ob = g.op(a), g.op(b)
    if a == b:
        raise TransformError(f"cannot fuse op {a} with itself")
    if not is_computation(oa.kind) or not is_computation(ob.kind):
        raise TransformError(f"op fusion requires computation ops: {a}, {b}")
    if oa.device.str() != ob.device.str():
        raise TransformError(f"ops {a} and {b} run on different devices")
    if not g.has_edge(a, b):
        raise TransformError(f"op fusion requires a direct edge {a} -> {b}")
    # second path a -> ... -> b: breadth-first over successor indices
    # (ascending index == id order, so the witness is the id-order BFS's)
    ia, ib = g.index_of(a), g.index_of(b)
    parent: dict[int, int] = {}
    frontier = deque()
    for s in g.succ_indices(ia):
        if s == ib:
            continue
        if s not in parent:
            parent[s] = ia
        frontier.append(s)
    while frontier:
        cur = frontier.popleft()
        if cur == ib:
            witness = [ib]
            x = parent[ib]
            while x != ia:
                witness.append(x)
                x = parent[x]
            witness.append(ia)
            witness.reverse()
            raise CycleError(f"fusing {a} and {b} would create a cycle",
                             [g.op_at(i).id for i in witness])
        for s in g.succ_indices(cur):
            if s not in parent:
                parent[s] = cur
                frontier.append(s)
    fused = copy.copy(oa)
    fused.id = fused_op_id(a, b)
    fused.dur = dur_us_override if dur_us_override >= 0 else round_us(cost.fused_dur_us(oa, ob))
    fused.produces = list(oa.produces) + list(ob.produces)
    if g.has_op(fused.id) and fused.id not in (a, b):
        raise TransformError(f"duplicate op id '{fused.id}'")
    return g.fused(ia, ib, fused)


def splice_topology(bld: GraphBuilder, topo: CommTopology, base: str, part_index: int,
                    part_count: int, vin: dict[str, str], vout: dict[str, str]) -> None:
    """optimize.cpp:325-361."""
    for op in topo.ops:
        bld.add_op(op)
    for x, y in topo.edges:
        bld.add_edge(x, y)
    unit = TensorUnit(topo.unit, base, topo.bytes, part_index, part_count, topo.ps_node,
                      sorted(op.id for op in topo.ops))
    for node, ids in topo.entry.items():
        if node not in vin:
            raise SpliceError(f"tensor {topo.unit} enters at node {node} which has no entry op")
        for i in ids:
            bld.add_edge(vin[node], i)
        unit.vin[node] = vin[node]
    for node, ids in topo.exit.items():
        if node not in vout:
            raise SpliceError(f"tensor {topo.unit} exits at node {node} which has no exit op")
        for i in ids:
            bld.add_edge(i, vout[node])
        unit.vout[node] = vout[node]
    bld.add_tensor_unit(unit)


def apply_tensor_fusion(g: GlobalDFG, t1: str, t2: str) -> GlobalDFG:
    """optimize.cpp:366-455: two unpartitioned tensors synchronize as one
    unit "t1+t2" with new IN/OUT splice points per worker."""
    if t1 == t2:
        raise TransformError(f"cannot fuse tensor {t1} with itself")
    if not g.has_base(t1):
        raise LookupError_(f"unknown tensor: {t1}")
    if not g.has_base(t2):
        raise LookupError_(f"unknown tensor: {t2}")
    n1, n2 = g.units_of_base(t1), g.units_of_base(t2)
    if len(n1) != 1 or len(n2) != 1:
        raise TransformError("tensor fusion needs unpartitioned inputs; merge "
                             f"{t1 if len(n1) != 1 else t2} back first")
    u1, u2 = g.tensor_unit(n1[0]), g.tensor_unit(n2[0])
    if sorted(u1.vin) != sorted(u2.vin) or sorted(u1.vout) != sorted(u2.vout):
        raise TransformError(f"tensors {t1} and {t2} attach to different worker sets")
    fused = f"{t1}+{t2}"
    bld = GraphBuilder(g)
    vin: dict[str, str] = {}
    vout: dict[str, str] = {}
    for node in sorted(u1.vin):
        dv = DeviceId.compute(node)
        in_op = Op(f"{node}->IN.{fused}", OpKind.VIRTUAL_IN, node, dv, 0, tensor=fused)
        out_op = Op(f"{node}->OUT.{fused}", OpKind.VIRTUAL_OUT, node, dv, 0, tensor=fused)
        bld.add_op(in_op)
        bld.add_op(out_op)
        vin[node], vout[node] = in_op.id, out_op.id
        for p in sorted(set(g.preds(u1.vin[node])) | set(g.preds(u2.vin[node]))):
            bld.add_edge(p, in_op.id)
        for t in sorted(set(g.succs(u1.vout[node])) | set(g.succs(u2.vout[node]))):
            bld.add_edge(out_op.id, t)
    gone = list(u1.comm_ops) + list(u2.comm_ops) + list(u1.vin.values()) + \
        list(u1.vout.values()) + list(u2.vin.values()) + list(u2.vout.values())
    bld.remove_ops(gone)
    bld.remove_tensor_unit(u1.name)
    bld.remove_tensor_unit(u2.name)
    topo = expand_tensor(fused, u1.bytes + u2.bytes, g.cluster())
    splice_topology(bld, topo, fused, 0, 1, vin, vout)
    for op in g.ops():  # producers now advertise the fused unit
        if not is_computation(op.kind):
            continue
        touched, produces = False, []
        for t in op.produces:
            if t in (t1, t2):
                if not touched:
                    produces.append(fused)
                touched = True
            else:
                produces.append(t)
        if touched:
            bld.op(op.id).produces = produces  # copy-on-write in GraphBuilder.op
    return bld.build()


def apply_tensor_partition(g: GlobalDFG, t: str, k: int) -> GlobalDFG:
    """optimize.cpp:459-492: tensor t synchronizes as k balanced units
    "t#p<i>" (or "t" for k = 1), spliced where its first unit was."""
    if not g.has_base(t):
        raise LookupError_(f"unknown tensor: {t}")
    nbytes = g.base_bytes(t)
    if k < 1:
        raise TransformError(f"partition count must be >= 1, got {k}")
    if k > nbytes:
        raise TransformError(f"cannot split {nbytes} bytes of {t} into {k} partitions")
    names = g.units_of_base(t)
    first = g.tensor_unit(names[0])
    if first.part_count == k:
        return g
    bld = GraphBuilder(g)
    gone = []
    for name in names:
        gone += g.tensor_unit(name).comm_ops
        bld.remove_tensor_unit(name)
    bld.remove_ops(gone)
    base, rem = divmod(nbytes, k)
    for i in range(k):
        name = t if k == 1 else f"{t}#p{i}"
        topo = expand_tensor(name, base + (1 if i < rem else 0), g.cluster())
        splice_topology(bld, topo, t, i, k, dict(first.vin), dict(first.vout))
    return bld.build()


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


def apply_strategy(g: GlobalDFG, s: Strategy, cost: CostModel | None = None,
                   meta: ModelMeta | None = None) -> GlobalDFG:
    """optimize.cpp:506-531."""
    if s.kind == StrategyKind.OP_FUSION:
        return apply_op_fusion(g, s.a, s.b, cost, s.dur_us)
    if s.kind == StrategyKind.TENSOR_FUSION:
        return apply_tensor_fusion(g, s.a, s.b)
    if s.kind == StrategyKind.PARTITION:
        return apply_tensor_partition(g, s.a, s.k)
    if s.kind == StrategyKind.RECOMPUTE:
        return apply_recompute(g)
    if s.kind == StrategyKind.GRAD_ACCUM:
        return apply_grad_accum(g, meta or ModelMeta())
    raise TransformError("unknown strategy kind")


def apply_strategy_set(g: GlobalDFG, strategies, cost: CostModel | None = None,
                       meta: ModelMeta | None = None) -> GlobalDFG:
    """optimize.cpp:535-541."""
    for s in strategies:
        g = apply_strategy(g, s, cost, meta)
    return g


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


def memory_pass_layered(model, cluster, budget_bytes: int, meta: ModelMeta, engine=None,
                        part_k=None):
    """memory_pass (optimize.cpp:972-1021) for a layered model at generator
    speed: the base graph and its recompute / grad-accum variants are
    generated natively (dpro_graph_layered_variant), replayed in ONE batch
    and their peaks computed by ONE K5 launch from natively resolved
    inputs. Returns (strategy or None, NativeGraph, max peak, makespan) with
    memory_pass's choice and BudgetError; usable at config-4/5 scale."""
    from .engine import default_engine
    from .ingest import layered_graph_variant
    from .memory import batch_peak_memory, native_inputs
    eng = engine or default_engine()
    names = ["none", "recompute", "grad-accum"]

    def gen(v):  # the native generator releases the GIL: build all three at once
        try:
            return layered_graph_variant(model, cluster, v, meta.microbatch_scale, part_k)
        except Error:
            return None  # the rewrite does not apply (e.g. one layer)

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(3) as ex:
        graphs = list(ex.map(gen, names))
    live = [g for g in graphs if g is not None]
    b = eng.batch([g.csr for g in live])
    b.replay(want_schedule=True)
    ms, st, *_ = b.results()
    if np.any(st != 0):
        raise Error(f"replay failed: statuses {st.tolist()}")
    parts = [native_inputs(g, meta) for g in live]
    peak = batch_peak_memory(b, np.concatenate([p[1] for p in parts]),
                             np.concatenate([p[2] for p in parts]),
                             np.array([len(p[0]) for p in parts], np.int32),
                             np.concatenate([p[3] for p in parts]))
    maxes, o = [], 0
    for p in parts:
        maxes.append(int(peak[o:o + len(p[0])].max()) if len(p[0]) else 0)
        o += len(p[0])
    res = {}
    k = 0
    for v, g in zip(names, graphs):
        if g is not None:
            res[v] = (g, maxes[k], int(ms[k]))
            k += 1
    base_g, base_peak, base_t = res["none"]
    if budget_bytes <= 0 or base_peak <= budget_bytes:
        return None, base_g, base_peak, base_t
    best = None
    for v in names[1:]:
        if v in res and res[v][1] <= budget_bytes and (best is None or res[v][2] < res[best][2]):
            best = v
    if best is None:
        reached = min([base_peak] + [res[v][1] for v in names[1:] if v in res])
        raise BudgetError(f"peak memory {base_peak} bytes exceeds budget {budget_bytes} "
                          "bytes and no rewrite closes the gap", reached)
    kind = StrategyKind.RECOMPUTE if best == "recompute" else StrategyKind.GRAD_ACCUM
    k = int(math.ceil(math.sqrt(model.layers))) if best == "recompute" else 2
    g, pk, t = res[best]
    return Strategy(kind, "", "", k, -1), g, pk, t
