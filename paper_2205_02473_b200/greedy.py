"""The reference's own search driver (proj/src/optimize.cpp:1196-1650,
Alg. 1: critical-path-guided greedy walk) with every replay, critical path
and t_sync evaluated on the GPU.

    SearchOptions             optimize.hpp:207-222
    reference_search(g, opt)  search(), optimize.cpp:1327-1650

    coarsen(g, cost)          optimize.cpp:580-684 (pre-fusion pass)
    detect_symmetry(g)        optimize.cpp:686-813
    symmetry replication      optimize.cpp:1070-1168, 1592-1621

The same options give the same strategies, in the same order, with the
same fused durations and the same before/after times as the reference
(tests/test_greedy.py): every decision depends only on bit-exact replays,
critical paths and t_sync values. Registered (non-builtin) passes are not
supported.
"""
from __future__ import annotations

import os
import time
from collections import deque
from dataclasses import dataclass, field

from .errors import Error
from .graph import GlobalDFG, OpKind, is_computation
from .memory import ModelMeta
from .replay import (critical_path, execution_graph, replay, replay_times,
                     sync_makespan_grid)
from .rewrite import (CostModel, Strategy, StrategyKind, apply_op_fusion, apply_strategy,
                      apply_tensor_fusion, apply_tensor_partition, fused_op_id, local_part,
                      memory_pass, topo_order)
from .search import opt_part_num, should_fuse_ops, should_fuse_tensors

# speculative gate batch width: starts at min, doubles while no candidate is
# accepted, up to max. An acceptance discards the rest of the batch, so a wide
# batch wastes candidate construction on walks that accept often. On the
# 16-worker x 24-layer ring graph (390 acceptances, tools/greedy_speed.py,
# B200) "1,1" ran 20.4 s, "1,16" 24.6 s, "4,64" 51.0 s: the default is
# sequential makespan-only gates. DPRO_SPEC="min,max".
_SPEC_MIN, _SPEC_MAX = (int(x) for x in os.environ.get("DPRO_SPEC", "1,1").split(","))


@dataclass
class SearchOptions:
    """optimize.hpp:207-222."""
    time_budget_s: float = 30.0
    memory_budget_bytes: int = 0
    kmax: int = 16
    use_coarsen: bool = True
    use_symmetry: bool = True
    use_partial_replay: bool = True
    use_theorems: bool = True
    passes: list[str] = field(default_factory=list)
    cost: CostModel = field(default_factory=CostModel)
    meta: ModelMeta = field(default_factory=ModelMeta)
    convergence_pct: float = 0.5
    convergence_rounds: int = 5


@dataclass
class SearchOutcome:
    graph: GlobalDFG
    strategies: list[Strategy]
    before_us: int
    after_us: int
    search_wall_s: float = 0.0


def _producers_of(g: GlobalDFG, base: str) -> dict[str, list[str]]:
    """optimize.cpp:1197-1207: node -> ops producing `base`."""
    out: dict[str, list[str]] = {}
    for op in g.ops():
        if not is_computation(op.kind):
            continue
        for t in op.produces:
            if t == base:
                out.setdefault(op.node, []).append(op.id)
    return dict(sorted(out.items()))


def _try_bundle(g: GlobalDFG, bundle: list[Strategy], opt: SearchOptions):
    """optimize.cpp:1211-1227 (fills fused durations into the bundle)."""
    cur = g
    for s in bundle:
        try:
            cur = apply_strategy(cur, s, opt.cost, opt.meta)
        except Error:
            return None
        if s.kind == StrategyKind.OP_FUSION and s.dur_us < 0:
            s.dur_us = cur.op(fused_op_id(s.a, s.b)).dur
    return cur


def _append_pairing(g: GlobalDFG, base_a: str, base_b: str, walked_node: str,
                    bundle: list[Strategy]) -> bool:
    """optimize.cpp:1229-1262."""
    pa_, pb_ = _producers_of(g, base_a), _producers_of(g, base_b)
    for node in sorted(set(pa_) | set(pb_)):
        if node == walked_node:
            continue
        if node not in pa_ or node not in pb_:
            return False
        if len(pa_[node]) != 1 or len(pb_[node]) != 1:
            return False
        a, b = pa_[node][0], pb_[node][0]
        if a == b:
            continue
        if g.op(a).device.str() != g.op(b).device.str():
            return False
        if g.has_edge(a, b):
            bundle.append(Strategy(StrategyKind.OP_FUSION, a, b, 1, -1))
        elif g.has_edge(b, a):
            bundle.append(Strategy(StrategyKind.OP_FUSION, b, a, 1, -1))
        else:
            return False
    return True


def _append_unpartitions(g: GlobalDFG, bases: list[str], bundle: list[Strategy]) -> None:
    """optimize.cpp:1264-1272."""
    for base in bases:
        if g.has_base(base) and len(g.units_of_base(base)) > 1:
            bundle.append(Strategy(StrategyKind.PARTITION, base, "", 1, -1))


def _op_bases(op) -> list[str]:
    out: list[str] = []
    for t in op.produces:
        if t not in out:
            out.append(t)
    return out


def _strategy_key(s: Strategy) -> str:
    return f"{s.kind}|{s.a}|{s.b}|{s.k}"


class _Ctx:
    """SearchCtx (optimize.cpp:1144-1168): memoized t_sync, time budget."""

    def __init__(self, opt: SearchOptions, cluster):
        self.opt, self.cluster = opt, cluster
        self.cache: dict[tuple[int, int], int] = {}
        self.started = time.monotonic()

    def elapsed(self) -> float:
        return time.monotonic() - self.started

    def out_of_time(self) -> bool:
        return self.elapsed() >= self.opt.time_budget_s

    def sync(self, nbytes: int, k: int) -> int:
        key = (int(nbytes), int(k))
        if key not in self.cache:
            # t_sync is a pure function of (bytes, k): a miss fills the
            # whole row k = 1..kmax (what opt_part_num asks next) in one
            # K2 grid launch instead of one launch per k
            ks = sorted({key[1]} | set(range(1, max(1, min(int(self.opt.kmax), key[0])) + 1)))
            ks = [x for x in ks if (key[0], x) not in self.cache]
            if key[1] < 1:
                ks = [key[1]]  # the reference's error, raised by the grid
            vals = sync_makespan_grid(self.cluster, [key[0]] * len(ks), ks)
            self.cache.update({(key[0], x): v for x, v in zip(ks, vals)})
        return self.cache[key]


def _finish_fusion_bundle(g: GlobalDFG, bundle: list[Strategy], bases: list[str], ctx: _Ctx):
    """optimize.cpp:1277-1314."""
    fused = bases[0]
    for b in bases[1:]:
        bundle.append(Strategy(StrategyKind.TENSOR_FUSION, fused, b, 1, -1))
        fused += "+" + b
    applied = _try_bundle(g, bundle, ctx.opt)
    if applied is None:
        return None
    if not applied.has_base(fused):
        return applied
    nbytes = applied.base_bytes(fused)
    best_k = 1
    if ctx.opt.use_partial_replay:
        best_k = opt_part_num(nbytes, ctx.opt.kmax, ctx.sync)
    else:
        cap = min(max(ctx.opt.kmax, 1), nbytes)
        best = replay(applied).iteration_time_us
        for k in range(2, cap + 1):
            t = replay(apply_tensor_partition(applied, fused, k)).iteration_time_us
            if t < best:
                best, best_k = t, k
    if best_k > 1:
        part = Strategy(StrategyKind.PARTITION, fused, "", best_k, -1)
        try:
            applied = apply_strategy(applied, part, ctx.opt.cost, ctx.opt.meta)
        except Error:
            return None
        bundle.append(part)
    return applied


def coarsen(g: GlobalDFG, cost: CostModel):
    """optimize.cpp:580-662: (graph, applied strategies) of the backtracking
    pre-fusion pass (the view's group tables are not needed by search)."""
    graph, applied = g, []
    merges = []
    order = topo_order(g)
    if order is not None:
        for idx in reversed(order):
            u = g.op_at(idx)
            if not is_computation(u.kind) or u.kind == OpKind.UPDATE or u.produces:
                continue
            comp = [x for x in g.succs(u.id) if is_computation(g.op(x).kind)]
            if len(comp) != 1:
                continue
            v = g.op(comp[0])
            if v.kind == OpKind.UPDATE or u.device.str() != v.device.str():
                continue
            merges.append((u.id, v.id))
    moved: dict[str, str] = {}
    for uid, vid in merges:
        cu, cv = moved.get(uid, uid), moved.get(vid, vid)
        if cu == cv:
            continue
        try:
            nxt = apply_op_fusion(graph, cu, cv, cost)
        except Error:
            continue
        fid = fused_op_id(cu, cv)
        applied.append(Strategy(StrategyKind.OP_FUSION, cu, cv, 1, nxt.op(fid).dur))
        for k, v in list(moved.items()):
            if v in (cu, cv):
                moved[k] = fid
        moved[uid] = moved[vid] = fid
        graph = nxt
    refused: set[tuple[str, str]] = set()
    changed = True
    while changed:  # fold multiple tensors of one producer into one unit
        changed = False
        for op in graph.ops():
            if not is_computation(op.kind) or len(op.produces) < 2:
                continue
            t1, t2 = op.produces[0], op.produces[1]
            if (t1, t2) in refused:
                continue
            try:
                nxt = apply_tensor_fusion(graph, t1, t2)
            except Error:
                refused.add((t1, t2))
                continue
            applied.append(Strategy(StrategyKind.TENSOR_FUSION, t1, t2, 1, -1))
            graph = nxt
            changed = True
            break
    return graph, applied


def _sig(g: GlobalDFG, op):
    sizes = sorted(g.base_bytes(b) if g.has_base(b) else 0 for b in op.produces)
    return (int(op.kind), int(op.dur), sizes)


def _sig_match(a, b) -> bool:
    if a[0] != b[0] or a[2] != b[2]:
        return False
    return abs(float(a[1] - b[1])) <= 0.01 * float(max(a[1], b[1])) + 1e-9


def _produced_bases(g: GlobalDFG, ops) -> list[str]:
    out: list[str] = []
    for oid in ops:
        for b in g.op(oid).produces:
            if b not in out:
                out.append(b)
    return out


def detect_symmetry(g: GlobalDFG) -> list[list[tuple[list[str], list[str]]]]:
    """optimize.cpp:715-813: groups of segments (ops, tensors)."""
    out = []
    order = topo_order(g)
    if order is None:
        return out
    chains: dict[str, list[str]] = {}
    for idx in order:
        op = g.op_at(idx)
        if is_computation(op.kind):
            chains.setdefault(op.node, []).append(op.id)
    chains = dict(sorted(chains.items()))
    sigs, sorted_ops = {}, {}
    for node, ids in chains.items():  # worker replicas
        by_local = sorted(ids, key=local_part)
        sorted_ops[node] = by_local
        sigs[node] = [_sig(g, g.op(i)) for i in by_local]
    node_groups: list[list[str]] = []
    for node, sig in sigs.items():
        for grp in node_groups:
            ref = sigs[grp[0]]
            if len(ref) == len(sig) and all(_sig_match(x, y) for x, y in zip(ref, sig)):
                grp.append(node)
                break
        else:
            node_groups.append([node])
    for grp in node_groups:
        if len(grp) >= 2:
            out.append([(sorted_ops[nd], _produced_bases(g, sorted_ops[nd])) for nd in grp])
    if chains:  # periodic blocks tiling the first worker's chain
        ids = next(iter(chains.values()))
        n = len(ids)
        items = [_sig(g, g.op(i)) for i in ids]
        for w in range(1, n // 2 + 1):
            if n % w:
                continue
            if all(_sig_match(items[j], items[b * w + j])
                   for b in range(1, n // w) for j in range(w)):
                out.append([(ids[b * w:(b + 1) * w], _produced_bases(g, ids[b * w:(b + 1) * w]))
                            for b in range(n // w)])
                break
    return out


def _symmetry_maps(groups):
    """optimize.cpp:1080-1105: (op map, tensor map) per ordered segment pair."""
    maps = []
    for segs in groups:
        for i, (fo, ft) in enumerate(segs):
            for j, (to, tt) in enumerate(segs):
                if i == j or len(fo) != len(to) or len(ft) != len(tt):
                    continue
                maps.append((dict(zip(fo, to)), dict(zip(ft, tt))))
    return maps


def _node_part(oid: str) -> str:
    a = oid.find("->")
    return "" if a < 0 else oid[:a]


def _map_op_id(oid: str, m):
    """optimize.cpp:1107-1126."""
    node = _node_part(oid)
    if not node:
        return None
    locals_, mapped_node = [], ""
    for piece in local_part(oid).split("+"):
        full = node + "->" + piece
        target = m[0].get(full, full)
        tnode = _node_part(target)
        if not mapped_node:
            mapped_node = tnode
        elif mapped_node != tnode:
            return None
        locals_.append(local_part(target))
    return mapped_node + "->" + "+".join(locals_)


def _map_tensor(name: str, m) -> str:
    return "+".join(m[1].get(p, p) for p in name.split("+"))


def _map_strategy(s: Strategy, m):
    """optimize.cpp:1136-1158."""
    if s.kind == StrategyKind.OP_FUSION:
        a, b = _map_op_id(s.a, m), _map_op_id(s.b, m)
        if a is None or b is None:
            return None
        return Strategy(s.kind, a, b, s.k, -1)
    if s.kind == StrategyKind.TENSOR_FUSION:
        return Strategy(s.kind, _map_tensor(s.a, m), _map_tensor(s.b, m), s.k, s.dur_us)
    if s.kind == StrategyKind.PARTITION:
        return Strategy(s.kind, _map_tensor(s.a, m), s.b, s.k, s.dur_us)
    return None


def reference_search(g: GlobalDFG, opt: SearchOptions | None = None) -> SearchOutcome:
    """search() of optimize.cpp:1327-1650 with use_coarsen = use_symmetry =
    False."""
    opt = opt or SearchOptions()
    builtin = ["op-fusion", "tensor-fusion", "partition", "memory"]
    for name in opt.passes:
        if name not in builtin:
            raise Error(f"unknown pass: {name}")

    def enabled(name: str) -> bool:
        return not opt.passes or name in opt.passes

    before = replay(g).iteration_time_us
    out = SearchOutcome(g, [], before, before)
    if opt.time_budget_s <= 0:
        return out
    ctx = _Ctx(opt, g.cluster())
    graph = g
    strategies: list[Strategy] = []
    if opt.memory_budget_bytes > 0 and enabled("memory"):
        graph = memory_pass(graph, opt.memory_budget_bytes, opt.meta, strategies)
    current = replay(graph).iteration_time_us
    if opt.use_coarsen and opt.memory_budget_bytes == 0 and enabled("op-fusion") and \
            enabled("tensor-fusion"):
        cg, applied = coarsen(graph, opt.cost)
        if applied:
            t = replay(cg).iteration_time_us
            if t <= current:
                graph, current = cg, t
                strategies.extend(applied)
    sym_maps = _symmetry_maps(detect_symmetry(graph)) if opt.use_symmetry else []
    seen: set[str] = set()

    def gate(bundle, applied) -> bool:
        nonlocal graph, current
        if applied is None:
            return False
        t = replay(applied).iteration_time_us
        if t >= current:
            return False
        graph, current = applied, t
        strategies.extend(bundle)
        seen.add(";".join(_strategy_key(s) for s in bundle) + ";")
        return True

    previous, flat, timed_out = current, 0, False
    while not timed_out:
        round_g = graph
        round_res = replay(round_g)
        path = critical_path(execution_graph(round_g, round_res), round_res)
        accepted = 0
        replication_queue: list[list[Strategy]] = []

        def accept(bundle, applied, t) -> None:
            nonlocal graph, current, accepted
            graph, current = applied, t
            strategies.extend(bundle)
            seen.add(";".join(_strategy_key(s) for s in bundle) + ";")
            accepted += 1
            replication_queue.append([Strategy(x.kind, x.a, x.b, x.k, x.dur_us)
                                      for x in bundle])

        def walk(items, make) -> bool:
            """The sequential loop `for it in items: if out_of_time: break;
            attempt(*make(it))`, with speculative batched gates: candidates
            are built against the current graph and replayed in one GPU
            launch, then gated in order. A rejection leaves the graph as it
            was, so the candidates after it are still the ones the sequential
            loop would build; after an acceptance they are discarded and the
            walk resumes from the next item on the new graph. Same decisions,
            same order; only the number of launches changes. Returns
            timed_out."""
            i, width = 0, _SPEC_MIN
            while i < len(items):
                pend, j, out = [], i, False
                while j < len(items) and len(pend) < width:
                    if ctx.out_of_time():
                        out = True
                        break
                    r = make(items[j])
                    if r is not None and r[1] is not None:
                        pend.append((j, r[0], r[1]))
                    j += 1
                try:
                    times = replay_times([c[2] for c in pend])
                except Error:  # re-run one by one: errors surface in order
                    times = [None] * len(pend)
                hit = None
                for (idx, bundle, applied), t in zip(pend, times):
                    if t is None:  # raises the reference's replay error, in order
                        t = replay(applied).iteration_time_us
                    if t < current:
                        accept(bundle, applied, t)
                        hit = idx
                        break
                if hit is None:
                    if out:
                        return True
                    i, width = j, min(2 * width, _SPEC_MAX)
                else:
                    i, width = hit + 1, _SPEC_MIN
            return False

        def make_opf(item):  # one step of optimize.cpp:1410-1466
            a, b = item
            if not graph.has_op(a) or not graph.has_op(b):
                return None
            pa, pb = graph.op(a), graph.op(b)
            if not is_computation(pa.kind) or not is_computation(pb.kind):
                return None
            if OpKind.UPDATE in (pa.kind, pb.kind):
                return None
            if pa.device.str() != pb.device.str() or not graph.has_edge(a, b):
                return None
            if opt.use_theorems:
                q_prev = 0
                if pa.produces:
                    base = pa.produces[0]
                    if not graph.has_base(base):
                        return None
                    q_prev = ctx.sync(graph.base_bytes(base), len(graph.units_of_base(base)))
                if not should_fuse_ops(pa.dur, pb.dur, opt.cost.fused_dur_us(pa, pb), q_prev):
                    return None
            bases = _op_bases(pa)
            for base in _op_bases(pb):
                if base not in bases:
                    bases.append(base)
            bundle: list[Strategy] = []
            _append_unpartitions(graph, bases, bundle)
            bundle.append(Strategy(StrategyKind.OP_FUSION, a, b, 1, -1))
            if pa.produces and pb.produces:
                if not enabled("tensor-fusion"):
                    return None
                if not _append_pairing(graph, pa.produces[0], pb.produces[0], pa.node, bundle):
                    return None
            if len(bases) >= 2:
                return bundle, _finish_fusion_bundle(graph, bundle, bases, ctx)
            return bundle, _try_bundle(graph, bundle, opt)

        if enabled("op-fusion"):  # computation runs, optimize.cpp:1410-1466
            items = [(run.ops[i], run.ops[i + 1]) for run in path.runs
                     if not run.communication for i in range(len(run.ops) - 1)]
            timed_out = walk(items, make_opf)

        def run_bases(runs):
            order = []
            for run in runs:
                for oid in run.ops:
                    op = round_g.op(oid)
                    if not op.tensor or not round_g.has_tensor_unit(op.tensor):
                        continue
                    base = round_g.tensor_unit(op.tensor).base
                    if base not in order:
                        order.append(base)
            return order

        def make_tf(item):  # one step of optimize.cpp:1468-1521
            u, v = item
            if not graph.has_base(u) or not graph.has_base(v):
                return None
            if opt.use_theorems:
                q_prev_end = 0
                for name in round_g.units_of_base(u):
                    for cid in round_g.tensor_unit(name).comm_ops:
                        q_prev_end = max(q_prev_end, round_res.schedule[cid].end)
                p_cur_end = 0
                for ids in _producers_of(round_g, v).values():
                    for oid in ids:
                        p_cur_end = max(p_cur_end, round_res.schedule[oid].end)
                if not should_fuse_tensors(q_prev_end, p_cur_end, round_g.base_bytes(u),
                                           round_g.base_bytes(v), opt.kmax, ctx.sync):
                    return None
            bundle = []
            _append_unpartitions(graph, [u, v], bundle)
            pairing: list[Strategy] = []
            if not _append_pairing(graph, u, v, "", pairing):
                return None
            if pairing and not enabled("op-fusion"):
                return None
            bundle += pairing
            return bundle, _finish_fusion_bundle(graph, bundle, [u, v], ctx)

        if enabled("tensor-fusion") and not timed_out:  # optimize.cpp:1468-1521
            items = []
            for run in path.runs:
                if run.communication:
                    order = run_bases([run])
                    items += [(order[i], order[i + 1]) for i in range(len(order) - 1)]
            timed_out = walk(items, make_tf)

        def make_part(base):  # one step of optimize.cpp:1523-1561
            if not graph.has_base(base):
                return None
            nbytes = graph.base_bytes(base)
            k_cur = len(graph.units_of_base(base))
            k_best = k_cur
            if opt.use_partial_replay:
                k_best = opt_part_num(nbytes, opt.kmax, ctx.sync)
            else:  # every k of the sweep in one batched launch
                cap = min(max(opt.kmax, 1), nbytes)
                ks = [k for k in range(1, cap + 1) if k != k_cur]
                gs = [apply_tensor_partition(graph, base, k) for k in ks]
                best = current
                for k, gk, t in zip(ks, gs, replay_times(gs)):
                    if t is None:
                        t = replay(gk).iteration_time_us
                    if t < best:
                        best, k_best = t, k
            if k_best == k_cur:
                return None
            bundle = [Strategy(StrategyKind.PARTITION, base, "", k_best, -1)]
            return bundle, _try_bundle(graph, bundle, opt)

        if enabled("partition") and not timed_out:  # optimize.cpp:1523-1561
            timed_out = walk(run_bases([r for r in path.runs if r.communication]), make_part)

        if sym_maps:  # replicate accepted bundles onto symmetric ops / tensors
            queue = deque(replication_queue)
            while queue and not timed_out:
                bundle = queue.popleft()
                for m in sym_maps:
                    timed_out = ctx.out_of_time()
                    if timed_out:
                        break
                    mapped = [_map_strategy(x, m) for x in bundle]
                    if any(x is None for x in mapped):
                        continue
                    key = ";".join(_strategy_key(x) for x in mapped) + ";"
                    if key in seen:
                        continue
                    seen.add(key)
                    applied = _try_bundle(graph, mapped, opt)
                    if gate(mapped, applied):
                        accepted += 1
                        queue.append(mapped)

        if accepted == 0:
            break
        change = 100.0 * (previous - current) / previous if previous > 0 else 0.0
        flat = flat + 1 if change < opt.convergence_pct else 0
        previous = current
        if flat >= opt.convergence_rounds:
            break
    return SearchOutcome(graph, strategies, before, current, ctx.elapsed())
