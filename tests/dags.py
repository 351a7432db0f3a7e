"""Random-graph families for parity tests (test infrastructure).

* `random_dag_ref`   -- proj/tests/test_replay.cpp:214-238 (2-12 ops, 1-3
  devices, durations 1..6, edge p=0.22, shuffled wiring).
* `acceptance_dag`   -- proj/tests/acceptance_main.cpp:293-320 (durations
  1..50, edge p=0.3, ids "<node>->opNN").
* `fuzz_dag`         -- beyond the reference's oracles: zero
  durations, virtual ops (each with >= 1 predecessor), link devices,
  shuffled multi-digit names (w10 < w2 byte order), wider graphs.
numpy RNGs replace std::mt19937, so the draws differ from the reference's
sequences; the families (shape, sizes, distributions) are the same.
"""
from __future__ import annotations

import numpy as np

from paper_2205_02473_b200.graph import DeviceId, GraphBuilder, Op, OpKind, comp


def random_dag_ref(rng: np.random.Generator):
    n = int(rng.integers(2, 13))
    devs = int(rng.integers(1, 4))
    b = GraphBuilder()
    names = []
    for i in range(n):
        name = chr(ord("a") + i)
        dev = chr(ord("A") + int(rng.integers(0, devs)))
        names.append(name)
        b.add_op(comp(name, dev, int(rng.integers(1, 7))))
    rng.shuffle(names)
    for i in range(n):
        for j in range(i + 1, n):
            if rng.random() < 0.22:
                b.add_edge(names[i], names[j])
    return b.build()


def acceptance_dag(rng: np.random.Generator):
    n = int(rng.integers(2, 13))
    devices = int(rng.integers(1, 4))
    b = GraphBuilder()
    ids = []
    for i in range(n):
        node = f"n{int(rng.integers(0, devices))}"
        name = f"{node}->op{i:02d}"
        ids.append(name)
        b.add_op(comp(name, node, int(rng.integers(1, 51))))
    for i in range(n):
        for j in range(i + 1, n):
            if rng.random() < 0.3:
                b.add_edge(ids[i], ids[j])
    return b.build()


def fuzz_dag(rng: np.random.Generator, max_ops: int = 40, zero_p: float = 0.3,
             virt_p: float = 0.15, edge_p: float | None = None, max_dur: int = 9):
    n = int(rng.integers(2, max_ops + 1))
    nodes = [f"w{i}" for i in range(int(rng.integers(1, 13)))]
    b = GraphBuilder()
    names = []
    ep = edge_p if edge_p is not None else float(rng.uniform(0.05, 0.35))
    order = rng.permutation(n)  # wiring order independent of names
    kinds = {}
    for i in range(n):
        name = f"op{int(rng.integers(0, 10**6))}_{i}"
        names.append(name)
    for pos, i in enumerate(order):
        name = names[i]
        # an op may be virtual only if it can get a predecessor
        virtual = pos > 0 and rng.random() < virt_p
        if virtual:
            node = nodes[int(rng.integers(0, len(nodes)))]
            kind = OpKind.VIRTUAL_IN if rng.random() < 0.5 else OpKind.VIRTUAL_OUT
            b.add_op(Op(id=name, kind=kind, node=node, device=DeviceId.compute(node), dur=0))
        else:
            src = nodes[int(rng.integers(0, len(nodes)))]
            if rng.random() < 0.4 and len(nodes) > 1:
                dst = nodes[int(rng.integers(0, len(nodes)))]
                while dst == src:
                    dst = nodes[int(rng.integers(0, len(nodes)))]
                dev = DeviceId.link(src, dst)
                kind = OpKind.RECV if rng.random() < 0.5 else OpKind.SEND
            else:
                dev = DeviceId.compute(src)
                kind = OpKind.FW
            dur = 0 if rng.random() < zero_p else int(rng.integers(1, max_dur + 1))
            b.add_op(Op(id=name, kind=kind, node=src, device=dev, dur=dur))
        kinds[name] = virtual
    for a in range(n):
        for c in range(a + 1, n):
            if rng.random() < ep:
                b.add_edge(names[order[a]], names[order[c]])
    # every virtual op gets >= 1 predecessor (else the init quirk may fire)
    for pos in range(1, n):
        nm = names[order[pos]]
        if kinds[nm] and not any(b.has_edge(names[order[a]], nm) for a in range(pos)):
            b.add_edge(names[order[int(rng.integers(0, pos))]], nm)
    return b.build()


def memory_dag(rng: np.random.Generator, max_ops: int = 30):
    """Graphs + ModelMeta json for estimate_peak_memory (memory.cpp:122-167):
    FW/BW/UPDATE ops named like the reference's ingest ("<node>->FW.t3",
    "@mb1" micro-batch copies, "RFW." recomputation, '+'-fused locals),
    communication and virtual ops in between, zero durations, and metas
    that sometimes miss an entry (MissingMetaError / UPDATE -> 0)."""
    n = int(rng.integers(2, max_ops + 1))
    nodes = [f"w{i}" for i in range(int(rng.integers(1, 5)))]
    b = GraphBuilder()
    ids, locals_ = [], set()
    for i in range(n):
        node = nodes[int(rng.integers(0, len(nodes)))]
        r = rng.random()
        if r < 0.12 and i > 0:
            kind = OpKind.VIRTUAL_IN
            oid, dev, dur = f"{node}->VIN.v{i}", DeviceId.compute(node), 0
        elif r < 0.24 and len(nodes) > 1:
            peer = nodes[(nodes.index(node) + 1) % len(nodes)]
            kind = OpKind.SEND if rng.random() < 0.5 else OpKind.RECV
            oid, dev = f"{node}->{kind.name}.t{i}", DeviceId.link(node, peer)
            dur = int(rng.integers(0, 10))
        else:
            kind = [OpKind.FW, OpKind.BW, OpKind.UPDATE][int(rng.choice(3, p=[0.45, 0.4, 0.15]))]
            tag = {OpKind.FW: "FW", OpKind.BW: "BW", OpKind.UPDATE: "UPDATE"}[kind]
            form = rng.random()
            if form < 0.15:
                local = f"{tag}.t{i}@mb{int(rng.integers(0, 2))}"
                locals_.add(f"{tag}.t{i}")
            elif form < 0.25 and kind == OpKind.FW:
                local = f"RFW.t{i}"
                locals_.add(f"FW.t{i}")
            elif form < 0.4:
                local = f"{tag}.t{i}+{tag}.u{i}"
                locals_.update({f"{tag}.t{i}", f"{tag}.u{i}"})
            else:
                local = f"{tag}.t{i}"
                locals_.add(local)
            oid, dev = f"{node}->{local}", DeviceId.compute(node)
            dur = 0 if rng.random() < 0.2 else int(rng.integers(1, 10))
        ids.append(oid)
        b.add_op(Op(id=oid, kind=kind, node=node, device=dev, dur=dur))
    order = rng.permutation(n)
    ep = float(rng.uniform(0.08, 0.4))
    for a in range(n):
        for c in range(a + 1, n):
            if rng.random() < ep:
                b.add_edge(ids[order[a]], ids[order[c]])
    for pos in range(1, n):  # virtual ops get a predecessor (init quirk)
        nm = ids[order[pos]]
        if "->VIN." in nm and not any(b.has_edge(ids[order[a]], nm) for a in range(pos)):
            b.add_edge(ids[order[int(rng.integers(0, pos))]], nm)
    miss = rng.random() < 0.15
    out = {}
    for loc in sorted(locals_):
        if miss and rng.random() < 0.2:
            continue
        out[loc] = int(rng.integers(0, 1000)) if rng.random() < 0.9 else 0
    for oid in ids:  # a few direct full-id entries win over locals
        if rng.random() < 0.1:
            out[oid] = int(rng.integers(0, 5000))
    pers = {nd: int(rng.integers(0, 10**6)) for nd in nodes
            if not (rng.random() < 0.05)}
    meta = {"output_bytes": out, "persistent_bytes": pers, "microbatch_scale": 0.5}
    return b.build(), meta


def rewrite_dag(rng: np.random.Generator):
    """Valid graphs for the memory rewrites (optimize.cpp:819-959): per node
    an FW chain, a mirrored BW chain, FW.l_i -> BW.l_i, UPDATE ops after
    their BW, plus random extra FW->BW / BW->UPDATE edges and cross-node
    edges; no comm or virtual ops (validate() would need tensor units)."""
    b = GraphBuilder()
    nodes = [f"w{i}" for i in range(int(rng.integers(1, 4)))]
    for nd in nodes:
        L = int(rng.integers(1, 11))
        for i in range(L):
            b.add_op(Op(f"{nd}->FW.l{i}", OpKind.FW, nd, DeviceId.compute(nd),
                        int(rng.integers(0, 50))))
            b.add_op(Op(f"{nd}->BW.l{i}", OpKind.BW, nd, DeviceId.compute(nd),
                        int(rng.integers(0, 80))))
            if rng.random() < 0.6:
                b.add_op(Op(f"{nd}->UPDATE.l{i}", OpKind.UPDATE, nd, DeviceId.compute(nd),
                            int(rng.integers(0, 9))))
                b.add_edge(f"{nd}->BW.l{i}", f"{nd}->UPDATE.l{i}")
        for i in range(L):
            if i > 0:
                b.add_edge(f"{nd}->FW.l{i - 1}", f"{nd}->FW.l{i}")
            if i + 1 < L:
                b.add_edge(f"{nd}->BW.l{i + 1}", f"{nd}->BW.l{i}")
            b.add_edge(f"{nd}->FW.l{i}", f"{nd}->BW.l{i}")
            for j in range(i + 1, L):  # skip connections used by later backward ops
                if rng.random() < 0.03:
                    b.add_edge(f"{nd}->FW.l{i}", f"{nd}->BW.l{j}")
        if len(nodes) > 1 and rng.random() < 0.5:  # a cross-node dependency
            other = nodes[(nodes.index(nd) + 1) % len(nodes)]
            if b.has_op(f"{other}->BW.l0") and not b.has_edge(f"{other}->BW.l0", f"{nd}->FW.l0"):
                b.add_edge(f"{nd}->FW.l0", f"{other}->BW.l0")
    return b.build()


def strategy_chain(rng: np.random.Generator, g, n: int = 6):
    """Random optimize.cpp strategies for a layered graph g: op fusion of
    computation pairs (valid chains, cross-device and cycle-closing pairs
    included), tensor fusion of two base tensors, partition with k in 1..4.
    Returned as (kind, a, b, k) tuples; errors are part of the test."""
    comp = [o.id for o in g.ops() if int(o.kind) in (0, 1, 2)]
    bases = sorted({u.base for u in g.tensor_units().values()})
    out = []
    for _ in range(n):
        r = rng.random()
        if r < 0.4 and comp:
            a = comp[int(rng.integers(0, len(comp)))]
            succ = [s for s in g.succs(a)] if g.has_op(a) else []
            if succ and rng.random() < 0.8:
                b = succ[int(rng.integers(0, len(succ)))]
            else:
                b = comp[int(rng.integers(0, len(comp)))]
            out.append((0, a, b, 1))
        elif r < 0.7 and len(bases) > 1:
            i, j = rng.choice(len(bases), 2, replace=False)
            out.append((1, bases[int(i)], bases[int(j)], 1))
        elif bases:
            out.append((2, bases[int(rng.integers(0, len(bases)))], "", int(rng.integers(1, 5))))
    return out
