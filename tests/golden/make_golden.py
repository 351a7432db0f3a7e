"""Generates the golden vectors in tests/golden/ by running the UNMODIFIED
reference (oracle/_ref/libdpro_ref.so, built from /root/reference/proj/src by
oracle/Makefile). Run here, where /root/reference exists:

    python tests/golden/make_golden.py

The JSON files are committed; the GPU box (no /root/reference) only reads
them. Every vector records the reference's outputs: iteration time, per-op
start/end, timeline positions, critical path (op indices, runs, conforming)
or the raised error (status, message, cycle ids).
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from dags import (acceptance_dag, fuzz_dag, memory_dag, random_dag_ref, rewrite_dag,
                  strategy_chain)  # noqa: E402
from golden_io import rows_digest  # noqa: E402
from oracle.oracle import RefError, RefGraph, ref_sync_makespan  # noqa: E402
from paper_2205_02473_b200.graph import (DeviceId, GraphBuilder, Op, OpKind, comp,  # noqa: E402
                                         synth_cluster)

OUT = Path(__file__).resolve().parent


def g_to_json(g):
    return {"ops": [[o.id, int(o.kind), int(o.device.kind), o.device.node, o.device.peer,
                     int(o.dur)] for o in g.ops()],
            "edges": [[g.op_at(i).id, g.op_at(s).id] for i in range(g.size())
                      for s in g.succ_indices(i)]}


def expect(rg: RefGraph) -> dict:
    try:
        T, s, e, tl, util = rg.replay()
    except RefError as err:
        return {"status": err.status, "message": err.msg, "cycle": err.cycle}
    cp = rg.critical_path()
    return {"status": 0, "T": T, "start": s.tolist(), "end": e.tolist(), "tl_pos": tl.tolist(),
            "util": [float(u) for u in util], "path": cp["path"].tolist(),
            "runs": cp["runs"], "conforming": cp["conforming"],
            "exec_edges": rg.exec_edge_count()}


def named_cases():
    cases = {}
    b = GraphBuilder()  # test_replay.cpp:251-261
    b.add_op(comp("x", "A", 10)); b.add_op(comp("y", "B", 5)); b.add_edge("x", "y")
    cases["chain_15"] = b.build()
    b = GraphBuilder()  # 263-272
    b.add_op(comp("p", "A", 10)); b.add_op(comp("q", "A", 5))
    cases["serialize_15"] = b.build()
    b = GraphBuilder()  # 274-304
    for n, d, t in [("a", "d1", 2), ("b", "d1", 3), ("c", "d2", 5), ("d", "d1", 1)]:
        b.add_op(comp(n, d, t))
    for x, y in [("a", "b"), ("a", "c"), ("c", "d")]:
        b.add_edge(x, y)
    cases["diamond_8"] = b.build()
    b = GraphBuilder()  # 306-322
    for n, t in [("x", 1), ("y", 2), ("z", 3)]:
        b.add_op(comp(n, "A", t))
    cases["serial_edges"] = b.build()
    b = GraphBuilder()  # 324-339
    b.add_op(comp("a", "A", 1)); b.add_op(comp("b", "B", 2)); b.add_op(comp("c", "A", 3))
    b.add_edge("a", "b"); b.add_edge("b", "c")
    cases["chain_path"] = b.build()
    b = GraphBuilder()  # 341-355
    for n, d, t in [("a", "A", 2), ("b", "B", 4), ("c", "C", 4), ("d", "A", 1)]:
        b.add_op(comp(n, d, t))
    for x, y in [("a", "b"), ("a", "c"), ("b", "d"), ("c", "d")]:
        b.add_edge(x, y)
    cases["equal_branches"] = b.build()
    b = GraphBuilder()  # 357-370
    for n, d, t in [("m", "D", 10), ("pa", "E", 2), ("pb", "F", 4), ("z", "D", 3), ("a", "D", 3)]:
        b.add_op(comp(n, d, t))
    b.add_edge("pa", "z"); b.add_edge("pb", "a")
    cases["earlier_ready"] = b.build()
    b = GraphBuilder()  # 372-393
    b.add_op(comp("a", "w0", 5))
    b.add_op(Op("v", OpKind.VIRTUAL_IN, "w0", DeviceId.compute("w0"), 0))
    b.add_op(comp("b", "w0", 3))
    b.add_edge("a", "v"); b.add_edge("v", "b")
    cases["virtual_no_device"] = b.build()
    b = GraphBuilder()  # 395-406
    b.add_op(comp("a", "A", 1)); b.add_op(comp("b", "A", 1))
    b.add_edge("a", "b"); b.add_edge("b", "a")
    cases["cycle"] = b.build()
    b = GraphBuilder()
    b.add_op(comp("a", "A", -1))
    cases["missing_duration"] = b.build()
    b = GraphBuilder()
    b.add_op(comp("a", "A", 3)); b.add_op(comp("b", "A", -1)); b.add_op(comp("c", "B", -5))
    b.add_op(Op("v", OpKind.VIRTUAL_OUT, "A", DeviceId.compute("A"), -3))
    cases["missing_first_index"] = b.build()
    b = GraphBuilder()
    for n, d, t in [("a", "A", 1), ("b", "A", 1), ("c", "B", 2), ("d", "B", 1)]:
        b.add_op(comp(n, d, t))
    b.add_edge("a", "b"); b.add_edge("c", "d"); b.add_edge("d", "c")
    cases["partial_cycle"] = b.build()
    # SURVEY Appendix A vectors
    b = GraphBuilder()  # Z1
    for n, t in [("a", 0), ("b", 3), ("c", 5)]:
        b.add_op(comp(n, "D", t))
    b.add_edge("a", "b")
    cases["Z1_zero_round"] = b.build()
    b = GraphBuilder()  # Z2
    lk = DeviceId.link("w0", "w1")
    for n, t, k in [("SEND.x1", 0, OpKind.SEND), ("SEND.x2", 0, OpKind.SEND),
                    ("RECV.x1", 10, OpKind.RECV), ("RECV.x2", 10, OpKind.RECV)]:
        b.add_op(Op(n, k, "w0", lk, t))
    b.add_edge("SEND.x1", "RECV.x1"); b.add_edge("SEND.x2", "RECV.x2")
    cases["Z2_link_queue"] = b.build()
    b = GraphBuilder()  # Z3
    b.add_op(comp("p", "A", 4))
    b.add_op(Op("v", OpKind.VIRTUAL_IN, "A", DeviceId.compute("A"), 0))
    b.add_op(comp("q", "B", 0)); b.add_op(comp("s", "B", 1)); b.add_op(comp("r", "B", 2))
    for x, y in [("p", "v"), ("v", "q"), ("v", "s"), ("q", "r")]:
        b.add_edge(x, y)
    cases["Z3_virtual_zero"] = b.build()
    b = GraphBuilder()  # Z4
    b.add_op(comp("pre", "F", 10)); b.add_op(comp("z0", "E", 0)); b.add_op(comp("y", "D", 1))
    b.add_op(comp("x", "D", 1)); b.add_op(comp("m", "D", 10))
    for x, y in [("pre", "z0"), ("pre", "y"), ("z0", "x")]:
        b.add_edge(x, y)
    cases["Z4_cross_round_tie"] = b.build()
    # init quirk: virtual a -> virtual b, a < b
    vin = lambda n: Op(n, OpKind.VIRTUAL_IN, "A", DeviceId.compute("A"), 0)
    b = GraphBuilder()
    b.add_op(vin("a")); b.add_op(vin("b")); b.add_edge("a", "b")
    cases["quirk_vv_throws"] = b.build()
    b = GraphBuilder()
    b.add_op(vin("b")); b.add_op(vin("a")); b.add_edge("b", "a")
    cases["quirk_vv_reversed"] = b.build()
    b = GraphBuilder()
    b.add_op(vin("a")); b.add_op(vin("b")); b.add_op(comp("x", "A", 3))
    b.add_op(vin("c")); b.add_op(vin("d"))
    for x, y in [("a", "b"), ("b", "x"), ("d", "c"), ("c", "x")]:
        b.add_edge(x, y)
    cases["quirk_chain_throws"] = b.build()
    b = GraphBuilder()  # double cascade readies s early, then another op stays stuck
    b.add_op(vin("a")); b.add_op(vin("b")); b.add_op(comp("s", "A", 2)); b.add_op(comp("x", "B", 5))
    b.add_op(comp("y", "C", 1))
    for x, y in [("a", "b"), ("b", "s"), ("x", "s"), ("b", "y"), ("y", "x"), ("x", "y")]:
        b.add_edge(x, y)
    cases["quirk_wrap"] = b.build()
    b = GraphBuilder()
    b.add_op(vin("a")); b.add_op(vin("b")); b.add_op(comp("s", "A", 2)); b.add_op(comp("x", "B", 5))
    for x, y in [("a", "b"), ("b", "s"), ("x", "s")]:
        b.add_edge(x, y)
    cases["quirk_premature"] = b.build()
    b = GraphBuilder()  # two double cascades cancel two stuck ops: "success"
    for n in "abcd":
        b.add_op(vin(n))
    b.add_op(comp("x", "A", 1)); b.add_op(comp("y", "A", 1))
    for x, y in [("a", "b"), ("c", "d"), ("x", "y"), ("y", "x")]:
        b.add_edge(x, y)
    cases["quirk_wrap_zero"] = b.build()
    b = GraphBuilder()
    cases["empty"] = b.build()
    return cases


def main():
    rng = np.random.default_rng(20260815)
    vectors = []
    for name, g in named_cases().items():
        vectors.append({"name": name, "graph": g_to_json(g), "expect": expect(RefGraph.from_dfg(g))})
    fam = [("random_dag_ref", random_dag_ref, 150), ("acceptance_dag", acceptance_dag, 100),
           ("fuzz_dag", fuzz_dag, 250)]
    for fname, fn, count in fam:
        for t in range(count):
            g = fn(rng)
            vectors.append({"name": f"{fname}_{t}", "graph": g_to_json(g),
                            "expect": expect(RefGraph.from_dfg(g))})
    (OUT / "replay_vectors.json").write_text(json.dumps(vectors, separators=(",", ":")))

    # t_sync: test_optimize.cpp:265-291, plus a ring/PS grid
    tsync = []
    clusters = {
        "ps_1x1_bw1": synth_cluster("ps", 1, 1, 1.0, 0.0),
        "ps_1x1_lat50": synth_cluster("ps", 1, 1, 1.0, 50.0),
        "ring12_bw1": synth_cluster("ring", 12, 0, 1.0, 0.0),
        "ring8_100g": synth_cluster("ring", 8, 0, 12500.0, 5.0),
        "ps16x4_100g": synth_cluster("ps", 16, 4, 12500.0, 5.0),
        "ring3_bw7": synth_cluster("ring", 3, 0, 7.0, 1.5),
    }
    grid = {
        "ps_1x1_bw1": [(100, k) for k in (1, 2, 3, 4, 10, 11, 12, 16)],
        "ps_1x1_lat50": [(100, k) for k in (1, 2, 3, 4)],
        "ring12_bw1": [(1000, 1), (1000, 2), (1000, 11), (1000, 12), (7, 3)],
        "ring8_100g": [(b, k) for b in (4096, 1 << 20, 102_760_448) for k in (1, 2, 3, 8, 11, 16)],
        "ps16x4_100g": [(b, k) for b in (4096, 2_359_296) for k in (1, 2, 4, 11, 16)],
        "ring3_bw7": [(b, k) for b in (1, 2, 5, 1000) for k in (1, 2, 3)],
    }
    for cname, c in clusters.items():
        for bytes_, k in grid[cname]:
            tsync.append({"cluster": cname, "bytes": bytes_, "k": k,
                          "expect": ref_sync_makespan(c.to_json(), bytes_, k)})
    (OUT / "tsync_vectors.json").write_text(json.dumps(
        {"clusters": {k: [v.scheme, len(v.workers()), len(v.ps_nodes()),
                          v.links[0].bandwidth_bytes_per_us, v.links[0].latency_us]
                      for k, v in clusters.items()},
         "cases": tsync}, indent=0))

    # layered synthetic graphs (ingest-built) + partitions: T, schedule digest
    synth = []
    srng = np.random.default_rng(3)
    for scheme, W, S, L in [("ring", 4, 0, 6), ("ring", 11, 0, 4), ("ps", 3, 2, 6),
                            ("ps", 16, 4, 5), ("ring", 8, 0, 12)]:
        fw = srng.integers(10, 400, L).tolist()
        bw = srng.integers(10, 800, L).tolist()
        tb = srng.integers(1000, 4_000_000, L).tolist()
        spec = {"layers": L, "fw_dur_us": fw, "bw_dur_us": bw, "tensor_bytes": tb,
                "update_dur_us": 5, "scheme": scheme, "workers": W, "ps_count": S,
                "bandwidth_bytes_per_us": 12500.0, "latency_us": 5.0}
        for variant in range(2):
            k = [1] * L if variant == 0 else srng.choice([1, 2, 3, 4, 11], L).tolist()
            rg = RefGraph.synth(spec)
            for i, ki in enumerate(k):
                rg = rg.partition(f"g{i}", int(ki))
            T, s, e, tl, util = rg.replay()
            cp = rg.critical_path()
            digest = hashlib.sha256(np.concatenate([s, e]).astype("<i8").tobytes()).hexdigest()
            synth.append({"spec": spec, "part_k": [int(x) for x in k], "n_ops": rg.n_ops,
                          "n_edges": rg.n_edges, "T": T, "schedule_sha256": digest,
                          "path": cp["path"].tolist(), "conforming": cp["conforming"],
                          "ops_sha256": hashlib.sha256("\n".join(rg.op_ids()).encode()).hexdigest()})
    (OUT / "synth_vectors.json").write_text(json.dumps(synth, indent=0))
    print(f"{len(vectors)} replay vectors, {len(tsync)} t_sync vectors, {len(synth)} synth vectors")


def memory_cases():
    """proj/tests/test_memory.cpp cases (graph, meta)."""
    cases = {}
    b = GraphBuilder()  # test_memory.cpp:58-70
    b.add_op(comp("w0->FW.a", "w0", 10)); b.add_op(comp("w0->FW.b", "w0", 10))
    b.add_edge("w0->FW.a", "w0->FW.b")
    cases["chained"] = (b.build(), {"output_bytes": {"FW.a": 10, "FW.b": 10},
                                    "persistent_bytes": {"w0": 100}})
    b = GraphBuilder()  # 72-79
    b.add_op(comp("w0->UPDATE.a", "w0", 5, OpKind.UPDATE))
    cases["persistent_only"] = (b.build(), {"persistent_bytes": {"w0": 77}})
    b = GraphBuilder()  # 81-94
    for n, t in [("a", 4), ("b", 4), ("c", 2)]:
        b.add_op(comp(f"w0->FW.{n}", "w0", t))
    b.add_edge("w0->FW.a", "w0->FW.c"); b.add_edge("w0->FW.b", "w0->FW.c")
    cases["fan_in"] = (b.build(), {"output_bytes": {"FW.a": 10, "FW.b": 10, "FW.c": 0},
                                   "persistent_bytes": {"w0": 100}})
    b = GraphBuilder()  # 96-108
    b.add_op(comp("w0->FW.a", "w0", 4))
    g = b.build()
    cases["missing_sizes"] = (g, {"persistent_bytes": {"w0": 1}})
    cases["missing_persistent"] = (g, {"output_bytes": {"FW.a": 10}})
    b = GraphBuilder()  # 110-128
    for n in "abcd":
        b.add_op(comp(f"w0->FW.{n}", "w0", 2))
    for x, y in [("a", "b"), ("a", "d"), ("b", "c"), ("c", "d")]:
        b.add_edge(f"w0->FW.{x}", f"w0->FW.{y}")
    cases["last_consumer"] = (b.build(), {"output_bytes": {"FW.a": 8, "FW.b": 2, "FW.c": 2,
                                                           "FW.d": 0},
                                          "persistent_bytes": {"w0": 0}})
    return cases


def memory_expect(g, meta):
    try:
        return {"status": 0, "peak": RefGraph.from_dfg(g).peak_memory(meta)}
    except RefError as err:
        return {"status": err.status, "message": err.msg}


def memory_main():
    """estimate_peak_memory vectors: test_memory.cpp cases, random
    memory_dag graphs, ingest-built layered graphs (with partitions)."""
    vecs = []
    for name, (g, meta) in memory_cases().items():
        vecs.append({"name": name, "graph": g_to_json(g), "meta": meta,
                     "expect": memory_expect(g, meta)})
    rng = np.random.default_rng(20261018)
    for t in range(300):
        g, meta = memory_dag(rng)
        vecs.append({"name": f"memory_dag_{t}", "graph": g_to_json(g), "meta": meta,
                     "expect": memory_expect(g, meta)})
    layered = []
    srng = np.random.default_rng(11)
    for scheme, W, S, L in [("ring", 4, 0, 6), ("ps", 3, 2, 6), ("ring", 8, 0, 12),
                            ("ps", 16, 4, 5)]:
        spec = {"layers": L, "fw_dur_us": srng.integers(10, 400, L).tolist(),
                "bw_dur_us": srng.integers(10, 800, L).tolist(),
                "tensor_bytes": srng.integers(1000, 4_000_000, L).tolist(),
                "update_dur_us": 5, "scheme": scheme, "workers": W, "ps_count": S,
                "bandwidth_bytes_per_us": 12500.0, "latency_us": 5.0}
        act = srng.integers(1, 1 << 24, L).tolist()
        meta = {"output_bytes": {**{f"FW.l{i}": act[i] for i in range(L)},
                                 **{f"BW.l{i}": act[i] // 2 for i in range(L)}},
                "persistent_bytes": {}}
        for variant in range(2):
            k = [1] * L if variant == 0 else srng.choice([1, 2, 3, 4], L).tolist()
            rg = RefGraph.synth(spec)
            for i, ki in enumerate(k):
                rg = rg.partition(f"g{i}", int(ki))
            nodes = sorted({d.split("->")[0] for d in rg.op_ids() if "->" in d})
            meta["persistent_bytes"] = {nd: 4 * sum(spec["tensor_bytes"]) for nd in nodes}
            layered.append({"spec": spec, "part_k": [int(x) for x in k], "meta": dict(meta),
                            "peak": rg.peak_memory(meta)})
    (OUT / "memory_vectors.json").write_text(json.dumps({"graphs": vecs, "layered": layered},
                                                        separators=(",", ":")))
    print(f"{len(vecs)} memory vectors, {len(layered)} layered memory vectors")


def ref_rows(rg):
    ex = rg.export()
    ids, ds = rg.op_ids(), rg.device_strs()
    so, su = ex["succ_off"], ex["succ"]
    return [(ids[i], int(ex["kind"][i]), ds[int(ex["dev"][i])], int(ex["dur"][i]),
             [ids[s] for s in su[so[i]:so[i + 1]]]) for i in range(len(ids))]


def _max_peak(rg, meta):
    return max(rg.peak_memory(meta).values(), default=0)


def rewrite_main():
    """apply_strategy(recompute | grad-accum) and memory_pass vectors
    (optimize.cpp:506-531, 819-1021) on layered synth graphs and random
    rewrite_dag graphs; rewritten graphs are pinned by a digest of their
    (id, kind, device, dur, successors) rows."""
    out = {"sources": [], "apply": [], "memory_pass": []}
    srng = np.random.default_rng(29)
    sources = []
    for scheme, W, S, L in [("ring", 4, 0, 6), ("ps", 3, 2, 9), ("ring", 8, 0, 16),
                            ("ring", 2, 0, 1), ("ps", 4, 1, 25)]:
        spec = {"layers": L, "fw_dur_us": srng.integers(10, 400, L).tolist(),
                "bw_dur_us": srng.integers(10, 800, L).tolist(),
                "tensor_bytes": srng.integers(1000, 4_000_000, L).tolist(),
                "update_dur_us": 5, "scheme": scheme, "workers": W, "ps_count": S,
                "bandwidth_bytes_per_us": 12500.0, "latency_us": 5.0}
        rg = RefGraph.synth(spec)
        act = srng.integers(1, 1 << 26, L).tolist()
        meta = {"output_bytes": {**{f"FW.l{i}": act[i] for i in range(L)},
                                 **{f"BW.l{i}": spec["tensor_bytes"][i] for i in range(L)}},
                "persistent_bytes": {f"w{i}": sum(spec["tensor_bytes"]) for i in range(W)},
                "microbatch_scale": float(srng.choice([0.5, 0.37]))}
        sources.append(({"synth": spec}, rg, meta))
    rng = np.random.default_rng(31)
    for t in range(120):
        g = rewrite_dag(rng)
        meta = {"output_bytes": {f"{k}.l{i}": int(rng.integers(0, 1 << 20))
                                 for k in ("FW", "BW") for i in range(10)},
                "persistent_bytes": {f"w{i}": int(rng.integers(0, 1 << 20)) for i in range(3)},
                "microbatch_scale": float(rng.choice([0.5, 0.25, 0.37]))}
        sources.append(({"graph": g_to_json(g)}, RefGraph.from_dfg(g), meta))
    for si, (src, rg, meta) in enumerate(sources):
        out["sources"].append({**src, "meta": meta})
        for kind in (3, 4):
            try:
                res = {"status": 0, "digest": rows_digest(ref_rows(rg.apply_memory_strategy(kind, meta)))}
            except RefError as err:
                res = {"status": err.status, "message": err.msg}
            out["apply"].append({"src": si, "kind": kind, "expect": res})
        base = _max_peak(rg, meta)
        peaks = []
        for kind in (3, 4):
            try:
                peaks.append(_max_peak(rg.apply_memory_strategy(kind, meta), meta))
            except RefError:
                pass
        budgets = sorted({0, base, base + 1, max(1, base - 1)} |
                         {p for p in peaks} | {max(1, min(peaks + [base]) - 1)})
        for budget in budgets:
            try:
                g2, kind, k = rg.memory_pass(budget, meta)
                res = {"status": 0, "kind": kind, "k": k, "digest": rows_digest(ref_rows(g2))}
            except RefError as err:
                res = {"status": err.status, "message": err.msg,
                       "best_peak": getattr(err, "best_peak", None)}
            out["memory_pass"].append({"src": si, "budget": int(budget), "expect": res})
    # strategy chains (op fusion, tensor fusion, partition) on layered synth
    # graphs, applied one by one; after an error the chain continues on the
    # last good graph
    from paper_2205_02473_b200.graph import synth_cluster
    from paper_2205_02473_b200.ingest import LayeredModel, layered_global_dfg
    out["chains"] = []
    crng = np.random.default_rng(41)
    for si, (src, rg0, meta) in enumerate(sources):
        if "synth" not in src:
            continue
        sp = src["synth"]
        g = layered_global_dfg(LayeredModel(sp["fw_dur_us"], sp["bw_dur_us"], sp["tensor_bytes"],
                                            sp["update_dur_us"]),
                               synth_cluster(sp["scheme"], sp["workers"], sp["ps_count"],
                                             sp["bandwidth_bytes_per_us"], sp["latency_us"]))
        for rep in range(6):
            chain = strategy_chain(crng, g, 6)
            rg, steps = rg0, []
            for kind, a, b, k in chain:
                try:
                    if kind == 0:
                        nrg = rg.op_fusion(a, b)
                    elif kind == 1:
                        nrg = rg.tensor_fusion(a, b)
                    else:
                        nrg = rg.partition(a, k)
                    rg = nrg
                    steps.append({"status": 0, "digest": rows_digest(ref_rows(rg))})
                except RefError as err:
                    steps.append({"status": err.status, "message": err.msg, "cycle": err.cycle})
            out["chains"].append({"src": si, "chain": chain, "steps": steps})
    (OUT / "rewrite_vectors.json").write_text(json.dumps(out, separators=(",", ":")))
    print(f"{len(out['apply'])} rewrite vectors, {len(out['memory_pass'])} memory_pass vectors, "
          f"{len(out['chains'])} strategy chains")


if __name__ == "__main__":
    if sys.argv[1:] == ["memory"]:
        memory_main()
    elif sys.argv[1:] == ["rewrite"]:
        rewrite_main()
    else:
        main()
        memory_main()
        rewrite_main()
