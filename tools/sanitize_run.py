"""Small workloads through every kernel path, sized for compute-sanitizer
(racecheck / synccheck / memcheck replay each kernel many times):

    compute-sanitizer --tool racecheck python tools/sanitize_run.py

Paths: fast kernel (1, 2, 4 warps), general kernel, 2-entry rings (in-launch
fallbacks), deep-ring pass, global counters, delta merge + pack, overlay
batches, critical path, peak memory. Every result is checked against the C
oracle, so a silent corruption also fails the run.
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    from dags import acceptance_dag, fuzz_dag, random_dag_ref
    from oracle import oracle
    from paper_2205_02473_b200.engine import Csr, Engine
    from paper_2205_02473_b200.graph import synth_cluster
    from paper_2205_02473_b200.ingest import LayeredBase, LayeredModel, layered_graph_variant
    eng = Engine(0)
    rng = np.random.default_rng(5)
    graphs = []
    for t in range(60):
        k = t % 3
        graphs.append(random_dag_ref(rng) if k == 0 else acceptance_dag(rng) if k == 1 else
                      fuzz_dag(rng, max_ops=60, zero_p=0.4, virt_p=0.2))
    want = [oracle.port_replay(g.to_csr()) for g in graphs]
    modes = [dict(fast=1, warps=1), dict(fast=1, warps=2), dict(fast=1, warps=4),
             dict(fast=0), dict(fast=1, ring=2), dict(fast=1, deep_first=1),
             dict(fast=1, gcnt=1)]
    for m in modes:
        for k, v in m.items():
            eng.set_option(k, v)
        b = eng.batch([Csr.from_dict(g.to_csr()) for g in graphs])
        b.replay(want_schedule=True)
        ms, st, er, s, e = b.results(schedule=True)
        paths = b.critical_paths()
        for i, w in enumerate(want):
            assert st[i] == w["status"], (m, i)
            if w["status"] == 0:
                a, z = int(b.op_off[i]), int(b.op_off[i + 1])
                assert ms[i] == w["T"] and np.array_equal(s[a:z], w["start"]), (m, i)
                assert np.array_equal(paths[i], w["path"]), (m, i)
        print("mode ok", m, flush=True)
        for k in ("fast", "warps", "ring", "deep_first", "gcnt"):
            eng.set_option(k, {"fast": 1, "warps": 0, "ring": 4, "deep_first": -1, "gcnt": 0}[k])
    # delta merge + pack, overlay batches
    L = 6
    model = LayeredModel(rng.integers(10, 300, L).tolist(), rng.integers(10, 600, L).tolist(),
                         rng.integers(1000, 900_000, L).tolist(), 5)
    for cl in (synth_cluster("ring", 5, 0, 12500.0, 5.0), synth_cluster("ps", 4, 2, 12500.0, 5.0)):
        base = LayeredBase(model, cl)
        specs = [([[0, 1], [2], [3, 4, 5]], [2, 1, 3]), ([[i] for i in range(L)], [1, 2] * 3)]
        fj = np.array([[1, 0, 0, 0, 0], [0, 0, 1, 0, 0]], np.uint8)
        res = eng.resident(base.graph().csr)
        full = base.candidates(specs, threads=2, fw_join=fj)
        for ov in (0, 1):
            eng.set_option("overlay", ov)
            db = eng.delta_batch(res, base.deltas(specs, threads=2, fw_join=fj))
            db.replay(want_schedule=True)
            ms, st, _, s, e = db.results(schedule=True)
            for i, g in enumerate(full):
                w = oracle.port_replay(g.csr)
                a, z = int(db.op_off[i]), int(db.op_off[i + 1])
                assert st[i] == 0 and ms[i] == w["T"] and np.array_equal(s[a:z], w["start"])
            eng.set_option("overlay", 0)
        vs = [layered_graph_variant(model, cl, v, 0.5) for v in ("recompute", "grad-accum")]
        eng.set_option("overlay", 1)
        db = eng.delta_batch(res, base.deltas_from_graphs(vs))
        db.replay(want_schedule=True)
        ms, st, _, s, e = db.results(schedule=True)
        eng.set_option("overlay", 0)
        for i, g in enumerate(vs):
            w = oracle.port_replay(g.csr)
            assert st[i] == 0 and ms[i] == w["T"]
        print("delta / overlay ok", cl.scheme, flush=True)
    print("sanitize run ok")


if __name__ == "__main__":
    main()
