"""Memory rewrites (recompute, grad-accum) and the memory pass against the
reference (optimize.cpp:506-531, 819-1021). Rewritten graphs are compared
row by row (id, kind, device, dur, successors) through a digest made by the
reference (tests/golden/rewrite_vectors.json); memory_pass runs its
replays and peak estimates on the GPU."""
import numpy as np
import pytest

from golden_io import dfg_rows, graph_from_json, rewrite_vectors, rows_digest
from paper_2205_02473_b200 import ModelMeta, TransformError
from paper_2205_02473_b200.graph import synth_cluster
from paper_2205_02473_b200.ingest import (LayeredModel, layered_global_dfg, layered_graph)
from paper_2205_02473_b200.rewrite import (BudgetError, StrategyKind, apply_grad_accum,
                                           apply_recompute, memory_pass)

_SRC_CACHE = {}


def _source(vecs, i):
    if i not in _SRC_CACHE:
        s = vecs["sources"][i]
        if "synth" in s:
            sp = s["synth"]
            c = synth_cluster(sp["scheme"], sp["workers"], sp["ps_count"],
                              sp["bandwidth_bytes_per_us"], sp["latency_us"])
            g = layered_global_dfg(LayeredModel(sp["fw_dur_us"], sp["bw_dur_us"],
                                                sp["tensor_bytes"], sp["update_dur_us"]), c)
        else:
            g = graph_from_json(s["graph"])
        _SRC_CACHE[i] = (g, ModelMeta.from_json(s["meta"]))
    return _SRC_CACHE[i]


def test_layered_global_dfg_matches_native_generator():
    rng = np.random.default_rng(1)
    for scheme, W, S, L in [("ring", 4, 0, 5), ("ps", 3, 2, 4), ("ring", 11, 0, 3)]:
        c = synth_cluster(scheme, W, S, 12500.0, 5.0)
        m = LayeredModel(rng.integers(10, 400, L).tolist(), rng.integers(10, 800, L).tolist(),
                         rng.integers(1000, 4_000_000, L).tolist(), 5)
        k = rng.choice([1, 2, 3], L).tolist()
        ng, g = layered_graph(m, c, k), layered_global_dfg(m, c, k)
        a = g.to_csr()
        assert [o.id for o in g.ops()] == ng.op_ids()
        for f in ("dur", "dev", "flags", "succ_off", "succ", "indeg"):
            assert np.array_equal(a[f], getattr(ng.csr, f)), f


def test_rewrites_match_reference_vectors():
    vecs = rewrite_vectors()
    for v in vecs["apply"]:
        g, meta = _source(vecs, v["src"])
        exp = v["expect"]
        fn = (lambda: apply_recompute(g)) if v["kind"] == 3 else (lambda: apply_grad_accum(g, meta))
        if exp["status"] == 0:
            assert rows_digest(dfg_rows(fn())) == exp["digest"], v
        else:
            assert exp["status"] == 5
            with pytest.raises(TransformError) as ei:
                fn()
            assert str(ei.value) == exp["message"]


def test_rewrites_match_live_reference(ref):
    from dags import rewrite_dag
    from golden.make_golden import ref_rows
    rng = np.random.default_rng(77)
    for t in range(80):
        g = rewrite_dag(rng)
        rg = ref.RefGraph.from_dfg(g)
        scale = float(rng.choice([0.5, 0.3, 0.7]))
        meta = ModelMeta(microbatch_scale=scale)
        for kind, fn in ((3, lambda: apply_recompute(g)), (4, lambda: apply_grad_accum(g, meta))):
            try:
                exp = ref_rows(rg.apply_memory_strategy(kind, meta.to_json()))
            except ref.RefError as err:
                exp = err.msg
            try:
                got = dfg_rows(fn())
            except TransformError as err:
                got = str(err)
            assert got == exp, (t, kind)


@pytest.mark.gpu
def test_memory_pass_matches_reference_vectors(engine):
    vecs = rewrite_vectors()
    n_applied = 0
    for v in vecs["memory_pass"]:
        g, meta = _source(vecs, v["src"])
        exp = v["expect"]
        applied = []
        if exp["status"] == 0:
            out = memory_pass(g, v["budget"], meta, applied)
            if exp["kind"] < 0:
                assert out is g and not applied, v
            else:
                n_applied += 1
                assert applied[0].kind == StrategyKind(exp["kind"]) and applied[0].k == exp["k"]
                assert rows_digest(dfg_rows(out)) == exp["digest"], v
        else:
            assert exp["status"] == 7
            with pytest.raises(BudgetError) as ei:
                memory_pass(g, v["budget"], meta, applied)
            assert str(ei.value) == exp["message"]
            assert ei.value.best_peak_bytes == exp["best_peak"]
    assert n_applied > 100


def _apply_chain(g, chain):
    from paper_2205_02473_b200 import CycleError, Error
    from paper_2205_02473_b200.errors import LookupError_
    from paper_2205_02473_b200.rewrite import (apply_op_fusion, apply_tensor_fusion,
                                               apply_tensor_partition)
    steps = []
    for kind, a, b, k in chain:
        try:
            if kind == 0:
                g = apply_op_fusion(g, a, b)
            elif kind == 1:
                g = apply_tensor_fusion(g, a, b)
            else:
                g = apply_tensor_partition(g, a, k)
            steps.append({"status": 0, "digest": rows_digest(dfg_rows(g))})
        except CycleError as e:
            steps.append({"status": 2, "message": str(e), "cycle": e.cycle})
        except LookupError_ as e:
            steps.append({"status": 4, "message": str(e)})
        except TransformError as e:
            steps.append({"status": 5, "message": str(e)})
        except Error as e:  # pragma: no cover - unexpected kind
            steps.append({"status": 3, "message": str(e)})
    return g, steps


def test_strategy_chains_match_reference_vectors():
    """op fusion / tensor fusion / partition chains (optimize.cpp:245-492)
    against the reference: every intermediate graph row by row, every
    error with its type, message and cycle witness."""
    vecs = rewrite_vectors()
    for v in vecs["chains"]:
        g, _ = _source(vecs, v["src"])
        _, steps = _apply_chain(g, [tuple(c) for c in v["chain"]])
        for got, exp in zip(steps, v["steps"]):
            exp = {k: x for k, x in exp.items() if not (k == "cycle" and exp["status"] != 2)}
            got = {k: x for k, x in got.items() if k in exp}
            assert got == exp, (v["chain"], got, exp)


def test_strategy_chains_match_live_reference(ref):
    from dags import strategy_chain
    from golden.make_golden import ref_rows
    rng = np.random.default_rng(5)
    for scheme, W, S, L in [("ring", 3, 0, 5), ("ps", 4, 2, 6)]:
        spec = {"layers": L, "fw_dur_us": rng.integers(10, 400, L).tolist(),
                "bw_dur_us": rng.integers(10, 800, L).tolist(),
                "tensor_bytes": rng.integers(1000, 4_000_000, L).tolist(),
                "update_dur_us": 5, "scheme": scheme, "workers": W, "ps_count": S,
                "bandwidth_bytes_per_us": 12500.0, "latency_us": 5.0}
        c = synth_cluster(scheme, W, S, 12500.0, 5.0)
        g0 = layered_global_dfg(LayeredModel(spec["fw_dur_us"], spec["bw_dur_us"],
                                             spec["tensor_bytes"], 5), c)
        for _ in range(8):
            chain = strategy_chain(rng, g0, 5)
            _, steps = _apply_chain(g0, chain)
            rg = ref.RefGraph.synth(spec)
            for (kind, a, b, k), got in zip(chain, steps):
                try:
                    rg = (rg.op_fusion(a, b) if kind == 0 else
                          rg.tensor_fusion(a, b) if kind == 1 else rg.partition(a, k))
                    exp = {"status": 0, "digest": rows_digest(ref_rows(rg))}
                except ref.RefError as e:
                    exp = {"status": e.status, "message": e.msg}
                assert {k2: got.get(k2) for k2 in exp} == exp, (chain, kind, a, b, k)


@pytest.mark.gpu
def test_rewritten_graphs_replay_like_reference(engine, ref):
    """GPU replay of rewritten graphs equals the reference replay of the
    same rewrite chain (makespan and every start/end)."""
    from paper_2205_02473_b200 import replay_many
    from golden.make_golden import ref_rows  # noqa: F401 - import check
    vecs = rewrite_vectors()
    graphs, exps = [], []
    for v in vecs["chains"][:12]:
        g, _ = _source(vecs, v["src"])
        g2, steps = _apply_chain(g, [tuple(c) for c in v["chain"]])
        graphs.append(g2)
        sp = vecs["sources"][v["src"]]["synth"]
        rg = ref.RefGraph.synth(sp)
        for kind, a, b, k in v["chain"]:
            try:
                rg = (rg.op_fusion(a, b) if kind == 0 else
                      rg.tensor_fusion(a, b) if kind == 1 else rg.partition(a, k))
            except ref.RefError:
                pass
        exps.append(rg.replay())
    for r, (T, s, e, _, _) in zip(replay_many(graphs), exps):
        assert r.iteration_time_us == T
        order = sorted(r.schedule)
        assert [r.schedule[i].start for i in order] == s.tolist()
        assert [r.schedule[i].end for i in order] == e.tolist()


@pytest.mark.parametrize("scheme,W,S,L", [("ring", 3, 0, 1), ("ring", 4, 0, 7), ("ps", 3, 2, 10),
                                          ("ring", 2, 0, 16)])
def test_native_memory_variants_match_rewrites(scheme, W, S, L):
    """dpro_graph_layered_variant == apply_recompute / apply_grad_accum on
    the same layered graph (those are pinned to the reference above)."""
    from paper_2205_02473_b200.ingest import layered_graph_variant
    rng = np.random.default_rng(L)
    c = synth_cluster(scheme, W, S, 12500.0, 5.0)
    m = LayeredModel(rng.integers(10, 400, L).tolist(), rng.integers(11, 801, L).tolist(),
                     rng.integers(1000, 4_000_000, L).tolist(), 5)
    k = rng.choice([1, 2, 3], L).tolist()
    g = layered_global_dfg(m, c, k)
    for var, fn in (("recompute", lambda: apply_recompute(g)),
                    ("grad-accum", lambda: apply_grad_accum(g, ModelMeta(microbatch_scale=0.37)))):
        try:
            exp = fn()
        except TransformError as e:
            with pytest.raises(Exception, match=str(e)):
                layered_graph_variant(m, c, var, 0.37, k)
            continue
        ng = layered_graph_variant(m, c, var, 0.37, k)
        a = exp.to_csr()
        assert [o.id for o in exp.ops()] == ng.op_ids()
        for f in ("dur", "dev", "flags", "succ_off", "succ", "indeg"):
            assert np.array_equal(a[f], getattr(ng.csr, f)), (var, f)


def test_native_memory_inputs_match_resolve():
    from paper_2205_02473_b200 import MissingMetaError
    from paper_2205_02473_b200.ingest import layered_graph_variant
    from paper_2205_02473_b200.memory import native_inputs, resolve
    L = 6
    c = synth_cluster("ps", 3, 2, 12500.0, 5.0)
    m = LayeredModel([100] * L, [200] * L, [1000 * (i + 1) for i in range(L)], 5)
    meta = ModelMeta({**{f"FW.l{i}": 10 * (i + 1) for i in range(L)},
                      **{f"BW.l{i}": 7 * (i + 1) for i in range(L)}},
                     {f"w{i}": 1000 for i in range(3)})
    for var in ("none", "recompute", "grad-accum"):
        ng = layered_graph_variant(m, c, var, 0.5)
        a, b = native_inputs(ng, meta), resolve(ng.to_global_dfg(c), meta)
        assert a[0] == b[0]
        for x, y in zip(a[1:], b[1:]):
            assert np.array_equal(x, y), var
    bad = ModelMeta({"FW.l0": 1}, {f"w{i}": 1 for i in range(3)})
    ng = layered_graph_variant(m, c, "none", 0.5)
    with pytest.raises(MissingMetaError) as e1:
        native_inputs(ng, bad)
    with pytest.raises(MissingMetaError) as e2:
        resolve(ng.to_global_dfg(c), bad)
    assert str(e1.value) == str(e2.value)


@pytest.mark.gpu
def test_memory_pass_layered_matches_memory_pass(engine):
    """memory_pass_layered (native graphs, one batch, one K5 launch) makes
    the same choice as memory_pass on the GlobalDFG for a range of budgets."""
    from paper_2205_02473_b200.rewrite import memory_pass_layered
    rng = np.random.default_rng(8)
    L = 9
    c = synth_cluster("ring", 4, 0, 12500.0, 5.0)
    m = LayeredModel(rng.integers(100, 400, L).tolist(), rng.integers(100, 800, L).tolist(),
                     rng.integers(1000, 4_000_000, L).tolist(), 5)
    act = rng.integers(1, 1 << 26, L).tolist()
    meta = ModelMeta({**{f"FW.l{i}": act[i] for i in range(L)},
                      **{f"BW.l{i}": int(m.tensor_bytes[i]) for i in range(L)}},
                     {f"w{i}": int(sum(m.tensor_bytes)) for i in range(4)}, 0.5)
    g = layered_global_dfg(m, c)
    _, base_g, base_peak, _ = memory_pass_layered(m, c, 0, meta, engine)
    for budget in (0, base_peak, base_peak - 1, base_peak // 2, 1):
        try:
            applied = []
            out = memory_pass(g, budget, meta, applied)
            exp = ("ok", [int(a.kind) for a in applied], [o.id for o in out.ops()])
        except BudgetError as e:
            exp = ("budget", str(e), e.best_peak_bytes)
        try:
            st, ng, _, _ = memory_pass_layered(m, c, budget, meta, engine)
            got = ("ok", [] if st is None else [int(st.kind)], ng.op_ids())
        except BudgetError as e:
            got = ("budget", str(e), e.best_peak_bytes)
        assert got == exp, budget
