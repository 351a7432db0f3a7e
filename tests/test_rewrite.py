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
