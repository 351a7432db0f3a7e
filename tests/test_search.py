"""Batched evaluator / search driver (search.py). CPU tests: the predicates
and opt_part_num exactly as proj/tests/test_optimize.cpp:246-291 states
them; GPU tests: the batched t_sync table and the MCMC driver, whose every
evaluated candidate must equal the reference's replay of the same rewrite
chain (apply_tensor_fusion + apply_tensor_partition)."""
import numpy as np
import pytest

from paper_2205_02473_b200.search import (SyncSearch, SyncTable, opt_part_num, should_fuse_ops,
                                          should_fuse_tensors)


def test_op_fusion_predicate():  # test_optimize.cpp:246-254
    assert should_fuse_ops(3, 4, 6.0, 1)
    assert not should_fuse_ops(3, 4, 6.0, 5)
    assert should_fuse_ops(3, 4, 6.0, 0)


def test_tensor_fusion_predicate():  # test_optimize.cpp:256-262
    sync = lambda b, k: b
    assert should_fuse_tensors(100, 50, 20, 40, 1, sync)
    assert not should_fuse_tensors(60, 50, 20, 40, 1, sync)


def test_opt_part_num_ties_and_cap():  # test_optimize.cpp:285-291
    assert opt_part_num(100, 4, lambda b, k: 7) == 1
    assert opt_part_num(2, 4, lambda b, k: 100 - k) == 2


@pytest.mark.gpu
def test_sync_table_grid(engine):  # test_optimize.cpp:265-283 on the GPU grid
    from paper_2205_02473_b200.graph import synth_cluster
    t = SyncTable(synth_cluster("ps", 1, 1, 1.0, 0.0), engine)
    assert t.opt_part_num_many([100], 4) == [4]
    assert [t(100, k) for k in (1, 2, 3, 4)] == [200, 150, 134, 125]
    t50 = SyncTable(synth_cluster("ps", 1, 1, 1.0, 50.0), engine)
    assert t50.opt_part_num_many([100, 1], 4) == [1, 1]


def _ref_chain(ref, spec, groups, ks):
    """The reference's own rewrite chain for a SyncState."""
    rg = ref.RefGraph.synth(spec)
    for g in groups:
        name = f"g{g[0]}"
        for i in g[1:]:
            rg = rg.tensor_fusion(name, f"g{i}")
            name = f"{name}+g{i}"
    for g, k in zip(groups, ks):
        if k > 1:
            rg = rg.partition("+".join(f"g{i}" for i in g), k)
    return rg


@pytest.mark.gpu
@pytest.mark.parametrize("scheme,W,S,guided", [("ring", 4, 0, 0.0), ("ps", 4, 2, 0.0),
                                               ("ring", 4, 0, 0.8)])
def test_search_candidates_match_reference(engine, ref, scheme, W, S, guided):
    from paper_2205_02473_b200.graph import synth_cluster
    from paper_2205_02473_b200.ingest import LayeredModel
    L = 6
    rng = np.random.default_rng(11)
    fw, bw = rng.integers(50, 400, L).tolist(), rng.integers(80, 900, L).tolist()
    tb = rng.integers(10_000, 3_000_000, L).tolist()
    spec = {"layers": L, "fw_dur_us": fw, "bw_dur_us": bw, "tensor_bytes": tb,
            "update_dur_us": 5, "scheme": scheme, "workers": W, "ps_count": S,
            "bandwidth_bytes_per_us": 1250.0, "latency_us": 5.0}
    s = SyncSearch(LayeredModel(fw, bw, tb, 5), synth_cluster(scheme, W, S, 1250.0, 5.0),
                   engine, kmax=8, beta=0.05, seed=3, threads=4, guided=guided)
    for _ in range(6):
        s.step(48)
    assert s.best.makespan <= s.log.history[0] or s.log.rounds == 6
    cands = [s.propose(s.state) for _ in range(12)] + [s.best]
    ms = s.evaluate(cands)
    for c, m in zip(cands, ms):
        T, *_ = _ref_chain(ref, spec, c.groups, c.ks).replay()
        assert T == int(m), (c.groups, c.ks)


@pytest.mark.gpu
def test_critical_layers_follow_the_critical_path(engine):
    """CandidateSelection input: the layers on K3's critical path of the
    current state; the path itself is checked against the reference in
    test_replay_gpu."""
    from paper_2205_02473_b200.graph import synth_cluster
    from paper_2205_02473_b200.ingest import LayeredModel
    from paper_2205_02473_b200.search import _layers_of_op
    L = 8
    m = LayeredModel([100] * L, [200] * L, [4_000_000] * (L - 1) + [40_000_000], 5)
    s = SyncSearch(m, synth_cluster("ring", 4, 0, 1250.0, 5.0), engine, guided=1.0, threads=2)
    crit = s.critical_layers(s.state)
    assert crit.dtype == bool and crit.any()
    # the huge last-layer gradient dominates the tail of the iteration
    assert crit[L - 1]
    assert _layers_of_op("RECV.g7#c0#s1#w1#w2") == [7]


@pytest.mark.gpu
def test_strategy_search_all_kinds_match_reference(engine, ref):
    """StrategySearch (op fusion, tensor fusion, partition, recompute,
    grad-accum on a GlobalDFG; candidates evaluated as deltas on the GPU):
    every evaluated makespan equals the reference replay of the same
    rewrite applied by the reference."""
    from golden.make_golden import ref_rows  # noqa: F401
    from paper_2205_02473_b200.graph import synth_cluster
    from paper_2205_02473_b200.ingest import LayeredModel, layered_global_dfg
    from paper_2205_02473_b200.memory import ModelMeta
    from paper_2205_02473_b200.rewrite import StrategyKind
    from paper_2205_02473_b200.search import StrategySearch
    L = 5
    rng = np.random.default_rng(21)
    spec = {"layers": L, "fw_dur_us": rng.integers(50, 400, L).tolist(),
            "bw_dur_us": rng.integers(80, 900, L).tolist(),
            "tensor_bytes": rng.integers(10_000, 3_000_000, L).tolist(),
            "update_dur_us": 5, "scheme": "ring", "workers": 3, "ps_count": 0,
            "bandwidth_bytes_per_us": 1250.0, "latency_us": 5.0}
    g0 = layered_global_dfg(LayeredModel(spec["fw_dur_us"], spec["bw_dur_us"],
                                         spec["tensor_bytes"], 5),
                            synth_cluster("ring", 3, 0, 1250.0, 5.0))
    s = StrategySearch(g0, engine, meta=ModelMeta(microbatch_scale=0.5), seed=4, beta=0.05)
    for _ in range(3):
        s.step(12)
    cands = s.propose(16)
    kinds = {int(st.kind) for st, _ in cands}
    ms = s.evaluate([c for _, c in cands])
    # the same strategies applied by the reference to the same current graph
    rg = ref.RefGraph.synth(spec)
    for st in s.applied:
        rg = (rg.op_fusion(st.a, st.b) if st.kind == StrategyKind.OP_FUSION else
              rg.tensor_fusion(st.a, st.b) if st.kind == StrategyKind.TENSOR_FUSION else
              rg.partition(st.a, st.k) if st.kind == StrategyKind.PARTITION else
              rg.apply_memory_strategy(int(st.kind), {"microbatch_scale": 0.5}))
    for (st, _), m in zip(cands, ms):
        r = (rg.op_fusion(st.a, st.b) if st.kind == StrategyKind.OP_FUSION else
             rg.tensor_fusion(st.a, st.b) if st.kind == StrategyKind.TENSOR_FUSION else
             rg.partition(st.a, st.k) if st.kind == StrategyKind.PARTITION else
             rg.apply_memory_strategy(int(st.kind), {"microbatch_scale": 0.5}))
        assert r.replay()[0] == int(m), st
    assert len(kinds) >= 3
