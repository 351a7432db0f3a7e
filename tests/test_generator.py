"""Host CSR generator (csrc/dfg_gen.cpp) vs the reference ingest/rewrite
path: identical op ids (hence index order), durations, devices and edges."""
import hashlib

import numpy as np
import pytest

from golden_io import synth_vectors
from paper_2205_02473_b200.graph import GraphBuilder, synth_cluster
from paper_2205_02473_b200.ingest import (LayeredModel, expand_tensor, layered_graph,
                                          layered_graphs, splice, tsync_graph)


def _model(s):
    return LayeredModel(s["fw_dur_us"], s["bw_dur_us"], s["tensor_bytes"], s["update_dur_us"])


def _cluster(s):
    return synth_cluster(s["scheme"], s["workers"], s["ps_count"], s["bandwidth_bytes_per_us"],
                         s["latency_us"])


def test_generator_matches_golden_op_order():
    for v in synth_vectors():
        ng = layered_graph(_model(v["spec"]), _cluster(v["spec"]), v["part_k"])
        assert ng.n_ops == v["n_ops"] and ng.n_edges == v["n_edges"]
        assert hashlib.sha256("\n".join(ng.op_ids()).encode()).hexdigest() == v["ops_sha256"]


def _same_csr(ex, ng, ref_graph):
    assert ref_graph.op_ids() == ng.op_ids()
    assert ref_graph.device_strs() == ng.device_strs()
    for k in ("dur", "succ_off", "succ", "dev", "flags"):
        assert np.array_equal(np.asarray(ex[k]), np.asarray(getattr(ng.csr, k))), k
    assert np.array_equal(ex["indeg"], ng.csr.indeg)


@pytest.mark.parametrize("scheme,W,S,L", [("ring", 2, 0, 3), ("ring", 13, 0, 3), ("ps", 5, 3, 7),
                                          ("ps", 1, 1, 2), ("ring", 10, 0, 2)])
def test_generator_matches_reference_ingest_and_partition(ref, scheme, W, S, L):
    rng = np.random.default_rng(W * 31 + L)
    spec = {"layers": L, "fw_dur_us": rng.integers(0, 99, L).tolist(),
            "bw_dur_us": rng.integers(1, 99, L).tolist(),
            "tensor_bytes": rng.integers(20, 90000, L).tolist(), "update_dur_us": 5,
            "scheme": scheme, "workers": W, "ps_count": S, "bandwidth_bytes_per_us": 33.0,
            "latency_us": 2.5}
    rg = ref.RefGraph.synth(spec)
    ng = layered_graph(_model(spec), _cluster(spec))
    _same_csr(rg.export(), ng, rg)
    ks = rng.choice([1, 2, 3, 10, 12], L).tolist()
    for i, k in enumerate(ks):
        rg = rg.partition(f"g{i}", int(k))
    ng = layered_graph(_model(spec), _cluster(spec), ks)
    _same_csr(rg.export(), ng, rg)


def test_generator_batch_equals_single():
    s = synth_vectors()[2]["spec"]
    pk = np.array([[1] * s["layers"], [2] * s["layers"], [3, 1] * (s["layers"] // 2)], np.int32)
    many = layered_graphs(_model(s), _cluster(s), pk, threads=3)
    for row, g in zip(pk, many):
        one = layered_graph(_model(s), _cluster(s), row)
        assert one.op_ids() == g.op_ids()
        assert np.array_equal(one.csr.succ, g.csr.succ)


@pytest.mark.parametrize("scheme,W,S,b,k", [("ring", 12, 0, 1000, 12), ("ps", 3, 2, 100, 11),
                                            ("ring", 4, 0, 5, 3), ("ps", 16, 4, 4096, 4)])
def test_tsync_graph_matches_reference(ref, scheme, W, S, b, k):
    c = synth_cluster(scheme, W, S, 1.0, 0.5)
    rg = ref.RefGraph.tsync(c.to_json(), b, k)
    ng = tsync_graph(c, b, k)
    _same_csr(rg.export(), ng, rg)


def test_python_expansion_matches_native():
    c = synth_cluster("ring", 11, 0, 7.0, 1.0)
    b = GraphBuilder()
    for i in range(3):
        splice(b, expand_tensor("tsync" if i == 0 else f"tsync#p{i}", 1000 + i, c))
    g = b.build()
    # native t_sync graph for k=1 has only the "tsync" unit
    ng = tsync_graph(c, 1000, 1)
    ids = [op.id for op in g.ops() if op.id.split(".", 1)[1].startswith("tsync#c")]
    assert ids == ng.op_ids()


def test_generator_errors():
    c = synth_cluster("ring", 1, 0, 1.0, 0.0)
    with pytest.raises(Exception, match="degenerate ring"):
        layered_graph(LayeredModel([1], [1], [10]), c)
    c = synth_cluster("ring", 3, 0, 1.0, 0.0)
    with pytest.raises(Exception, match="cannot split 10 bytes"):
        layered_graph(LayeredModel([1], [1], [10]), c, [11])


@pytest.mark.parametrize("scheme,W,S", [("ring", 4, 0), ("ps", 5, 2), ("ring", 11, 0)])
def test_generator_tensor_fusion_matches_reference(ref, scheme, W, S):
    """apply_tensor_fusion chains (+ a partition of the fused unit) through the
    reference vs the generator's fused groups."""
    from paper_2205_02473_b200.ingest import layered_graph_groups
    L = 6
    rng = np.random.default_rng(W)
    spec = {"layers": L, "fw_dur_us": rng.integers(1, 99, L).tolist(),
            "bw_dur_us": rng.integers(1, 99, L).tolist(),
            "tensor_bytes": rng.integers(20, 90000, L).tolist(), "update_dur_us": 5,
            "scheme": scheme, "workers": W, "ps_count": S, "bandwidth_bytes_per_us": 33.0,
            "latency_us": 2.5}
    rg = ref.RefGraph.synth(spec)
    rg = rg.tensor_fusion("g1", "g2").tensor_fusion("g1+g2", "g3")
    rg = rg.tensor_fusion("g5", "g0").partition("g5+g0", 3).partition("g4", 2)
    groups = [[1, 2, 3], [5, 0], [4]]
    ng = layered_graph_groups(_model(spec), _cluster(spec), groups, [1, 3, 2])
    _same_csr(rg.export(), ng, rg)


@pytest.mark.parametrize("scheme,W,S,L", [("ring", 8, 0, 12), ("ps", 16, 4, 9), ("ring", 11, 0, 6),
                                          ("ps", 3, 2, 7)])
def test_delta_construction_equals_full_build(scheme, W, S, L):
    """Candidates built as base + delta (dpro_graph_from_base_batch) are the
    exact CSR of a full rebuild (same ids, devices, durations, edges)."""
    from paper_2205_02473_b200.ingest import LayeredBase, layered_graphs_groups
    rng = np.random.default_rng(L * 7 + W)
    model = LayeredModel(rng.integers(10, 900, L).tolist(), rng.integers(10, 900, L).tolist(),
                         rng.integers(100, 4_000_000, L).tolist(), 5)
    cluster = synth_cluster(scheme, W, S, 12500.0, 5.0)
    specs = []
    for _ in range(24):
        groups, i = [], 0
        while i < L:
            n = int(rng.choice([1, 1, 1, 2, 3]))
            groups.append(list(range(i, min(L, i + n))))
            i += n
        ks = [int(rng.choice([1, 1, 2, 3, 4, 12])) for _ in groups]
        specs.append((groups, ks))
    specs.append(([[i] for i in range(L)], [1] * L))  # the base itself
    full = layered_graphs_groups(model, cluster, specs, threads=4)
    delta = LayeredBase(model, cluster).candidates(specs, threads=4)
    for a, b in zip(full, delta):
        assert a.op_ids() == b.op_ids()
        assert a.device_strs() == b.device_strs()
        for k in ("dur", "dev", "flags", "succ_off", "succ", "indeg"):
            assert np.array_equal(getattr(a.csr, k), getattr(b.csr, k)), k
