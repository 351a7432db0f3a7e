"""K5 (batched peak-memory estimate) against the reference's
estimate_peak_memory (proj/src/memory.cpp:122-167). Mirrors
proj/tests/test_memory.cpp, plus random graphs and ingest-built layered
graphs from tests/golden/memory_vectors.json (made by the reference)."""
import json

import numpy as np
import pytest

from golden_io import GOLDEN, graph_from_json
from paper_2205_02473_b200 import (CycleError, MissingMetaError, ModelMeta, OpKind, comp,
                                   estimate_peak_memory, estimate_peak_memory_many,
                                   output_bytes_for, replay, replay_many)
from paper_2205_02473_b200.graph import synth_cluster
from paper_2205_02473_b200.ingest import LayeredModel, layered_graph
from paper_2205_02473_b200.memory import resolve


def _vectors():
    return json.loads((GOLDEN / "memory_vectors.json").read_text())


def _port_args(g):
    ops = [(o.id, int(o.kind), o.node) for o in g.ops()]
    succ = [list(g.succ_indices(i)) for i in range(g.size())]
    return ops, succ


# ---- host side (CPU) ----------------------------------------------------

def test_model_meta_json_round_trip(tmp_path):
    """test_memory.cpp:37-46."""
    m = ModelMeta({"FW.a": 10, "BW.a": 4}, {"w0": 100}, 0.25)
    back = ModelMeta.from_json(m.to_json())
    assert back == m
    m.save(str(tmp_path / "m.json"))
    assert ModelMeta.load(str(tmp_path / "m.json")) == m


def test_output_bytes_fall_back_across_id_forms():
    """test_memory.cpp:48-56, plus the '+'-fused rule (memory.cpp:104-118)."""
    m = ModelMeta({"FW.a": 10, "w0->FW.b": 20, "FW.c": 3})
    assert output_bytes_for(m, "w0->FW.a") == 10
    assert output_bytes_for(m, "w0->FW.b") == 20
    assert output_bytes_for(m, "w0->FW.a@mb1") == 5
    assert output_bytes_for(m, "w0->RFW.a") == 10
    assert output_bytes_for(m, "w0->FW.zzz") == -1
    assert output_bytes_for(m, "w0->FW.a+FW.c") == 13
    assert output_bytes_for(m, "w0->FW.a+FW.zzz") == -1


def test_missing_metadata_is_reported_in_reference_order():
    """test_memory.cpp:96-108: resolve() raises before any GPU work."""
    from paper_2205_02473_b200 import GraphBuilder
    b = GraphBuilder()
    b.add_op(comp("w0->FW.a", "w0", 4))
    g = b.build()
    with pytest.raises(MissingMetaError, match="no output bytes for op w0->FW.a"):
        resolve(g, ModelMeta(persistent_bytes={"w0": 1}))
    with pytest.raises(MissingMetaError, match="no persistent bytes for node w0"):
        resolve(g, ModelMeta(output_bytes={"FW.a": 10}))


def test_port_matches_reference_memory_vectors(port):
    """The oracle restatement against every reference-made vector."""
    n = 0
    for v in _vectors()["graphs"]:
        exp = v["expect"]
        if exp["status"] == 2:
            continue  # replay itself raises (covered by the replay vectors)
        g = graph_from_json(v["graph"])
        got = port.port_replay(_csr(g))
        ops, succ = _port_args(g)
        if exp["status"] == 6:
            with pytest.raises(KeyError) as ei:
                port.port_peak_memory(ops, succ, got["start"], got["end"], v["meta"])
            assert ei.value.args[0] == exp["message"], v["name"]
        else:
            assert port.port_peak_memory(ops, succ, got["start"], got["end"],
                                         v["meta"]) == exp["peak"], v["name"]
        n += 1
    assert n > 250


def _csr(g):
    from paper_2205_02473_b200.engine import Csr
    return Csr.from_dict(g.to_csr())


def test_port_matches_live_reference_on_random_graphs(ref, port):
    from dags import memory_dag
    rng = np.random.default_rng(99)
    for t in range(60):
        g, meta = memory_dag(rng, max_ops=60)
        rg = ref.RefGraph.from_dfg(g)
        try:
            exp = rg.peak_memory(meta)
        except ref.RefError as err:
            if err.status != 6:
                continue
            exp = err.msg
        got = port.port_replay(_csr(g))
        ops, succ = _port_args(g)
        try:
            res = port.port_peak_memory(ops, succ, got["start"], got["end"], meta)
        except KeyError as e:
            res = e.args[0]
        assert res == exp, t


# ---- GPU (K5) -------------------------------------------------------------

@pytest.mark.gpu
def test_memory_cases_of_reference_tests(engine):
    """test_memory.cpp:58-128 on the GPU."""
    for v in _vectors()["graphs"][:6]:
        g = graph_from_json(v["graph"])
        meta = ModelMeta.from_json(v["meta"])
        r = replay(g)
        if v["expect"]["status"] == 6:
            with pytest.raises(MissingMetaError) as ei:
                estimate_peak_memory(g, r, meta)
            assert str(ei.value) == v["expect"]["message"]
        else:
            assert estimate_peak_memory(g, r, meta) == v["expect"]["peak"], v["name"]


@pytest.mark.gpu
def test_batched_memory_matches_reference_vectors(engine):
    """All random vectors in ONE replay batch + ONE K5 launch."""
    vs = [v for v in _vectors()["graphs"] if v["expect"]["status"] == 0]
    graphs = [graph_from_json(v["graph"]) for v in vs]
    results = replay_many(graphs)
    peaks = estimate_peak_memory_many(graphs, results,
                                      [ModelMeta.from_json(v["meta"]) for v in vs])
    for v, p in zip(vs, peaks):
        assert p == v["expect"]["peak"], v["name"]


@pytest.mark.gpu
def test_memory_errors_match_reference(engine):
    for v in _vectors()["graphs"]:
        st = v["expect"]["status"]
        if st == 0:
            continue
        g = graph_from_json(v["graph"])
        if st == 2:
            with pytest.raises(CycleError):
                replay(g)
            continue
        with pytest.raises(MissingMetaError) as ei:
            estimate_peak_memory(g, replay(g), ModelMeta.from_json(v["meta"]))
        assert str(ei.value) == v["expect"]["message"], v["name"]


@pytest.mark.gpu
def test_memory_on_layered_graphs(engine):
    for v in _vectors()["layered"]:
        s = v["spec"]
        c = synth_cluster(s["scheme"], s["workers"], s["ps_count"], s["bandwidth_bytes_per_us"],
                          s["latency_us"])
        ng = layered_graph(LayeredModel(s["fw_dur_us"], s["bw_dur_us"], s["tensor_bytes"],
                                        s["update_dur_us"]), c, v["part_k"])
        g = ng.to_global_dfg(c)
        assert estimate_peak_memory(g, replay(g), ModelMeta.from_json(v["meta"])) == v["peak"]


@pytest.mark.gpu
@pytest.mark.parametrize("workers,layers", [(8, 24), (32, 48)])
def test_memory_at_scale_matches_port(engine, port, workers, layers):
    """Larger layered graphs (thousands of ops, many events per node)
    against the oracle restatement on the same schedule."""
    rng = np.random.default_rng(workers)
    c = synth_cluster("ring", workers, 0, 12500.0, 5.0)
    m = LayeredModel(rng.integers(10, 400, layers).tolist(), rng.integers(10, 800, layers).tolist(),
                     rng.integers(1000, 4_000_000, layers).tolist(), 5)
    ng = layered_graph(m, c, rng.choice([1, 2, 3, 4], layers).tolist())
    g = ng.to_global_dfg(c)
    meta = ModelMeta({**{f"FW.l{i}": int(x) for i, x in enumerate(rng.integers(1, 1 << 30, layers))},
                      **{f"BW.l{i}": int(x) for i, x in enumerate(rng.integers(0, 1 << 30, layers))}},
                     {f"w{i}": 7 * i for i in range(workers)})
    r = replay(g)
    got = estimate_peak_memory(g, r, meta)
    start = np.array([r.schedule[o.id].start for o in g.ops()])
    end = np.array([r.schedule[o.id].end for o in g.ops()])
    ops, succ = _port_args(g)
    assert got == port.port_peak_memory(ops, succ, start, end, meta.to_json())
