"""The CPU oracles, pinned before they are trusted (no GPU needed).

* the C port (oracle/replay_oracle.c) against the reference's golden
  vectors (tests/golden, generated from the compiled reference);
* the port against the live reference (oracle/_ref) on fresh fuzz graphs,
  when the reference library is built (this container).
"""
import numpy as np
import pytest

from dags import acceptance_dag, fuzz_dag, random_dag_ref
from golden_io import graph_from_json, replay_vectors, synth_vectors
from paper_2205_02473_b200.graph import synth_cluster
from paper_2205_02473_b200.ingest import LayeredModel, layered_graph


def _check_port_against(expect, g, got):
    if expect["status"] != 0:
        assert got["status"] == expect["status"]
        if expect["status"] == 1:
            assert expect["message"] == f"op {g.op_at(int(got['err'])).id} has no duration"
        else:
            stuck = [g.op_at(i).id for i in np.flatnonzero(got["scheduled"] == 0)]
            assert stuck == expect["cycle"]
            assert f"; {got['err']} ops never became ready" in expect["message"]
        return
    assert got["status"] == 0
    assert got["T"] == expect["T"]
    assert got["start"].tolist() == expect["start"]
    assert got["end"].tolist() == expect["end"]
    assert got["tl_pos"].tolist() == expect["tl_pos"]
    assert got["path"].tolist() == expect["path"]


def test_port_matches_reference_golden_vectors(port):
    vecs = replay_vectors()
    assert len(vecs) > 500
    for v in vecs:
        g = graph_from_json(v["graph"])
        got = port.port_replay(g.to_csr())
        try:
            _check_port_against(v["expect"], g, got)
        except AssertionError as e:  # pragma: no cover - message helper
            raise AssertionError(f"vector {v['name']}: {e}") from e


@pytest.mark.parametrize("family,count", [(random_dag_ref, 200), (acceptance_dag, 200),
                                          (fuzz_dag, 400)])
def test_port_matches_live_reference_on_fuzz(ref, port, family, count):
    rng = np.random.default_rng(7 + count)
    for _ in range(count):
        g = family(rng)
        rg = ref.RefGraph.from_dfg(g)
        got = port.port_replay(g.to_csr())
        try:
            T, s, e, tl, util = rg.replay()
        except ref.RefError as err:
            assert got["status"] == err.status
            continue
        assert got["status"] == 0 and got["T"] == T
        assert np.array_equal(got["start"], s) and np.array_equal(got["end"], e)
        assert np.array_equal(got["tl_pos"], tl)
        assert np.array_equal(got["path"], rg.critical_path()["path"])


def test_port_on_ingest_built_graphs_matches_golden(port):
    import hashlib
    for v in synth_vectors():
        s = v["spec"]
        c = synth_cluster(s["scheme"], s["workers"], s["ps_count"], s["bandwidth_bytes_per_us"],
                          s["latency_us"])
        ng = layered_graph(LayeredModel(s["fw_dur_us"], s["bw_dur_us"], s["tensor_bytes"],
                                        s["update_dur_us"]), c, v["part_k"])
        got = port.port_replay(ng.csr)
        assert got["status"] == 0 and got["T"] == v["T"]
        digest = hashlib.sha256(np.concatenate([got["start"], got["end"]]).astype("<i8").tobytes())
        assert digest.hexdigest() == v["schedule_sha256"]
        assert got["path"].tolist() == v["path"]
