"""Timeline writer (report.py) byte for byte against the reference CLI's
timeline.json (proj/tools/dpro_main.cpp:64-116) on the same graphs."""
import numpy as np
import pytest

from paper_2205_02473_b200.graph import synth_cluster
from paper_2205_02473_b200.ingest import LayeredModel, layered_global_dfg
from paper_2205_02473_b200.report import timeline_json, timeline_text

SPECS = [("ring", 2, 0, 2), ("ring", 4, 0, 5), ("ps", 3, 2, 4)]


def _spec(scheme, W, S, L, seed):
    rng = np.random.default_rng(seed)
    return {"layers": L, "fw_dur_us": rng.integers(10, 400, L).tolist(),
            "bw_dur_us": rng.integers(10, 800, L).tolist(),
            "tensor_bytes": rng.integers(1000, 4_000_000, L).tolist(), "update_dur_us": 5,
            "scheme": scheme, "workers": W, "ps_count": S, "bandwidth_bytes_per_us": 12500.0,
            "latency_us": 5.0}


def test_timeline_shape():
    class R:  # minimal result stand-in
        pass
    sp = _spec("ring", 2, 0, 2, 1)
    g = layered_global_dfg(LayeredModel(sp["fw_dur_us"], sp["bw_dur_us"], sp["tensor_bytes"], 5),
                           synth_cluster("ring", 2, 0, 12500.0, 5.0))
    from paper_2205_02473_b200.replay import ScheduleEntry
    r = R()
    r.schedule = {o.id: ScheduleEntry(0, int(o.dur), o.device) for o in g.ops()}
    j = timeline_json(g, r)
    assert j["displayTimeUnit"] == "ms"
    assert all(e["ph"] == "X" for e in j["traceEvents"])
    assert not any(e["cat"].startswith("VIRTUAL") for e in j["traceEvents"])


@pytest.mark.gpu
@pytest.mark.parametrize("scheme,W,S,L", SPECS)
def test_timeline_bytes_match_reference_cli(engine, ref, scheme, W, S, L):
    from paper_2205_02473_b200 import replay
    sp = _spec(scheme, W, S, L, L + W)
    g = layered_global_dfg(LayeredModel(sp["fw_dur_us"], sp["bw_dur_us"], sp["tensor_bytes"], 5),
                           synth_cluster(scheme, W, S, 12500.0, 5.0))
    text = timeline_text(g, replay(g)).encode()
    assert text == ref.RefGraph.synth(sp).timeline_json()


@pytest.mark.parametrize("scheme,W,S,L", SPECS)
def test_timeline_bytes_match_reference_cli_on_oracle_schedule(ref, port, scheme, W, S, L):
    """Same bytes with the schedule of the C oracle (CPU, no GPU)."""
    from paper_2205_02473_b200.engine import Csr
    from paper_2205_02473_b200.replay import ScheduleEntry

    class R:
        pass
    sp = _spec(scheme, W, S, L, L + W)
    g = layered_global_dfg(LayeredModel(sp["fw_dur_us"], sp["bw_dur_us"], sp["tensor_bytes"], 5),
                           synth_cluster(scheme, W, S, 12500.0, 5.0))
    o = port.port_replay(Csr.from_dict(g.to_csr()))
    r = R()
    r.schedule = {op.id: ScheduleEntry(int(o["start"][i]), int(o["end"][i]), op.device)
                  for i, op in enumerate(g.ops())}
    assert timeline_text(g, r).encode() == ref.RefGraph.synth(sp).timeline_json()


@pytest.mark.parametrize("scheme,W,S,L", SPECS)
def test_native_timeline_writer_matches_reference(ref, port, tmp_path, scheme, W, S, L):
    """dpro_graph_write_timeline (streamed, for 10^6+-op schedules) writes
    the reference CLI's bytes; candidates built as host-merged deltas carry
    the same comm metadata."""
    from paper_2205_02473_b200.engine import Csr
    from paper_2205_02473_b200.ingest import LayeredBase, layered_graph
    sp = _spec(scheme, W, S, L, L + W)
    m = LayeredModel(sp["fw_dur_us"], sp["bw_dur_us"], sp["tensor_bytes"], 5)
    c = synth_cluster(scheme, W, S, 12500.0, 5.0)
    ng = layered_graph(m, c)
    o = port.port_replay(ng.csr)
    path = tmp_path / "t.json"
    ng.write_timeline(str(path), o["start"], o["end"])
    assert path.read_bytes() == ref.RefGraph.synth(sp).timeline_json()
    # a partition + fusion candidate (host-merged delta) against the Python
    # writer on the same graph (which the reference pins above)
    from paper_2205_02473_b200.replay import ScheduleEntry
    base = LayeredBase(m, c)
    groups = [[0, 1]] + [[i] for i in range(2, L)]
    cand = base.candidates([(groups, [2] + [1] * (L - 2))])[0]
    o2 = port.port_replay(cand.csr)
    cand.write_timeline(str(path), o2["start"], o2["end"])
    g = cand.to_global_dfg(c)

    class R:
        pass
    r = R()
    r.schedule = {op.id: ScheduleEntry(int(o2["start"][i]), int(o2["end"][i]), op.device)
                  for i, op in enumerate(g.ops())}
    assert path.read_text() == timeline_text(g, r)
