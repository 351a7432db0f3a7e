"""t_sync grid (sync_makespan / partial_replay) on the GPU vs the reference's
values (golden vectors from the compiled reference; test_optimize.cpp:265-291
and SURVEY Appendix A Z5/Z6 are among them)."""
import hashlib

import numpy as np
import pytest

from golden_io import synth_vectors, tsync_vectors
from paper_2205_02473_b200 import (Error, GraphBuilder, LookupError_, TensorUnit, partial_replay,
                                   replay, sync_makespan, sync_makespan_grid)
from paper_2205_02473_b200.engine import Csr
from paper_2205_02473_b200.graph import DeviceId, Op, OpKind, synth_cluster
from paper_2205_02473_b200.ingest import LayeredModel, expand_ps, layered_graph, splice

pytestmark = pytest.mark.gpu


def test_tsync_golden_grid():
    clusters, cases = tsync_vectors()
    by_cluster = {}
    for c in cases:
        by_cluster.setdefault(c["cluster"], []).append(c)
    for name, cs in by_cluster.items():
        got = sync_makespan_grid(clusters[name], [c["bytes"] for c in cs], [c["k"] for c in cs])
        assert got == [c["expect"] for c in cs], name


def test_partition_grid_pipeline_schedule():
    c = synth_cluster("ps", 1, 1, 1.0, 0.0)
    assert [sync_makespan(c, 100, k) for k in (1, 2, 3, 4)] == [200, 150, 134, 125]
    with pytest.raises(Error, match="partition count must be >= 1"):
        sync_makespan(c, 100, 0)


def _ps_fixture():
    """test_replay.cpp:472-490: one worker, one server, 1 B/us, 100 B tensor."""
    c = synth_cluster("ps", 1, 1, 1.0, 0.0)
    b = GraphBuilder()
    b.set_cluster(c)
    b.add_op(Op("w0->BW.a", OpKind.BW, "w0", DeviceId.compute("w0"), 10))
    b.add_op(Op("w0->IN.g0", OpKind.VIRTUAL_IN, "w0", DeviceId.compute("w0"), 0))
    b.add_op(Op("w0->OUT.g0", OpKind.VIRTUAL_OUT, "w0", DeviceId.compute("w0"), 0))
    b.add_edge("w0->BW.a", "w0->IN.g0")
    splice(b, expand_ps("g0", 100, c))
    return b.build()


def test_partial_replay_of_ps_tensor():
    g = _ps_fixture()
    assert partial_replay(g, "g0", 1) == 200
    assert partial_replay(g, "g0", 2) == 150
    with pytest.raises(LookupError_):
        partial_replay(g, "nope", 1)
    with pytest.raises(Error):
        partial_replay(g, "g0", 0)
    assert replay(g).iteration_time_us == 210


@pytest.mark.parametrize("fast", [1, 0])
def test_ingest_built_graphs_on_gpu(engine, fast):
    engine.set_option("fast", fast)
    vs = synth_vectors()
    graphs = []
    for v in vs:
        s = v["spec"]
        c = synth_cluster(s["scheme"], s["workers"], s["ps_count"], s["bandwidth_bytes_per_us"],
                          s["latency_us"])
        graphs.append(layered_graph(LayeredModel(s["fw_dur_us"], s["bw_dur_us"],
                                                 s["tensor_bytes"], s["update_dur_us"]), c,
                                    v["part_k"]))
    batch = engine.batch([g.csr for g in graphs])
    batch.replay(True)
    ms, st, er, start, end = batch.results(schedule=True)
    paths = batch.critical_paths()
    for i, v in enumerate(vs):
        a, b = int(batch.op_off[i]), int(batch.op_off[i + 1])
        assert st[i] == 0 and ms[i] == v["T"]
        d = hashlib.sha256(np.concatenate([start[a:b], end[a:b]]).astype("<i8").tobytes())
        assert d.hexdigest() == v["schedule_sha256"]
        assert paths[i].tolist() == v["path"]
    if fast:
        assert batch.stats()["fallbacks"] <= len(vs)  # ring queues > 4 deep fall back
    engine.set_option("fast", 1)


@pytest.mark.parametrize("scheme,W,S,bw,lat,ks", [
    ("ring", 12, 0, 1.0, 0.0, [1, 2, 10, 11, 12]),
    ("ring", 4, 0, 33.0, 2.5, [1, 3, 16]),
    ("ps", 3, 2, 1.0, 0.5, [1, 2, 11, 12]),
    ("ps", 16, 4, 12500.0, 5.0, [1, 4, 7]),
    ("ps", 1, 1, 1.0, 0.0, [1, 2, 3, 4])])
def test_device_generated_tsync_graphs_match_host(engine, port, scheme, W, S, bw, lat, ks):
    """K2: the graphs generated on the GPU (dpro_cuda_batch_create_tsync)
    replay to the same schedule, position by position (so the same index
    order, devices and durations), as the host generator's graphs replayed
    by the C oracle; the grid API agrees with the host-built path."""
    from paper_2205_02473_b200.graph import synth_cluster
    from paper_2205_02473_b200.ingest import tsync_graph
    c = synth_cluster(scheme, W, S, bw, lat)
    grid = [(b, k) for b in (1, 100, 4096, 123457) for k in ks]
    b = engine.tsync_batch(c, [x for x, _ in grid], [k for _, k in grid])
    b.replay(want_schedule=True)
    ms, st, _, start, end = b.results(schedule=True)
    for i, (by, k) in enumerate(grid):
        g = tsync_graph(c, by, k)
        o = port.port_replay(g.csr)
        a, z = int(b.op_off[i]), int(b.op_off[i + 1])
        assert st[i] == 0 and ms[i] == o["T"], (by, k)
        assert z - a == g.n_ops and int(b.n_edges[i]) == g.n_edges
        assert np.array_equal(start[a:z], o["start"]) and np.array_equal(end[a:z], o["end"])
        order, dev_off, busy = b.timelines(i)
        assert int(b.n_devices[i]) == g.csr.n_devices
    engine.set_option("tsync_host", 1)
    try:
        host, _ = engine.tsync_grid(c, [x for x, _ in grid], [k for _, k in grid])
    finally:
        engine.set_option("tsync_host", 0)
    dev, _ = engine.tsync_grid(c, [x for x, _ in grid], [k for _, k in grid])
    assert np.array_equal(host, dev) and np.array_equal(dev, ms)
