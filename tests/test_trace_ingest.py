"""trace_ingest.ingest_bundle against the reference's ingest_bundle
(proj/src/ingest.cpp:452-493) on the reference generator's own trace
bundles: identical graphs row by row (ids, kinds, devices, durations,
edges)."""
import pytest

from golden_io import dfg_rows, rows_digest
from paper_2205_02473_b200.graph import synth_cluster
from paper_2205_02473_b200.trace_ingest import DependencySpec, TraceEvent, ingest_bundle

SPECS = [("ring", 2, 0, 2, 100.0, [10, 20], [30, 40], [1000, 2000]),
         ("ring", 4, 0, 5, 12500.0, [120, 80, 300, 50, 90], [200, 150, 600, 90, 100],
          [1_000_000, 30_000, 4_000_000, 7, 250_000]),
         ("ps", 3, 2, 4, 1250.0, [100, 200, 300, 400], [150, 250, 350, 450],
          [10_000, 20_000, 30_000, 40_000])]


@pytest.mark.parametrize("scheme,W,S,L,bw,fw,bwd,tb", SPECS)
def test_ingest_bundle_matches_reference(ref, scheme, W, S, L, bw, fw, bwd, tb):
    from golden.make_golden import ref_rows
    spec = {"layers": L, "fw_dur_us": fw, "bw_dur_us": bwd, "tensor_bytes": tb,
            "update_dur_us": 5, "scheme": scheme, "workers": W, "ps_count": S,
            "bandwidth_bytes_per_us": bw, "latency_us": 5.0}
    bundle = ref.ref_synth_bundle(spec)
    events = [TraceEvent.from_dict(e) for e in bundle["events"]]
    deps = DependencySpec.from_json(bundle["deps"])
    g = ingest_bundle(events, deps, synth_cluster(scheme, W, S, bw, 5.0))
    assert rows_digest(dfg_rows(g)) == rows_digest(ref_rows(ref.RefGraph.synth(spec)))


@pytest.mark.parametrize("seed", range(6))
def test_ingest_noisy_multi_iteration_bundles(ref, seed):
    """Bundles with several iterations and jittered durations / starts:
    mean durations (round half even), RECV service time after its SEND,
    missing SENDs -- against the reference's ingest_bundle on the same
    bundle."""
    import numpy as np
    from golden.make_golden import ref_rows
    rng = np.random.default_rng(seed)
    scheme, W, S = [("ring", 3, 0), ("ps", 3, 2), ("ring", 4, 0)][seed % 3]
    L = int(rng.integers(2, 5))
    spec = {"layers": L, "fw_dur_us": rng.integers(10, 300, L).tolist(),
            "bw_dur_us": rng.integers(10, 600, L).tolist(),
            "tensor_bytes": rng.integers(1000, 2_000_000, L).tolist(), "update_dur_us": 5,
            "scheme": scheme, "workers": W, "ps_count": S,
            "bandwidth_bytes_per_us": 1250.0, "latency_us": 5.0}
    base = ref.ref_synth_bundle(spec)
    events = []
    for it in range(3):
        for e in base["events"]:
            if e["kind"] == 3 and rng.random() < 0.1:
                continue  # a missing SEND: the RECV keeps its own start
            d = dict(e)
            d["iteration"] = it
            d["dur"] = max(0, int(e["dur"]) + int(rng.integers(-3, 4)))
            d["start"] = int(e["start"]) + it * 100_000 + int(rng.integers(0, 3))
            events.append(d)
    bundle = {"events": events, "deps": base["deps"]}
    cluster = synth_cluster(scheme, W, S, 1250.0, 5.0)
    g = ingest_bundle([TraceEvent.from_dict(e) for e in events],
                      DependencySpec.from_json(base["deps"]), cluster)
    exp = ref.RefGraph.ingest(bundle, cluster.to_json())
    assert rows_digest(dfg_rows(g)) == rows_digest(ref_rows(exp))
