"""The reference's search driver (greedy.reference_search, optimize.cpp:
1327-1650 with coarsening / symmetry off) against the reference's own
search(): the same strategies in the same order (kind, operands, k, fused
durations) and the same before/after iteration times."""
import numpy as np
import pytest

from paper_2205_02473_b200.graph import synth_cluster
from paper_2205_02473_b200.ingest import LayeredModel, layered_global_dfg

CASES = [("ring", 4, 0, 6, 1250.0, 3), ("ring", 3, 0, 8, 500.0, 5), ("ps", 3, 2, 6, 1250.0, 7),
         ("ring", 4, 0, 5, 12500.0, 9),
         # PS graphs where partition, op fusion and tensor fusion are all accepted
         ("ps", 4, 2, 4, 300.0, 1), ("ps", 4, 2, 6, 100.0, 2), ("ps", 4, 2, 4, 2000.0, 2)]


def _spec(scheme, W, S, L, bw, seed):
    rng = np.random.default_rng(seed)
    return {"layers": L, "fw_dur_us": rng.integers(50, 400, L).tolist(),
            "bw_dur_us": rng.integers(80, 900, L).tolist(),
            "tensor_bytes": rng.integers(10_000, 3_000_000, L).tolist(), "update_dur_us": 5,
            "scheme": scheme, "workers": W, "ps_count": S, "bandwidth_bytes_per_us": bw,
            "latency_us": 5.0}


@pytest.mark.gpu
@pytest.mark.parametrize("scheme,W,S,L,bw,seed", CASES)
@pytest.mark.parametrize("theorems,full", [(True, False), (False, False), (True, True),
                                           (False, True)])
def test_reference_search_matches_reference(engine, ref, scheme, W, S, L, bw, seed, theorems,
                                            full):
    """full: the reference's default options (coarsening + symmetry
    replication on); else its ablation switches off."""
    from paper_2205_02473_b200.greedy import SearchOptions, reference_search
    sp = _spec(scheme, W, S, L, bw, seed)
    g = layered_global_dfg(LayeredModel(sp["fw_dur_us"], sp["bw_dur_us"], sp["tensor_bytes"], 5),
                           synth_cluster(scheme, W, S, bw, 5.0))
    opts = {"time_budget_s": 600.0, "use_coarsen": full, "use_symmetry": full,
            "use_theorems": theorems, "kmax": 8}
    exp = ref.RefGraph.synth(sp).search(opts)
    got = reference_search(g, SearchOptions(time_budget_s=600.0, use_theorems=theorems, kmax=8,
                                            use_coarsen=full, use_symmetry=full))
    assert got.before_us == exp["before_us"]
    assert [{"kind": str(s.kind), "a": s.a, "b": s.b, "k": s.k, "dur_us": s.dur_us}
            for s in got.strategies] == exp["strategies"]
    assert got.after_us == exp["after_us"]
