"""reference_search (GPU replays) vs the reference's search() (CPU) on a
layered graph: python tools/greedy_speed.py [WORKERS] [LAYERS]"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    from oracle import oracle
    from paper_2205_02473_b200.graph import synth_cluster
    from paper_2205_02473_b200.greedy import SearchOptions, reference_search
    from paper_2205_02473_b200.ingest import LayeredModel, layered_global_dfg
    W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    L = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    rng = np.random.default_rng(1)
    spec = {"layers": L, "fw_dur_us": rng.integers(50, 400, L).tolist(),
            "bw_dur_us": rng.integers(80, 900, L).tolist(),
            "tensor_bytes": rng.integers(10_000, 3_000_000, L).tolist(), "update_dur_us": 5,
            "scheme": "ring", "workers": W, "ps_count": 0, "bandwidth_bytes_per_us": 1250.0,
            "latency_us": 5.0}
    g = layered_global_dfg(LayeredModel(spec["fw_dur_us"], spec["bw_dur_us"],
                                        spec["tensor_bytes"], 5),
                           synth_cluster("ring", W, 0, 1250.0, 5.0))
    from paper_2205_02473_b200.engine import default_engine
    default_engine()  # CUDA context + library load: once per process, not timed
    t = time.perf_counter()
    ours = reference_search(g, SearchOptions(time_budget_s=600.0))
    t_ours = time.perf_counter() - t
    res = {"ops": g.size(), "ours_s": round(t_ours, 2), "ours": [ours.before_us, ours.after_us,
                                                                 len(ours.strategies)]}
    if oracle.ref_available():
        t = time.perf_counter()
        r = oracle.RefGraph.synth(spec).search({"time_budget_s": 600.0})
        res["reference_s"] = round(time.perf_counter() - t, 2)
        res["reference"] = [r["before_us"], r["after_us"], len(r["strategies"])]
    print(res)


if __name__ == "__main__":
    main()
