"""StrategySearch (op fusion + recompute + grad-accum + tensor fusion +
partition) on a GPT-2-medium-shaped layered graph scaled to fit host
rewrites: LAYERS layers (default 24), WORKERS-worker ring (default 4).
Prints one JSON line: per-round host rewrite / delta / GPU time."""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    from paper_2205_02473_b200.engine import Engine
    from paper_2205_02473_b200.graph import synth_cluster
    from paper_2205_02473_b200.ingest import LayeredModel, layered_global_dfg
    from paper_2205_02473_b200.memory import ModelMeta
    from paper_2205_02473_b200.search import StrategySearch
    from paper_2205_02473_b200.workloads import gpt2_medium_tensors
    L = int(os.environ.get("LAYERS", "24"))
    W = int(os.environ.get("WORKERS", "4"))
    rounds = int(os.environ.get("ROUNDS", "5"))
    batch = int(os.environ.get("BATCH", "64"))
    t = gpt2_medium_tensors()
    tb = [int(sum(t[i::L])) for i in range(L)]  # tensors folded onto L layers
    rng = np.random.default_rng(4)
    m = LayeredModel(rng.integers(8000, 16000, L).tolist(), rng.integers(15000, 30000, L).tolist(),
                     tb, 5)
    g = layered_global_dfg(m, synth_cluster("ring", W, 0, 12_500.0, 5.0))
    eng = Engine(0)
    s = StrategySearch(g, eng, meta=ModelMeta(microbatch_scale=0.5), seed=1, beta=0.001)
    t_rw = t_ev = 0.0
    orig_p, orig_e = s.propose, s.evaluate

    def prop(n):
        nonlocal t_rw
        t0 = time.perf_counter()
        out = orig_p(n)
        t_rw += time.perf_counter() - t0
        return out

    def ev(graphs):
        nonlocal t_ev
        t0 = time.perf_counter()
        out = orig_e(graphs)
        t_ev += time.perf_counter() - t0
        return out

    s.propose, s.evaluate = prop, ev
    s.step(batch)
    t_rw = t_ev = 0.0
    t0 = time.perf_counter()
    for _ in range(rounds):
        s.step(batch)
    el = time.perf_counter() - t0
    print(json.dumps({"workload": f"GPT-2-medium-shaped layered DFG, {L} layers, {W}-worker ring, "
                                  f"{g.size()} ops", "rounds": rounds, "batch": batch,
                      "round_s": el / rounds, "host_rewrite_s_per_round": t_rw / rounds,
                      "delta_upload_replay_s_per_round": t_ev / rounds,
                      "initial_makespan_us": s.log.history[0], "best_makespan_us": s.best[1],
                      "applied": [str(x.kind) for x in s.best[2]]}))


if __name__ == "__main__":
    main()
