"""memory_pass at BASELINE config-4/5 scale (GPT-2 medium 64-worker ring,
4.8M ops; BERT-large 128-worker ring, 10M ops): base, recompute and
grad-accum graphs generated natively, replayed in one GPU batch, peak memory
by one K5 launch. Usage: python tools/memory_pass_scale.py CONFIG"""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    from paper_2205_02473_b200.engine import Engine
    from paper_2205_02473_b200.memory import ModelMeta
    from paper_2205_02473_b200.rewrite import BudgetError, memory_pass_layered
    from paper_2205_02473_b200.workloads import workload
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    w = workload(cfg)
    L = w.layers
    tb = [int(x) for x in w.model.tensor_bytes]
    act = [4 * x for x in tb]  # activations: 4x the layer's parameter bytes
    meta = ModelMeta({**{f"FW.l{i}": act[i] for i in range(L)},
                      **{f"BW.l{i}": tb[i] for i in range(L)}},
                     {n.id: int(sum(tb)) for n in w.cluster.nodes}, 0.5)
    eng = Engine(0)
    t0 = time.perf_counter()
    _, g, base_peak, base_t = memory_pass_layered(w.model, w.cluster, 0, meta, eng)
    t_base = time.perf_counter() - t0
    out = {"workload": w.description, "ops": g.n_ops, "base_peak_bytes": base_peak,
           "base_makespan_us": base_t, "probe_s": round(t_base, 2)}
    for frac in (0.9, 0.75, 0.5):
        budget = int(base_peak * frac)
        t0 = time.perf_counter()
        try:
            st, g2, pk, t = memory_pass_layered(w.model, w.cluster, budget, meta, eng)
            out[f"budget_{frac}"] = {"applied": str(st.kind) if st else None, "peak": pk,
                                     "makespan_us": t, "ops": g2.n_ops,
                                     "s": round(time.perf_counter() - t0, 2)}
        except BudgetError as e:
            out[f"budget_{frac}"] = {"BudgetError": str(e), "best_peak": e.best_peak_bytes,
                                     "s": round(time.perf_counter() - t0, 2)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
