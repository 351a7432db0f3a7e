"""Small driver for ncu: builds a config batch and replays it a few times.

    python tools/profile_replay.py [--config 2] [--batch 1024] [--iters 3]
"""
import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--schedule", type=int, default=1)
    a = ap.parse_args()
    import numpy as np
    from paper_2205_02473_b200.engine import Engine
    from paper_2205_02473_b200.ingest import layered_graphs
    from paper_2205_02473_b200.workloads import workload
    w = workload(a.config)
    graphs = layered_graphs(w.model, w.cluster, w.candidate_partitions(a.batch), threads=16)
    eng = Engine(0)
    import os
    for key in ("warps", "ring", "fast"):
        if os.environ.get("DPRO_" + key.upper()):
            eng.set_option(key, int(os.environ["DPRO_" + key.upper()]))
    b = eng.batch([g.csr for g in graphs])
    for _ in range(a.iters):
        t = time.perf_counter()
        b.replay(bool(a.schedule))
        ms, st, *_ = b.results()
        print(f"replay {1e3 * (time.perf_counter() - t):.2f} ms, ok={int((st == 0).sum())}, "
              f"makespan[0]={ms[0]} V={int(b.n_ops.mean())} stats={b.stats()}")


if __name__ == "__main__":
    main()
