"""Replay kernel time vs warps per candidate (config 2, 1024 delta
candidates): python tools/warps_sweep.py [CONFIG]"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    from paper_2205_02473_b200.engine import Engine
    from paper_2205_02473_b200.ingest import LayeredBase
    from paper_2205_02473_b200.workloads import workload
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    w = workload(cfg)
    pk = w.candidate_partitions(1024)
    specs = [([[i] for i in range(w.layers)], pk[c].tolist()) for c in range(1024)]
    base = LayeredBase(w.model, w.cluster)
    eng = Engine(0)
    res = eng.resident(base.graph().csr)
    b = eng.delta_batch(res, base.deltas(specs, threads=16))
    ref = None
    for nw in (0, 1, 2, 4, 8):
        eng.set_option("warps", nw)
        ts = []
        for _ in range(6):
            torch.cuda.synchronize()
            t = time.perf_counter()
            b.replay(want_schedule=True)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t)
        ms = b.results()[0]
        ref = ms if ref is None else ref
        assert np.array_equal(ms, ref)
        print(f"warps {nw}: {np.median(ts[1:]) * 1e3:.2f} ms  stats {b.stats()}")


if __name__ == "__main__":
    main()
