"""Replay-path statistics for op-fusion candidates (fallbacks, deep-ring
retries, timing). python tools/opf_stats.py CONFIG P [B]"""
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
    cfg, p = int(sys.argv[1]), float(sys.argv[2])
    B = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
    w = workload(cfg)
    L = w.layers
    base = LayeredBase(w.model, w.cluster)
    rng = np.random.default_rng(0)
    specs = [([[i] for i in range(L)], [1] * L)] * B
    fj = (rng.random((B, L - 1)) < p).astype(np.uint8)
    bj = (rng.random((B, L - 1)) < p).astype(np.uint8)
    eng = Engine(0)
    res = eng.resident(base.graph().csr)
    b = eng.delta_batch(res, base.deltas(specs, threads=16, fw_join=fj, bw_join=bj))
    for _ in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        b.replay(want_schedule=False)
        torch.cuda.synchronize()
        el = time.perf_counter() - t
    info = b.pack_info()
    print(f"config {cfg} p={p}: replay {el * 1e3:.2f} ms for {B}; stats {b.stats()}; "
          f"not_fast values {np.unique(info[:, 1]).tolist()}")


if __name__ == "__main__":
    main()
