"""Overlay vs materialized delta batches on a config (timing + equality).

    python tools/overlay_bench.py CONFIG B [iters]
"""
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    cfg, B = int(sys.argv[1]), int(sys.argv[2])
    iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    import torch
    from paper_2205_02473_b200.engine import Engine
    from paper_2205_02473_b200.ingest import LayeredBase
    from paper_2205_02473_b200.workloads import workload
    w = workload(cfg)
    base = LayeredBase(w.model, w.cluster)
    t = time.perf_counter()
    deltas, descs = w.candidate_deltas(base, B, threads=16,
                                       variants=not os.environ.get("NO_VARIANTS"))
    print(f"deltas {time.perf_counter() - t:.2f} s", flush=True)
    eng = Engine(0)
    for key in ("ring", "warps", "deep_first", "gring0"):
        if os.environ.get("DPRO_" + key.upper()):
            eng.set_option(key, int(os.environ["DPRO_" + key.upper()]))
    res = eng.resident(base.graph().csr)
    out = {}
    for ov in ((1, 0) if not os.environ.get("MAT_ONLY") else (0,)):
        if ov == 0 and (B > 296 or os.environ.get('OV_ONLY')):
            continue
        eng.set_option("overlay", ov)
        t = time.perf_counter()
        b = eng.delta_batch(res, deltas)
        torch.cuda.synchronize()
        tc = time.perf_counter() - t
        for it in range(iters):
            t = time.perf_counter()
            b.prepare()
            torch.cuda.synchronize()
            tp = time.perf_counter() - t
            t = time.perf_counter()
            b.replay(want_schedule=True)
            torch.cuda.synchronize()
            tr = time.perf_counter() - t
            print(f"overlay={ov} B={B}: create {tc:.2f} s, prepare {tp * 1e3:.1f} ms, replay "
                  f"{tr * 1e3:.1f} ms -> {B / (tp + tr):.0f} replays/s (replay only "
                  f"{B / tr:.0f}/s); stats {b.stats()} diag {b.diag()}", flush=True)
        ms, st, *_ = b.results()
        out[ov] = ms
        print("status ok", int((st == 0).sum()), "of", B, flush=True)
        del b
    if 0 in out:
        n = min(len(out[0]), len(out[1]))
        print("overlay == materialized makespans:", bool(np.array_equal(out[0][:n], out[1][:n])))


if __name__ == "__main__":
    main()
