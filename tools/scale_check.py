"""Configs 4/5 (4.7M / ~10M-op DFGs): native build time, GPU replay (one
batch of B candidates) vs the C oracle on the same graph. Usage:
python tools/scale_check.py CONFIG [B]"""
import hashlib
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    cfg = int(sys.argv[1])
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    from oracle import oracle
    from paper_2205_02473_b200.engine import Engine
    from paper_2205_02473_b200.ingest import LayeredBase
    from paper_2205_02473_b200.workloads import workload
    w = workload(cfg)
    t = time.perf_counter()
    base = LayeredBase(w.model, w.cluster)
    bg = base.graph()
    t_base = time.perf_counter() - t
    print(f"config {cfg}: base graph V={bg.n_ops} E={bg.n_edges} D={bg.csr.n_devices} "
          f"built in {t_base:.2f} s", flush=True)
    pk = w.candidate_partitions(B, tensors_per_cand=8)
    specs = [([[i] for i in range(w.layers)], pk[c].tolist()) for c in range(B)]
    t = time.perf_counter()
    deltas = base.deltas(specs, threads=16)
    t_d = time.perf_counter() - t
    eng = Engine(0)
    import os
    if os.environ.get("WARPS"):
        eng.set_option("warps", int(os.environ["WARPS"]))
    res = eng.resident(bg.csr)
    t = time.perf_counter()
    b = eng.delta_batch(res, deltas)
    t_up = time.perf_counter() - t
    import torch
    torch.cuda.synchronize()
    t = time.perf_counter()
    b.replay(want_schedule=True)
    torch.cuda.synchronize()
    t_rep = time.perf_counter() - t
    t = time.perf_counter()
    ms, st, er, s, e = b.results(schedule=True)
    t_d2h = time.perf_counter() - t
    print("pack info [first_missing, not_fast, n_cnt, n_src]:", b.pack_info()[:2].tolist())
    print(f"deltas {t_d:.2f} s, upload+merge+pack {t_up:.2f} s, replay {t_rep * 1e3:.1f} ms "
          f"for {B} candidates ({B / t_rep:.0f} replays/s, "
          f"{B * bg.n_ops / t_rep / 1e9:.2f} G node-updates/s); schedule D2H {t_d2h:.1f} s; "
          f"all ok: {bool((st == 0).all())}; stats {b.stats()}", flush=True)
    # parity of candidate 0 with the C oracle on the host-merged CSR
    g0 = base.candidates(specs[:1], threads=16)[0]
    t = time.perf_counter()
    ref = oracle.port_replay(g0.csr)
    t_port = time.perf_counter() - t
    n0 = int(b.op_off[1])
    ok = ref["T"] == ms[0] and np.array_equal(ref["start"], s[:n0]) and np.array_equal(ref["end"], e[:n0])
    print(f"C oracle: T={ref['T']} in {t_port:.1f} s; GPU T={ms[0]}; start/end equal: {ok}")
    assert ok


if __name__ == "__main__":
    main()
