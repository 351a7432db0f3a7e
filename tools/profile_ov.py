"""One overlay replay of a config batch (for ncu):
    python tools/profile_ov.py CONFIG B [replays]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    cfg, B = int(sys.argv[1]), int(sys.argv[2])
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    import torch
    from paper_2205_02473_b200.engine import Engine
    from paper_2205_02473_b200.ingest import LayeredBase
    from paper_2205_02473_b200.workloads import workload
    w = workload(cfg)
    base = LayeredBase(w.model, w.cluster)
    deltas, _ = w.candidate_deltas(base, B, threads=16)
    eng = Engine(0)
    eng.set_option("overlay", 1)
    res = eng.resident(base.graph().csr)
    b = eng.delta_batch(res, deltas)
    for _ in range(reps):
        b.replay(want_schedule=True)
        torch.cuda.synchronize()
    print("diag", b.diag(), "stats", b.stats())


if __name__ == "__main__":
    main()
