"""BASELINE config 3: VGG-16 tensor-fusion + tensor-partition MCMC search,
4096 candidates per round, 8-worker ring. Prints one JSON line with per-round
timings (host candidate construction vs GPU replay). Multi-GPU via torchrun:
each rank proposes its own 4096 candidates; the best is agreed with one
NCCL MIN all-reduce + broadcast per round."""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    rounds = int(os.environ.get("ROUNDS", "5"))
    batch = int(os.environ.get("BATCH", "4096"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2205_02473_b200.engine import Engine
    from paper_2205_02473_b200.search import SyncSearch
    from paper_2205_02473_b200.workloads import workload
    w = workload(int(os.environ.get("CONFIG", "3")))
    eng = Engine(local)
    threads = max(1, (os.cpu_count() or 8) // world)
    s = SyncSearch(w.model, w.cluster, eng, kmax=16, beta=0.002, seed=3, threads=threads,
                   dist=dist, rank=rank, guided=float(os.environ.get("GUIDED", "0")),
                   op_fusion=os.environ.get("OPF", "0") == "1")
    # split timing: wrap the batched evaluation
    t_gen = t_gpu = 0.0

    def timed(cuts, kl, fj=None, bj=None):
        nonlocal t_gen, t_gpu
        t0 = time.perf_counter()
        deltas = s.base.deltas_from_arrays(*s._spec_arrays(cuts, kl), threads=threads,
                                           fw_join=fj, bw_join=bj)
        t1 = time.perf_counter()
        b = eng.delta_batch(s.resident, deltas)
        t1b = time.perf_counter()
        b.replay(want_schedule=False)
        ms, st, *_ = b.results()
        t2 = time.perf_counter()
        if os.environ.get("STATS"):
            print(json.dumps({"prepare_s": round(t1b - t1, 4), "replay_s": round(t2 - t1b, 4),
                              **b.stats()}), file=sys.stderr)
        t_gen += t1 - t0
        t_gpu += t2 - t1
        s.log.evaluated += len(ms)
        return ms

    s.evaluate_arrays = timed
    s.step(batch)  # warm-up round
    t_gen = t_gpu = 0.0
    t0 = time.perf_counter()
    for _ in range(rounds):
        s.step(batch)
    el = time.perf_counter() - t0
    if rank == 0:
        print(json.dumps({"workload": w.description, "gpus": world, "rounds": rounds,
                          "candidates_per_round_per_gpu": batch,
                          "round_s": el / rounds,
                          "candidates_per_s": world * batch * rounds / el,
                          "host_construction_s_per_round": t_gen / rounds,
                          "upload_replay_s_per_round": t_gpu / rounds,
                          "initial_makespan_us": s.log.history[0] if s.log.history else None,
                          "best_makespan_us": s.best.makespan,
                          "accepted": s.log.accepted}))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
