"""Benchmark: batched candidate-DFG replay (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 2] [--batch B]

Workload (N=1 line = BASELINE configs[1]): BERT-base parameter-server DFG,
16 workers / 4 servers, 199 tensors, a batch of 1024 candidate graphs (each
re-partitions 8 seeded tensors with k in {1,2,4}, the reference's
apply_tensor_partition rewrite). Candidates are deltas of
one resident base graph (include/dpro_cuda.h dpro_delta). One step = the
device-side merge of every delta (K0) + the pack kernel + one exact replay
of every candidate (K1: per-op start/end + makespan) + the per-round
best-cost exchange (argmin; NCCL MIN all-reduce across ranks when N > 1),
with the inputs (base graph + deltas) resident in HBM. The per-step working
set (merged CSR + packed records, ~3.9 GB) is larger than L2: no flush.

Multi-GPU: one process per GPU (torchrun), each rank replays its own 1024
candidates (weak scaling); timing is the max over ranks of CUDA-event time.

--impl reference: the reference's own CPU replayer (oracle/_ref, the
unmodified proj/src/replay.cpp) on all host cores, same workload/metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "candidate DFG replays/sec"
UNIT = "replays/s"


def _peak_hbm() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def _ncu_traffic() -> float | None:
    p = ROOT / "profiles" / "ncu_traffic.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["dram_bytes_per_launch"])
        except Exception:
            return None
    return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        for line in (getattr(self, "out", "") or "").strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for name, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                                "sw_power_cap"), f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def build_candidates(config: int, batch: int, rank: int, threads: int):
    from paper_2205_02473_b200.ingest import layered_graphs
    from paper_2205_02473_b200.workloads import workload
    w = workload(config)
    pk = w.candidate_partitions(batch, rank=rank)
    graphs = layered_graphs(w.model, w.cluster, pk, threads=threads)
    return w, graphs


def ref_graphs(graphs, threads: int):
    """The reference's own graph objects (oracle/_ref) for the bounded
    sample, built once per run; None when the reference library is absent."""
    from oracle import oracle
    if not oracle.ref_available():
        return None
    sample = graphs[: max(threads * 2, 8)]
    refs = []
    for g in sample:
        devs = g.device_strs()
        ids = g.op_ids()
        ops = []
        for i, id_ in enumerate(ids):
            ds = devs[int(g.csr.dev[i])]
            if ">" in ds:
                a, b = ds.split(">", 1)
                dk, dn, dp = 1, a, b
            else:
                dk, dn, dp = 0, ds, ""
            ops.append((id_, g.op_kind(i), dk, dn, dp, int(g.csr.dur[i])))
        so, su = g.csr.succ_off, g.csr.succ
        edges = [(ids[i], ids[int(s)]) for i in range(len(ids)) for s in su[so[i]:so[i + 1]]]
        refs.append(oracle.RefGraph.from_ops(ops, edges))
    return refs


def cpu_reference_time(graphs, budget_s: float, threads: int, refs=None):
    """Times the reference replay() (oracle/_ref) on a bounded sample; falls
    back to the C port when the reference library is absent."""
    from oracle import oracle
    sample = graphs[: max(threads * 2, 8)]
    if refs is None:
        refs = ref_graphs(graphs, threads)
    if refs is not None:
        # calibrate: one round of len(refs) replays, then size to the budget
        sec, _ = oracle.ref_replay_bench(refs, len(refs), threads)
        per = sec / len(refs)
        n = int(max(len(refs), min(budget_s / max(per, 1e-9), 100_000)))
        sec, ms = oracle.ref_replay_bench(refs, n, threads)
        return {"value": n / sec, "unit": UNIT, "cores": threads, "kind": "reference",
                "sample": f"{n} dpro::replay() calls over {len(refs)} of the workload's "
                          f"candidate graphs on {threads} std::threads ({sec:.1f} s); graph "
                          f"construction excluded",
                "makespans": ms[: len(refs)].tolist()}
    t0 = time.perf_counter()
    n = 0
    while time.perf_counter() - t0 < budget_s:
        oracle.port_replay(sample[n % len(sample)].csr)
        n += 1
    sec = time.perf_counter() - t0
    return {"value": n / sec, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{n} C-oracle replays (1 thread, {sec:.1f} s)"}


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    w, graphs = build_candidates(args.config, min(args.batch, 4 * threads), 0, threads)
    vals = []
    cpu = None
    per_step = min(args.ref_seconds, 150.0 / max(1, args.warmup + args.steps))
    refs = ref_graphs(graphs, threads)  # once: the steps time only replay()
    for step in range(args.warmup + args.steps):
        cpu = cpu_reference_time(graphs, budget_s=per_step, threads=threads, refs=refs)
        if step >= args.warmup:
            vals.append(cpu["value"])
    value = float(np.mean(vals))
    cpu = {k: v for k, v in cpu.items() if k != "makespans"}
    cpu["value"] = value
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * args.batch / value, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": w.description, "batch": args.batch, "model": w.name,
                   "n_ops": int(np.mean([g.n_ops for g in graphs]))},
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def run_ours(args) -> None:
    import ctypes as C

    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2205_02473_b200 import _native as N
    from paper_2205_02473_b200.engine import Engine
    from paper_2205_02473_b200.ingest import LayeredBase
    from paper_2205_02473_b200.workloads import workload

    threads = max(1, (os.cpu_count() or 8) // max(world, 1))
    w = workload(args.config)
    pk = w.candidate_partitions(args.batch, rank=rank)
    specs = [([[i] for i in range(w.layers)], pk[c].tolist()) for c in range(args.batch)]
    t0 = time.perf_counter()
    base = LayeredBase(w.model, w.cluster)
    deltas = base.deltas(specs, threads=threads)  # candidates as deltas of the base
    t_build = time.perf_counter() - t0
    stream = torch.cuda.current_stream()
    eng = Engine(local)
    eng.set_stream(stream.cuda_stream)
    resident = eng.resident(base.graph().csr)  # base graph: uploaded once, stays in HBM
    batch = eng.delta_batch(resident, deltas)   # deltas uploaded once: inputs in HBM
    algo_bytes = batch.algorithmic_bytes()
    B = batch.n
    mk_view = _device_view(batch.device_results()["makespan"], B, local)

    def exchange():
        # per-round best-cost exchange (K4): argmin over this rank's
        # candidates, one packed int64 MIN all-reduce across ranks
        best = torch.min(mk_view, dim=0)
        key = (best.values << 24) | (rank << 20) | best.indices
        if dist is not None:
            dist.all_reduce(key, op=dist.ReduceOp.MIN)
        return key

    def step():
        batch.prepare()                    # K0 delta merge + pack kernel
        batch.replay(want_schedule=True)   # K1 replay: makespan + per-op start/end
        return exchange()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        for i in range(args.steps):
            ev[i][0].record(stream)
            batch.prepare()
            ev[i][1].record(stream)
            batch.replay(want_schedule=True)
            ev[i][2].record(stream)
            exchange()
            ev[i][3].record(stream)
        torch.cuda.synchronize()
    prep_ms = [e[0].elapsed_time(e[1]) for e in ev]
    kern_ms = [e[1].elapsed_time(e[2]) for e in ev]
    total_ms = ev[0][0].elapsed_time(ev[-1][3])
    if dist is not None:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms, st, er, _, _ = batch.results()
    ok = int((st == 0).sum())
    kstats = batch.stats()

    # e2e through the C ABI with HOST buffers: the search's call
    # (dpro_cuda_replay_delta_batch: H2D of the deltas, merge, pack, replay,
    # D2H of makespan/status/err), and for reference the full-CSR call
    # (dpro_cuda_replay_batch: H2D of every candidate's CSR)
    hm = np.zeros(B, np.int64)
    hs = np.zeros(B, np.int32)
    he = np.zeros(B, np.int64)

    def timed(fn):
        out = []
        for i in range(max(2, min(args.steps, 5)) + 1):
            torch.cuda.synchronize()
            if dist is not None:
                dist.barrier()
            t0 = time.perf_counter()
            assert fn() == 0
            el = time.perf_counter() - t0
            if i > 0:
                out.append(el)
        e = float(np.median(out))
        if dist is not None:
            t = torch.tensor([e], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e = float(t.item())
        return e

    e2e_s = timed(lambda: N.lib.dpro_cuda_replay_delta_batch(
        eng.ctx, resident.handle, C.cast(deltas.array, C.c_void_p), B, N.ptr(hm), N.ptr(hs),
        N.ptr(he)))
    assert np.array_equal(hm, ms), "e2e makespans differ from the device-resident run"
    graphs = base.candidates(specs, threads=threads)  # host-merged full CSRs
    arr = (N.DproCsr * B)(*[g.csr.as_struct() for g in graphs])
    hm2 = np.zeros(B, np.int64)
    full_s = timed(lambda: N.lib.dpro_cuda_replay_batch(eng.ctx, arr, B, N.DPRO_HOST,
                                                        N.ptr(hm2), None, None, N.ptr(hs),
                                                        N.ptr(he)))
    assert np.array_equal(hm2, ms), "full-CSR makespans differ from the delta run"
    h2d = int(sum(_delta_bytes(deltas[i]) for i in range(B)))
    d2h = B * (8 + 4 + 8)

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    peak, peak_src = _peak_hbm()
    kmean = float(np.mean(kern_ms)) / 1e3
    achieved = algo_bytes / kmean / 1e9
    value = world * B * args.steps / (total_ms / 1e3)
    cpu = cpu_reference_time(graphs, budget_s=args.cpu_seconds, threads=os.cpu_count() or 1)
    mk_cpu = cpu.pop("makespans", None)
    if mk_cpu is not None:
        assert mk_cpu == ms[: len(mk_cpu)].tolist(), "GPU makespans differ from the reference"
    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic",
        "config": {"workload": w.description, "model": w.name, "batch_per_gpu": B,
                   "global_batch": B * world, "n_ops_mean": float(batch.n_ops.mean()),
                   "n_edges_mean": float(batch.n_edges.mean()),
                   "parallelism": f"candidates sharded over {world} GPU(s)",
                   "step": "delta merge (K0) + pack + replay (K1, per-op start/end) + "
                           "best-cost exchange, inputs (base graph + deltas) resident in HBM",
                   "l2": "per-step working set (%.2f GB of merged CSR + packed records) "
                         "larger than L2; no flush" % (algo_bytes * 3 / 1e9),
                   "node_updates_per_s": value * float(batch.n_ops.mean()),
                   "prepare_ms_mean": float(np.mean(prep_ms)),
                   "replay_ms_mean": kmean * 1e3,
                   "replay_only_per_s": world * B / kmean,
                   "build_s": round(t_build, 2), "status_ok": ok,
                   "kernel": "replay_fast_kernel (general-path fallbacks: %d)" % kstats["fallbacks"],
                   "fast_smem_bytes_per_candidate": kstats["fast_smem_bytes"],
                   "fast_candidates_per_sm": kstats["fast_blocks_per_sm"]},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": _ncu_traffic(),
                     "kernel": "replay_fast_kernel",
                     "algorithmic_bytes_per_launch": algo_bytes, "peak_source": peak_src,
                     "kernel_ms_mean": kmean * 1e3},
        "cpu_baseline": cpu,
        "e2e": {"value": world * B / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "note": "dpro_cuda_replay_delta_batch with host deltas (H2D + merge + pack + "
                        "replay, makespan-only) per step",
                "full_csr": {"value": world * B / full_s,
                             "h2d_bytes_per_step": int(sum(_packed_bytes(g) for g in graphs)),
                             "note": "dpro_cuda_replay_batch with every candidate's host CSR"}},
        # per step: delta_merge_kernel, pack_kernel, replay_fast_kernel pass 0 +
        # deep-ring pass 1 (profiles/r01_delta_launches.csv)
        "gpu_launches": 4 * args.steps,
        "clocks": clocks,
    }
    print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


def _delta_bytes(d) -> int:
    import ctypes as C
    a = lambda x: (x + 15) & ~15
    nn = d.n_new
    ne = C.cast(d.new_succ_off, C.POINTER(C.c_uint32))[nn] if d.new_succ_off else 0
    return (a(4 * d.n_removed) + a(4 * nn) + a(8 * nn) + a(2 * nn) + a(nn) + a(4 * (nn + 1)) +
            a(4 * ne) + 2 * a(4 * d.n_extra) + a(4 * d.n_cut))


def _packed_bytes(g) -> int:
    n, e = g.n_ops, g.n_edges
    a = lambda x: (x + 15) & ~15
    return a(4 * n) + a(2 * n) + a(n) + a(4 * (n + 1)) + a(4 * e) + a(4 * n)


def _device_view(ptr: int, n: int, device: int):
    """torch int64 tensor aliasing engine-owned device memory (no copy)."""
    import torch

    class _Cai:
        def __init__(self):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i8",
                                             "data": (ptr, False), "version": 3,
                                             "strides": None}
    return torch.as_tensor(_Cai(), device=f"cuda:{device}")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-seconds", type=float, default=10.0)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
