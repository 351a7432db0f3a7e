"""Benchmark: batched candidate-DFG replay (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 4] [--batch B]

Workload (default: BASELINE configs[3], the largest single-GPU config):
GPT-2 medium 64-worker ring-all-reduce DFG (292 tensors, 4.80M ops, 6.0M
edges, 128 devices) and its per-round candidate mix:
the recompute candidate, the grad-accum candidate and 1774 single-worker
adjacent op-fusion pairs -- 1776 candidates per GPU, all resident at once
(12 per SM, 2-warp CTAs; ~170 GB of schedules and timelines).
Candidates are deltas of one resident base graph (include/dpro_cuda.h
dpro_delta), replayed on the base's packed layout plus per-candidate
overlays (csrc/overlay.h). One step = the overlay upload + one exact replay
of every candidate (K1: per-op start/end + makespan) + the per-round
best-cost exchange (argmin; two NCCL MIN all-reduces across ranks when
N > 1), with the inputs (base graph + overlays) resident in HBM. The step's
working set is far larger than L2: no flush needed. Smaller configs
(--config 1-3) use per-candidate merged copies (delta merge K0 + pack)
instead of overlays.

Multi-GPU: one process per GPU (torchrun), each rank replays its own batch
(weak scaling); time is the max over ranks of CUDA-event time.

--impl reference: the reference's own CPU replayer (oracle/_ref: the
unmodified proj/src, compiled by oracle/Makefile) on all host cores, over
the same workload's candidates built by the reference's own generator and
rewrites (RefGraph.synth + apply_op_fusion / apply_strategy); it never
imports the product package.
"""
from __future__ import annotations

import argparse
import importlib.util
import json
import os
import platform
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


def _specs_module():
    """paper_2205_02473_b200/workloads.py loaded by path: the workload
    definitions without importing the product package (no libdpro_cuda.so)."""
    p = ROOT / "paper_2205_02473_b200" / "workloads.py"
    spec = importlib.util.spec_from_file_location("_bench_workloads", p)
    mod = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = mod  # dataclasses resolve their module here
    spec.loader.exec_module(mod)
    return mod


def bench_config(spec: dict, batch: int, world: int) -> dict:
    """The `config` object -- identical in both arms."""
    return {"workload": spec["description"], "model": spec["name"],
            "batch_per_gpu": batch, "global_batch": batch * world,
            "parallelism": f"candidates sharded over {world} GPU(s)",
            "l2": "working set (merged CSRs, packed records, schedules) far larger than L2; "
                  "no flush"}


def _cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def _peak_hbm() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def _ncu_traffic(config: int) -> dict | None:
    """DRAM bytes per launch of the replay kernel from the committed
    `ncu --set full` capture of this config (profiles/ncu_traffic.json)."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get(f"config{config}")
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
                 "--format=csv,noheader,nounits", "-lms", "20"],
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


# --------------------------------------------------------------------------
# the reference, built and run through oracle/_ref only
# --------------------------------------------------------------------------
def ref_sample_graphs(specs_mod, spec: dict, descs: list[tuple], log=print):
    """The reference's own graphs for `descs`: RefGraph.synth (the reference
    generator: synth.cpp + ingest) and the reference rewrites
    (apply_op_fusion, apply_strategy kRecompute / kGradAccum, apply_partition)."""
    from oracle import oracle
    t0 = time.perf_counter()
    base = oracle.RefGraph.synth(specs_mod.synth_spec(spec))
    log(f"reference synth: {base.n_ops} ops in {time.perf_counter() - t0:.1f} s")
    out = []
    for d in descs:
        t1 = time.perf_counter()
        if d[0] == "recompute":
            g = base.apply_memory_strategy(3, {})
        elif d[0] == "grad-accum":
            g = base.apply_memory_strategy(4, {})
        elif d[0] == "opf":
            g = base.op_fusion(*specs_mod.opf_pair(d))
        else:  # ("partition", ks)
            g = base
            for i, k in enumerate(d[1]):
                if k != 1:
                    g = g.partition(f"g{i}", int(k))
        out.append(g)
        log(f"reference candidate {d}: {g.n_ops} ops in {time.perf_counter() - t1:.1f} s")
    return out, time.perf_counter() - t0


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    S = _specs_module()
    spec = S.workload_spec(args.config)
    B = args.batch or spec["batch"]
    threads = os.cpu_count() or 1
    if spec["mix"] == "op_fusion":
        descs = S.op_fusion_mix(spec["seed"], spec["workers"], spec["layers"], B, 0)
        # the reference's apply_strategy(kGradAccum) on the 4.8M-op graph did
        # not finish within 40 min on the GPU box's host: the sample is the
        # recompute candidate and op-fusion pairs (1,478 of the 1,480)
        descs = [d for d in descs if d[0] != "grad-accum"]
        n_sample = args.ref_sample or 4
    else:
        pk = S.partition_specs(spec["seed"], spec["layers"], B, 0)
        descs = [("partition", tuple(r)) for r in pk.tolist()]
        n_sample = args.ref_sample or max(8, 2 * threads)
    sample = descs[:n_sample]  # config 4: recompute, grad-accum, then op fusion
    from oracle import oracle
    graphs, build_s = ref_sample_graphs(S, spec, sample, log=lambda m: print(m, file=sys.stderr))
    # replays per step: every thread busy for graphs that fit the caches; a
    # config-4 graph (4.8M ops, ~12 GB of std::map-based GlobalDFG) is DRAM
    # bound on the host -- 16 concurrent replays take as long as 16 serial
    # ones -- so there a step replays each sample graph once, one per thread
    big = spec["mix"] == "op_fusion"
    per_step = len(graphs) if big else max(threads, len(graphs))
    threads = min(threads, per_step)
    vals, step_ms = [], []
    for step in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        sec, ms = oracle.ref_replay_bench(graphs, per_step, threads)
        wall = time.perf_counter() - t0
        if step >= args.warmup:
            vals.append(per_step / sec)
            step_ms.append(1e3 * wall)
    value = float(np.mean(vals))
    cpu = {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
           "sample": f"each step: {per_step} dpro::replay() calls on {threads} std::threads over "
                     f"{len(graphs)} of the workload's candidates ({[d[0] for d in sample]}), "
                     f"built by the reference's generator + rewrites in {build_s:.0f} s "
                     f"(excluded)",
           "cpu_model": _cpu_model()}
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": float(np.mean(step_ms)), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": bench_config(spec, B, args.gpus),
        "cpu_baseline": cpu,
        "reference_makespans": [int(x) for x in ms[: len(graphs)]],
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def cpu_reference_sample(S, spec, descs, gpu_ms: np.ndarray, threads: int, budget_s: float):
    """cpu_baseline of our line: the reference replay (oracle/_ref) timed on a
    bounded sample of this batch's candidates, built by the reference; its
    makespans must equal the GPU's for the same candidates."""
    from oracle import oracle
    if not oracle.ref_available():
        return None, "oracle/_ref/libdpro_ref.so absent"
    big = spec["mix"] == "op_fusion"
    idx = [2, 3] if big and len(descs) > 3 else list(range(min(len(descs), max(8, threads))))
    graphs, build_s = ref_sample_graphs(S, spec, [descs[i] for i in idx],
                                        log=lambda m: print(m, file=sys.stderr))
    # single thread: one replay
    sec1, ms1 = oracle.ref_replay_bench(graphs[:1], 1, 1)
    # all threads: as many concurrent replays as fit the budget
    n = len(graphs) if big else max(len(graphs), int(budget_s / max(sec1, 1e-9)) * threads)
    n = max(n, min(threads, len(graphs)))
    secp, msp = oracle.ref_replay_bench(graphs, n, min(threads, n))
    ok = all(int(msp[k]) == int(gpu_ms[idx[k % len(idx)]]) for k in range(len(graphs)))
    assert ok, f"GPU makespans differ from the reference: {msp[:len(graphs)]} vs {gpu_ms[idx]}"
    per_thread = 1.0 / sec1
    used = min(threads, n)
    measured = n / secp
    out = {"value": measured, "unit": UNIT,
           "cores": used, "kind": "reference", "cpu_model": _cpu_model(),
           "single_thread_replays_per_s": per_thread,
           "sample": (f"reference dpro::replay() on candidates {idx} of this batch, built by "
                      f"the reference's generator + rewrites ({build_s:.0f} s, excluded); "
                      f"1 replay on 1 thread: {sec1:.1f} s; {n} replays on {used} threads: "
                      f"{secp:.1f} s ({measured:.3f}/s)" +
                      ("; more threads do not help: a 4.8M-op reference graph is DRAM bound "
                       "on the host" if big else "")),
           "parity": f"reference makespans {[int(x) for x in msp[:len(graphs)]]} == GPU"}
    return out, None


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------
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
    from paper_2205_02473_b200.exchange import exchange_best
    from paper_2205_02473_b200.ingest import LayeredBase
    from paper_2205_02473_b200.workloads import workload

    threads = max(1, (os.cpu_count() or 8) // max(world, 1))
    w = workload(args.config)
    B = args.batch or w.batch
    t0 = time.perf_counter()
    base = LayeredBase(w.model, w.cluster)
    deltas, descs = w.candidate_deltas(base, B, rank=rank, threads=threads)
    t_build = time.perf_counter() - t0
    stream = torch.cuda.current_stream()
    eng = Engine(local)
    eng.set_stream(stream.cuda_stream)
    # multi-million-op graphs: replay on the resident base + per-candidate
    # overlays (csrc/overlay.h) instead of a merged copy per candidate
    overlay = w.spec["layers"] * w.spec["workers"] * w.spec["workers"] > 1_000_000
    eng.set_option("overlay", 1 if overlay else 0)
    resident = eng.resident(base.graph().csr)  # base graph: uploaded once, stays in HBM
    batch = eng.delta_batch(resident, deltas)   # deltas uploaded once: inputs in HBM
    algo_bytes = batch.algorithmic_bytes()
    mk_view = _device_view(batch.device_results()["makespan"], B, local)
    dev = f"cuda:{local}"

    def exchange():
        # per-round best-cost exchange (K4): argmin over this rank's
        # candidates, then MIN makespan / MIN (rank, index) across ranks
        best = torch.min(mk_view, dim=0)
        if dist is not None:
            return exchange_best(dist, int(best.values), int(best.indices), rank, dev)
        return best

    for _ in range(args.warmup):
        batch.prepare()
        batch.replay(want_schedule=True)
        exchange()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        for i in range(args.steps):
            ev[i][0].record(stream)
            batch.prepare()                    # K0 delta merge + pack kernel
            ev[i][1].record(stream)
            batch.replay(want_schedule=True)   # K1 replay: makespan + per-op start/end
            ev[i][2].record(stream)
            exchange()
            ev[i][3].record(stream)
        torch.cuda.synchronize()
    prep_ms = [e[0].elapsed_time(e[1]) for e in ev]
    kern_ms = [e[1].elapsed_time(e[2]) for e in ev]
    total_ms = ev[0][0].elapsed_time(ev[-1][3])
    if dist is not None:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms, st, er, _, _ = batch.results()
    ok = int((st == 0).sum())
    assert ok == B, f"{B - ok} candidates failed"
    kstats = batch.stats()
    kdiag = batch.diag()
    n_ops_mean = float(batch.n_ops.mean())
    n_edges_mean = float(batch.n_edges.mean())
    batch.close()  # the e2e call below allocates its own batch

    # e2e through the C ABI with HOST buffers: the search's call
    # (dpro_cuda_replay_delta_batch: H2D of the deltas, merge, pack, replay,
    # D2H of makespan/status/err)
    hm = np.zeros(B, np.int64)
    hs = np.zeros(B, np.int32)
    he = np.zeros(B, np.int64)

    def timed(fn, reps):
        out = []
        for i in range(reps + 1):
            torch.cuda.synchronize()
            if dist is not None:
                dist.barrier()
            t0 = time.perf_counter()
            rc = fn()
            assert rc == 0, f"e2e call failed ({rc}): {N.lib.dpro_cuda_last_error(eng.ctx)}"
            el = time.perf_counter() - t0
            if i > 0:
                out.append(el)
        e = float(np.median(out))
        if dist is not None:
            t = torch.tensor([e], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e = float(t.item())
        return e

    e2e_s = timed(lambda: N.lib.dpro_cuda_replay_delta_batch(
        eng.ctx, resident.handle, C.cast(deltas.array, C.c_void_p), B, N.ptr(hm), N.ptr(hs),
        N.ptr(he)), max(2, min(args.steps, 3)))
    assert np.array_equal(hm, ms), "e2e makespans differ from the device-resident run"
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
    cpu, why = (None, "skipped (--cpu-seconds 0)" if world == 1 else
                "measured at N=1 only (rank 0 of a single-GPU run)")
    if args.cpu_seconds > 0 and world == 1:
        S = _specs_module()
        cpu, why = cpu_reference_sample(S, S.workload_spec(args.config), descs, ms,
                                        os.cpu_count() or 1, args.cpu_seconds)
    traffic = _ncu_traffic(args.config)
    clocks = clk.summary()
    n_ops = n_ops_mean
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic",
        "config": bench_config(w.spec, B, world),
        "details": {
            "candidates": {k: sum(1 for d in descs if d[0] == k)
                           for k in sorted({d[0] for d in descs})},
            "n_ops_mean": n_ops, "n_edges_mean": n_edges_mean,
            "engine": "overlay batches (resident base + per-candidate overlays)" if overlay
                      else "delta merge + pack per candidate",
            "pass_ms_last_step": kdiag["pass_ms"],
            "step": ("overlay upload + replay (K1 on base + overlays, per-op start/end) + "
                     "best-cost exchange, inputs (base graph + overlays) resident in HBM"
                     if overlay else
                     "delta merge (K0) + pack + replay (K1, per-op start/end) + best-cost "
                     "exchange, inputs (base graph + deltas) resident in HBM"),
            "node_updates_per_s": value * n_ops,
            "prepare_ms_mean": float(np.mean(prep_ms)),
            "replay_ms_mean": kmean * 1e3,
            "replay_only_per_s": world * B / kmean,
            "build_s": round(t_build, 2), "status_ok": ok,
            "kernel": "%s (general/materialized hand-offs: %d)" % (
                "replay_ov_kernel" if overlay else "replay_fast_kernel", kstats["fallbacks"]),
            "fast_smem_bytes_per_candidate": kstats["fast_smem_bytes"],
            "fast_candidates_per_sm": kstats["fast_blocks_per_sm"],
            "deep_ring_candidates": kstats["deep_ring_retries"]},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak,
                     "traffic": traffic["dram_bytes_per_launch"] if traffic else None,
                     "traffic_source": traffic.get("source") if traffic else None,
                     "kernel": "replay_ov_kernel" if overlay else "replay_fast_kernel",
                     "algorithmic_bytes_per_launch": algo_bytes,
                     "algorithmic_bytes": "32 V + 4 E per candidate (BASELINE.md section 2)",
                     "peak_source": peak_src, "kernel_ms_mean": kmean * 1e3},
        "cpu_baseline": cpu if cpu is not None else {"value": None, "unit": UNIT,
                                                     "cores": 0, "kind": "reference",
                                                     "sample": why},
        "e2e": {"value": world * B / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "note": ("dpro_cuda_replay_delta_batch with host deltas per step: overlay build on "
                         "host threads + H2D + replay (makespan only) + D2H" if overlay else
                         "dpro_cuda_replay_delta_batch with host deltas per step: H2D + merge + "
                         "pack + replay (makespan only) + D2H")},
        # per step -- overlay: replay_ov_kernel x4 (global-ring side pass,
        # residency pass, deep-ring pass, global-ring pass); merged: delta
        # merge, pack, replay_fast_kernel x3 + the general hand-off
        # (profiles/r02_*launches.csv)
        "gpu_launches": (4 if overlay else 6) * args.steps,
        "clocks": clocks,
    }
    print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


def _delta_bytes(d) -> int:
    import ctypes as C
    a = lambda x: (x + 15) & ~15  # noqa: E731
    nn = d.n_new
    ne = C.cast(d.new_succ_off, C.POINTER(C.c_uint32))[nn] if d.new_succ_off else 0
    return (a(4 * d.n_removed) + a(4 * nn) + a(8 * nn) + a(2 * nn) + a(nn) + a(4 * (nn + 1)) +
            a(4 * ne) + 2 * a(4 * d.n_extra) + a(4 * d.n_cut))


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
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--batch", type=int, default=0, help="candidates per GPU (0: the config's)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0,
                    help="cpu_baseline budget (0: skip)")
    ap.add_argument("--ref-sample", type=int, default=0,
                    help="reference arm: candidate graphs built through oracle/_ref")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
