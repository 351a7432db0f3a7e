"""Synthetic DFG workloads of BASELINE.json `configs`.

Shape: the reference generator's layered model (proj/src/synth.cpp:200-217):
FW chain, mirrored BW chain, one gradient tensor per layer, UPDATE gated on
its synchronization; one layer per parameter tensor, in forward order.
Tensor bytes are the real fp32 parameter sizes; per-layer FW/BW durations are
total / L x U(0.8, 1.2) (seeded), with totals from PAPER.md:1312-1318
(ResNet-50 FW 34.78 ms / BW 71.34 ms; BERT-base 107.49 / 185.66 ms) and
FLOP-scaled for the other models. Cluster: synth_cluster full mesh,
12,500 B/us (100 Gbps) and 5 us latency (synth.cpp:65-86).
Durations are integer microseconds (the reference's unit).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Any

import numpy as np

# This module imports nothing from the product package at module level:
# bench.py's reference arm loads it by file path (workload_spec,
# op_fusion_mix, partition_specs) to build the SAME workload through the
# reference library alone, without loading libdpro_cuda.so.

F32 = 4


def resnet50_tensors() -> list[int]:
    """161 tensors: 53 conv + 53 BN (gamma, beta) + FC weight/bias."""
    t = [7 * 7 * 3 * 64 * F32, 64 * F32, 64 * F32]
    cin = 64
    for width, blocks in zip((64, 128, 256, 512), (3, 4, 6, 3)):
        for b in range(blocks):
            for k, ci, co in ((1, cin, width), (3, width, width), (1, width, 4 * width)):
                t += [k * k * ci * co * F32, co * F32, co * F32]
            if b == 0:
                t += [cin * 4 * width * F32, 4 * width * F32, 4 * width * F32]
            cin = 4 * width
    t += [2048 * 1000 * F32, 1000 * F32]
    assert len(t) == 161
    return t


def bert_tensors(layers: int, hidden: int, inter: int, vocab: int = 30522,
                 max_pos: int = 512) -> list[int]:
    """Embeddings (5) + 16 per encoder layer + pooler (2)."""
    h = hidden
    t = [vocab * h * F32, max_pos * h * F32, 2 * h * F32, h * F32, h * F32]
    for _ in range(layers):
        for _qkvo in range(4):
            t += [h * h * F32, h * F32]
        t += [h * F32, h * F32, h * inter * F32, inter * F32, inter * h * F32, h * F32,
              h * F32, h * F32]
    t += [h * h * F32, h * F32]
    return t


def vgg16_tensors() -> list[int]:
    cfg = [64, 64, 128, 128, 256, 256, 256, 512, 512, 512, 512, 512, 512]
    t, cin = [], 3
    for co in cfg:
        t += [3 * 3 * cin * co * F32, co * F32]
        cin = co
    for ci, co in ((25088, 4096), (4096, 4096), (4096, 1000)):
        t += [ci * co * F32, co * F32]
    assert len(t) == 32
    return t


def gpt2_medium_tensors() -> list[int]:
    d, t = 1024, [50257 * 1024 * F32, 1024 * 1024 * F32]
    for _ in range(24):
        t += [d * F32, d * F32, d * 3 * d * F32, 3 * d * F32, d * d * F32, d * F32,
              d * F32, d * F32, d * 4 * d * F32, 4 * d * F32, 4 * d * d * F32, d * F32]
    t += [d * F32, d * F32]
    assert len(t) == 292
    return t


def bert_large_units(n_units: int = 152) -> list[int]:
    """391 BERT-large tensors bucketed into contiguous fused units."""
    t = bert_tensors(24, 1024, 4096)
    assert len(t) == 391
    return [int(sum(part)) for part in np.array_split(np.array(t, np.int64), n_units)]


def partition_specs(seed: int, layers: int, n: int, rank: int = 0, tensors_per_cand: int = 8,
                    choices=(1, 2, 4)) -> np.ndarray:
    """[n, L] partition counts: each candidate re-partitions
    `tensors_per_cand` seeded tensors with k in `choices`
    (apply_tensor_partition, optimize.cpp:459-492)."""
    rng = np.random.default_rng([seed, rank])
    pk = np.ones((n, layers), np.int32)
    for c in range(n):
        idx = rng.choice(layers, size=min(tensors_per_cand, layers), replace=False)
        pk[c, idx] = rng.choice(choices, size=len(idx))
    return pk


def op_fusion_mix(seed: int, workers: int, layers: int, n: int, rank: int = 0) -> list[tuple]:
    """BASELINE config 4's per-round candidate mix:
    the recompute candidate (optimize.cpp:819-881), the grad-accum candidate
    (883-959) and n - 2 distinct adjacent op-fusion pairs, each fusing
    FW.l<i>+FW.l<i+1> or BW.l<i+1>+BW.l<i> on ONE worker w<k> -- the
    reference's own apply_op_fusion(g, a, b) candidate (245-318).
    -> [("recompute",), ("grad-accum",), ("opf", k, "FW"|"BW", i), ...]"""
    rng = np.random.default_rng([seed, rank, 4])
    out: list[tuple] = [("recompute",), ("grad-accum",)][:n]
    seen = set()
    while len(out) < n:
        c = ("opf", int(rng.integers(0, workers)), "FW" if rng.random() < 0.5 else "BW",
             int(rng.integers(0, layers - 1)))
        if c not in seen:
            seen.add(c)
            out.append(c)
    return out


def opf_pair(desc: tuple) -> tuple[str, str]:
    """The two op ids apply_op_fusion(g, a, b) fuses for an ("opf", ...) desc."""
    _, k, kind, i = desc
    w = f"w{k}"
    return (f"{w}->FW.l{i}", f"{w}->FW.l{i + 1}") if kind == "FW" else \
        (f"{w}->BW.l{i + 1}", f"{w}->BW.l{i}")


def workload_spec(config: int) -> dict[str, Any]:
    """BASELINE.json configs[config-1] as a plain spec: the layered model,
    the synth_cluster parameters (synth.cpp:65-86) and the candidate mix.
    Keys of the model/cluster part are the reference generator's
    (ref_synth_graph / gen_synthetic)."""
    if config == 1:
        t = resnet50_tensors()
        fw, bw = _durations(34_780, 71_340, len(t), 1)
        s = dict(name="resnet50_ring8", scheme="ring", workers=8, ps_count=0, batch=4096, seed=1,
                 mix="partition",
                 description="ResNet-50 DP DFG, 8-worker ring all-reduce (161 tensors), "
                             "partition candidates")
    elif config == 2:
        t = bert_tensors(12, 768, 3072)
        fw, bw = _durations(107_490, 185_660, len(t), 2)
        s = dict(name="bert_base_ps16x4", scheme="ps", workers=16, ps_count=4, batch=1024, seed=2,
                 mix="partition",
                 description="BERT-base PS DFG, 16 workers / 4 servers (199 tensors), batch of "
                             "1024 candidate replays (each re-partitions 8 tensors, k in {1,2,4})")
    elif config == 3:
        t = vgg16_tensors()
        fw, bw = _durations(132_000, 271_000, len(t), 3)
        s = dict(name="vgg16_ring8", scheme="ring", workers=8, ps_count=0, batch=4096, seed=3,
                 mix="partition",
                 description="VGG-16 ring-8 DFG (32 tensors), 4096 partition candidates/round")
    elif config == 4:
        t = gpt2_medium_tensors()
        fw, bw = _durations(344_000, 594_000, len(t), 4)
        s = dict(name="gpt2_medium_ring64", scheme="ring", workers=64, ps_count=0, batch=1776,
                 seed=4, mix="op_fusion",
                 description="GPT-2 medium 64-worker ring DFG (292 tensors, 4.80M ops), "
                             "op-fusion + recomputation + gradient-accumulation candidates")
    elif config == 5:
        t = bert_large_units()
        fw, bw = _durations(332_000, 575_000, len(t), 5)
        s = dict(name="bert_large_ring128", scheme="ring", workers=128, ps_count=0, batch=8192,
                 seed=5, mix="partition",
                 description="BERT-large 128-worker ring DFG (152 fused units, ~10M ops)")
    else:
        raise ValueError(f"unknown config {config}")
    s.update(layers=len(t), fw_dur_us=fw, bw_dur_us=bw, tensor_bytes=t, update_dur_us=5,
             bandwidth_bytes_per_us=12_500.0, latency_us=5.0)
    return s


def synth_spec(spec: dict) -> dict:
    """The reference generator's spec (ref_synth_graph: synth.cpp + ingest) of a workload."""
    keys = ("layers", "fw_dur_us", "bw_dur_us", "tensor_bytes", "update_dur_us", "scheme",
            "workers", "ps_count", "bandwidth_bytes_per_us", "latency_us")
    return {k: spec[k] for k in keys}


@dataclass
class Workload:
    name: str
    model: Any      # ingest.LayeredModel
    cluster: Any    # graph.ClusterSpec
    batch: int
    description: str
    seed: int
    spec: dict

    @property
    def layers(self) -> int:
        return self.model.layers

    def candidate_partitions(self, n: int, rank: int = 0, tensors_per_cand: int = 8,
                             choices=(1, 2, 4)) -> np.ndarray:
        return partition_specs(self.seed, self.layers, n, rank, tensors_per_cand, choices)

    def op_fusion_mix(self, n: int, rank: int = 0) -> list[tuple]:
        return op_fusion_mix(self.seed, len(self.cluster.workers()), self.layers, n, rank)

    def candidate_deltas(self, base, n: int, rank: int = 0, threads: int = 8,
                         variants: bool = True):
        """The workload's candidate batch as deltas against `base` (a
        LayeredBase of this workload) -> (deltas, descriptions). Config 4:
        op_fusion_mix(); the others: candidate_partitions()."""
        from .ingest import ConcatDeltas, layered_graph_variant
        L = self.layers
        if self.spec["mix"] != "op_fusion":
            pk = self.candidate_partitions(n, rank=rank)
            specs = [([[i] for i in range(L)], pk[c].tolist()) for c in range(n)]
            return base.deltas(specs, threads=threads), [("partition", tuple(r)) for r in pk.tolist()]
        descs = self.op_fusion_mix(n, rank)
        if not variants:  # op-fusion candidates only (measurements)
            descs = [d for d in self.op_fusion_mix(n + 2, rank) if d[0] == "opf"][:n]
        opf = [d for d in descs if d[0] == "opf"]
        fj = np.zeros((len(opf), L - 1), np.uint8)
        bj = np.zeros((len(opf), L - 1), np.uint8)
        for r, (_, wk, kind, i) in enumerate(opf):
            (fj if kind == "FW" else bj)[r, i] = 1
        specs = [([[i] for i in range(L)], [1] * L)] * len(opf)
        parts = []
        variants = [layered_graph_variant(self.model, self.cluster, d[0], 0.5)
                    for d in descs if d[0] != "opf"]
        if variants:
            parts.append(base.deltas_from_graphs(variants, threads=threads))
        if opf:
            parts.append(base.deltas(specs, threads=threads, fw_join=fj, bw_join=bj,
                                     join_worker=[d[1] for d in opf]))
        return ConcatDeltas(parts), descs


def _durations(total_fw_us: float, total_bw_us: float, L: int, seed: int):
    rng = np.random.default_rng(seed)
    fw = np.rint(total_fw_us / L * rng.uniform(0.8, 1.2, L)).astype(np.int64)
    bw = np.rint(total_bw_us / L * rng.uniform(0.8, 1.2, L)).astype(np.int64)
    return fw.tolist(), bw.tolist()


def workload(config: int) -> Workload:
    """BASELINE.json configs[config-1] with the product's model and cluster
    objects."""
    from .graph import synth_cluster
    from .ingest import LayeredModel
    s = workload_spec(config)
    return Workload(s["name"], LayeredModel(s["fw_dur_us"], s["bw_dur_us"], s["tensor_bytes"],
                                            s["update_dur_us"]),
                    synth_cluster(s["scheme"], s["workers"], s["ps_count"],
                                  s["bandwidth_bytes_per_us"], s["latency_us"]),
                    s["batch"], s["description"], s["seed"], s)
