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

import numpy as np

from .graph import ClusterSpec, synth_cluster
from .ingest import LayeredModel

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


@dataclass
class Workload:
    name: str
    model: LayeredModel
    cluster: ClusterSpec
    batch: int
    description: str
    seed: int

    @property
    def layers(self) -> int:
        return self.model.layers

    def candidate_partitions(self, n: int, rank: int = 0, tensors_per_cand: int = 8,
                             choices=(1, 2, 4)) -> np.ndarray:
        """[n, L] partition counts: each candidate re-partitions
        `tensors_per_cand` seeded tensors with k in `choices`
        (apply_tensor_partition, optimize.cpp:459-492)."""
        rng = np.random.default_rng([self.seed, rank])
        pk = np.ones((n, self.layers), np.int32)
        for c in range(n):
            idx = rng.choice(self.layers, size=min(tensors_per_cand, self.layers), replace=False)
            pk[c, idx] = rng.choice(choices, size=len(idx))
        return pk


def _durations(total_fw_us: float, total_bw_us: float, L: int, seed: int):
    rng = np.random.default_rng(seed)
    fw = np.rint(total_fw_us / L * rng.uniform(0.8, 1.2, L)).astype(np.int64)
    bw = np.rint(total_bw_us / L * rng.uniform(0.8, 1.2, L)).astype(np.int64)
    return fw.tolist(), bw.tolist()


def workload(config: int) -> Workload:
    """BASELINE.json configs[config-1]."""
    if config == 1:
        t = resnet50_tensors()
        fw, bw = _durations(34_780, 71_340, len(t), 1)
        return Workload("resnet50_ring8", LayeredModel(fw, bw, t, 5),
                        synth_cluster("ring", 8, 0, 12_500.0, 5.0), 4096,
                        "ResNet-50 DP DFG, 8-worker ring all-reduce (161 tensors)", 1)
    if config == 2:
        t = bert_tensors(12, 768, 3072)
        fw, bw = _durations(107_490, 185_660, len(t), 2)
        return Workload("bert_base_ps16x4", LayeredModel(fw, bw, t, 5),
                        synth_cluster("ps", 16, 4, 12_500.0, 5.0), 1024,
                        "BERT-base PS DFG, 16 workers / 4 servers (199 tensors), batch of "
                        "1024 candidate replays (each re-partitions 8 tensors, k in {1,2,4})", 2)
    if config == 3:
        t = vgg16_tensors()
        fw, bw = _durations(132_000, 271_000, len(t), 3)
        return Workload("vgg16_ring8", LayeredModel(fw, bw, t, 5),
                        synth_cluster("ring", 8, 0, 12_500.0, 5.0), 4096,
                        "VGG-16 ring-8 DFG (32 tensors), 4096 partition candidates/round", 3)
    if config == 4:
        t = gpt2_medium_tensors()
        fw, bw = _durations(344_000, 594_000, len(t), 4)
        return Workload("gpt2_medium_ring64", LayeredModel(fw, bw, t, 5),
                        synth_cluster("ring", 64, 0, 12_500.0, 5.0), 8,
                        "GPT-2 medium 64-worker ring DFG (292 tensors)", 4)
    if config == 5:
        t = bert_large_units()
        fw, bw = _durations(332_000, 575_000, len(t), 5)
        return Workload("bert_large_ring128", LayeredModel(fw, bw, t, 5),
                        synth_cluster("ring", 128, 0, 12_500.0, 5.0), 8192,
                        "BERT-large 128-worker ring DFG (152 fused units, ~10M ops)", 5)
    raise ValueError(f"unknown config {config}")
