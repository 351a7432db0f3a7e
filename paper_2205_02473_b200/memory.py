"""Peak-memory estimate on replayed schedules (proj/include/dpro/memory.hpp,
proj/src/memory.cpp) -- the memory term of the search objective.

    ModelMeta                   memory.cpp:24-69 (json round trip, load/save)
    output_bytes_for(meta, op)  memory.cpp:71-119 (id -> local -> @mb -> RFW.
                                -> '+'-fused fallbacks)
    estimate_peak_memory(g, r, meta)   memory.cpp:122-167, on the GPU (K5)
    estimate_peak_memory_many(graphs, results, metas)  -- batched form

Byte resolution and the MissingMetaError checks are string work on the host
(same order and messages as the reference); the event construction, the
per-node sort and the running-maximum scan run on the schedule already in
HBM (csrc/memory_kernel.cuh). No CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _native as N
from .engine import Batch, _check
from .errors import IoError, MissingMetaError, ParseError
from .graph import GlobalDFG, OpKind


def is_computation(kind: OpKind) -> bool:
    """graph.hpp:43-45."""
    return kind in (OpKind.FW, OpKind.BW, OpKind.UPDATE)


@dataclass
class ModelMeta:
    """memory.hpp:30-45."""
    output_bytes: dict[str, int] = field(default_factory=dict)
    persistent_bytes: dict[str, int] = field(default_factory=dict)
    microbatch_scale: float = 0.5

    def to_json(self) -> dict:
        return {"schema_version": 1, "output_bytes": dict(self.output_bytes),
                "persistent_bytes": dict(self.persistent_bytes),
                "microbatch_scale": self.microbatch_scale}

    @staticmethod
    def from_json(j: dict) -> "ModelMeta":
        m = ModelMeta()
        m.output_bytes = {k: int(v) for k, v in j.get("output_bytes", {}).items()}
        m.persistent_bytes = {k: int(v) for k, v in j.get("persistent_bytes", {}).items()}
        if "microbatch_scale" in j:
            m.microbatch_scale = float(j["microbatch_scale"])
        return m

    @staticmethod
    def load(path: str) -> "ModelMeta":
        try:
            with open(path) as f:
                text = f.read()
        except OSError as e:
            raise IoError(f"cannot open model meta: {path}") from e
        try:
            return ModelMeta.from_json(json.loads(text))
        except json.JSONDecodeError as e:
            raise ParseError(f"invalid model meta in {path}: {e.msg}", e.pos) from e

    def save(self, path: str) -> None:
        try:
            with open(path, "w") as f:
                f.write(json.dumps(self.to_json(), indent=2) + "\n")
        except OSError as e:
            raise IoError(f"cannot write model meta: {path}") from e


def _local_output_bytes(meta: ModelMeta, local: str) -> int:
    """memory.cpp:73-92."""
    v = meta.output_bytes.get(local, -1)
    if v >= 0:
        return v
    at = local.rfind("@mb")
    if at >= 0:
        local = local[:at]
        v = meta.output_bytes.get(local, -1)
        if v >= 0:
            return (v + 1) // 2  # a micro-batch copy carries half the batch
    if local.startswith("RFW."):
        return meta.output_bytes.get("FW." + local[4:], -1)
    return -1


def output_bytes_for(meta: ModelMeta, op) -> int:
    """memory.cpp:96-119; -1 when unresolvable."""
    op_id = op if isinstance(op, str) else op.id
    if op_id in meta.output_bytes:
        return meta.output_bytes[op_id]
    arrow = op_id.find("->")
    local = op_id[arrow + 2:] if arrow >= 0 else op_id
    v = _local_output_bytes(meta, local)
    if v >= 0:
        return v
    if "+" in local:  # fused ops keep their constituents joined with '+'
        total = 0
        for piece in local.split("+"):
            pb = _local_output_bytes(meta, piece)
            if pb < 0:
                return -1
            total += pb
        return total
    return -1


def resolve(g: GlobalDFG, meta: ModelMeta):
    """Host half of memory.cpp:122-157: per-op output bytes and dense
    compute-node index, per-node persistent bytes. Raises MissingMetaError
    in the reference's order (ops first, then nodes in name order)."""
    ops = g.ops()
    n = len(ops)
    op_bytes = np.zeros(n, np.int64)
    op_node = np.full(n, -1, np.int32)
    nodes = sorted({op.node for op in ops if is_computation(op.kind)})
    index = {nd: i for i, nd in enumerate(nodes)}
    for i, op in enumerate(ops):
        if not is_computation(op.kind):
            continue
        op_node[i] = index[op.node]
        b = output_bytes_for(meta, op)
        if b < 0:
            if op.kind != OpKind.UPDATE:
                raise MissingMetaError(f"no output bytes for op {op.id}")
            b = 0
        op_bytes[i] = b
    pers = np.zeros(len(nodes), np.int64)
    for i, nd in enumerate(nodes):
        if nd not in meta.persistent_bytes:
            raise MissingMetaError(f"no persistent bytes for node {nd}")
        pers[i] = meta.persistent_bytes[nd]
    return nodes, op_bytes, op_node, pers


def native_inputs(graph, meta: ModelMeta):
    """resolve() for a generated graph (ingest.NativeGraph), natively:
    (nodes, op_bytes, op_node, persistent) for batch_peak_memory."""
    keys = list(meta.output_bytes)
    karr = (C.c_char_p * max(1, len(keys)))(*[k.encode() for k in keys])
    barr = np.ascontiguousarray([meta.output_bytes[k] for k in keys], np.int64)
    n = graph.n_ops
    op_bytes = np.zeros(max(1, n), np.int64)
    op_node = np.zeros(max(1, n), np.int32)
    nn, miss = C.c_int32(0), C.c_uint32(0)
    rc = N.lib.dpro_graph_memory_inputs(graph.handle, len(keys), karr, N.ptr(barr),
                                        N.ptr(op_bytes), N.ptr(op_node), C.byref(nn),
                                        C.byref(miss))
    if rc != N.DPRO_OK:
        raise MissingMetaError(f"no output bytes for op {graph.op_id(miss.value)}")
    nodes = [N.lib.dpro_graph_memory_node(graph.handle, i).decode() for i in range(nn.value)]
    pers = np.zeros(len(nodes), np.int64)
    for i, nd in enumerate(nodes):
        if nd not in meta.persistent_bytes:
            raise MissingMetaError(f"no persistent bytes for node {nd}")
        pers[i] = meta.persistent_bytes[nd]
    return nodes, op_bytes[:n], op_node[:n], pers


def batch_peak_memory(batch: Batch, op_bytes: np.ndarray, op_node: np.ndarray,
                      n_nodes: np.ndarray, persistent: np.ndarray) -> np.ndarray:
    """K5 on a batch replayed with want_schedule=True. Flat inputs in batch
    order (see include/dpro_cuda.h); returns peaks [sum n_nodes]."""
    op_bytes = np.ascontiguousarray(op_bytes, np.int64)
    op_node = np.ascontiguousarray(op_node, np.int32)
    n_nodes = np.ascontiguousarray(n_nodes, np.int32)
    persistent = np.ascontiguousarray(persistent, np.int64)
    if op_bytes.size != int(batch.op_off[-1]) or op_node.size != op_bytes.size:
        raise ValueError("op_bytes/op_node must cover every op of the batch")
    if n_nodes.size != batch.n or persistent.size != int(n_nodes.sum()):
        raise ValueError("n_nodes/persistent do not match the batch")
    peak = np.zeros(max(1, persistent.size), np.int64)
    _check(batch.engine.ctx,
           N.lib.dpro_cuda_batch_peak_memory(batch.engine.ctx, batch.handle, N.ptr(op_bytes),
                                             N.ptr(op_node), N.ptr(n_nodes), N.ptr(persistent),
                                             N.ptr(peak)),
           "batch_peak_memory")
    return peak[: persistent.size]


def estimate_peak_memory_many(graphs: Sequence[GlobalDFG], results, metas) -> list[dict]:
    """estimate_peak_memory for results of one replay_many() call (one K5
    launch). `metas` is one ModelMeta or one per graph."""
    if not graphs:
        return []
    if isinstance(metas, ModelMeta):
        metas = [metas] * len(graphs)
    batch = results[0]._batch  # noqa: SLF001
    if batch is None or any(r._batch is not batch for r in results):  # noqa: SLF001
        raise ValueError("results must come from one replay_many() call")
    if len(results) != batch.n or any(r._cand != i for i, r in enumerate(results)):  # noqa: SLF001
        raise ValueError("results must cover the whole batch in order")
    parts = [resolve(g, m) for g, m in zip(graphs, metas)]
    peak = batch_peak_memory(batch, np.concatenate([p[1] for p in parts]),
                             np.concatenate([p[2] for p in parts]),
                             np.array([len(p[0]) for p in parts], np.int32),
                             np.concatenate([p[3] for p in parts]))
    out, o = [], 0
    for nodes, *_ in parts:
        out.append({nd: int(peak[o + i]) for i, nd in enumerate(nodes)})
        o += len(nodes)
    return out


def estimate_peak_memory(g: GlobalDFG, result, meta: ModelMeta) -> dict[str, int]:
    """dpro::estimate_peak_memory (memory.hpp:56-58): node -> peak bytes."""
    b = result._batch  # noqa: SLF001
    if b is None:
        raise ValueError("result does not come from this engine's replay()")
    nodes, op_bytes, op_node, pers = resolve(g, meta)
    # the result may be one candidate of a larger batch: pad the others
    # with no computation ops and no nodes
    nb = np.zeros(int(b.op_off[-1]), np.int64)
    nn = np.full(int(b.op_off[-1]), -1, np.int32)
    a = int(b.op_off[result._cand])  # noqa: SLF001
    nb[a:a + op_bytes.size] = op_bytes
    nn[a:a + op_node.size] = op_node
    counts = np.zeros(b.n, np.int32)
    counts[result._cand] = len(nodes)  # noqa: SLF001
    peak = batch_peak_memory(b, nb, nn, counts, pers)
    return {nd: int(peak[i]) for i, nd in enumerate(nodes)}
