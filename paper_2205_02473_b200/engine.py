"""Batched replay engine: the host side over the C ABI (include/dpro_cuda.h).

`Engine` owns one dpro_ctx (one GPU). `Batch` is a registered set of
candidate CSR graphs (host arrays uploaded once, or device arrays used in
place) that can be replayed repeatedly; results stay on the device until
asked for. This is the interface the search loop drives in bulk; the
reference-shaped single-graph API lives in replay.py.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _native as N
from .errors import EngineError


@dataclass
class Csr:
    """Index-ordered CSR of one DFG (numpy, host)."""
    dur: np.ndarray        # int64 [n]
    dev: np.ndarray        # uint16 [n]
    flags: np.ndarray      # uint8 [n]
    succ_off: np.ndarray   # uint32 [n+1]
    succ: np.ndarray       # uint32 [e]
    indeg: np.ndarray | None
    n_devices: int

    @property
    def n_ops(self) -> int:
        return int(self.dur.shape[0])

    @property
    def n_edges(self) -> int:
        return int(self.succ.shape[0])

    @staticmethod
    def from_dict(d: dict) -> "Csr":
        return Csr(d["dur"], d["dev"], d["flags"], d["succ_off"], d["succ"],
                   d.get("indeg"), int(d["n_devices"]))

    def algorithmic_bytes(self) -> int:
        """B = 32 V + 4 E per replay."""
        return 32 * self.n_ops + 4 * self.n_edges

    def as_struct(self) -> N.DproCsr:
        for a, dt in ((self.dur, np.int64), (self.dev, np.uint16), (self.flags, np.uint8),
                      (self.succ_off, np.uint32), (self.succ, np.uint32)):
            if a.dtype != dt or not a.flags["C_CONTIGUOUS"]:
                raise ValueError(f"CSR array must be contiguous {np.dtype(dt)}")
        return N.DproCsr(self.n_ops, self.n_edges, self.n_devices, 64,
                         N.ptr(self.dur), N.ptr(self.dev), N.ptr(self.flags),
                         N.ptr(self.succ_off), N.ptr(self.succ),
                         N.ptr(self.indeg) if self.indeg is not None else None)


def _check(ctx, rc: int, what: str) -> None:
    if rc != N.DPRO_OK:
        msg = N.lib.dpro_cuda_last_error(ctx).decode(errors="replace")
        raise EngineError(f"{what} failed ({rc}): {msg}")


class Engine:
    """One dpro_ctx on one CUDA device."""

    def __init__(self, device: int = 0):
        self.device = device
        self.ctx = N.lib.dpro_cuda_create(device)
        if not self.ctx:
            raise EngineError(f"dpro_cuda_create({device}) failed: no usable CUDA device")

    def close(self) -> None:
        if self.ctx:
            N.lib.dpro_cuda_destroy(self.ctx)
            self.ctx = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_handle: int | None) -> None:
        _check(self.ctx, N.lib.dpro_cuda_set_stream(self.ctx, stream_handle), "set_stream")

    def set_option(self, key: str, value: int) -> None:
        """'fast' (1 on-chip fast path + exact fallback, 0 general kernel),
        'ring' (fast-path queue capacity per device)."""
        _check(self.ctx, N.lib.dpro_cuda_set_option(self.ctx, key.encode(), int(value)),
               f"set_option({key})")

    def batch(self, cands: Sequence[Csr] | Sequence[N.DproCsr],
              memspace: int = N.DPRO_HOST) -> "Batch":
        return Batch(self, cands, memspace)

    def resident(self, base: Csr | N.DproCsr) -> "Resident":
        """Uploads a base graph that stays in HBM for delta batches."""
        return Resident(self, base)

    def delta_batch(self, resident: "Resident", deltas) -> "Batch":
        """Batch of candidates given as deltas against `resident` (a
        DeltaSet or a ctypes array of N.DproDelta): merged on the GPU."""
        return Batch(self, deltas, N.DPRO_DEVICE, resident=resident)

    def tsync_batch(self, cluster, bytes_: Sequence[int], ks: Sequence[int]) -> "Batch":
        """The comm-only graphs of sync_makespan over a (bytes, k) grid as a
        batch, generated on the GPU (dpro_cuda_batch_create_tsync, K2)."""
        holder = N.ClusterDescHolder(cluster)
        b = np.ascontiguousarray(bytes_, dtype=np.int64)
        k = np.ascontiguousarray(ks, dtype=np.int32)
        h = N.lib.dpro_cuda_batch_create_tsync(self.ctx, C.byref(holder.desc), N.ptr(b), N.ptr(k),
                                               len(b))
        if not h:
            _check(self.ctx, N.DPRO_EINVAL, "batch_create_tsync")
        return Batch.from_handle(self, h, len(b))

    def tsync_grid(self, cluster, bytes_: Sequence[int], ks: Sequence[int]):
        """dpro_cuda_tsync_grid: (makespans, statuses)."""
        holder = N.ClusterDescHolder(cluster)
        b = np.ascontiguousarray(bytes_, dtype=np.int64)
        k = np.ascontiguousarray(ks, dtype=np.int32)
        out = np.zeros(len(b), np.int64)
        st = np.zeros(len(b), np.int32)
        rc = N.lib.dpro_cuda_tsync_grid(self.ctx, C.byref(holder.desc), N.ptr(b), N.ptr(k),
                                        len(b), N.ptr(out), N.ptr(st))
        if rc not in (N.DPRO_OK, N.DPRO_EINVAL):
            _check(self.ctx, rc, "tsync_grid")
        return out, st


class Resident:
    """A base graph resident in HBM (dpro_cuda_resident_create)."""

    def __init__(self, engine: Engine, base):
        self.engine = engine
        self._keep = base
        st = base.as_struct() if isinstance(base, Csr) else base
        self.n_ops = int(st.n_ops)
        self.handle = N.lib.dpro_cuda_resident_create(engine.ctx, C.byref(st))
        if not self.handle:
            _check(engine.ctx, N.DPRO_EINVAL, "resident_create")

    def close(self) -> None:
        if self.handle:
            N.lib.dpro_cuda_resident_destroy(self.engine.ctx, self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


class Batch:
    def __init__(self, engine: Engine, cands, memspace: int, resident: Resident | None = None):
        self.engine = engine
        self._keep = cands if resident is not None else list(cands)
        self._resident = resident  # prepare() re-reads the base graph in HBM
        self.with_schedule = False
        self.handle = None
        if resident is not None:  # delta batch
            arr, n = (cands.array, cands.n) if hasattr(cands, "array") else (cands, len(cands))
            self.n = n
            counts = [(resident.n_ops - arr[i].n_removed + arr[i].n_new, arr[i].n_devices)
                      for i in range(n)]
            self.n_ops = np.array([c[0] for c in counts], np.int64)
            self.n_devices = np.array([c[1] for c in counts], np.int64)
            self.handle = N.lib.dpro_cuda_batch_create_delta(engine.ctx, resident.handle,
                                                             C.cast(arr, C.c_void_p), n)
            if not self.handle:
                _check(engine.ctx, N.DPRO_EINVAL, "batch_create_delta")
            ne = np.zeros(max(1, n), np.uint32)
            N.lib.dpro_cuda_batch_sizes(self.handle, None, N.ptr(ne), None)
            self.n_edges = ne[:n].astype(np.int64)
        else:
            structs = [c.as_struct() if isinstance(c, Csr) else c for c in cands]
            self.n = len(structs)
            self.n_ops = np.array([s.n_ops for s in structs], np.int64)
            self.n_edges = np.array([s.n_edges for s in structs], np.int64)
            self.n_devices = np.array([s.n_devices for s in structs], np.int64)
            arr = (N.DproCsr * max(1, self.n))(*structs)
            self.handle = N.lib.dpro_cuda_batch_create(engine.ctx, arr, self.n, memspace)
            if not self.handle:
                _check(engine.ctx, N.DPRO_EINVAL, "batch_create")
        self.op_off = np.zeros(self.n + 1, np.int64)
        self.op_off[1:] = np.cumsum(self.n_ops)

    @classmethod
    def from_handle(cls, engine: Engine, handle: int, n: int) -> "Batch":
        """A batch the engine built itself (e.g. t_sync graphs on the GPU)."""
        self = cls.__new__(cls)
        self.engine, self._keep, self._resident = engine, None, None
        self.with_schedule = False
        self.handle, self.n = handle, n
        no = np.zeros(max(1, n), np.uint32)
        ne = np.zeros(max(1, n), np.uint32)
        nd = np.zeros(max(1, n), np.uint32)
        N.lib.dpro_cuda_batch_sizes(handle, N.ptr(no), N.ptr(ne), N.ptr(nd))
        self.n_ops = no[:n].astype(np.int64)
        self.n_edges = ne[:n].astype(np.int64)
        self.n_devices = nd[:n].astype(np.int64)
        self.op_off = np.zeros(n + 1, np.int64)
        self.op_off[1:] = np.cumsum(self.n_ops)
        return self

    def close(self) -> None:
        if self.handle:
            N.lib.dpro_cuda_batch_destroy(self.engine.ctx, self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def algorithmic_bytes(self) -> int:
        return int(32 * self.n_ops.sum() + 4 * self.n_edges.sum())

    def prepare(self) -> None:
        """Re-runs the device-side preparation (delta merge, pack) on the
        inputs already in HBM."""
        _check(self.engine.ctx, N.lib.dpro_cuda_batch_prepare(self.engine.ctx, self.handle),
               "batch_prepare")

    def replay(self, want_schedule: bool = True) -> None:
        """Asynchronous on the engine's stream."""
        _check(self.engine.ctx,
               N.lib.dpro_cuda_batch_replay(self.engine.ctx, self.handle, int(want_schedule)),
               "batch_replay")
        self.with_schedule = want_schedule

    def stats(self) -> dict:
        st = np.zeros(5, np.int64)
        _check(self.engine.ctx, N.lib.dpro_cuda_batch_stats(self.engine.ctx, self.handle,
                                                            N.ptr(st)), "batch_stats")
        return {"fallbacks": int(st[0]), "fast_smem_bytes": int(st[1]),
                "fast_blocks_per_sm": int(st[2]), "ring": int(st[3]),
                "deep_ring_retries": int(st[4])}

    def diag(self) -> dict:
        """Why candidates left the residency pass (dpro_cuda_batch_diag)."""
        d = np.zeros(10, np.int64)
        _check(self.engine.ctx, N.lib.dpro_cuda_batch_diag(self.engine.ctx, self.handle,
                                                           N.ptr(d), 10), "batch_diag")
        return {"pass0_ring": int(d[0]), "pass0_rl": int(d[1]), "deep_ring": int(d[2]),
                "deep_rl": int(d[3]), "overlay": bool(d[4]), "materialized": int(d[5]),
                "pass_ms": [round(x / 1e3, 3) for x in d[6:10].tolist()]}

    def pack_info(self) -> np.ndarray:
        """[n, 4]: first op without duration, not-fast bits, multi-pred ops, sources."""
        out = np.zeros((max(1, self.n), 4), np.uint32)
        N.lib.dpro_cuda_batch_pack_info(self.handle, N.ptr(out))
        return out[: self.n]

    def device_results(self) -> dict:
        ps = [C.c_void_p() for _ in range(5)]
        N.lib.dpro_cuda_batch_device_results(self.handle, *[C.byref(p) for p in ps])
        return dict(zip(("makespan", "status", "err", "start", "end"),
                        [p.value for p in ps]))

    def results(self, schedule: bool = False):
        ms = np.zeros(self.n, np.int64)
        st = np.zeros(self.n, np.int32)
        er = np.zeros(self.n, np.int64)
        start = end = None
        if schedule:
            start = np.zeros(int(self.op_off[-1]), np.int64)
            end = np.zeros(int(self.op_off[-1]), np.int64)
        _check(self.engine.ctx,
               N.lib.dpro_cuda_batch_results(self.engine.ctx, self.handle, N.ptr(ms), N.ptr(st),
                                             N.ptr(er), N.ptr(start), N.ptr(end)),
               "batch_results")
        return ms, st, er, start, end

    def timelines(self, cand: int):
        n, d = int(self.n_ops[cand]), int(self.n_devices[cand])
        order = np.zeros(max(n, 1), np.uint32)
        dev_off = np.zeros(d + 1, np.uint32)
        busy = np.zeros(max(d, 1), np.int64)
        _check(self.engine.ctx,
               N.lib.dpro_cuda_batch_timelines(self.engine.ctx, self.handle, cand, N.ptr(order),
                                               N.ptr(dev_off), N.ptr(busy)),
               "batch_timelines")
        return order, dev_off, busy[:d]

    def scheduled(self, cand: int) -> np.ndarray:
        m = np.zeros(max(1, int(self.n_ops[cand])), np.uint8)
        _check(self.engine.ctx,
               N.lib.dpro_cuda_batch_scheduled(self.engine.ctx, self.handle, cand, N.ptr(m)),
               "batch_scheduled")
        return m[: int(self.n_ops[cand])]

    def critical_paths(self):
        """List of per-candidate path index arrays (empty on error status)."""
        paths = np.zeros(max(1, int(self.op_off[-1])), np.uint32)
        lens = np.zeros(self.n, np.int64)
        _check(self.engine.ctx,
               N.lib.dpro_cuda_batch_critical_paths(self.engine.ctx, self.handle, N.ptr(paths),
                                                    N.ptr(lens)),
               "batch_critical_paths")
        return [paths[self.op_off[i]: self.op_off[i] + lens[i]].copy() for i in range(self.n)]


_default: Engine | None = None


def default_engine() -> Engine:
    global _default
    if _default is None:
        _default = Engine(0)
    return _default
