"""Deltas between two GlobalDFGs (include/dpro_cuda.h `dpro_delta`), so any
rewrite of `rewrite.py` (op fusion, tensor fusion, partition, recompute,
grad-accum) can be evaluated against a base graph resident in HBM.

    d = make_delta(base, cand)            # host, O(V + E) dict work
    ds = DeltaList([make_delta(base, c) for c in cands])
    b = engine.delta_batch(engine.resident(Csr.from_dict(base.to_csr())), ds)

An op whose id is in both graphs but whose kind / device / duration changed
is removed and re-added (same id, same position). Base edges between kept
ops that the candidate lacks are `cut`; out-edges of kept ops the base lacks
are `extra`. The candidate's own index order (its sorted ids) is the merge's
order, so replay results equal a replay of `cand` itself.
"""
from __future__ import annotations

import bisect
import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .graph import GlobalDFG, is_communication, is_virtual


@dataclass
class DeltaArrays:
    n_devices: int
    removed: np.ndarray       # u32, ascending base indices
    new_pos: np.ndarray       # u32
    new_dur: np.ndarray       # i64
    new_dev: np.ndarray       # u16
    new_flags: np.ndarray     # u8
    new_succ_off: np.ndarray  # u32 [n_new + 1]
    new_succ: np.ndarray      # u32
    extra_src: np.ndarray     # u32
    extra_dst: np.ndarray     # u32
    cut: np.ndarray           # u32, ascending positions in the base succ array

    def struct(self) -> N.DproDelta:
        p = lambda a: a.ctypes.data if a.size else None  # noqa: E731
        return N.DproDelta(self.n_devices, self.removed.size, p(self.removed), self.new_pos.size,
                           p(self.new_pos), p(self.new_dur), p(self.new_dev), p(self.new_flags),
                           self.new_succ_off.ctypes.data, p(self.new_succ), self.extra_src.size,
                           p(self.extra_src), p(self.extra_dst), self.cut.size, p(self.cut))


def _flags(op) -> int:
    return (N.FLAG_VIRTUAL if is_virtual(op.kind) else 0) | \
        (N.FLAG_COMM if is_communication(op.kind) else 0)


def make_delta(base: GlobalDFG, cand: GlobalDFG) -> DeltaArrays:
    bops, cops = base.ops(), cand.ops()
    bids = [o.id for o in bops]
    bdevs = base.devices()
    dindex = {d: i for i, d in enumerate(bdevs)}
    extra_devs: list = []
    for o in cops:
        if o.device not in dindex:
            dindex[o.device] = len(bdevs) + len(extra_devs)
            extra_devs.append(o.device)
    cindex = {o.id: i for i, o in enumerate(cops)}
    same = np.zeros(len(bops), bool)
    for b, o in enumerate(bops):
        c = cindex.get(o.id)
        if c is not None:
            oc = cops[c]
            same[b] = oc.kind == o.kind and oc.device == o.device and oc.dur == o.dur
    removed = np.flatnonzero(~same).astype(np.uint32)
    kept_ids = {bids[b] for b in np.flatnonzero(same)}
    new = [i for i, o in enumerate(cops) if o.id not in kept_ids]  # candidate order = id order
    new_pos = np.array([bisect.bisect_left(bids, cops[i].id) for i in new], np.uint32)
    new_succ_off = np.zeros(len(new) + 1, np.uint32)
    lists = [cand.succ_indices(i) for i in new]
    new_succ_off[1:] = np.cumsum([len(x) for x in lists], dtype=np.uint64)
    new_succ = np.array([t for x in lists for t in x], np.uint32)
    # edges out of kept base ops: cut (base-only) and extra (candidate-only)
    bso = base.to_csr()["succ_off"]
    cut, xs, xd = [], [], []
    for b in np.flatnonzero(same).tolist():
        c = cindex[bids[b]]
        csucc = set(cand.succ_indices(c))
        bsucc_final = set()
        for k, s in enumerate(base.succ_indices(b)):
            if same[s]:
                f = cindex[bids[s]]
                if f in csucc:
                    bsucc_final.add(f)
                else:
                    cut.append(int(bso[b]) + k)
        for t in sorted(csucc - bsucc_final):
            xs.append(b)
            xd.append(t)
    return DeltaArrays(
        len(bdevs) + len(extra_devs), removed, new_pos,
        np.array([cops[i].dur for i in new], np.int64),
        np.array([dindex[cops[i].device] for i in new], np.uint16),
        np.array([_flags(cops[i]) for i in new], np.uint8),
        new_succ_off, new_succ, np.array(xs, np.uint32), np.array(xd, np.uint32),
        np.array(sorted(cut), np.uint32))


class DeltaList:
    """A ctypes dpro_delta array over DeltaArrays (kept alive here); pass to
    Engine.delta_batch like a DeltaSet."""

    def __init__(self, deltas: list[DeltaArrays]):
        self._keep = deltas
        self.n = len(deltas)
        self.array = (N.DproDelta * max(1, self.n))(*[d.struct() for d in deltas])

    def __len__(self) -> int:
        return self.n

    def __getitem__(self, i: int) -> N.DproDelta:
        return self.array[i]
