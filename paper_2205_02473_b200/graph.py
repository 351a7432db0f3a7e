"""Graph model of the reference, proj/include/dpro/graph.hpp:30-212 and
proj/include/dpro/cluster.hpp:25-65, restricted to what the Replayer path
consumes. GlobalDFG keeps ops in byte-lexicographic id order
(proj/src/graph.cpp:278-297) -- the replay tie-break order -- and compiles to
the CSR the C ABI takes (include/dpro_cuda.h: dpro_csr)."""
from __future__ import annotations

import bisect
import enum
import math
from dataclasses import dataclass, field
from typing import Iterable

import numpy as np

from .errors import LookupError_, TopologyError, TransformError


class OpKind(enum.IntEnum):
    """graph.hpp:30-38 (enumerator order is part of the C ABI)."""
    FW = 0
    BW = 1
    UPDATE = 2
    SEND = 3
    RECV = 4
    VIRTUAL_IN = 5
    VIRTUAL_OUT = 6


def is_computation(k: OpKind) -> bool:
    return k in (OpKind.FW, OpKind.BW, OpKind.UPDATE)


def is_communication(k: OpKind) -> bool:
    return k in (OpKind.SEND, OpKind.RECV)


def is_virtual(k: OpKind) -> bool:
    return k in (OpKind.VIRTUAL_IN, OpKind.VIRTUAL_OUT)


class DeviceKind(enum.IntEnum):
    COMPUTE = 0
    LINK = 1


@dataclass(frozen=True, order=True)
class DeviceId:
    """graph.hpp:57-72; ordering = (kind, node, peer) like operator<=>."""
    kind: DeviceKind = DeviceKind.COMPUTE
    node: str = ""
    peer: str = ""

    @staticmethod
    def compute(node: str) -> "DeviceId":
        return DeviceId(DeviceKind.COMPUTE, node, "")

    @staticmethod
    def link(src: str, dst: str) -> "DeviceId":
        return DeviceId(DeviceKind.LINK, src, dst)

    def str(self) -> str:  # noqa: A003 - reference name
        return self.node if self.kind == DeviceKind.COMPUTE else f"{self.node}>{self.peer}"


@dataclass
class Op:
    """graph.hpp:74-86."""
    id: str
    kind: OpKind = OpKind.FW
    node: str = ""
    device: DeviceId = field(default_factory=DeviceId)
    dur: int = 0
    produces: list[str] = field(default_factory=list)
    tensor: str = ""
    bytes: int = 0
    transaction: str = ""


@dataclass
class TensorUnit:
    """graph.hpp:88-99 (fields the replay path reads)."""
    name: str
    base: str
    bytes: int = 0
    part_index: int = 0
    part_count: int = 1
    ps_node: str = ""
    comm_ops: list[str] = field(default_factory=list)
    vin: dict[str, str] = field(default_factory=dict)
    vout: dict[str, str] = field(default_factory=dict)


# --------------------------------------------------------------------------
# cluster (cluster.hpp:25-65)
# --------------------------------------------------------------------------
@dataclass
class NodeSpec:
    id: str
    machine: str = ""
    role: str = "worker"


@dataclass
class LinkSpec:
    src: str
    dst: str
    bandwidth_bytes_per_us: float = 1.0
    latency_us: float = 0.0


@dataclass
class ClusterSpec:
    scheme: str = "ring"  # "ring" | "ps"  (cluster.cpp:25-33)
    nodes: list[NodeSpec] = field(default_factory=list)
    links: list[LinkSpec] = field(default_factory=list)
    ring_order: list[str] = field(default_factory=list)
    chunks_per_tensor: int = 0

    def workers(self) -> list[str]:
        return [n.id for n in self.nodes if n.role == "worker"]

    def ps_nodes(self) -> list[str]:
        return [n.id for n in self.nodes if n.role == "ps"]

    def find_link(self, src: str, dst: str) -> LinkSpec | None:
        for l in self.links:  # first match wins, cluster.cpp:60-65
            if l.src == src and l.dst == dst:
                return l
        return None

    def check(self) -> None:
        """cluster.cpp:67-114 (topology subset)."""
        ids = [n.id for n in self.nodes]
        if len(set(ids)) != len(ids):
            raise TopologyError("duplicate node id")
        for l in self.links:
            if l.src not in ids or l.dst not in ids:
                raise TopologyError(f"link {l.src}->{l.dst} references unknown node")
            if l.bandwidth_bytes_per_us <= 0.0:
                raise TopologyError(f"link {l.src}->{l.dst} has non-positive bandwidth")
        if self.scheme == "ring":
            w = self.workers()
            if len(w) < 2:
                raise TopologyError(f"degenerate ring: {len(w)} worker(s)")
            if self.ring_order and sorted(self.ring_order) != sorted(w):
                raise TopologyError("ring_order is not a permutation of workers")
        else:
            if not self.ps_nodes():
                raise TopologyError("ps scheme with no ps node")
            if not self.workers():
                raise TopologyError("ps scheme with no worker")

    def to_json(self) -> dict:
        j = {"schema_version": 1, "scheme": self.scheme,
             "nodes": [{"id": n.id, "machine": n.machine or n.id, "role": n.role}
                       for n in self.nodes],
             "links": [{"src": l.src, "dst": l.dst,
                        "bandwidth_bytes_per_us": l.bandwidth_bytes_per_us,
                        "latency_us": l.latency_us} for l in self.links],
             "chunks_per_tensor": self.chunks_per_tensor}
        if self.ring_order:
            j["ring_order"] = list(self.ring_order)
        return j


def synth_cluster(scheme: str, workers: int, ps_count: int,
                  bandwidth_bytes_per_us: float, latency_us: float) -> ClusterSpec:
    """Full mesh, one machine per node (proj/src/synth.cpp:65-86)."""
    c = ClusterSpec(scheme=scheme)
    for i in range(workers):
        c.nodes.append(NodeSpec(f"w{i}", f"w{i}", "worker"))
    if scheme == "ps":
        for i in range(ps_count):
            c.nodes.append(NodeSpec(f"ps{i}", f"ps{i}", "ps"))
    for a in c.nodes:
        for b in c.nodes:
            if a.id != b.id:
                c.links.append(LinkSpec(a.id, b.id, bandwidth_bytes_per_us, latency_us))
    return c


def round_us(value: float) -> int:
    """Round half to even, time_util.hpp:28-35."""
    f = math.floor(value)
    frac = value - f
    lo = int(f)
    if frac > 0.5:
        return lo + 1
    if frac < 0.5:
        return lo
    return lo if lo % 2 == 0 else lo + 1


def fnv1a(text: str) -> int:
    """graph.cpp:57-64."""
    h = 1469598103934665603
    for c in text.encode():
        h ^= c
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def base_of_unit_name(name: str) -> str:
    """graph.cpp:66-73."""
    pos = name.rfind("#p")
    if pos < 0 or pos + 2 == len(name) or not name[pos + 2:].isdigit():
        return name
    return name[:pos]


# --------------------------------------------------------------------------
# GlobalDFG / GraphBuilder (graph.hpp:106-202)
# --------------------------------------------------------------------------
def _op_id(op: "Op") -> str:
    return op.id


class _CsrLists:
    """Per-op index lists held as one CSR (flat, off): list i is sliced out
    on access, so building a graph creates no per-op lists."""
    __slots__ = ("flat_np", "off_np", "flat", "off")

    def __init__(self, flat: np.ndarray, off: np.ndarray):
        self.flat_np, self.off_np = flat, off
        self.flat, self.off = flat.tolist(), off.tolist()

    def __getitem__(self, i: int) -> list[int]:
        return self.flat[self.off[i]:self.off[i + 1]]

    def __len__(self) -> int:
        return len(self.off) - 1

    def __iter__(self):
        fl, o = self.flat, self.off
        return (fl[o[i]:o[i + 1]] for i in range(len(o) - 1))


class GlobalDFG:
    """Immutable graph: ops sorted by id, ascending pred/succ index lists."""

    def __init__(self, ops: list[Op], succs: list[list[int]],
                 tensors: dict[str, TensorUnit], cluster: ClusterSpec,
                 index: dict[str, int] | None = None, edge_count: int | None = None):
        self._ops = ops
        self._index = index if index is not None else {op.id: i for i, op in enumerate(ops)}
        self._succs = succs
        self._preds_cache: list[list[int]] | None = None  # built on first use
        self._edge_count = (edge_count if edge_count is not None
                            else sum(len(s) for s in succs))
        self._tensors = dict(sorted(tensors.items()))
        self._cluster = cluster
        self._csr = None

    @property
    def _preds(self) -> list[list[int]]:
        # ascending: successors are visited in index order
        if self._preds_cache is None:
            sc = self._succs
            if isinstance(sc, _CsrLists):
                # the transpose of the successor CSR: a stable sort of the
                # heads keeps each predecessor list ascending
                n = len(self._ops)
                flat = np.asarray(sc.flat_np, np.int64)
                tails = np.repeat(np.arange(n, dtype=np.int64), np.diff(sc.off_np))
                order = np.argsort(flat, kind="stable")
                off = np.zeros(n + 1, np.int64)
                np.cumsum(np.bincount(flat, minlength=n), out=off[1:])
                self._preds_cache = _CsrLists(tails[order], off)
            else:
                preds: list[list[int]] = [[] for _ in self._ops]
                for a, ss in enumerate(sc):
                    for b in ss:
                        preds[b].append(a)
                self._preds_cache = preds
        return self._preds_cache

    def size(self) -> int:
        return len(self._ops)

    def __len__(self) -> int:
        return len(self._ops)

    def ops(self) -> list[Op]:
        return self._ops

    def has_op(self, id_: str) -> bool:
        return id_ in self._index

    def index_of(self, id_: str) -> int:
        try:
            return self._index[id_]
        except KeyError:
            raise LookupError_(f"no op '{id_}' in graph") from None

    def op(self, id_: str) -> Op:
        return self._ops[self.index_of(id_)]

    def op_at(self, i: int) -> Op:
        return self._ops[i]

    def succ_indices(self, i: int) -> list[int]:
        return self._succs[i]

    def pred_indices(self, i: int) -> list[int]:
        return self._preds[i]

    def succs(self, id_: str) -> list[str]:
        return [self._ops[i].id for i in self._succs[self.index_of(id_)]]

    def preds(self, id_: str) -> list[str]:
        return [self._ops[i].id for i in self._preds[self.index_of(id_)]]

    def has_edge(self, a: str, b: str) -> bool:
        if a not in self._index or b not in self._index:
            return False
        return self._index[b] in self._succs[self._index[a]]

    def edge_count(self) -> int:
        return self._edge_count

    def edge_set(self) -> frozenset:
        """All edges as (pred id, succ id) pairs (cached; the graph is immutable)."""
        if getattr(self, "_edges", None) is None:
            ids = [op.id for op in self._ops]
            self._edges = frozenset((ids[a], ids[b]) for a, ss in enumerate(self._succs)
                                    for b in ss)
        return self._edges

    def cluster(self) -> ClusterSpec:
        return self._cluster

    def tensor_units(self) -> dict[str, TensorUnit]:
        return self._tensors

    def has_tensor_unit(self, name: str) -> bool:
        return name in self._tensors

    def tensor_unit(self, name: str) -> TensorUnit:
        if name not in self._tensors:
            raise LookupError_(f"no tensor unit '{name}' in graph")
        return self._tensors[name]

    def has_base(self, base: str) -> bool:
        return any(u.base == base for u in self._tensors.values())

    def units_of_base(self, base: str) -> list[str]:
        """graph.cpp:119-125 (unit names in name order)."""
        return [n for n, u in self._tensors.items() if u.base == base]

    def base_bytes(self, base: str) -> int:
        units = [u for u in self._tensors.values() if u.base == base]
        if not units:
            raise LookupError_(f"no tensor '{base}' in graph")
        return sum(u.bytes for u in units)

    def fused(self, a: int, b: int, op: Op) -> "GlobalDFG":
        """The graph with ops a and b (indices) replaced by op, which takes
        their predecessors and successors (other than a and b): what
        GraphBuilder(g).remove_ops([a, b]); add_op(op); add_edge(...)
        builds for op fusion (optimize.cpp:245-317), computed on the index
        arrays instead of string-keyed edge sets. op must be on the device
        of a (fusion joins two ops of one device)."""
        ops, n = self._ops, len(self._ops)
        lo, hi = (a, b) if a < b else (b, a)
        keep = ops[:lo] + ops[lo + 1:hi] + ops[hi + 1:]
        pos = bisect.bisect_left(keep, op.id, key=_op_id)
        new_ops = keep[:pos] + [op] + keep[pos:]
        m = np.arange(n, dtype=np.int64)
        m -= (m > lo).astype(np.int64) + (m > hi)
        m += m >= pos
        sc = self._succs
        if isinstance(sc, _CsrLists):
            heads = np.asarray(sc.flat_np, np.int64)
            tails = np.repeat(np.arange(n, dtype=np.int64), np.diff(sc.off_np))
        else:
            heads = np.fromiter((x for ss in sc for x in ss), np.int64, self._edge_count)
            tails = np.repeat(np.arange(n, dtype=np.int64), [len(ss) for ss in sc])
        gone = (tails == a) | (tails == b)
        into = (heads == a) | (heads == b)
        preds = np.unique(tails[into & ~gone])
        succs = np.unique(heads[gone & ~into])
        keep_e = ~(gone | into)
        n2 = n - 1
        key = np.concatenate([m[tails[keep_e]] * n2 + m[heads[keep_e]],
                              m[preds] * n2 + pos, pos * n2 + m[succs]])
        key.sort()
        off = np.zeros(n2 + 1, np.int64)
        np.cumsum(np.bincount(key // n2, minlength=n2), out=off[1:])
        g = GlobalDFG(new_ops, _CsrLists(key % n2, off), self._tensors, self._cluster,
                      {o.id: i for i, o in enumerate(new_ops)}, int(key.size))
        if self._csr is not None:
            c = self._csr
            dindex = {d: i for i, d in enumerate(c["devices"])}
            if op.device in dindex:
                fl = (1 if is_virtual(op.kind) else 0) | (2 if is_communication(op.kind) else 0)
                succ = (key % n2).astype(np.uint32)
                g._csr = {"dur": np.insert(np.delete(c["dur"], [lo, hi]), pos, op.dur),
                          "dev": np.insert(np.delete(c["dev"], [lo, hi]), pos,
                                           dindex[op.device]),
                          "flags": np.insert(np.delete(c["flags"], [lo, hi]), pos, fl),
                          "succ_off": off.astype(np.uint32), "succ": succ,
                          "indeg": np.bincount(succ, minlength=n2).astype(np.uint32),
                          "devices": c["devices"], "n_devices": c["n_devices"]}
        return g

    # ---- CSR for the engine -------------------------------------------
    def devices(self) -> list[DeviceId]:
        """Dense device ids: DeviceId order over all ops."""
        return self.to_csr()["devices"]

    def to_csr(self) -> dict:
        if self._csr is None:
            devs = sorted({op.device for op in self._ops})
            if len(devs) > 65535:
                raise TransformError("more than 65535 devices")
            dindex = {d: i for i, d in enumerate(devs)}
            n = len(self._ops)
            dur = np.fromiter((op.dur for op in self._ops), np.int64, n)
            dev = np.fromiter((dindex[op.device] for op in self._ops), np.uint16, n)
            flags = np.fromiter(
                ((1 if is_virtual(op.kind) else 0) | (2 if is_communication(op.kind) else 0)
                 for op in self._ops), np.uint8, n)
            if isinstance(self._succs, _CsrLists):
                succ_off = self._succs.off_np.astype(np.uint32)
                succ = self._succs.flat_np.astype(np.uint32)
                indeg = np.bincount(succ, minlength=n).astype(np.uint32)
            else:
                succ_off = np.zeros(n + 1, np.uint32)
                succ_off[1:] = np.cumsum([len(s) for s in self._succs], dtype=np.uint64)
                succ = np.fromiter((s for ss in self._succs for s in ss), np.uint32,
                                   self._edge_count)
                indeg = np.fromiter((len(p) for p in self._preds), np.uint32, n)
            self._csr = {"dur": dur, "dev": dev, "flags": flags, "succ_off": succ_off,
                         "succ": succ, "indeg": indeg, "devices": devs,
                         "n_devices": len(devs)}
        return self._csr


class GraphBuilder:
    """Mutable, string-keyed construction buffer (graph.hpp:165-202)."""

    def __init__(self, g: GlobalDFG | None = None):
        self._ops: dict[str, Op] = {}
        self._edges: set[tuple[str, str]] = set()
        self._tensors: dict[str, TensorUnit] = {}
        self._cluster = ClusterSpec()
        self._shared: set[str] = set()  # ops still shared with the source graph
        self._src_ids: list[str] | None = None  # the source graph's op order
        if g is not None:
            self._cluster = g.cluster()
            # copy-on-write: GlobalDFG ops are immutable, so the builder shares
            # them and copies one only when op(id) hands it out for mutation
            for op in g.ops():
                self._ops[op.id] = op
            self._shared = set(self._ops)
            self._src_ids = list(self._ops)  # sorted: build() merges added ids into it
            self._edges = set(g.edge_set())
            self._tensors = dict(g.tensor_units())

    def set_cluster(self, c: ClusterSpec) -> None:
        self._cluster = c

    def add_op(self, op: Op) -> None:
        if not op.id:
            raise TransformError("op with empty id")
        if op.id in self._ops:
            raise TransformError(f"duplicate op id '{op.id}'")
        self._ops[op.id] = op

    def has_op(self, id_: str) -> bool:
        return id_ in self._ops

    def op(self, id_: str) -> Op:
        """The builder's op, mutable (GraphBuilder::op); a shared op is copied
        first so the source graph is never changed."""
        if id_ not in self._ops:
            raise LookupError_(f"no op '{id_}' in builder")
        if id_ in self._shared:
            import copy
            self._ops[id_] = copy.copy(self._ops[id_])
            self._shared.discard(id_)
        return self._ops[id_]

    def remove_op(self, id_: str) -> None:
        self.remove_ops([id_])

    def remove_ops(self, ids) -> None:
        """remove_op for several ops with one pass over the edges."""
        gone = set()
        for id_ in ids:
            if id_ not in self._ops:
                raise LookupError_(f"no op '{id_}' to remove")
            del self._ops[id_]
            self._shared.discard(id_)
            gone.add(id_)
        if gone:
            self._edges = {e for e in self._edges if e[0] not in gone and e[1] not in gone}

    def remove_tensor_unit(self, name: str) -> None:
        if name not in self._tensors:
            raise LookupError_(f"no tensor unit '{name}' to remove")
        del self._tensors[name]

    def preds(self, id_: str) -> list[str]:
        return sorted(a for a, b in self._edges if b == id_)

    def succs(self, id_: str) -> list[str]:
        return sorted(b for a, b in self._edges if a == id_)

    def add_edge(self, a: str, b: str) -> None:
        if a not in self._ops:
            raise LookupError_(f"edge tail '{a}' unknown")
        if b not in self._ops:
            raise LookupError_(f"edge head '{b}' unknown")
        if a == b:
            raise TransformError(f"self edge on '{a}'")
        self._edges.add((a, b))

    def remove_edge(self, a: str, b: str) -> None:
        self._edges.discard((a, b))

    def has_edge(self, a: str, b: str) -> bool:
        return (a, b) in self._edges

    def add_tensor_unit(self, unit: TensorUnit) -> None:
        if unit.name in self._tensors:
            raise TransformError(f"duplicate tensor unit '{unit.name}'")
        self._tensors[unit.name] = unit

    def build(self) -> GlobalDFG:
        ops = self._ops
        if self._src_ids is not None:
            # the source's order minus removed ops, then the added ids:
            # two sorted runs, which sort() merges in linear time
            src = self._src_ids
            ids = [k for k in src if k in ops]
            if len(ids) != len(ops):
                kept = set(ids)
                ids += sorted(k for k in ops if k not in kept)
                ids.sort()
        else:
            ids = sorted(ops)  # std::map order == byte order for str
        index = {k: i for i, k in enumerate(ids)}
        n, m = len(ids), len(self._edges)
        if m:
            # edges -> (tail, head) indices with C-level lookups, one sort of
            # tail * n + head, then ascending per-op lists sliced out of it
            heads, tails = zip(*self._edges)
            key = np.fromiter(map(index.__getitem__, heads), np.int64, m) * n
            key += np.fromiter(map(index.__getitem__, tails), np.int64, m)
            key.sort()
            off = np.zeros(n + 1, np.int64)
            np.cumsum(np.bincount(key // n, minlength=n), out=off[1:])
            succs = _CsrLists(key % n, off)
        else:
            succs = [[] for _ in ids]
        g = GlobalDFG([ops[k] for k in ids], succs, self._tensors, self._cluster, index,
                      len(self._edges))
        g._edges = frozenset(self._edges)  # edge_set() cache for the next builder
        return g


def comp(id_: str, dev: str, dur: int, kind: OpKind = OpKind.FW) -> Op:
    """Test helper of proj/tests/test_replay.cpp:32-41."""
    return Op(id=id_, kind=kind, node=dev, device=DeviceId.compute(dev), dur=dur)


def ops_from(iterable: Iterable[Op]) -> GraphBuilder:
    b = GraphBuilder()
    for op in iterable:
        b.add_op(op)
    return b
