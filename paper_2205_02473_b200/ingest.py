"""Comm-topology expansion and layered-model graphs.

* `expand_*` mirror proj/src/ingest.cpp:268-384 on the Python graph model
  (small graphs: fixtures, partial_replay tensors).
* `NativeGraph` wraps the C++ CSR generator of libdpro_cuda.so
  (csrc/dfg_gen.cpp) that builds the ingest/partition graphs of
  proj/src/ingest.cpp:187-454 and proj/src/optimize.cpp:459-492 straight in
  index order -- used for the large synthetic workloads.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _native as N
from .engine import Csr
from .errors import Error, TopologyError
from .graph import (ClusterSpec, DeviceId, GlobalDFG, GraphBuilder, Op, OpKind,
                    TensorUnit, base_of_unit_name, fnv1a, round_us)


@dataclass
class CommTopology:
    unit: str
    bytes: int = 0
    part_index: int = 0
    part_count: int = 1
    ps_node: str = ""
    ops: list[Op] = field(default_factory=list)
    edges: list[tuple[str, str]] = field(default_factory=list)
    entry: dict[str, list[str]] = field(default_factory=dict)
    exit: dict[str, list[str]] = field(default_factory=dict)


def _hop_dur(bytes_: int, cluster: ClusterSpec, src: str, dst: str) -> int:
    l = cluster.find_link(src, dst)  # ingest.cpp:37-48
    bw, lat = (l.bandwidth_bytes_per_us, l.latency_us) if l else (1.0, 0.0)
    return round_us(float(bytes_) / bw + lat)


def _comm_op(kind: OpKind, src: str, dst: str, tensor: str, bytes_: int, txn: str,
             dur: int) -> Op:
    return Op(id=f"{kind.name}.{txn}", kind=kind, node=src if kind == OpKind.SEND else dst,
              device=DeviceId.link(src, dst), dur=dur, tensor=tensor, bytes=bytes_,
              transaction=txn)


def expand_ring_allreduce(tensor: str, bytes_: int, cluster: ClusterSpec) -> CommTopology:
    """ingest.cpp:268-315."""
    order = list(cluster.ring_order) or sorted(cluster.workers())
    n = len(order)
    if n < 2:
        raise TopologyError(
            f"degenerate ring: allreduce needs at least 2 workers, got {n}")
    chunks = cluster.chunks_per_tensor if cluster.chunks_per_tensor > 0 else n
    steps = 2 * (n - 1)
    base, rem = divmod(bytes_, chunks) if bytes_ >= 0 else (int(bytes_ / chunks), 0)
    topo = CommTopology(tensor, bytes_)
    for c in range(chunks):
        cb = base + (1 if c < rem else 0)
        prev = None
        for s in range(steps):
            src, dst = order[(c + s) % n], order[(c + s + 1) % n]
            txn = f"{tensor}#c{c}#s{s}#{src}#{dst}"
            snd = _comm_op(OpKind.SEND, src, dst, tensor, cb, txn, 0)
            rcv = _comm_op(OpKind.RECV, src, dst, tensor, cb, txn,
                           _hop_dur(cb, cluster, src, dst))
            topo.edges.append((snd.id, rcv.id))
            if s == 0:
                topo.entry.setdefault(src, []).append(snd.id)
            else:
                topo.edges.append((prev, snd.id))
            if s >= n - 2:
                topo.exit.setdefault(dst, []).append(rcv.id)
            prev = rcv.id
            topo.ops += [snd, rcv]
    for ids in topo.exit.values():
        ids.sort()
    return topo


def ps_node_for(tensor: str, cluster: ClusterSpec) -> str:
    servers = sorted(cluster.ps_nodes())  # ingest.cpp:317-325
    if not servers:
        raise TopologyError("parameter-server scheme requires at least one ps node")
    return servers[fnv1a(tensor) % len(servers)]


def expand_ps(tensor: str, bytes_: int, cluster: ClusterSpec) -> CommTopology:
    """ingest.cpp:327-373."""
    server = ps_node_for(tensor, cluster)
    workers = sorted(cluster.workers())
    if not workers:
        raise TopologyError("parameter-server scheme requires at least one worker")
    topo = CommTopology(tensor, bytes_, ps_node=server)
    push_recvs, pull_sends = [], []
    for w in workers:
        push = f"{tensor}#push#{w}#{server}"
        ps = _comm_op(OpKind.SEND, w, server, tensor, bytes_, push, 0)
        pr = _comm_op(OpKind.RECV, w, server, tensor, bytes_, push,
                      _hop_dur(bytes_, cluster, w, server))
        topo.edges.append((ps.id, pr.id))
        topo.entry.setdefault(w, []).append(ps.id)
        push_recvs.append(pr.id)
        pull = f"{tensor}#pull#{server}#{w}"
        ls = _comm_op(OpKind.SEND, server, w, tensor, bytes_, pull, 0)
        lr = _comm_op(OpKind.RECV, server, w, tensor, bytes_, pull,
                      _hop_dur(bytes_, cluster, server, w))
        topo.edges.append((ls.id, lr.id))
        topo.exit.setdefault(w, []).append(lr.id)
        pull_sends.append(ls.id)
        topo.ops += [ps, pr, ls, lr]
    for pull in pull_sends:
        for push in push_recvs:
            topo.edges.append((push, pull))
    return topo


def expand_tensor(tensor: str, bytes_: int, cluster: ClusterSpec) -> CommTopology:
    if cluster.scheme == "ring":
        return expand_ring_allreduce(tensor, bytes_, cluster)
    return expand_ps(tensor, bytes_, cluster)


def splice(b: GraphBuilder, topo: CommTopology, base: str | None = None) -> None:
    """Adds a topology and hooks it onto <node>->IN./OUT.<base> when those
    ops exist (assemble_global_dfg, ingest.cpp:404-441)."""
    base = base or base_of_unit_name(topo.unit)
    for op in topo.ops:
        b.add_op(op)
    for x, y in topo.edges:
        b.add_edge(x, y)
    unit = TensorUnit(topo.unit, base, topo.bytes, topo.part_index, topo.part_count,
                      topo.ps_node, sorted(op.id for op in topo.ops))
    for node, ids in topo.entry.items():
        vin = f"{node}->IN.{base}"
        if b.has_op(vin):
            for i in ids:
                b.add_edge(vin, i)
            unit.vin[node] = vin
    for node, ids in topo.exit.items():
        vout = f"{node}->OUT.{base}"
        if b.has_op(vout):
            for i in ids:
                b.add_edge(i, vout)
            unit.vout[node] = vout
    b.add_tensor_unit(unit)


# --------------------------------------------------------------------------
# native generator
# --------------------------------------------------------------------------
class NativeGraph:
    """Owning handle of a dpro_graph (host CSR built by csrc/dfg_gen.cpp)."""

    def __init__(self, handle: int):
        if not handle:
            raise Error(N.lib.dpro_graph_last_error().decode())
        self.handle = handle
        s = N.DproCsr()
        N.lib.dpro_graph_csr(handle, C.byref(s))
        self.struct = s
        n, e = s.n_ops, s.n_edges

        def view(p, dt, cnt):
            if cnt == 0:
                return np.zeros(0, dt)
            return np.ctypeslib.as_array(
                C.cast(p, C.POINTER(np.ctypeslib.as_ctypes_type(dt))), (cnt,))

        self.csr = Csr(view(s.dur, np.int64, n), view(s.dev, np.uint16, n),
                       view(s.flags, np.uint8, n), view(s.succ_off, np.uint32, n + 1),
                       view(s.succ, np.uint32, e), view(s.indeg, np.uint32, n),
                       int(s.n_devices))

    def __del__(self):  # pragma: no cover
        if getattr(self, "handle", None):
            N.lib.dpro_graph_free(self.handle)
            self.handle = None

    @property
    def n_ops(self) -> int:
        return self.struct.n_ops

    @property
    def n_edges(self) -> int:
        return self.struct.n_edges

    def op_id(self, i: int) -> str:
        return N.lib.dpro_graph_op_id(self.handle, i).decode()

    def op_kind(self, i: int) -> int:
        return N.lib.dpro_graph_op_kind(self.handle, i)

    def op_ids(self) -> list[str]:
        return [self.op_id(i) for i in range(self.n_ops)]

    def device_strs(self) -> list[str]:
        return [N.lib.dpro_graph_device_str(self.handle, d).decode()
                for d in range(self.csr.n_devices)]

    def write_timeline(self, path: str, start: np.ndarray, end: np.ndarray) -> None:
        """The CLI's timeline.json for a replayed schedule, streamed natively
        (dpro_graph_write_timeline); byte-identical to report.write_timeline."""
        st = np.ascontiguousarray(start, np.int64)
        en = np.ascontiguousarray(end, np.int64)
        if st.size != self.n_ops or en.size != self.n_ops:
            raise ValueError("start/end must cover every op")
        if N.lib.dpro_graph_write_timeline(self.handle, N.ptr(st), N.ptr(en),
                                           str(path).encode()) != N.DPRO_OK:
            raise Error(N.lib.dpro_graph_last_error().decode())

    def to_global_dfg(self, cluster: ClusterSpec | None = None) -> GlobalDFG:
        """Python graph object (small graphs: tests / reference-shaped API)."""
        devs = self.device_strs()
        ids = self.op_ids()
        ops = []
        b = C.c_int64(0)
        for i, id_ in enumerate(ids):
            ds = devs[int(self.csr.dev[i])]
            dev = DeviceId.link(*ds.split(">", 1)) if ">" in ds else DeviceId.compute(ds)
            kind = OpKind(self.op_kind(i))
            node = dev.peer if kind == OpKind.RECV else dev.node  # Op::node of a RECV: receiver
            op = Op(id=id_, kind=kind, node=node, device=dev, dur=int(self.csr.dur[i]))
            unit = N.lib.dpro_graph_comm_info(self.handle, i, C.byref(b))
            if unit is not None:  # comm op: tensor unit, bytes, transaction
                op.tensor, op.bytes, op.transaction = unit.decode(), int(b.value), id_[5:]
            ops.append(op)
        so, su = self.csr.succ_off, self.csr.succ
        succs = [su[so[i]:so[i + 1]].tolist() for i in range(len(ids))]
        return GlobalDFG(ops, succs, {}, cluster or ClusterSpec())


@dataclass
class LayeredModel:
    """SynthSpec's layered model (proj/include/dpro/synth.hpp:32-44)."""
    fw_dur: Sequence[int]
    bw_dur: Sequence[int]
    tensor_bytes: Sequence[int]
    update_dur: int = 5

    @property
    def layers(self) -> int:
        return len(self.fw_dur)

    def struct(self):
        """ctypes view; the arrays live on the returned struct (thread-safe:
        concurrent generator calls each own their copies)."""
        fw = np.ascontiguousarray(self.fw_dur, np.int64)
        bw = np.ascontiguousarray(self.bw_dur, np.int64)
        tb = np.ascontiguousarray(self.tensor_bytes, np.int64)
        P = C.POINTER(C.c_int64)
        st = N.DproLayeredModel(self.layers, fw.ctypes.data_as(P), bw.ctypes.data_as(P),
                                tb.ctypes.data_as(P), int(self.update_dur))
        st._keep = (fw, bw, tb)
        return st


def layered_graph(model: LayeredModel, cluster: ClusterSpec,
                  part_k: Sequence[int] | None = None) -> NativeGraph:
    m = model.struct()
    holder = N.ClusterDescHolder(cluster)
    pk = None if part_k is None else np.ascontiguousarray(part_k, np.int32)
    st = C.c_int32(0)
    h = N.lib.dpro_graph_layered(C.byref(m), C.byref(holder.desc), N.ptr(pk), C.byref(st))
    return NativeGraph(h)


def layered_graph_variant(model: LayeredModel, cluster: ClusterSpec, variant: str,
                          microbatch_scale: float = 0.5,
                          part_k: Sequence[int] | None = None) -> NativeGraph:
    """The layered graph with "recompute" or "grad-accum" applied while
    generating it (dpro_graph_layered_variant) -- the graph
    rewrite.apply_recompute / apply_grad_accum produce, at native speed."""
    m = model.struct()
    holder = N.ClusterDescHolder(cluster)
    pk = None if part_k is None else np.ascontiguousarray(part_k, np.int32)
    st = C.c_int32(0)
    v = {"none": 0, "recompute": 1, "grad-accum": 2}[variant]
    h = N.lib.dpro_graph_layered_variant(C.byref(m), C.byref(holder.desc), N.ptr(pk), v,
                                         float(microbatch_scale), C.byref(st))
    return NativeGraph(h)


def layered_graph_groups(model: LayeredModel, cluster: ClusterSpec,
                         groups: Sequence[Sequence[int]],
                         ks: Sequence[int] | None = None) -> NativeGraph:
    """Tensor-fusion + partition candidate: groups[q] lists the layers fused
    into unit q in fusion order ("g3+g4"), ks[q] its partition count."""
    m = model.struct()
    holder = N.ClusterDescHolder(cluster)
    off = np.zeros(len(groups) + 1, np.int32)
    off[1:] = np.cumsum([len(g) for g in groups])
    mem = np.ascontiguousarray([i for g in groups for i in g], np.int32)
    kk = None if ks is None else np.ascontiguousarray(ks, np.int32)
    st = C.c_int32(0)
    h = N.lib.dpro_graph_layered_groups(C.byref(m), C.byref(holder.desc), len(groups),
                                        N.ptr(off), N.ptr(mem), N.ptr(kk), C.byref(st))
    return NativeGraph(h)


def layered_graphs_groups(model: LayeredModel, cluster: ClusterSpec,
                          specs: Sequence[tuple[Sequence[Sequence[int]], Sequence[int]]],
                          threads: int = 8) -> list[NativeGraph]:
    """Batch of fusion/partition candidates [(groups, ks), ...] built on
    native threads (no Python per candidate)."""
    m = model.struct()
    holder = N.ClusterDescHolder(cluster)
    n = len(specs)
    n_groups = np.array([len(g) for g, _ in specs], np.int32)
    spec_off = np.zeros(n, np.int64)
    spec_off[1:] = np.cumsum(n_groups[:-1])
    sizes = [len(m_) for g, _ in specs for m_ in g]
    group_off = np.zeros(len(sizes) + 1, np.int32)
    group_off[1:] = np.cumsum(sizes)
    members = np.ascontiguousarray([i for g, _ in specs for m_ in g for i in m_], np.int32)
    ks = np.ascontiguousarray([k for _, kk in specs for k in kk], np.int32)
    out = (C.c_void_p * n)()
    rc = N.lib.dpro_graph_layered_groups_batch(C.byref(m), C.byref(holder.desc), n,
                                               N.ptr(n_groups), N.ptr(spec_off),
                                               N.ptr(group_off), N.ptr(members), N.ptr(ks),
                                               threads, out)
    if rc != N.DPRO_OK:
        raise Error(N.lib.dpro_graph_last_error().decode())
    return [NativeGraph(out[i]) for i in range(n)]


class LayeredBase:
    """Base graph for delta construction (dpro_base_layered)."""

    def __init__(self, model: LayeredModel, cluster: ClusterSpec):
        self.model, self.cluster = model, cluster
        self._m = model.struct()
        self._layers = model.layers
        self._holder = N.ClusterDescHolder(cluster)
        st = C.c_int32(0)
        self.handle = N.lib.dpro_base_layered(C.byref(self._m), C.byref(self._holder.desc),
                                              C.byref(st))
        if not self.handle:
            raise Error(N.lib.dpro_graph_last_error().decode())

    def __del__(self):  # pragma: no cover
        if getattr(self, "handle", None):
            N.lib.dpro_base_free(self.handle)
            self.handle = None

    @staticmethod
    def _spec_arrays(specs):
        n = len(specs)
        n_groups = np.array([len(g) for g, _ in specs], np.int32)
        spec_off = np.zeros(n, np.int64)
        spec_off[1:] = np.cumsum(n_groups[:-1])
        sizes = [len(m_) for g, _ in specs for m_ in g]
        group_off = np.zeros(len(sizes) + 1, np.int32)
        group_off[1:] = np.cumsum(sizes)
        members = np.ascontiguousarray([i for g, _ in specs for m_ in g for i in m_], np.int32)
        ks = np.ascontiguousarray([k for _, kk in specs for k in kk], np.int32)
        return n_groups, spec_off, group_off, members, ks

    def _joins(self, n, fw_join, bw_join):
        L = self._layers
        conv = lambda j: None if j is None else np.ascontiguousarray(  # noqa: E731
            np.asarray(j, np.uint8).reshape(n, max(L - 1, 0)))
        return conv(fw_join), conv(bw_join)

    def candidates(self, specs: Sequence[tuple[Sequence[Sequence[int]], Sequence[int]]],
                   threads: int = 8, fw_join=None, bw_join=None) -> list[NativeGraph]:
        """[(groups, ks), ...] -> graphs by delta construction (merged on the
        host); fw_join / bw_join [n, L-1]: op fusion of adjacent FW / BW ops
        on every worker (dpro_graph_from_base_batch_ops)."""
        n = len(specs)
        n_groups, spec_off, group_off, members, ks = self._spec_arrays(specs)
        fj, bj = self._joins(n, fw_join, bw_join)
        out = (C.c_void_p * n)()
        rc = N.lib.dpro_graph_from_base_batch_ops(self.handle, n, N.ptr(n_groups),
                                                  N.ptr(spec_off), N.ptr(group_off),
                                                  N.ptr(members), N.ptr(ks), N.ptr(fj), N.ptr(bj),
                                                  threads, out)
        if rc != N.DPRO_OK:
            raise Error(N.lib.dpro_graph_last_error().decode())
        return [NativeGraph(out[i]) for i in range(n)]


    def deltas(self, specs: Sequence[tuple[Sequence[Sequence[int]], Sequence[int]]],
               threads: int = 8, fw_join=None, bw_join=None, join_worker=None) -> "DeltaSet":
        """[(groups, ks), ...] -> unmerged deltas for Engine.delta_batch
        (fw_join / bw_join as in candidates(); join_worker as in
        deltas_from_arrays())."""
        return self.deltas_from_arrays(*self._spec_arrays(specs), threads=threads,
                                       fw_join=fw_join, bw_join=bw_join,
                                       join_worker=join_worker)

    def deltas_from_graphs(self, graphs: Sequence["NativeGraph"], threads: int = 8) -> "DeltaSet":
        """Any generated graphs (recompute / grad-accum variants, ...) as
        deltas against this base (dpro_base_delta_from_graphs)."""
        n = len(graphs)
        arr = (C.c_void_p * max(1, n))(*[g.handle for g in graphs])
        out = C.c_void_p()
        rc = N.lib.dpro_base_delta_from_graphs(self.handle, arr, n, threads, C.byref(out))
        if rc != N.DPRO_OK:
            raise Error(N.lib.dpro_graph_last_error().decode())
        ds = DeltaSet(out.value, self)
        ds._graphs = list(graphs)
        return ds

    def worker(self, k: int) -> str:
        """Name of the k-th worker (the join_worker ordinal)."""
        name = N.lib.dpro_base_worker(self.handle, k)
        if name is None:
            raise IndexError(k)
        return name.decode()

    def deltas_from_arrays(self, n_groups, spec_off, group_off, members, ks,
                           threads: int = 8, fw_join=None, bw_join=None,
                           join_worker=None) -> "DeltaSet":
        """Same, from the flattened spec arrays of dpro_base_delta_batch;
        join_worker [n]: the worker ordinal the candidate's op-fusion joins
        apply to (-1 = every worker; None = every worker for all)."""
        n = len(n_groups)
        fj, bj = self._joins(n, fw_join, bw_join)
        jw = None if join_worker is None else np.ascontiguousarray(join_worker, np.int32)
        n_groups = np.ascontiguousarray(n_groups, np.int32)
        spec_off = np.ascontiguousarray(spec_off, np.int64)
        group_off = np.ascontiguousarray(group_off, np.int32)
        members = np.ascontiguousarray(members, np.int32)
        ks = np.ascontiguousarray(ks, np.int32)
        out = C.c_void_p()
        if jw is None and not hasattr(N.lib, "dpro_base_delta_batch_ex"):  # older builds
            rc = N.lib.dpro_base_delta_batch_ops(self.handle, n, N.ptr(n_groups),
                                                 N.ptr(spec_off), N.ptr(group_off),
                                                 N.ptr(members), N.ptr(ks), N.ptr(fj),
                                                 N.ptr(bj), threads, C.byref(out))
        else:
            rc = N.lib.dpro_base_delta_batch_ex(self.handle, n, N.ptr(n_groups),
                                                N.ptr(spec_off), N.ptr(group_off),
                                                N.ptr(members), N.ptr(ks), N.ptr(fj), N.ptr(bj),
                                                N.ptr(jw), threads, C.byref(out))
        if rc != N.DPRO_OK:
            raise Error(N.lib.dpro_graph_last_error().decode())
        return DeltaSet(out.value, self)

    def graph(self) -> "BaseGraphView":
        """The base graph's CSR / ids (owned by the base)."""
        return BaseGraphView(N.lib.dpro_base_graph(self.handle), self)


class BaseGraphView(NativeGraph):
    """Non-owning NativeGraph over a base's graph."""

    def __init__(self, handle: int, owner):
        self._owner = owner
        super().__init__(handle)

    def __del__(self):  # pragma: no cover - owned by the base
        self.handle = None


class ConcatDeltas:
    """Several delta sets as one candidate batch (a ctypes dpro_delta array
    over their views; the sets stay alive here). Engine.delta_batch takes it
    like a DeltaSet."""

    def __init__(self, sets):
        self._sets = list(sets)
        items = [(s, i) for s in self._sets for i in range(len(s))]
        self.n = len(items)
        self.array = (N.DproDelta * max(1, self.n))(*[s[i] for s, i in items])
        self._where = items

    def __len__(self) -> int:
        return self.n

    def __getitem__(self, i: int) -> N.DproDelta:
        return self.array[i]

    def device_str(self, cand: int, d: int) -> str:
        s, i = self._where[cand]
        return s.device_str(i, d)


class DeltaSet:
    """Owning handle of a dpro_delta_set (candidates as deltas)."""

    def __init__(self, handle: int, base: LayeredBase):
        self.handle, self._base = handle, base
        self.n = N.lib.dpro_delta_set_size(handle)
        self.array = C.cast(N.lib.dpro_delta_set_deltas(handle),
                            C.POINTER(N.DproDelta * max(1, self.n))).contents

    def __len__(self) -> int:
        return self.n

    def __getitem__(self, i: int) -> N.DproDelta:
        return self.array[i]

    def device_str(self, cand: int, d: int) -> str:
        return N.lib.dpro_delta_set_device_str(self.handle, cand, d).decode()

    def __del__(self):  # pragma: no cover
        if getattr(self, "handle", None):
            N.lib.dpro_delta_set_free(self.handle)
            self.handle = None


def layered_graphs(model: LayeredModel, cluster: ClusterSpec, part_k: np.ndarray,
                   threads: int = 8) -> list[NativeGraph]:
    """Candidate batch: one graph per row of part_k [n, layers]."""
    m = model.struct()
    holder = N.ClusterDescHolder(cluster)
    pk = np.ascontiguousarray(part_k, np.int32)
    n = pk.shape[0]
    out = (C.c_void_p * n)()
    rc = N.lib.dpro_graph_layered_batch(C.byref(m), C.byref(holder.desc), N.ptr(pk), n,
                                        threads, out)
    if rc != N.DPRO_OK:
        raise Error(N.lib.dpro_graph_last_error().decode())
    return [NativeGraph(out[i]) for i in range(n)]


def tsync_graph(cluster: ClusterSpec, bytes_: int, k: int) -> NativeGraph:
    holder = N.ClusterDescHolder(cluster)
    st = C.c_int32(0)
    return NativeGraph(N.lib.dpro_graph_tsync(C.byref(holder.desc), int(bytes_), int(k),
                                              C.byref(st)))


def layered_global_dfg(model: LayeredModel, cluster: ClusterSpec,
                       part_k: Sequence[int] | None = None) -> GlobalDFG:
    """The same layered graph as layered_graph(), built op by op through
    GraphBuilder with full Op fields and tensor units (synth.cpp:200-217 deps
    through build_local_dfg + assemble_global_dfg, ingest.cpp:243-265,
    404-441). Small models only: the graph rewrites of rewrite.py and the
    reference-shaped API take this form; the search uses the native one."""
    b = GraphBuilder()
    b.set_cluster(cluster)
    L = model.layers
    for w in cluster.workers():
        dv = DeviceId.compute(w)
        for i in range(L):
            b.add_op(Op(f"{w}->FW.l{i}", OpKind.FW, w, dv, int(model.fw_dur[i])))
            b.add_op(Op(f"{w}->BW.l{i}", OpKind.BW, w, dv, int(model.bw_dur[i]),
                        produces=[f"g{i}"]))
            b.add_op(Op(f"{w}->UPDATE.l{i}", OpKind.UPDATE, w, dv, int(model.update_dur)))
            b.add_op(Op(f"{w}->IN.g{i}", OpKind.VIRTUAL_IN, w, dv, 0))
            b.add_op(Op(f"{w}->OUT.g{i}", OpKind.VIRTUAL_OUT, w, dv, 0))
        for i in range(L):
            if i > 0:
                b.add_edge(f"{w}->FW.l{i - 1}", f"{w}->FW.l{i}")
            if i + 1 < L:
                b.add_edge(f"{w}->BW.l{i + 1}", f"{w}->BW.l{i}")
            b.add_edge(f"{w}->FW.l{i}", f"{w}->BW.l{i}")
            b.add_edge(f"{w}->BW.l{i}", f"{w}->IN.g{i}")
            b.add_edge(f"{w}->OUT.g{i}", f"{w}->UPDATE.l{i}")
    for i in range(L):
        k = int(part_k[i]) if part_k is not None else 1
        nbytes = int(model.tensor_bytes[i])
        base, rem = divmod(nbytes, k)
        for p in range(k):
            unit = f"g{i}" if k == 1 else f"g{i}#p{p}"
            topo = expand_tensor(unit, base + (1 if p < rem else 0), cluster)
            topo.part_index, topo.part_count = p, k
            splice(b, topo, f"g{i}")
    return b.build()
