"""TEST INFRASTRUCTURE ONLY -- the checkers for the CUDA Replayer.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
arm may import this module, and only as the checker or the timed CPU
baseline; the product package never does.

Two oracles:
* `ref`   -- the UNMODIFIED reference library (proj/src/*.cpp compiled by
             oracle/Makefile into oracle/_ref/libdpro_ref.so) behind the
             extern "C" shim oracle/ref_capi.cpp. Ground truth.
* `port`  -- oracle/replay_oracle.c, a plain-C restatement of
             proj/src/replay.cpp:37-226 over CSR (oracle/liboracle.so).
             Pinned against `ref` and the reference's golden vectors by
             tests/test_oracle.py.
"""
from __future__ import annotations

import ctypes as C
import json
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SO = HERE / "_ref" / "libdpro_ref.so"
PORT_SO = HERE / "liboracle.so"

_P, _I32, _I64 = C.c_void_p, C.c_int32, C.c_int64
_ref = None
_port = None


def _ptr(a):
    return None if a is None else a.ctypes.data


def ref_available() -> bool:
    return REF_SO.exists()


def port_available() -> bool:
    return PORT_SO.exists()


def ref_lib():
    global _ref
    if _ref is None:
        lib = C.CDLL(str(REF_SO))
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_last_cycle_len": (_I64, []),
            "ref_last_cycle_id": (C.c_char_p, [_I64]),
            "ref_graph_from_arrays": (_P, [_I64, _P, _P, _P, _P, _P, _P, _I64, _P, _P, _P]),
            "ref_synth_graph": (_P, [C.c_char_p, _P]),
            "ref_apply_partition": (_P, [_P, C.c_char_p, _I32, _P]),
            "ref_apply_tensor_fusion": (_P, [_P, C.c_char_p, C.c_char_p, _P]),
            "ref_apply_op_fusion": (_P, [_P, C.c_char_p, C.c_char_p, _I64, _P]),
            "ref_with_durations": (_P, [_P, _P, _P]),
            "ref_graph_free": (None, [_P]),
            "ref_graph_num_ops": (_I64, [_P]),
            "ref_graph_num_edges": (_I64, [_P]),
            "ref_graph_num_devices": (_I32, [_P]),
            "ref_graph_op_id": (C.c_char_p, [_P, _I64]),
            "ref_graph_device_str": (C.c_char_p, [_P, _I32]),
            "ref_graph_device_kind": (_I32, [_P, _I32]),
            "ref_graph_hash": (C.c_uint64, [_P]),
            "ref_graph_export": (None, [_P, _P, _P, _P, _P, _P, _P]),
            "ref_replay": (_I32, [_P, _P, _P, _P, _P, _P]),
            "ref_critical_path": (_I32, [_P, _P, _P, _P, _P, _P, _P, _P, _P]),
            "ref_execution_graph_edges": (_I64, [_P]),
            "ref_sync_makespan": (_I32, [C.c_char_p, _I64, _I32, _P]),
            "ref_peak_memory": (_I32, [_P, C.c_char_p, _P, _P]),
            "ref_peak_node": (C.c_char_p, [_I32]),
            "ref_apply_memory_strategy": (_P, [_P, _I32, C.c_char_p, _P]),
            "ref_timeline_json": (_I64, [_P, _P, _I64, _P]),
            "ref_search": (_I64, [_P, C.c_char_p, _P, _I64, _P]),
            "ref_synth_bundle": (_I64, [C.c_char_p, _P, _I64, _P]),
            "ref_ingest": (_P, [C.c_char_p, C.c_char_p, _P]),
            "ref_memory_pass": (_P, [_P, _I64, C.c_char_p, _P, _P, _P, _P]),
            "ref_partial_replay": (_I32, [_P, C.c_char_p, _I32, _P]),
            "ref_tsync_graph": (_P, [C.c_char_p, _I64, _I32, _P]),
            "ref_replay_bench": (_I32, [_P, _I64, _I64, _I32, _P, _P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype, fn.argtypes = res, args
        _ref = lib
    return _ref


class RefError(Exception):
    def __init__(self, status: int, msg: str, cycle=None):
        super().__init__(f"[{status}] {msg}")
        self.status, self.msg, self.cycle = status, msg, cycle or []


def _raise(lib, st: int):
    if st:
        cyc = [lib.ref_last_cycle_id(i).decode() for i in range(lib.ref_last_cycle_len())]
        raise RefError(st, lib.ref_last_error().decode(), cyc)


class RefGraph:
    """A reference GlobalDFG (heap handle in libdpro_ref.so)."""

    def __init__(self, handle):
        self.lib = ref_lib()
        if not handle:
            raise RefError(3, self.lib.ref_last_error().decode())
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_graph_free(self.h)
            self.h = None

    # --- construction ---------------------------------------------------
    @staticmethod
    def from_ops(ops, edges) -> "RefGraph":
        """ops: iterable of (id, kind:int, dev_kind:int, dev_node, dev_peer, dur)."""
        lib = ref_lib()
        ops = list(ops)
        edges = list(edges)
        n, m = len(ops), len(edges)
        enc = lambda xs: (C.c_char_p * max(1, len(xs)))(*[x.encode() for x in xs])
        ids = enc([o[0] for o in ops])
        kinds = np.array([o[1] for o in ops], np.int32)
        dk = np.array([o[2] for o in ops], np.int32)
        dn = enc([o[3] for o in ops])
        dp = enc([o[4] for o in ops])
        dur = np.array([o[5] for o in ops], np.int64)
        ea = enc([e[0] for e in edges])
        eb = enc([e[1] for e in edges])
        st = C.c_int32(0)
        h = lib.ref_graph_from_arrays(n, ids, _ptr(kinds), _ptr(dk), dn, dp, _ptr(dur), m, ea,
                                      eb, C.byref(st))
        _raise(lib, st.value)
        return RefGraph(h)

    @staticmethod
    def from_dfg(g) -> "RefGraph":
        """From a paper_2205_02473_b200.graph.GlobalDFG (small graphs)."""
        ops = [(o.id, int(o.kind), int(o.device.kind), o.device.node, o.device.peer, int(o.dur))
               for o in g.ops()]
        edges = [(g.op_at(i).id, g.op_at(s).id) for i in range(g.size())
                 for s in g.succ_indices(i)]
        return RefGraph.from_ops(ops, edges)

    @staticmethod
    def synth(spec: dict) -> "RefGraph":
        lib = ref_lib()
        st = C.c_int32(0)
        h = lib.ref_synth_graph(json.dumps(spec).encode(), C.byref(st))
        _raise(lib, st.value)
        return RefGraph(h)

    @staticmethod
    def ingest(bundle: dict, cluster_json: dict) -> "RefGraph":
        """ingest_bundle on {events, deps} + a cluster (ClusterSpec JSON)."""
        lib = ref_lib()
        st = C.c_int32(0)
        h = lib.ref_ingest(json.dumps(bundle).encode(), json.dumps(cluster_json).encode(),
                           C.byref(st))
        _raise(lib, st.value)
        return RefGraph(h)

    @staticmethod
    def tsync(cluster_json: dict, bytes_: int, k: int) -> "RefGraph":
        lib = ref_lib()
        st = C.c_int32(0)
        h = lib.ref_tsync_graph(json.dumps(cluster_json).encode(), bytes_, k, C.byref(st))
        _raise(lib, st.value)
        return RefGraph(h)

    def partition(self, tensor: str, k: int) -> "RefGraph":
        st = C.c_int32(0)
        h = self.lib.ref_apply_partition(self.h, tensor.encode(), k, C.byref(st))
        _raise(self.lib, st.value)
        return RefGraph(h)

    def op_fusion(self, a: str, b: str, dur_override: int = -1) -> "RefGraph":
        """apply_op_fusion with the default CostModel (ratio 0.8)."""
        st = C.c_int32(0)
        h = self.lib.ref_apply_op_fusion(self.h, a.encode(), b.encode(), dur_override,
                                         C.byref(st))
        _raise(self.lib, st.value)
        return RefGraph(h)

    def tensor_fusion(self, t1: str, t2: str) -> "RefGraph":
        st = C.c_int32(0)
        h = self.lib.ref_apply_tensor_fusion(self.h, t1.encode(), t2.encode(), C.byref(st))
        _raise(self.lib, st.value)
        return RefGraph(h)

    def search(self, options: dict) -> dict:
        """dpro::search(g, options) -> {before_us, after_us, strategies}."""
        st = C.c_int32(0)
        o = json.dumps(options).encode()
        n = self.lib.ref_search(self.h, o, None, 0, C.byref(st))
        _raise(self.lib, st.value)
        buf = C.create_string_buffer(n)
        self.lib.ref_search(self.h, o, buf, n, C.byref(st))
        return json.loads(buf.raw[:n].decode())

    def timeline_json(self) -> bytes:
        """The CLI's timeline.json bytes for replay(g) (dpro_main.cpp:90-116)."""
        st = C.c_int32(0)
        n = self.lib.ref_timeline_json(self.h, None, 0, C.byref(st))
        _raise(self.lib, st.value)
        buf = C.create_string_buffer(n)
        self.lib.ref_timeline_json(self.h, buf, n, C.byref(st))
        return buf.raw[:n]

    def apply_memory_strategy(self, kind: int, meta: dict) -> "RefGraph":
        """apply_strategy(kRecompute=3 | kGradAccum=4)."""
        st = C.c_int32(0)
        h = self.lib.ref_apply_memory_strategy(self.h, kind, json.dumps(meta).encode(),
                                               C.byref(st))
        _raise(self.lib, st.value)
        return RefGraph(h)

    def memory_pass(self, budget: int, meta: dict):
        """-> (graph, applied kind or -1, k); RefError status 7 carries
        best_peak in .best_peak."""
        st, kind, k, best = C.c_int32(0), C.c_int32(-1), C.c_int32(0), C.c_int64(0)
        h = self.lib.ref_memory_pass(self.h, budget, json.dumps(meta).encode(), C.byref(st),
                                     C.byref(kind), C.byref(k), C.byref(best))
        try:
            _raise(self.lib, st.value)
        except RefError as e:
            e.best_peak = best.value
            raise
        return RefGraph(h), kind.value, k.value

    def with_durations(self, dur: np.ndarray) -> "RefGraph":
        st = C.c_int32(0)
        d = np.ascontiguousarray(dur, np.int64)
        h = self.lib.ref_with_durations(self.h, _ptr(d), C.byref(st))
        _raise(self.lib, st.value)
        return RefGraph(h)

    # --- inspection -----------------------------------------------------
    @property
    def n_ops(self) -> int:
        return self.lib.ref_graph_num_ops(self.h)

    @property
    def n_edges(self) -> int:
        return self.lib.ref_graph_num_edges(self.h)

    @property
    def n_devices(self) -> int:
        return self.lib.ref_graph_num_devices(self.h)

    def op_ids(self) -> list[str]:
        return [self.lib.ref_graph_op_id(self.h, i).decode() for i in range(self.n_ops)]

    def device_strs(self) -> list[str]:
        return [self.lib.ref_graph_device_str(self.h, d).decode() for d in range(self.n_devices)]

    def content_hash(self) -> int:
        return self.lib.ref_graph_hash(self.h)

    def export(self) -> dict:
        """Index-ordered CSR (+ kind, bytes) in the engine's dtypes."""
        n, e = self.n_ops, self.n_edges
        dur = np.zeros(n, np.int64)
        kind = np.zeros(n, np.int32)
        dev = np.zeros(n, np.int32)
        so = np.zeros(n + 1, np.uint32)
        su = np.zeros(max(e, 1), np.uint32)
        by = np.zeros(n, np.int64)
        self.lib.ref_graph_export(self.h, _ptr(dur), _ptr(kind), _ptr(dev), _ptr(so), _ptr(su),
                                  _ptr(by))
        flags = (np.isin(kind, (5, 6)).astype(np.uint8) | (np.isin(kind, (3, 4)).astype(np.uint8) << 1))
        indeg = np.bincount(su[:e], minlength=n).astype(np.uint32) if n else np.zeros(0, np.uint32)
        return {"dur": dur, "kind": kind, "dev": dev.astype(np.uint16), "flags": flags,
                "succ_off": so, "succ": su[:e].copy(), "indeg": indeg, "bytes": by,
                "n_devices": self.n_devices}

    # --- the reference Replayer -----------------------------------------
    def replay(self):
        """(T, start, end, tl_pos, util) or raises RefError."""
        n = self.n_ops
        start = np.zeros(n, np.int64)
        end = np.zeros(n, np.int64)
        tl = np.zeros(n, np.int32)
        util = np.zeros(max(1, self.n_devices), np.float64)
        T = C.c_int64(0)
        st = self.lib.ref_replay(self.h, _ptr(start), _ptr(end), C.byref(T), _ptr(tl), _ptr(util))
        _raise(self.lib, st)
        return T.value, start, end, tl, util[: self.n_devices]

    def critical_path(self):
        n = self.n_ops
        path = np.zeros(max(n, 1), np.uint32)
        plen = C.c_int64(0)
        total = C.c_int64(0)
        conf = C.c_int32(0)
        rc = np.zeros(max(n, 1), np.int32)
        rd = np.zeros(max(n, 1), np.int64)
        rl = np.zeros(max(n, 1), np.int64)
        nr = C.c_int64(0)
        st = self.lib.ref_critical_path(self.h, _ptr(path), C.byref(plen), C.byref(total),
                                        C.byref(conf), _ptr(rc), _ptr(rd), _ptr(rl), C.byref(nr))
        _raise(self.lib, st)
        k = nr.value
        return {"path": path[: plen.value].copy(), "total": total.value,
                "conforming": bool(conf.value),
                "runs": list(zip(rc[:k].tolist(), rd[:k].tolist(), rl[:k].tolist()))}

    def peak_memory(self, meta: dict) -> dict:
        """estimate_peak_memory(g, replay(g), meta) -> {node: peak bytes}."""
        peaks = np.zeros(4096, np.int64)
        nn = C.c_int32(0)
        _raise(self.lib, self.lib.ref_peak_memory(self.h, json.dumps(meta).encode(), _ptr(peaks),
                                                  C.byref(nn)))
        return {self.lib.ref_peak_node(i).decode(): int(peaks[i]) for i in range(nn.value)}

    def exec_edge_count(self) -> int:
        return self.lib.ref_execution_graph_edges(self.h)

    def partial_replay(self, tensor: str, k: int) -> int:
        out = C.c_int64(0)
        _raise(self.lib, self.lib.ref_partial_replay(self.h, tensor.encode(), k, C.byref(out)))
        return out.value


def port_peak_memory(ops, succ, start, end, meta: dict) -> dict:
    """Restatement of estimate_peak_memory (proj/src/memory.cpp:122-167) and
    output_bytes_for (memory.cpp:71-119) in plain Python, for checking.
    ops: [(id, kind, node)] (kind as the OpKind int: FW=0, BW=1, UPDATE=2),
    succ: successor index lists, start/end: the replayed schedule, meta: the
    ModelMeta json. Returns {node: peak} or raises KeyError(message) where
    the reference raises MissingMetaError."""
    out_b = meta.get("output_bytes", {})
    pers = meta.get("persistent_bytes", {})

    def local_bytes(local):  # memory.cpp:73-92
        if out_b.get(local, -1) >= 0:
            return out_b[local]
        at = local.rfind("@mb")
        if at >= 0 and out_b.get(local[:at], -1) >= 0:
            return (out_b[local[:at]] + 1) // 2
        if local.startswith("RFW."):
            return out_b.get("FW." + local[4:], -1)
        return -1

    def bytes_for(op_id):  # memory.cpp:96-119
        if op_id in out_b:
            return out_b[op_id]
        local = op_id.split("->", 1)[1] if "->" in op_id else op_id
        v = local_bytes(local)
        if v >= 0 or "+" not in local:
            return v
        parts = [local_bytes(p) for p in local.split("+")]
        return -1 if min(parts) < 0 else sum(parts)

    comp = lambda k: k in (0, 1, 2)  # noqa: E731  graph.hpp:43-45
    events: dict[str, list] = {}
    for i, (oid, kind, node) in enumerate(ops):
        if not comp(kind):
            continue
        events.setdefault(node, [])
        b = bytes_for(oid)
        if b < 0:
            if kind != 2:
                raise KeyError(f"no output bytes for op {oid}")
            b = 0
        if b == 0:
            continue
        freed = int(end[i])
        for s in succ[i]:
            if comp(ops[s][1]):
                freed = max(freed, int(end[s]))
        events[node] += [(int(start[i]), b), (freed, -b)]
    peak = {}
    for node in sorted(events):
        if node not in pers:
            raise KeyError(f"no persistent bytes for node {node}")
        live = best = 0
        for _, d in sorted(events[node]):
            live += d
            best = max(best, live)
        peak[node] = pers[node] + best
    return peak


def ref_synth_bundle(spec: dict) -> dict:
    """The reference generator's trace events + dependency spec (JSON)."""
    lib = ref_lib()
    st = C.c_int32(0)
    o = json.dumps(spec).encode()
    n = lib.ref_synth_bundle(o, None, 0, C.byref(st))
    _raise(lib, st.value)
    buf = C.create_string_buffer(n)
    lib.ref_synth_bundle(o, buf, n, C.byref(st))
    return json.loads(buf.raw[:n].decode())


def ref_sync_makespan(cluster_json: dict, bytes_: int, k: int) -> int:
    lib = ref_lib()
    out = C.c_int64(0)
    _raise(lib, lib.ref_sync_makespan(json.dumps(cluster_json).encode(), bytes_, k, C.byref(out)))
    return out.value


def ref_replay_bench(graphs: list[RefGraph], n_replays: int, threads: int):
    """Times dpro::replay over n_replays graphs (round-robin) on `threads`
    std::threads; returns (seconds, makespans)."""
    lib = ref_lib()
    hs = (C.c_void_p * len(graphs))(*[g.h for g in graphs])
    ms = np.zeros(n_replays, np.int64)
    sec = C.c_double(0)
    _raise(lib, lib.ref_replay_bench(hs, len(graphs), n_replays, threads, _ptr(ms), C.byref(sec)))
    return sec.value, ms


# --------------------------------------------------------------------------
# the C restatement ("port")
# --------------------------------------------------------------------------
def port_lib():
    global _port
    if _port is None:
        lib = C.CDLL(str(PORT_SO))
        lib.orc_replay.restype = _I32
        lib.orc_replay.argtypes = [C.c_uint32, _P, _P, _P, C.c_uint32, _P, _P, _P, _P, _P, _P,
                                   _P, _P, _P]
        lib.orc_critical_path.restype = _I64
        lib.orc_critical_path.argtypes = [C.c_uint32, _P, C.c_uint32, _P, _P, _P, _P, _I64, _P,
                                          _P]
        _port = lib
    return _port


def port_replay(csr) -> dict:
    """csr: dict or engine.Csr-like with dur/dev/flags/succ_off/succ/n_devices."""
    get = (lambda k: csr[k]) if isinstance(csr, dict) else (lambda k: getattr(csr, k))
    dur = np.ascontiguousarray(get("dur"), np.int64)
    n = dur.shape[0]
    dev = np.ascontiguousarray(get("dev"), np.uint32)
    flags = np.ascontiguousarray(get("flags"), np.uint8)
    so = np.ascontiguousarray(get("succ_off"), np.uint32)
    su = np.ascontiguousarray(get("succ"), np.uint32)
    nd = int(get("n_devices"))
    start = np.zeros(n, np.int64)
    end = np.zeros(n, np.int64)
    tl = np.zeros(n, np.int32)
    busy = np.zeros(max(nd, 1), np.int64)
    sched = np.zeros(max(n, 1), np.uint8)
    T = C.c_int64(0)
    err = C.c_int64(0)
    lib = port_lib()
    st = lib.orc_replay(n, _ptr(dur), _ptr(dev), _ptr(flags), nd, _ptr(so), _ptr(su),
                        _ptr(start), _ptr(end), C.byref(T), _ptr(tl), _ptr(busy), _ptr(sched),
                        C.byref(err))
    out = {"status": st, "err": err.value, "T": T.value, "start": start, "end": end,
           "tl_pos": tl, "busy": busy[:nd], "scheduled": sched[:n]}
    if st == 0:
        path = np.zeros(max(n, 1), np.uint32)
        L = lib.orc_critical_path(n, _ptr(dev), nd, _ptr(so), _ptr(su), _ptr(start), _ptr(end),
                                  T.value, _ptr(tl), _ptr(path))
        out["path"] = path[:L].copy()
    return out
