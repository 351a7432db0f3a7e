"""ctypes binding of libdpro_cuda.so (include/dpro_cuda.h).

The product path has no CPU fallback: if the in-tree library is missing the
import of this module raises, and every replay entry point fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
# DPRO_LIB: an alternative build of the same library (kernel A/B experiments)
LIB_PATH = Path(os.environ.get("DPRO_LIB", str(_HERE / "libdpro_cuda.so")))

DPRO_OK, DPRO_MISSING_PROFILE, DPRO_CYCLE, DPRO_EINVAL = 0, 1, 2, 3
DPRO_ECUDA, DPRO_ENOMEM, DPRO_EUNSUPPORTED = 4, 5, 6
DPRO_HOST, DPRO_DEVICE = 0, 1
FLAG_VIRTUAL, FLAG_COMM = 0x1, 0x2


class DproCsr(C.Structure):
    _fields_ = [
        ("n_ops", C.c_uint32),
        ("n_edges", C.c_uint32),
        ("n_devices", C.c_uint32),
        ("dur_bits", C.c_int32),
        ("dur", C.c_void_p),
        ("dev", C.c_void_p),
        ("flags", C.c_void_p),
        ("succ_off", C.c_void_p),
        ("succ", C.c_void_p),
        ("indeg", C.c_void_p),
    ]


class DproClusterDesc(C.Structure):
    _fields_ = [
        ("scheme", C.c_int32),
        ("n_nodes", C.c_int32),
        ("node_ids", C.POINTER(C.c_char_p)),
        ("node_role", C.POINTER(C.c_int32)),
        ("n_links", C.c_int32),
        ("link_src", C.POINTER(C.c_int32)),
        ("link_dst", C.POINTER(C.c_int32)),
        ("link_bw", C.POINTER(C.c_double)),
        ("link_lat", C.POINTER(C.c_double)),
        ("n_ring", C.c_int32),
        ("ring_order", C.POINTER(C.c_int32)),
        ("chunks_per_tensor", C.c_int32),
    ]


class DproLayeredModel(C.Structure):
    _fields_ = [
        ("layers", C.c_int32),
        ("fw_dur", C.POINTER(C.c_int64)),
        ("bw_dur", C.POINTER(C.c_int64)),
        ("tensor_bytes", C.POINTER(C.c_int64)),
        ("update_dur", C.c_int64),
    ]


class DproDelta(C.Structure):
    _fields_ = [
        ("n_devices", C.c_uint32),
        ("n_removed", C.c_uint32), ("removed", C.c_void_p),
        ("n_new", C.c_uint32), ("new_pos", C.c_void_p), ("new_dur", C.c_void_p),
        ("new_dev", C.c_void_p), ("new_flags", C.c_void_p), ("new_succ_off", C.c_void_p),
        ("new_succ", C.c_void_p),
        ("n_extra", C.c_uint32), ("extra_src", C.c_void_p), ("extra_dst", C.c_void_p),
        ("n_cut", C.c_uint32), ("cut", C.c_void_p),
    ]


# (name, restype, argtypes) for every symbol include/dpro_cuda.h declares.
_P, _I32, _I64, _U32 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32
SIGNATURES = {
    "dpro_cuda_abi_version": (C.c_int, []),
    "dpro_cuda_create": (_P, [C.c_int]),
    "dpro_cuda_destroy": (None, [_P]),
    "dpro_cuda_set_stream": (C.c_int, [_P, _P]),
    "dpro_cuda_set_option": (C.c_int, [_P, C.c_char_p, _I64]),
    "dpro_cuda_batch_stats": (C.c_int, [_P, _P, _P]),
    "dpro_cuda_batch_diag": (C.c_int, [_P, _P, _P, _I32]),
    "dpro_cuda_last_error": (C.c_char_p, [_P]),
    "dpro_cuda_batch_create": (_P, [_P, C.POINTER(DproCsr), _I32, _I32]),
    "dpro_cuda_batch_destroy": (None, [_P, _P]),
    "dpro_cuda_batch_replay": (C.c_int, [_P, _P, _I32]),
    "dpro_cuda_batch_device_results": (C.c_int, [_P, _P, _P, _P, _P, _P]),
    "dpro_cuda_batch_results": (C.c_int, [_P, _P, _P, _P, _P, _P, _P]),
    "dpro_cuda_batch_timelines": (C.c_int, [_P, _P, _I32, _P, _P, _P]),
    "dpro_cuda_batch_critical_paths": (C.c_int, [_P, _P, _P, _P]),
    "dpro_cuda_batch_scheduled": (C.c_int, [_P, _P, _I32, _P]),
    "dpro_cuda_batch_peak_memory": (C.c_int, [_P, _P, _P, _P, _P, _P, _P]),
    "dpro_cuda_critical_path": (C.c_int, [_P, C.POINTER(DproCsr), _P, _P, _I64, _P, _P]),
    "dpro_cuda_replay_batch": (C.c_int, [_P, C.POINTER(DproCsr), _I32, _I32, _P, _P, _P, _P, _P]),
    "dpro_cuda_resident_create": (_P, [_P, C.POINTER(DproCsr)]),
    "dpro_cuda_resident_destroy": (None, [_P, _P]),
    "dpro_cuda_batch_create_delta": (_P, [_P, _P, _P, _I32]),
    "dpro_cuda_batch_prepare": (C.c_int, [_P, _P]),
    "dpro_cuda_batch_sizes": (C.c_int, [_P, _P, _P, _P]),
    "dpro_cuda_batch_pack_info": (C.c_int, [_P, _P]),
    "dpro_cuda_replay_delta_batch": (C.c_int, [_P, _P, _P, _I32, _P, _P, _P]),
    "dpro_base_delta_batch": (C.c_int, [_P, _I32, _P, _P, _P, _P, _P, _I32, _P]),
    "dpro_base_delta_batch_ops": (C.c_int, [_P, _I32, _P, _P, _P, _P, _P, _P, _P, _I32, _P]),
    "dpro_base_delta_batch_ex": (C.c_int, [_P, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _I32, _P]),
    "dpro_base_worker": (C.c_char_p, [_P, _I32]),
    "dpro_base_delta_from_graphs": (C.c_int, [_P, _P, _I32, _I32, _P]),
    "dpro_graph_from_base_batch_ops": (C.c_int, [_P, _I32, _P, _P, _P, _P, _P, _P, _P, _I32, _P]),
    "dpro_delta_set_deltas": (_P, [_P]),
    "dpro_delta_set_size": (_I32, [_P]),
    "dpro_delta_set_device_str": (C.c_char_p, [_P, _I32, _U32]),
    "dpro_delta_set_free": (None, [_P]),
    "dpro_base_graph": (_P, [_P]),
    "dpro_cuda_batch_create_tsync": (_P, [_P, C.POINTER(DproClusterDesc), _P, _P, _I32]),
    "dpro_cuda_tsync_grid": (C.c_int, [_P, C.POINTER(DproClusterDesc), _P, _P, _I32, _P, _P]),
    "dpro_graph_layered": (_P, [C.POINTER(DproLayeredModel), C.POINTER(DproClusterDesc), _P, _P]),
    "dpro_graph_layered_variant": (_P, [C.POINTER(DproLayeredModel), C.POINTER(DproClusterDesc), _P, _I32, C.c_double, _P]),
    "dpro_graph_memory_inputs": (C.c_int, [_P, _I32, _P, _P, _P, _P, _P, _P]),
    "dpro_graph_memory_node": (C.c_char_p, [_P, _I32]),
    "dpro_graph_comm_info": (C.c_char_p, [_P, _U32, _P]),
    "dpro_graph_write_timeline": (C.c_int, [_P, _P, _P, C.c_char_p]),
    "dpro_graph_layered_batch": (C.c_int, [C.POINTER(DproLayeredModel), C.POINTER(DproClusterDesc), _P, _I32, _I32, _P]),
    "dpro_graph_layered_groups": (_P, [C.POINTER(DproLayeredModel), C.POINTER(DproClusterDesc), _I32, _P, _P, _P, _P]),
    "dpro_graph_layered_groups_batch": (C.c_int, [C.POINTER(DproLayeredModel), C.POINTER(DproClusterDesc), _I32, _P, _P, _P, _P, _P, _I32, _P]),
    "dpro_base_layered": (_P, [C.POINTER(DproLayeredModel), C.POINTER(DproClusterDesc), _P]),
    "dpro_base_free": (None, [_P]),
    "dpro_graph_from_base_batch": (C.c_int, [_P, _I32, _P, _P, _P, _P, _P, _I32, _P]),
    "dpro_graph_tsync": (_P, [C.POINTER(DproClusterDesc), _I64, _I32, _P]),
    "dpro_graph_csr": (C.c_int, [_P, C.POINTER(DproCsr)]),
    "dpro_graph_op_id": (C.c_char_p, [_P, _U32]),
    "dpro_graph_op_kind": (_I32, [_P, _U32]),
    "dpro_graph_device_str": (C.c_char_p, [_P, _U32]),
    "dpro_graph_free": (None, [_P]),
    "dpro_graph_last_error": (C.c_char_p, []),
}


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make -C paper_2205_02473_b200` "
            "or __graft_entry__.build(); there is no CPU fallback")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        if "DPRO_LIB" in os.environ and not hasattr(lib, name):
            continue  # A/B experiments against an older build of the library
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def ptr(a: np.ndarray | None) -> int | None:
    return None if a is None else a.ctypes.data


class ClusterDescHolder:
    """Keeps the ctypes arrays of a dpro_cluster_desc alive."""

    def __init__(self, cluster) -> None:
        ids = [n.id for n in cluster.nodes]
        index = {nid: i for i, nid in enumerate(ids)}
        self._ids = (C.c_char_p * max(1, len(ids)))(*[s.encode() for s in ids])
        self._role = (C.c_int32 * max(1, len(ids)))(
            *[0 if n.role == "worker" else 1 for n in cluster.nodes])
        L = cluster.links
        self._src = (C.c_int32 * max(1, len(L)))(*[index[l.src] for l in L])
        self._dst = (C.c_int32 * max(1, len(L)))(*[index[l.dst] for l in L])
        self._bw = (C.c_double * max(1, len(L)))(*[l.bandwidth_bytes_per_us for l in L])
        self._lat = (C.c_double * max(1, len(L)))(*[l.latency_us for l in L])
        ring = [index[w] for w in cluster.ring_order]
        self._ring = (C.c_int32 * max(1, len(ring)))(*ring)
        self.desc = DproClusterDesc(
            1 if cluster.scheme == "ps" else 0, len(ids), self._ids, self._role,
            len(L), self._src, self._dst, self._bw, self._lat, len(ring),
            self._ring, int(cluster.chunks_per_tensor))


def check_symbols() -> list[str]:
    """Names declared in include/dpro_cuda.h that the library fails to export."""
    header = (_HERE.parent / "include" / "dpro_cuda.h").read_text()
    import re
    declared = set(re.findall(r"\b(dpro_(?:cuda|graph|base)_\w+)\s*\(", header))
    missing = [n for n in sorted(declared) if not hasattr(lib, n)]
    return missing + [n for n in sorted(declared) if n not in SIGNATURES]


if os.environ.get("DPRO_CHECK_SYMBOLS"):
    _m = check_symbols()
    if _m:
        raise ImportError(f"libdpro_cuda.so misses {_m}")
