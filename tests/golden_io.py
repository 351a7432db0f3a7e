"""Loading the committed golden vectors (test infrastructure)."""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from paper_2205_02473_b200.graph import DeviceId, DeviceKind, GraphBuilder, Op, OpKind, synth_cluster

GOLDEN = Path(__file__).resolve().parent / "golden"


def graph_from_json(j):
    b = GraphBuilder()
    for id_, kind, dk, node, peer, dur in j["ops"]:
        dev = DeviceId(DeviceKind(dk), node, peer)
        b.add_op(Op(id=id_, kind=OpKind(kind), node=node, device=dev, dur=int(dur)))
    for a, c in j["edges"]:
        b.add_edge(a, c)
    return b.build()


def replay_vectors():
    return json.loads((GOLDEN / "replay_vectors.json").read_text())


def tsync_vectors():
    j = json.loads((GOLDEN / "tsync_vectors.json").read_text())
    clusters = {k: synth_cluster(s, w, p, bw, lat) for k, (s, w, p, bw, lat) in j["clusters"].items()}
    return clusters, j["cases"]


def synth_vectors():
    return json.loads((GOLDEN / "synth_vectors.json").read_text())


def tl_pos_from(order, dev_off, n):
    tl = np.full(n, -1, np.int64)
    for d in range(len(dev_off) - 1):
        a, b = int(dev_off[d]), int(dev_off[d + 1])
        for p in range(a, b):
            tl[int(order[p])] = p - a
    return tl


def rows_digest(rows) -> str:
    """sha256 over (id, kind, device, dur, successor ids) rows in index order."""
    import hashlib
    h = hashlib.sha256()
    for oid, kind, dev, dur, succ in rows:
        h.update(f"{oid}|{kind}|{dev}|{dur}|{','.join(succ)}\n".encode())
    return h.hexdigest()


def dfg_rows(g):
    c = g.to_csr()
    ds = [d.str() for d in c["devices"]]
    return [(o.id, int(o.kind), ds[int(c["dev"][i])], int(o.dur),
             [g.op_at(s).id for s in g.succ_indices(i)]) for i, o in enumerate(g.ops())]


def rewrite_vectors():
    return json.loads((GOLDEN / "rewrite_vectors.json").read_text())
