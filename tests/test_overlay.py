"""Overlay batches (engine option "overlay"): delta candidates replayed on the
resident base's packed layout + per-candidate overlays (csrc/overlay.h),
bit-exact against the materialized delta path (merge + pack + replay) and
the C oracle -- every start/end, makespan, timeline and busy sum."""
import numpy as np
import pytest

from paper_2205_02473_b200.delta import DeltaList, make_delta
from paper_2205_02473_b200.engine import Csr
from paper_2205_02473_b200.graph import synth_cluster
from paper_2205_02473_b200.ingest import (ConcatDeltas, LayeredBase, LayeredModel,
                                          layered_graph_variant)
from paper_2205_02473_b200.workloads import workload

pytestmark = pytest.mark.gpu


def _replay(engine, res, deltas, overlay):
    engine.set_option("overlay", 1 if overlay else 0)
    try:
        b = engine.delta_batch(res, deltas)
        b.replay(want_schedule=True)
        out = b.results(schedule=True)
        tls = [b.timelines(i) for i in range(b.n)]
        st = b.stats()
    finally:
        engine.set_option("overlay", 0)
    return b, out, tls, st


def _same(engine, res, deltas, port=None, graphs=None, expect_fast=True):
    b1, (m1, s1, e1, a1, z1), t1, _ = _replay(engine, res, deltas, False)
    b2, (m2, s2, e2, a2, z2), t2, st = _replay(engine, res, deltas, True)
    assert np.array_equal(s1, s2) and np.array_equal(e1, e2)
    for i in range(b2.n):
        if s1[i] != 0:  # errors: status and err only (no schedule is defined)
            continue
        a, z = int(b2.op_off[i]), int(b2.op_off[i + 1])
        assert m1[i] == m2[i], i
        assert np.array_equal(a1[a:z], a2[a:z]) and np.array_equal(z1[a:z], z2[a:z]), i
        (o1, d1, u1), (o2, d2, u2) = t1[i], t2[i]
        assert np.array_equal(o1, o2) and np.array_equal(d1, d2) and np.array_equal(u1, u2), i
    if graphs is not None:
        for i, g in enumerate(graphs):
            o = port.port_replay(g.csr)
            a, z = int(b2.op_off[i]), int(b2.op_off[i + 1])
            assert m2[i] == o["T"] and np.array_equal(a2[a:z], o["start"])
    return b2, st


def _setup(scheme, W, S, L, seed):
    rng = np.random.default_rng(seed)
    c = synth_cluster(scheme, W, S, 12500.0, 5.0)
    m = LayeredModel(rng.integers(10, 400, L).tolist(), rng.integers(10, 800, L).tolist(),
                     rng.integers(1000, 4_000_000, L).tolist(), 5)
    return rng, LayeredBase(m, c)


@pytest.mark.parametrize("scheme,W,S,L", [("ring", 4, 0, 8), ("ps", 4, 2, 10),
                                          ("ring", 11, 0, 6), ("ps", 16, 4, 12)])
def test_overlay_matches_materialized_mixed_candidates(engine, port, scheme, W, S, L):
    """Tensor fusion + partition specs, single- and all-worker op fusion,
    recompute / grad-accum variants (graph -> delta), and the base itself."""
    rng, base = _setup(scheme, W, S, L, W * 100 + L)
    specs, fjs, bjs, jws = [], [], [], []
    for k in range(24):
        cuts = sorted(rng.choice(np.arange(1, L), int(rng.integers(0, L // 2)), replace=False).tolist())
        groups, a = [], 0
        for cp in cuts + [L]:
            groups.append(list(range(a, cp)))
            a = cp
        specs.append((groups, [int(rng.integers(1, 5)) for _ in groups]))
        fjs.append((rng.random(L - 1) < 0.2).astype(np.uint8))
        bjs.append((rng.random(L - 1) < 0.2).astype(np.uint8))
        jws.append(int(rng.integers(-1, W)))
    d1 = base.deltas(specs, threads=4, fw_join=np.array(fjs), bw_join=np.array(bjs),
                     join_worker=jws)
    variants = [layered_graph_variant(base.model, base.cluster, v, 0.5)
                for v in ("recompute", "grad-accum")] + [base.graph()]
    d2 = base.deltas_from_graphs(variants, threads=3)
    res = engine.resident(base.graph().csr)
    full = base.candidates(specs, threads=4, fw_join=np.array(fjs), bw_join=np.array(bjs))
    _same(engine, res, ConcatDeltas([d1, d2]))
    # port check on the non-op-fusion-worker subset (full graphs exist for them)
    plain = [i for i in range(len(specs)) if jws[i] == -1]
    if plain:
        sub = ConcatDeltas([base.deltas([specs[i] for i in plain], threads=2,
                                        fw_join=np.array([fjs[i] for i in plain]),
                                        bw_join=np.array([bjs[i] for i in plain]))])
        _same(engine, res, sub, port, [full[i] for i in plain])


def test_overlay_generic_rewrites_and_errors(engine):
    """Generic GlobalDFG rewrites (delta.make_delta) incl. cut edges, and a
    candidate with a cycle / a missing duration: the overlay batch hands
    those to the materialized path and reports the same statuses."""
    from paper_2205_02473_b200.ingest import layered_global_dfg
    from paper_2205_02473_b200.rewrite import apply_grad_accum, apply_recompute
    from paper_2205_02473_b200.memory import ModelMeta
    rng, base = _setup("ring", 4, 0, 6, 7)
    g = layered_global_dfg(base.model, base.cluster)
    cands = [apply_recompute(g), apply_grad_accum(g, ModelMeta())]
    res = engine.resident(Csr.from_dict(g.to_csr()))
    ds = [make_delta(g, c) for c in cands]
    # missing duration: a new op with dur -1
    bad = make_delta(g, cands[0])
    bad.new_dur = bad.new_dur.copy()
    nv = np.flatnonzero((bad.new_flags & 1) == 0)
    bad.new_dur[nv[0]] = -1
    ds.append(bad)
    # cycle: an extra edge from a late op back to a source
    cyc = make_delta(g, g)
    csr = g.to_csr()
    src = int(np.flatnonzero(np.bincount(csr["succ"], minlength=g.size()) == 0)[0])
    last = int(np.argmax(csr["succ_off"][1:] - csr["succ_off"][:-1] == 0))  # an op without succs
    cyc.extra_src = np.array([last], np.uint32)
    cyc.extra_dst = np.array([src], np.uint32)
    ds.append(cyc)
    b, st = _same(engine, res, DeltaList(ds))
    ms, status, err, *_ = b.results()
    assert status.tolist()[:2] == [0, 0] and status[2] == 1 and status[3] == 2


def test_overlay_config4_scale(engine, port):
    """Config 4 (4.8M ops): the bench's candidate mix in overlay mode equals
    the materialized path, the grad-accum variant (230-deep link queue)
    included; op-fusion candidates stay on the overlay fast path."""
    w = workload(4)
    base = LayeredBase(w.model, w.cluster)
    deltas, descs = w.candidate_deltas(base, 12, threads=16)
    res = engine.resident(base.graph().csr)
    b, st = _same(engine, res, deltas)
    assert st["fallbacks"] == 0
