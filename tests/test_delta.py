"""Resident base graph + per-candidate deltas (dpro_delta): the host delta
emission against the full rebuild (CPU), and the GPU merge + replay against
the host-merged candidates (bit-exact start/end/makespan, GPU)."""
import ctypes as C

import numpy as np
import pytest

from paper_2205_02473_b200 import _native as N
from paper_2205_02473_b200.graph import synth_cluster
from paper_2205_02473_b200.ingest import LayeredBase, LayeredModel


def _arr(p, dt, n):
    if n == 0:
        return np.zeros(0, dt)
    return np.ctypeslib.as_array(C.cast(p, C.POINTER(np.ctypeslib.as_ctypes_type(dt))),
                                 (n,)).copy()


def merge_host(bc, nb, d):
    """Checker: the merge include/dpro_cuda.h defines for a dpro_delta."""
    rem = _arr(d.removed, np.uint32, d.n_removed)
    pos = _arr(d.new_pos, np.uint32, d.n_new)
    keep = np.ones(nb, bool)
    keep[rem] = False
    b = np.arange(nb)
    fb = b - np.searchsorted(rem, b, "left") + np.searchsorted(pos, b, "right")
    fn = pos - np.searchsorted(rem, pos, "left") + np.arange(d.n_new)
    n = nb - d.n_removed + d.n_new
    dur = np.zeros(n, np.int64)
    dev = np.zeros(n, np.uint16)
    fl = np.zeros(n, np.uint8)
    dur[fb[keep]], dev[fb[keep]], fl[fb[keep]] = bc.dur[keep], bc.dev[keep], bc.flags[keep]
    dur[fn] = _arr(d.new_dur, np.int64, d.n_new)
    dev[fn] = _arr(d.new_dev, np.uint16, d.n_new)
    fl[fn] = _arr(d.new_flags, np.uint8, d.n_new)
    succ = [[] for _ in range(n)]
    cut = set(_arr(d.cut, np.uint32, d.n_cut).tolist())
    for x in np.flatnonzero(keep):
        a = int(bc.succ_off[x])
        succ[fb[x]] += [int(fb[s]) for k, s in enumerate(bc.succ[a:int(bc.succ_off[x + 1])])
                        if keep[s] and a + k not in cut]
    nso = _arr(d.new_succ_off, np.uint32, d.n_new + 1)
    ns = _arr(d.new_succ, np.uint32, int(nso[-1]))
    for k in range(d.n_new):
        succ[fn[k]] += ns[nso[k]:nso[k + 1]].tolist()
    for a, c in zip(_arr(d.extra_src, np.uint32, d.n_extra), _arr(d.extra_dst, np.uint32, d.n_extra)):
        succ[fb[a]].append(int(c))
    return dur, dev, fl, [sorted(x) for x in succ]


def _setup(scheme, W, S, L, n, seed):
    rng = np.random.default_rng(seed)
    c = synth_cluster(scheme, W, S, 12500.0, 5.0)
    m = LayeredModel(rng.integers(10, 400, L).tolist(), rng.integers(10, 800, L).tolist(),
                     rng.integers(1000, 4_000_000, L).tolist(), 5)
    specs = []
    for _ in range(n):
        cuts = sorted(rng.choice(np.arange(1, L), int(rng.integers(0, L // 2)),
                                 replace=False).tolist())
        groups, a = [], 0
        for cp in cuts + [L]:
            groups.append(list(range(a, cp)))
            a = cp
        specs.append((groups, [int(rng.integers(1, 5)) for _ in groups]))
    return LayeredBase(m, c), specs


CASES = [("ring", 4, 0, 8), ("ps", 4, 2, 10), ("ring", 8, 0, 16), ("ps", 16, 4, 12)]


@pytest.mark.parametrize("scheme,W,S,L", CASES)
def test_deltas_merge_to_the_full_candidates(scheme, W, S, L):
    base, specs = _setup(scheme, W, S, L, 12, W * L)
    bv = base.graph()
    full = base.candidates(specs)
    ds = base.deltas(specs)
    for i, g in enumerate(full):
        dur, dev, fl, succ = merge_host(bv.csr, bv.n_ops, ds[i])
        cs = g.csr
        assert len(dur) == g.n_ops
        assert np.array_equal(dur, cs.dur) and np.array_equal(fl, cs.flags)
        strs = g.device_strs()
        assert [ds.device_str(i, int(x)) for x in dev] == [strs[int(x)] for x in cs.dev]
        for k in range(g.n_ops):
            assert succ[k] == cs.succ[cs.succ_off[k]:cs.succ_off[k + 1]].tolist(), (i, k)


def test_delta_symbols_are_exported():
    for name in ("dpro_cuda_resident_create", "dpro_cuda_batch_create_delta",
                 "dpro_cuda_replay_delta_batch", "dpro_base_delta_batch"):
        assert hasattr(N.lib, name)


@pytest.mark.gpu
@pytest.mark.parametrize("scheme,W,S,L", CASES + [("ring", 8, 0, 48)])
def test_gpu_merge_replays_like_full_candidates(engine, scheme, W, S, L):
    base, specs = _setup(scheme, W, S, L, 64, 1000 + W * L)
    full = base.candidates(specs)
    fb = engine.batch([g.csr for g in full])
    fb.replay(want_schedule=True)
    ms0, st0, er0, s0, e0 = fb.results(schedule=True)
    res = engine.resident(base.graph().csr)
    db = engine.delta_batch(res, base.deltas(specs))
    db.replay(want_schedule=True)
    ms1, st1, er1, s1, e1 = db.results(schedule=True)
    assert np.array_equal(st0, st1) and np.all(st0 == 0)
    assert np.array_equal(ms0, ms1)
    assert np.array_equal(s0, s1) and np.array_equal(e0, e1)
    # critical paths on the merged CSR equal those of the host-merged ones
    for p0, p1 in zip(fb.critical_paths(), db.critical_paths()):
        assert np.array_equal(p0, p1)


@pytest.mark.gpu
def test_gpu_delta_one_shot_and_makespan_only(engine):
    base, specs = _setup("ps", 16, 4, 24, 256, 7)
    full = base.candidates(specs)
    fb = engine.batch([g.csr for g in full])
    fb.replay(want_schedule=False)
    ms0, *_ = fb.results()
    res = engine.resident(base.graph().csr)
    ds = base.deltas(specs)
    ms = np.zeros(len(specs), np.int64)
    st = np.zeros(len(specs), np.int32)
    er = np.zeros(len(specs), np.int64)
    rc = N.lib.dpro_cuda_replay_delta_batch(engine.ctx, res.handle, C.cast(ds.array, C.c_void_p),
                                            len(specs), N.ptr(ms), N.ptr(st), N.ptr(er))
    assert rc == 0 and np.all(st == 0)
    assert np.array_equal(ms, ms0)


@pytest.mark.gpu
def test_config4_scale_candidates_match_oracle(engine, port):
    """BASELINE config 4 shape (GPT-2 medium, 64-worker ring, 4.8M ops):
    delta candidates on the fast path (u16 counters in global scratch,
    deep-ring pass) equal the C oracle on the host-merged CSR."""
    from paper_2205_02473_b200.workloads import workload
    w = workload(4)
    base = LayeredBase(w.model, w.cluster)
    pk = w.candidate_partitions(2, tensors_per_cand=8)
    specs = [([[i] for i in range(w.layers)], pk[c].tolist()) for c in range(2)]
    res = engine.resident(base.graph().csr)
    b = engine.delta_batch(res, base.deltas(specs, threads=16))
    b.replay(want_schedule=True)
    ms, st, er, s, e = b.results(schedule=True)
    assert b.stats()["fallbacks"] == 0 and np.all(st == 0)
    full = base.candidates(specs, threads=16)
    for i, g in enumerate(full):
        exp = port.port_replay(g.csr)
        a, z = int(b.op_off[i]), int(b.op_off[i + 1])
        assert ms[i] == exp["T"]
        assert np.array_equal(s[a:z], exp["start"]) and np.array_equal(e[a:z], exp["end"])


@pytest.mark.gpu
def test_peak_memory_on_delta_batches(engine, port):
    """K5 on the schedules of a delta batch (merged in HBM) equals the
    oracle restatement on the host-merged candidates (memory.cpp:122-167)."""
    from paper_2205_02473_b200.memory import ModelMeta, batch_peak_memory, resolve
    from paper_2205_02473_b200.graph import synth_cluster
    base, specs = _setup("ps", 4, 2, 10, 24, 77)
    cluster = synth_cluster("ps", 4, 2, 12500.0, 5.0)
    L = 10
    meta = ModelMeta({**{f"FW.l{i}": 1000 * (i + 1) for i in range(L)},
                      **{f"BW.l{i}": 300 * (i + 2) for i in range(L)}},
                     {f"w{i}": 5000 * i for i in range(4)})
    graphs = [g.to_global_dfg(cluster) for g in base.candidates(specs)]
    res = engine.resident(base.graph().csr)
    b = engine.delta_batch(res, base.deltas(specs))
    b.replay(want_schedule=True)
    ms, st, er, s, e = b.results(schedule=True)
    parts = [resolve(g, meta) for g in graphs]
    peak = batch_peak_memory(b, np.concatenate([p[1] for p in parts]),
                             np.concatenate([p[2] for p in parts]),
                             np.array([len(p[0]) for p in parts], np.int32),
                             np.concatenate([p[3] for p in parts]))
    o = 0
    for i, (g, (nodes, *_)) in enumerate(zip(graphs, parts)):
        a, z = int(b.op_off[i]), int(b.op_off[i + 1])
        ops = [(op.id, int(op.kind), op.node) for op in g.ops()]
        succ = [list(g.succ_indices(k)) for k in range(g.size())]
        exp = port.port_peak_memory(ops, succ, s[a:z], e[a:z], meta.to_json())
        assert {nd: int(peak[o + j]) for j, nd in enumerate(nodes)} == exp
        o += len(nodes)


def _rewrite_pairs(seed: int, count: int):
    """(base, candidate) GlobalDFG pairs from the reference-pinned rewrites:
    recompute (drops edges between kept ops: cut), grad-accum (replaces
    every FW/BW op), op fusion / tensor fusion / partition on layered
    graphs."""
    from dags import rewrite_dag, strategy_chain
    from paper_2205_02473_b200.graph import synth_cluster as sc
    from paper_2205_02473_b200.ingest import layered_global_dfg
    from paper_2205_02473_b200.memory import ModelMeta
    from paper_2205_02473_b200.rewrite import (apply_op_fusion, apply_tensor_fusion,
                                               apply_tensor_partition, grad_accum_candidate,
                                               recompute_candidate)
    from paper_2205_02473_b200 import Error
    rng = np.random.default_rng(seed)
    pairs = []
    while len(pairs) < count:
        g = rewrite_dag(rng)
        for c in (recompute_candidate(g), grad_accum_candidate(g, ModelMeta())):
            if c is not None:
                pairs.append((g, c[0]))
        L = int(rng.integers(3, 7))
        m = LayeredModel(rng.integers(10, 400, L).tolist(), rng.integers(10, 800, L).tolist(),
                         rng.integers(1000, 4_000_000, L).tolist(), 5)
        lg = layered_global_dfg(m, sc("ring", 3, 0, 12500.0, 5.0))
        cg = lg
        for kind, a, b, k in strategy_chain(rng, lg, 4):
            try:
                cg = (apply_op_fusion(cg, a, b) if kind == 0 else
                      apply_tensor_fusion(cg, a, b) if kind == 1 else
                      apply_tensor_partition(cg, a, k))
            except Error:
                pass
        pairs.append((lg, cg))
    return pairs[:count]


def test_make_delta_merges_to_the_candidate():
    from paper_2205_02473_b200.delta import DeltaList, make_delta
    from paper_2205_02473_b200.engine import Csr
    pairs = _rewrite_pairs(3, 40)
    n_cut = 0
    for base, cand in pairs:
        dl = DeltaList([make_delta(base, cand)])  # owns the arrays d points into
        d = dl[0]
        n_cut += d.n_cut
        bc = Csr.from_dict(base.to_csr())
        dur, dev, fl, succ = merge_host(bc, base.size(), d)
        cc = cand.to_csr()
        assert np.array_equal(dur, cc["dur"]) and np.array_equal(fl, cc["flags"])
        bdevs = base.devices()
        extra = [dv for dv in cc["devices"] if dv not in bdevs]
        allv = bdevs + extra
        assert [allv[int(x)] for x in dev] == [cc["devices"][int(x)] for x in cc["dev"]]
        for k in range(cand.size()):
            assert succ[k] == sorted(cand.succ_indices(k)), k
    assert n_cut > 0  # the cut path is exercised


@pytest.mark.gpu
def test_gpu_replay_of_generic_deltas(engine):
    """Rewritten GlobalDFGs evaluated as deltas of their base (cut edges,
    removed/changed ops, new devices) replay exactly like the candidates."""
    from paper_2205_02473_b200 import replay_many
    from paper_2205_02473_b200.delta import DeltaList, make_delta
    from paper_2205_02473_b200.engine import Csr
    pairs = _rewrite_pairs(9, 30)
    by_base = {}
    for base, cand in pairs:
        by_base.setdefault(id(base), (base, []))[1].append(cand)
    for base, cands in by_base.values():
        res = engine.resident(Csr.from_dict(base.to_csr()))
        b = engine.delta_batch(res, DeltaList([make_delta(base, c) for c in cands]))
        b.replay(want_schedule=True)
        ms, st, er, s, e = b.results(schedule=True)
        for i, r in enumerate(replay_many(cands)):
            a, z = int(b.op_off[i]), int(b.op_off[i + 1])
            assert st[i] == 0 and ms[i] == r.iteration_time_us
            ids = [o.id for o in cands[i].ops()]
            assert s[a:z].tolist() == [r.schedule[x].start for x in ids]
            assert e[a:z].tolist() == [r.schedule[x].end for x in ids]


def _op_fusion_chain(g, workers, L, fj, bj):
    """The reference's sequential op fusions for fw/bw joins (left to right
    on FW chains, top-down on BW chains) via rewrite.apply_op_fusion."""
    from paper_2205_02473_b200.rewrite import apply_op_fusion
    for w in sorted(workers):
        a = 0
        while a < L:
            b = a
            while b + 1 < L and fj[b]:
                b += 1
            cur = f"{w}->FW.l{a}"
            for j in range(a + 1, b + 1):
                g = apply_op_fusion(g, cur, f"{w}->FW.l{j}")
                cur += f"+FW.l{j}"
            a = b + 1
        top = L - 1
        while top >= 0:
            lo = top
            while lo - 1 >= 0 and bj[lo - 1]:
                lo -= 1
            cur = f"{w}->BW.l{top}"
            for j in range(top - 1, lo - 1, -1):
                g = apply_op_fusion(g, cur, f"{w}->BW.l{j}")
                cur += f"+BW.l{j}"
            top = lo - 1
    return g


@pytest.mark.parametrize("scheme,W,S,L", [("ring", 3, 0, 6), ("ps", 3, 2, 7), ("ring", 4, 0, 9)])
def test_native_op_fusion_candidates_match_rewrite_chain(scheme, W, S, L):
    """dpro_graph_from_base_batch_ops / dpro_base_delta_batch_ops with op
    fusion (+ tensor fusion + partition) == the reference-pinned rewrite
    chain (apply_tensor_fusion / apply_tensor_partition / apply_op_fusion)."""
    from paper_2205_02473_b200.graph import synth_cluster as sc
    from paper_2205_02473_b200.ingest import layered_global_dfg
    from paper_2205_02473_b200.rewrite import apply_tensor_fusion, apply_tensor_partition
    rng = np.random.default_rng(L * 7 + W)
    c = sc(scheme, W, S, 12500.0, 5.0)
    m = LayeredModel(rng.integers(10, 400, L).tolist(), rng.integers(11, 801, L).tolist(),
                     rng.integers(1000, 4_000_000, L).tolist(), 5)
    base = LayeredBase(m, c)
    bv = base.graph()
    workers = [n.id for n in c.nodes if n.role == "worker"]
    specs, fjs, bjs, exps = [], [], [], []
    for t in range(6):
        fj = (rng.random(L - 1) < 0.4).astype(np.uint8)
        bj = (rng.random(L - 1) < 0.4).astype(np.uint8)
        cut = int(rng.integers(1, L - 1))
        groups = [list(range(0, cut + 1))] + [[i] for i in range(cut + 1, L)] if t % 2 else \
            [[i] for i in range(L)]
        ks = [int(rng.integers(1, 4)) for _ in groups]
        g = layered_global_dfg(m, c)
        if len(groups[0]) > 1:
            name = "g0"
            for i in groups[0][1:]:
                g = apply_tensor_fusion(g, name, f"g{i}")
                name += f"+g{i}"
        for grp, k in zip(groups, ks):
            g = apply_tensor_partition(g, "+".join(f"g{i}" for i in grp), k)
        exps.append(_op_fusion_chain(g, workers, L, fj, bj))
        specs.append((groups, ks))
        fjs.append(fj)
        bjs.append(bj)
    full = base.candidates(specs, fw_join=fjs, bw_join=bjs)
    ds = base.deltas(specs, fw_join=fjs, bw_join=bjs)
    for i, (ng, g) in enumerate(zip(full, exps)):
        a = g.to_csr()
        assert [o.id for o in g.ops()] == ng.op_ids(), i
        for f in ("dur", "dev", "flags", "succ_off", "succ", "indeg"):
            assert np.array_equal(a[f], getattr(ng.csr, f)), (i, f)
        dur, dev, fl, succ = merge_host(bv.csr, bv.n_ops, ds[i])  # the delta form too
        assert np.array_equal(dur, ng.csr.dur) and np.array_equal(fl, ng.csr.flags)
        for k in range(ng.n_ops):
            assert succ[k] == ng.csr.succ[ng.csr.succ_off[k]:ng.csr.succ_off[k + 1]].tolist()


@pytest.mark.gpu
def test_gpu_op_fusion_deltas_replay_like_full(engine):
    base, specs = _setup("ring", 8, 0, 24, 64, 5)
    rng = np.random.default_rng(1)
    fj = (rng.random((64, 23)) < 0.3).astype(np.uint8)
    bj = (rng.random((64, 23)) < 0.3).astype(np.uint8)
    full = base.candidates(specs, fw_join=fj, bw_join=bj)
    fb = engine.batch([g.csr for g in full])
    fb.replay(want_schedule=True)
    ms0, st0, _, s0, e0 = fb.results(schedule=True)
    res = engine.resident(base.graph().csr)
    db = engine.delta_batch(res, base.deltas(specs, fw_join=fj, bw_join=bj))
    db.replay(want_schedule=True)
    ms1, st1, _, s1, e1 = db.results(schedule=True)
    assert np.all(st0 == 0) and np.array_equal(ms0, ms1)
    assert np.array_equal(s0, s1) and np.array_equal(e0, e1)


@pytest.mark.gpu
def test_delta_batch_edge_cases(engine):
    """Empty batches and malformed deltas: empty results, or the engine's
    EINVAL with the reason (no device work, no crash)."""
    from paper_2205_02473_b200.delta import DeltaArrays, DeltaList, make_delta
    from paper_2205_02473_b200.engine import Csr
    from paper_2205_02473_b200.errors import Error
    base, specs = _setup("ring", 4, 0, 5, 2, 3)
    res = engine.resident(base.graph().csr)
    b = engine.delta_batch(res, DeltaList([]))
    b.replay(want_schedule=False)
    ms, st, *_ = b.results()
    assert ms.size == 0 and st.size == 0
    # a no-op delta replays the base itself
    g = base.graph().to_global_dfg()
    d0 = make_delta(g, g)
    assert d0.removed.size == 0 and d0.new_pos.size == 0
    b = engine.delta_batch(res, DeltaList([d0]))
    b.replay(want_schedule=False)
    fb = engine.batch([base.graph().csr])
    fb.replay(want_schedule=False)
    assert b.results()[0].tolist() == fb.results()[0].tolist()
    # malformed: removed index out of range, new_pos not sorted, bad successor
    u32 = lambda x: np.array(x, np.uint32)  # noqa: E731
    empty = dict(new_pos=u32([]), new_dur=np.zeros(0, np.int64), new_dev=np.zeros(0, np.uint16),
                 new_flags=np.zeros(0, np.uint8), new_succ_off=u32([0]), new_succ=u32([]),
                 extra_src=u32([]), extra_dst=u32([]), cut=u32([]))
    n = base.graph().n_ops
    bad = [DeltaArrays(d0.n_devices, u32([n + 5]), **empty),
           DeltaArrays(d0.n_devices, u32([]), **{**empty, "new_pos": u32([3, 1]),
                                                  "new_dur": np.ones(2, np.int64),
                                                  "new_dev": np.zeros(2, np.uint16),
                                                  "new_flags": np.zeros(2, np.uint8),
                                                  "new_succ_off": u32([0, 0, 0])}),
           DeltaArrays(d0.n_devices, u32([]), **{**empty, "new_pos": u32([0]),
                                                  "new_dur": np.ones(1, np.int64),
                                                  "new_dev": np.zeros(1, np.uint16),
                                                  "new_flags": np.zeros(1, np.uint8),
                                                  "new_succ_off": u32([0, 1]),
                                                  "new_succ": u32([n + 7])})]
    for d in bad:
        with pytest.raises(Error, match="delta 0"):
            engine.delta_batch(res, DeltaList([d]))
    # the engine stays usable afterwards
    b = engine.delta_batch(res, base.deltas(specs))
    b.replay(want_schedule=False)
    assert np.all(b.results()[1] == 0)


@pytest.mark.parametrize("scheme,W,S,L", [("ring", 4, 0, 8), ("ps", 3, 2, 7), ("ring", 11, 0, 5)])
def test_graph_variants_as_deltas_merge_exactly(scheme, W, S, L):
    """dpro_base_delta_from_graphs: recompute / grad-accum / partitioned /
    fused graphs against the base; merging the delta gives the graph's own
    CSR and device names."""
    from paper_2205_02473_b200.ingest import layered_graph, layered_graph_variant
    base, specs = _setup(scheme, W, S, L, 3, W + 7 * L)
    m, c = base.model, base.cluster
    graphs = [layered_graph_variant(m, c, "recompute", 0.5),
              layered_graph_variant(m, c, "grad-accum", 0.55),
              layered_graph_variant(m, c, "grad-accum", 0.5, [2] * L),
              layered_graph(m, c, [3] * L)] + base.candidates(specs)
    bv = base.graph()
    ds = base.deltas_from_graphs(graphs, threads=3)
    for i, g in enumerate(graphs):
        dur, dev, fl, succ = merge_host(bv.csr, bv.n_ops, ds[i])
        cs = g.csr
        assert len(dur) == g.n_ops
        assert np.array_equal(dur, cs.dur) and np.array_equal(fl, cs.flags)
        strs = g.device_strs()
        assert [ds.device_str(i, int(x)) for x in dev] == [strs[int(x)] for x in cs.dev]
        for k in range(g.n_ops):
            assert succ[k] == cs.succ[cs.succ_off[k]:cs.succ_off[k + 1]].tolist(), (i, k)
    same_set = base.deltas_from_graphs([bv])
    same = same_set[0]
    assert same.n_removed == same.n_new == same.n_extra == same.n_cut == 0


def test_single_worker_op_fusion_deltas_match_reference_rewrite(ref):
    """join_worker: the reference's own op-fusion candidate, apply_op_fusion
    (optimize.cpp:245-318) of two adjacent ops of ONE worker."""
    spec = {"layers": 6, "fw_dur_us": [11, 23, 35, 47, 59, 61], "bw_dur_us": [13, 27, 31, 43, 57, 69],
            "tensor_bytes": [1000, 25000, 3000, 40000, 500, 60000], "update_dur_us": 5,
            "scheme": "ring", "workers": 11, "ps_count": 0, "bandwidth_bytes_per_us": 125.0,
            "latency_us": 5.0}
    m = LayeredModel(spec["fw_dur_us"], spec["bw_dur_us"], spec["tensor_bytes"], 5)
    c = synth_cluster("ring", 11, 0, 125.0, 5.0)
    base = LayeredBase(m, c)
    L = 6
    cases = [(3, "FW", 2), (10, "BW", 4), (0, "FW", 0), (7, "BW", 0)]
    fj = np.zeros((len(cases), L - 1), np.uint8)
    bj = np.zeros((len(cases), L - 1), np.uint8)
    for r, (wk, kind, i) in enumerate(cases):
        (fj if kind == "FW" else bj)[r, i] = 1
    specs = [([[i] for i in range(L)], [1] * L)] * len(cases)
    ds = base.deltas(specs, fw_join=fj, bw_join=bj, join_worker=[wk for wk, _, _ in cases])
    bv = base.graph()
    rg0 = ref.RefGraph.synth(spec)
    for r, (wk, kind, i) in enumerate(cases):
        w = base.worker(wk)
        a, b = (f"{w}->FW.l{i}", f"{w}->FW.l{i + 1}") if kind == "FW" else \
            (f"{w}->BW.l{i + 1}", f"{w}->BW.l{i}")
        rg = rg0.op_fusion(a, b)
        ex = rg.export()
        dur, dev, fl, succ = merge_host(bv.csr, bv.n_ops, ds[r])
        assert np.array_equal(dur, ex["dur"]) and np.array_equal(fl, ex["flags"])
        rstr = rg.device_strs()
        assert [ds.device_str(r, int(x)) for x in dev] == [rstr[int(x)] for x in ex["dev"]]
        for k in range(len(dur)):
            assert succ[k] == ex["succ"][ex["succ_off"][k]:ex["succ_off"][k + 1]].tolist()
