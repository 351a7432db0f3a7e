"""Parity at BASELINE scale: the product path -- candidates
as deltas of an HBM-resident base, merged (K0), packed and replayed (K1) on
the GPU, critical path by K3 -- against the reference itself (oracle/_ref:
the unmodified proj/src) on the SAME candidates built by the reference's own
generator and rewrites (RefGraph.synth + apply_tensor_partition /
apply_op_fusion / apply_strategy). Every start/end, the makespan and the
critical path are compared. Config 5 (10M ops) runs against the pinned C
port (tests/test_oracle.py); ns-scaled durations (x1000, the north_star's
integer-ns unit) must run on the fast path and give exactly 1000x the us
schedule (replay.cpp only adds and compares times)."""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from paper_2205_02473_b200.engine import Csr
from paper_2205_02473_b200.ingest import LayeredBase, layered_graph_variant
from paper_2205_02473_b200.workloads import opf_pair, synth_spec, workload

pytestmark = pytest.mark.gpu


def _ref_candidates(ref, spec, descs, threads=16):
    base = ref.RefGraph.synth(synth_spec(spec))

    def build(d):
        if d[0] == "recompute":
            return base.apply_memory_strategy(3, {})
        if d[0] == "grad-accum":
            return base.apply_memory_strategy(4, {})
        if d[0] == "opf":
            return base.op_fusion(*opf_pair(d))
        g = base
        for i, k in enumerate(d[1]):
            if k != 1:
                g = g.partition(f"g{i}", int(k))
        return g
    with ThreadPoolExecutor(threads) as ex:
        return list(ex.map(build, descs))


def _gpu_delta_batch(engine, w, n, rank=0):
    base = LayeredBase(w.model, w.cluster)
    deltas, descs = w.candidate_deltas(base, n, rank=rank, threads=16)
    res = engine.resident(base.graph().csr)
    b = engine.delta_batch(res, deltas)
    b.replay(want_schedule=True)
    ms, st, _, start, end = b.results(schedule=True)
    return base, deltas, descs, b, ms, st, start, end


def _compare_with_ref(b, i, ms, st, start, end, paths, rg):
    T, rs, re, _, _ = rg.replay()
    a, z = int(b.op_off[i]), int(b.op_off[i + 1])
    assert st[i] == 0, i
    assert ms[i] == T, (i, ms[i], T)
    assert z - a == rg.n_ops
    assert np.array_equal(start[a:z], rs), i
    assert np.array_equal(end[a:z], re), i
    assert np.array_equal(paths[i], rg.critical_path()["path"]), i


@pytest.mark.parametrize("config,n", [(1, 64), (2, 64), (3, 64)])
def test_full_size_configs_vs_reference(engine, ref, config, n):
    """Configs 1-3 at full size, 64 candidates each (delta path), against
    dpro::replay + dpro::critical_path on the reference-built candidates."""
    w = workload(config)
    base, deltas, descs, b, ms, st, start, end = _gpu_delta_batch(engine, w, n)
    assert b.stats()["fallbacks"] == 0
    paths = b.critical_paths()
    rgs = _ref_candidates(ref, w.spec, descs)
    with ThreadPoolExecutor(16) as ex:
        list(ex.map(lambda i: _compare_with_ref(b, i, ms, st, start, end, paths, rgs[i]),
                    range(n)))


def test_config4_candidates_vs_reference_and_port(engine, ref, port):
    """Config 4 (GPT-2 medium ring-64, 4.80M ops): the batch's candidate mix
    on the GPU. One op-fusion candidate against the reference itself (built
    by RefGraph.synth + apply_op_fusion: ~2.5 min of host time), the
    recompute / grad-accum candidates and one more op fusion against the
    pinned C port on the same CSRs."""
    w = workload(4)
    base, deltas, descs, b, ms, st, start, end = _gpu_delta_batch(engine, w, 6)
    assert (st == 0).all()
    paths = b.critical_paths()
    assert [d[0] for d in descs[:2]] == ["recompute", "grad-accum"]
    # candidate 2 (single-worker op fusion) vs the reference
    rg = _ref_candidates(ref, w.spec, [descs[2]])[0]
    _compare_with_ref(b, 2, ms, st, start, end, paths, rg)
    # candidates 0, 1 (memory variants, generated natively) and 3 vs the port
    cands = [layered_graph_variant(w.model, w.cluster, "recompute", 0.5),
             layered_graph_variant(w.model, w.cluster, "grad-accum", 0.5)]
    for i, g in ((0, cands[0]), (1, cands[1])):
        o = port.port_replay(g.csr)
        a, z = int(b.op_off[i]), int(b.op_off[i + 1])
        assert ms[i] == o["T"] and np.array_equal(start[a:z], o["start"])
        assert np.array_equal(end[a:z], o["end"]) and np.array_equal(paths[i], o["path"])


def test_config5_scale_vs_port(engine, port):
    """Config 5 (BERT-large ring-128, ~10M ops), two partition candidates as
    deltas, every start/end against the C port."""
    w = workload(5)
    base = LayeredBase(w.model, w.cluster)
    pk = w.candidate_partitions(2)
    specs = [([[i] for i in range(w.layers)], pk[c].tolist()) for c in range(2)]
    res = engine.resident(base.graph().csr)
    b = engine.delta_batch(res, base.deltas(specs, threads=16))
    b.replay(want_schedule=True)
    ms, st, _, start, end = b.results(schedule=True)
    full = base.candidates(specs, threads=2)
    for i, g in enumerate(full):
        o = port.port_replay(g.csr)
        a, z = int(b.op_off[i]), int(b.op_off[i + 1])
        assert st[i] == 0 and ms[i] == o["T"]
        assert np.array_equal(start[a:z], o["start"]) and np.array_equal(end[a:z], o["end"])


def _scaled(csr: Csr, f: int) -> Csr:
    return Csr(np.ascontiguousarray(csr.dur * f, np.int64), csr.dev, csr.flags, csr.succ_off,
               csr.succ, csr.indeg, csr.n_devices)


@pytest.mark.parametrize("config,n", [(2, 32), (4, 2)])
def test_ns_durations_on_the_fast_path(engine, config, n):
    """Durations x1000 (us -> ns): sum(dur) is far above 2^31 (config 4:
    ~10^12 ns), yet every candidate stays on the fast path (no general-path
    fallback) and the schedule is exactly 1000x the us one."""
    w = workload(config)
    base = LayeredBase(w.model, w.cluster)
    pk = w.candidate_partitions(n)
    specs = [([[i] for i in range(w.layers)], pk[c].tolist()) for c in range(n)]
    graphs = base.candidates(specs, threads=8)
    us = engine.batch([g.csr for g in graphs])
    us.replay(want_schedule=True)
    ms_us, st_us, _, s_us, e_us = us.results(schedule=True)
    ns = engine.batch([_scaled(g.csr, 1000) for g in graphs])
    ns.replay(want_schedule=True)
    ms_ns, st_ns, _, s_ns, e_ns = ns.results(schedule=True)
    assert ns.stats()["fallbacks"] == 0
    assert (st_us == 0).all() and (st_ns == 0).all()
    assert int(graphs[0].csr.dur.sum()) * 1000 > 2 ** 31  # the old fast-path limit
    assert np.array_equal(ms_ns, ms_us * 1000)
    assert np.array_equal(s_ns, s_us * 1000) and np.array_equal(e_ns, e_us * 1000)
    for i in range(n):
        o1, d1, b1 = us.timelines(i)
        o2, d2, b2 = ns.timelines(i)
        assert np.array_equal(o1, o2) and np.array_equal(b2, b1 * 1000)
