"""GlobalDFG.fused (the index-array op fusion behind rewrite.apply_op_fusion)
equals the GraphBuilder construction it replaces: same ops in the same
order, same edges, same tensors, same engine CSR -- on layered ring / PS
graphs, with and without a cached CSR, including chains of fusions."""
import numpy as np
import pytest

from paper_2205_02473_b200.errors import CycleError, TransformError
from paper_2205_02473_b200.graph import GraphBuilder, synth_cluster
from paper_2205_02473_b200.ingest import LayeredModel, layered_global_dfg
from paper_2205_02473_b200.rewrite import apply_op_fusion, fused_op_id


def _builder_fusion(g, a, b, fused):
    preds = (set(g.preds(a)) | set(g.preds(b))) - {a, b}
    succs = (set(g.succs(a)) | set(g.succs(b))) - {a, b}
    bld = GraphBuilder(g)
    bld.remove_ops([a, b])
    bld.add_op(fused)
    for p in preds:
        bld.add_edge(p, fused.id)
    for t in succs:
        bld.add_edge(fused.id, t)
    return bld.build()


def _same(x, y):
    assert [o.id for o in x.ops()] == [o.id for o in y.ops()]
    assert [o.dur for o in x.ops()] == [o.dur for o in y.ops()]
    assert x.edge_count() == y.edge_count()
    for i in range(x.size()):
        assert list(x.succ_indices(i)) == list(y.succ_indices(i)), i
        assert list(x.pred_indices(i)) == list(y.pred_indices(i)), i
    assert x.edge_set() == y.edge_set()
    assert x.tensor_units().keys() == y.tensor_units().keys()
    cx, cy = x.to_csr(), y.to_csr()
    for k in ("dur", "dev", "flags", "succ_off", "succ", "indeg"):
        assert np.array_equal(cx[k], cy[k]), k
    assert cx["devices"] == cy["devices"]


@pytest.mark.parametrize("scheme,W,S,L,seed", [("ring", 4, 0, 8, 1), ("ps", 4, 2, 6, 2),
                                               ("ring", 8, 0, 12, 3)])
def test_fused_equals_builder(scheme, W, S, L, seed):
    rng = np.random.default_rng(seed)
    m = LayeredModel(rng.integers(10, 400, L).tolist(), rng.integers(10, 800, L).tolist(),
                     rng.integers(1000, 4_000_000, L).tolist(), 5)
    g = layered_global_dfg(m, synth_cluster(scheme, W, S, 12500.0, 5.0))
    done = 0
    for step in range(40):
        if step % 2:
            g.to_csr()  # exercise the carried CSR
        comp = [o.id for o in g.ops() if o.kind.name in ("FW", "BW")]
        a = comp[int(rng.integers(len(comp)))]
        ss = [s for s in g.succs(a) if g.op(s).kind.name in ("FW", "BW")
              and g.op(s).device == g.op(a).device]
        if not ss:
            continue
        b = ss[int(rng.integers(len(ss)))]
        try:
            h = apply_op_fusion(g, a, b)
        except (CycleError, TransformError):
            continue
        fused = h.op(fused_op_id(a, b))
        _same(h, _builder_fusion(g, a, b, fused))
        g = h
        done += 1
    assert done >= 5
