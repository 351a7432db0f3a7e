import sys; sys.path.insert(0, '/root/repo')
from paper_2205_02473_b200 import (GraphBuilder, comp, replay, execution_graph, critical_path,
                                   sync_makespan, ModelMeta, estimate_peak_memory, memory_pass,
                                   write_timeline)
b = GraphBuilder()
b.add_op(comp("w0->FW.a", "w0", 10)); b.add_op(comp("w0->FW.b", "w0", 10))
b.add_edge("w0->FW.a", "w0->FW.b")
g = b.build()
r = replay(g)
path = critical_path(execution_graph(g, r), r)
peaks = estimate_peak_memory(g, r, ModelMeta({"FW.a": 10, "FW.b": 10}, {"w0": 100}))
write_timeline("/tmp/timeline.json", g, r)
print(r.iteration_time_us, [p.op for p in path.ops], peaks)
from paper_2205_02473_b200.engine import Engine
from paper_2205_02473_b200.ingest import LayeredBase
from paper_2205_02473_b200.workloads import workload
w = workload(2)
base = LayeredBase(w.model, w.cluster)
specs = [([[i] for i in range(w.layers)], list(k)) for k in w.candidate_partitions(1024)]
eng = Engine(0)
batch = eng.delta_batch(eng.resident(base.graph().csr), base.deltas(specs))
batch.replay(want_schedule=False)
makespans, status, *_ = batch.results()
print(makespans[:3], int((status == 0).sum()))
from paper_2205_02473_b200.search import SyncSearch
best = SyncSearch(w.model, w.cluster, eng, op_fusion=True).run(rounds=3, batch=256)
print(best.makespan)
