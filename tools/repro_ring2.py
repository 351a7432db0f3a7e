import sys, os
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1])); sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from dags import random_dag_ref, acceptance_dag, fuzz_dag
from paper_2205_02473_b200.engine import Engine, Csr
w = int(sys.argv[1]); which = sys.argv[2]
rng = np.random.default_rng(1000)
graphs = []
for t in range(1500):
    k = t % 5
    if k == 0: graphs.append(random_dag_ref(rng))
    elif k == 1: graphs.append(acceptance_dag(rng))
    elif k == 2: graphs.append(fuzz_dag(rng, max_ops=80, zero_p=0.5, virt_p=0.2))
    elif k == 3: graphs.append(fuzz_dag(rng, max_ops=200, zero_p=0.2, virt_p=0.1, edge_p=0.03, max_dur=3))
    else: graphs.append(fuzz_dag(rng, max_ops=30, zero_p=0.8, virt_p=0.3))
if which != "all":
    a, z = (int(x) for x in which.split(":"))
    graphs = graphs[a:z]
e = Engine(0); e.set_option("ring", 2); e.set_option("warps", w)
b = e.batch([Csr.from_dict(g.to_csr()) for g in graphs])
b.replay(True)
ms, st, er, s, en = b.results(schedule=True)
print("warps", w, "ok", (st == 0).sum(), "fallbacks", b.stats()["fallbacks"])
if len(graphs) == 1:
    g = graphs[0]
    print("n", g.size(), "devs", g.to_csr()["n_devices"], "edges", g.edge_count())
    import json
    print(json.dumps({"ops": [[o.id, int(o.kind), int(o.device.kind), o.device.node, o.device.peer, int(o.dur)] for o in g.ops()],
                      "edges": [[g.op_at(i).id, g.op_at(s).id] for i in range(g.size()) for s in g.succ_indices(i)]}))
