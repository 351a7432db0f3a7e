import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2205_02473_b200.engine import Engine
from paper_2205_02473_b200.ingest import layered_graphs
from paper_2205_02473_b200.workloads import workload
cfg = int(sys.argv[1])
w = workload(cfg)
pk = w.candidate_partitions(1024)
graphs = layered_graphs(w.model, w.cluster, pk, threads=16)
eng = Engine(0)
for ring in (64,):
    for i, g in enumerate(graphs):
        b = eng.batch([g.csr]); b.replay(False); b.results()
        st = b.stats()
        if st["fallbacks"]:
            ks = {int(j): int(pk[i][j]) for j in np.flatnonzero(pk[i] > 1)}
            print(i, "V", g.n_ops, "ring", st["ring"], "parts", ks, "max indeg", int(g.csr.indeg.max()),
                  "max outdeg", int(np.diff(g.csr.succ_off.astype(np.int64)).max()))
