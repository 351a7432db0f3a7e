"""Times the pieces of the e2e path (host CSR -> makespans) for config 2."""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2205_02473_b200 import _native as N  # noqa: E402
from paper_2205_02473_b200.engine import Engine  # noqa: E402
from paper_2205_02473_b200.ingest import layered_graphs  # noqa: E402
from paper_2205_02473_b200.workloads import workload  # noqa: E402

w = workload(2)
graphs = layered_graphs(w.model, w.cluster, w.candidate_partitions(1024), threads=16)
eng = Engine(0)
B = len(graphs)
arr = (N.DproCsr * B)(*[g.csr.as_struct() for g in graphs])
ms = np.zeros(B, np.int64); st = np.zeros(B, np.int32); er = np.zeros(B, np.int64)
for it in range(4):
    t0 = time.perf_counter()
    b = N.lib.dpro_cuda_batch_create(eng.ctx, arr, B, N.DPRO_HOST)
    t1 = time.perf_counter()
    N.lib.dpro_cuda_batch_replay(eng.ctx, b, 0)
    N.lib.dpro_cuda_batch_results(eng.ctx, b, N.ptr(ms), N.ptr(st), N.ptr(er), None, None)
    t2 = time.perf_counter()
    N.lib.dpro_cuda_batch_destroy(eng.ctx, b)
    t3 = time.perf_counter()
    print(f"create(pack+H2D+pack kernel) {1e3*(t1-t0):.1f} ms, replay+D2H {1e3*(t2-t1):.1f} ms, "
          f"destroy {1e3*(t3-t2):.1f} ms, total {1e3*(t3-t0):.1f} ms")
