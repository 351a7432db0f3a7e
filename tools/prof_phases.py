"""Phase breakdown of the fast replay (needs a -DDPRO_PROFILE build in DPRO_LIB)."""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2205_02473_b200 import _native as N  # noqa: E402
from paper_2205_02473_b200.engine import Engine  # noqa: E402
from paper_2205_02473_b200.ingest import layered_graphs  # noqa: E402
from paper_2205_02473_b200.workloads import workload  # noqa: E402

cfg = int(os.environ.get("CFG", "2"))
nb = int(os.environ.get("NB", "1024"))
w = workload(cfg)
eng = Engine(0)
eng.set_option("warps", int(os.environ.get("DPRO_WARPS", "4")))
if os.environ.get("OVERLAY"):  # the bench's candidate mix on overlay batches
    from paper_2205_02473_b200.ingest import LayeredBase
    base = LayeredBase(w.model, w.cluster)
    deltas, _ = w.candidate_deltas(base, nb, threads=16, variants=False)
    eng.set_option("overlay", 1)
    res = eng.resident(base.graph().csr)
    b = eng.delta_batch(res, deltas)
else:
    graphs = layered_graphs(w.model, w.cluster, w.candidate_partitions(nb), threads=16)
    b = eng.batch([g.csr for g in graphs])
fn = N.lib.dpro_debug_prof
fn.argtypes = [C.c_void_p]
buf = np.zeros(16, np.uint64)
b.replay(True); b.results(); fn(buf.ctypes.data)
b.replay(True); b.results(); fn(buf.ctypes.data)
rounds, zr = int(buf[0]), int(buf[1])
print(f"candidates {nb}: rounds/cand {rounds/nb:.0f} (zero rounds {zr/nb:.0f})")
names = ["reduce+zero-check", "collect ranges", "expand", "dispatch"]
tot = sum(int(buf[i]) for i in range(2, 6))
for i, nm in enumerate(names):
    v = int(buf[2 + i])
    print(f"  {nm:18s} {v/rounds:8.1f} cycles/round ({100*v/tot:4.1f}%)")
print(f"  expand passes/round {int(buf[8])/rounds:.2f}, records/round {int(buf[9])/rounds:.1f}, "
      f"thread0 work {int(buf[10])/rounds:.0f} cyc/round, barrier wait {int(buf[11])/rounds:.0f} cyc/round")
print(f"  thread0: waiting for record loads {int(buf[12])/rounds:.0f} cyc/round, applying {int(buf[13])/rounds:.0f} cyc/round")
print(f"  total {tot/rounds:.1f} cycles/round; ranges/round {int(buf[6])/rounds:.2f}; "
      f"dispatching lanes/round {int(buf[7])/rounds:.2f}")
