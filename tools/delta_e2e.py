"""Config-2 e2e: full host CSR vs resident base + deltas (timing sketch)."""
import ctypes as C, os, sys, time
import numpy as np
sys.path.insert(0, '.')
from paper_2205_02473_b200 import _native as N
from paper_2205_02473_b200.engine import Engine
from paper_2205_02473_b200.ingest import LayeredBase, layered_graphs
from paper_2205_02473_b200.workloads import workload

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
w = workload(cfg)
pk = w.candidate_partitions(B)
t = time.perf_counter(); graphs = layered_graphs(w.model, w.cluster, pk, threads=os.cpu_count()); t_full = time.perf_counter() - t
base = LayeredBase(w.model, w.cluster)
specs = [([[i] for i in range(w.layers)], pk[c].tolist()) for c in range(B)]
t = time.perf_counter(); ds = base.deltas(specs, threads=os.cpu_count()); t_delta = time.perf_counter() - t
print(f"build full {t_full:.3f}s  deltas {t_delta:.3f}s")
eng = Engine(0)
res = eng.resident(base.graph().csr)
arr = (N.DproCsr * B)(*[g.csr.as_struct() for g in graphs])
hm = np.zeros(B, np.int64); hs = np.zeros(B, np.int32); he = np.zeros(B, np.int64)
dm = np.zeros(B, np.int64)
def full():
    assert N.lib.dpro_cuda_replay_batch(eng.ctx, arr, B, N.DPRO_HOST, N.ptr(hm), None, None, N.ptr(hs), N.ptr(he)) == 0
def delta():
    assert N.lib.dpro_cuda_replay_delta_batch(eng.ctx, res.handle, C.cast(ds.array, C.c_void_p), B, N.ptr(dm), N.ptr(hs), N.ptr(he)) == 0
for name, fn in (("full", full), ("delta", delta)):
    fn()
    ts = []
    for _ in range(5):
        t = time.perf_counter(); fn(); ts.append(time.perf_counter() - t)
    print(f"{name}: {np.median(ts)*1e3:.2f} ms/step  {B/np.median(ts):.0f} replays/s")
assert np.array_equal(hm, dm) and np.all(hs == 0)
blob = sum(4*d.n_removed + 15*d.n_new + 4*(d.n_new+1) + 4*int(np.ctypeslib.as_array(C.cast(d.new_succ_off, C.POINTER(C.c_uint32)), (d.n_new+1,))[-1]) + 8*d.n_extra for d in ds.array)
print("delta bytes/step", blob)
os.environ["DPRO_TRACE"] = "1"
