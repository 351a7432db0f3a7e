"""Native timeline writer throughput on a BASELINE config graph:
python tools/timeline_speed.py CONFIG [PATH]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    from paper_2205_02473_b200.engine import Engine
    from paper_2205_02473_b200.ingest import layered_graph
    from paper_2205_02473_b200.workloads import workload
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    path = sys.argv[2] if len(sys.argv) > 2 else "/dev/null"
    w = workload(cfg)
    g = layered_graph(w.model, w.cluster)
    eng = Engine(0)
    b = eng.batch([g.csr])
    b.replay(want_schedule=True)
    _, st, _, s, e = b.results(schedule=True)
    t = time.perf_counter()
    g.write_timeline(path, s, e)
    el = time.perf_counter() - t
    size = Path(path).stat().st_size if path != "/dev/null" else -1
    print(f"config {cfg}: {g.n_ops} ops, timeline written in {el:.2f} s "
          f"({g.n_ops / el / 1e6:.2f} M ops/s), {size} bytes")


if __name__ == "__main__":
    main()
