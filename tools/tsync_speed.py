"""t_sync grid throughput (sync_makespan over a (bytes, k) grid): K2 (graphs
generated on the GPU) vs the host-built graphs, same values.

    python tools/tsync_speed.py [scheme W S n_bytes kmax]"""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    a = sys.argv[1:]
    scheme = a[0] if a else "ring"
    W, S = (int(a[1]), int(a[2])) if len(a) > 2 else (8, 0)
    nb, kmax = (int(a[3]), int(a[4])) if len(a) > 4 else (256, 16)
    from paper_2205_02473_b200.engine import Engine
    from paper_2205_02473_b200.graph import synth_cluster
    c = synth_cluster(scheme, W, S, 12500.0, 5.0)
    rng = np.random.default_rng(1)
    sizes = rng.integers(1000, 400_000_000, nb)
    b = np.repeat(sizes, kmax)
    k = np.tile(np.arange(1, kmax + 1), nb)
    eng = Engine(0)
    out = {"grid": int(len(b)), "cluster": f"{scheme} W={W} S={S}"}
    for host in (0, 1):
        eng.set_option("tsync_host", host)
        eng.tsync_grid(c, b[:64], k[:64])  # warm-up
        t = time.perf_counter()
        ms, st = eng.tsync_grid(c, b, k)
        el = time.perf_counter() - t
        out["host" if host else "device"] = {"seconds": el, "t_sync_per_s": len(b) / el,
                                             "ok": int((st == 0).sum())}
        out.setdefault("values", []).append(ms)
    eng.set_option("tsync_host", 0)
    out["equal"] = bool(np.array_equal(out["values"][0], out["values"][1]))
    del out["values"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
