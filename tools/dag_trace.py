"""Summarise a task-graph POTRF trace (DIAM_B200_DAG_TRACE=<csv>).

    DIAM_B200_DAG_TRACE=/tmp/dag.csv python tools/bench_diag.py 1024
    python tools/dag_trace.py /tmp/dag.csv
"""
import collections
import sys

import numpy as np


def main():
    rows = np.loadtxt(sys.argv[1], delimiter=",", dtype=np.float64)
    typ = rows[:, 0].astype(int)
    grab, deps, done = rows[:, 5], rows[:, 6], rows[:, 7]
    t0 = grab.min()
    print(f"{len(rows)} tasks, span {(done.max() - t0) / 1e3:.1f} us")
    names = {0: "POTRF", 1: "TRSM", 2: "UPDATE"}
    for k in sorted(names):
        m = typ == k
        if not m.any():
            continue
        ex = (done[m] - deps[m]) / 1e3
        wt = (deps[m] - grab[m]) / 1e3
        print(f"  {names[k]:6s} n={m.sum():6d} exec mean {ex.mean():7.1f} us (p50 {np.median(ex):6.1f}, max {ex.max():7.1f})"
              f"  wait mean {wt.mean():7.1f} us  busy {ex.sum() / 1e3:8.2f} ms")
    busy = (done - deps).sum()
    waits = (deps - grab).sum()
    print(f"  worker time: exec {busy / 1e6:.2f} ms, dependency waits {waits / 1e6:.2f} ms")
    # per-k POTRF completion times (critical path progress)
    pk = collections.defaultdict(list)
    for r in rows[typ == 0]:
        pk[int(r[4])].append(r[7] - t0)
    print("  POTRF(k) done (us, max over chains): " +
          " ".join(f"{k}:{max(v) / 1e3:.0f}" for k, v in sorted(pk.items())))


if __name__ == "__main__":
    main()
