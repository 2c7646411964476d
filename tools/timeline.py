"""GPU timeline of one batch from the engine's CUDA events (profiling mode).

    DIAM_B200_GROUPS=4 python tools/timeline.py [--config d1024]

Prints, per kernel class, the time covered and the union of busy time over all
streams, so idle gaps (host round trips, dependency stalls) become visible.
"""
import argparse
import collections
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="d1024")
    ap.add_argument("--phases", action="store_true", help="per-stream start/end of every class")
    args = ap.parse_args()
    path = os.path.join(tempfile.gettempdir(), f"diam_timeline_{os.getpid()}.csv")
    os.environ["DIAM_B200_TIMELINE"] = path
    import bench
    import paper_1506_05741_b200 as pkg
    cfg = bench.CONFIGS[args.config]
    kind, d, per_gpu, n_lag, M = cfg
    lib = pkg.load()
    tp = bench.make_target_file(kind, d)
    t = lib.target_load(tp)
    eng = lib.engine(t, **bench.run_options(cfg, per_gpu))
    eng.run_batches(2)
    eng.set_profiling(True)
    ms = eng.run_batches(1)
    eng.stat("gemm_target")  # resolves the events -> CSV
    rows = []
    for line in open(path):
        name, stream, a, b = line.strip().split(",")
        rows.append((name, stream, float(a), float(b)))
    os.unlink(path)
    os.unlink(tp)
    rows.sort(key=lambda r: r[2])
    end = max(r[3] for r in rows)
    # union of busy intervals
    busy, cur_s, cur_e = 0.0, None, None
    for _, _, a, b in rows:
        if cur_s is None or a > cur_e:
            if cur_s is not None:
                busy += cur_e - cur_s
            cur_s, cur_e = a, b
        else:
            cur_e = max(cur_e, b)
    busy += cur_e - cur_s
    per = collections.defaultdict(float)
    for n, _, a, b in rows:
        per[n] += b - a
    print(f"batch {ms:.2f} ms (events span {end:.2f} ms); union of instrumented kernels busy {busy:.2f} ms "
          f"({100 * busy / end:.1f}%)")
    for n, v in sorted(per.items(), key=lambda kv: -kv[1]):
        print(f"  {n:14s} {v:8.2f} ms summed over streams")
    streams = sorted({r[1] for r in rows})
    if args.phases:
        for si, st in enumerate(streams):
            rs = [r for r in rows if r[1] == st]
            print(f"stream {si}: " + " ".join(f"{n[:4]}@{a:.1f}-{b:.1f}" for n, _, a, b in rs))
    for s in streams:
        rs = [r for r in rows if r[1] == s]
        span = rs[-1][3] - rs[0][2]
        work = sum(r[3] - r[2] for r in rs)
        print(f"  stream {s}: {len(rs)} events, covered {work:.2f} ms of {span:.2f} ms")


if __name__ == "__main__":
    main()
