"""Marginal cost of each kernel class in the grouped engine (timing experiment).

    python tools/twice_sweep.py [--config d1024] [--batches 5]

Runs the bench workload with DIAM_B200_TWICE=<class> (the class's idempotent step is
launched twice, so the run itself is unchanged) and prints the batch time against the plain
run: the difference is what one instance of the class costs in the real, overlapped
schedule -- unlike the single-stream per-class times of bench.py's profile pass.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1506_05741_b200 as pkg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="d1024", choices=sorted(bench.CONFIGS))
    ap.add_argument("--batches", type=int, default=5)
    ap.add_argument("--sets", default="none,normals,trmm,target,potrf")
    ap.add_argument("--twice", action="store_true", default=True, help="DIAM_B200_TWICE (the only mode)")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    kind, d, per_gpu, n_lag, M = cfg
    lib = pkg.load()
    path = bench.make_target_file(kind, d)
    t = lib.target_load(path)
    base = None
    for s in args.sets.split(","):
        var = "DIAM_B200_TWICE"
        if s == "none":
            os.environ.pop(var, None)
        else:
            os.environ[var] = s
        eng = lib.engine(t, **bench.run_options(cfg, per_gpu))
        eng.run_batches(2)
        ms = eng.run_batches(args.batches) / args.batches
        del eng
        if base is None:
            base = ms
        print(f"{'twice' if args.twice else 'skip'} {s:24s} {ms:7.2f} ms/batch  (delta {ms - base:+6.2f})", flush=True)
    os.environ.pop(var, None)
    os.unlink(path)


if __name__ == "__main__":
    main()
