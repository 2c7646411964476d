"""Marginal cost of each kernel class in the grouped engine (timing experiment).

    python tools/skip_sweep.py [--config d1024] [--batches 5]

Runs the bench workload with DIAM_B200_SKIP=<class> (the class is not launched at all;
results are discarded) and prints the batch time against the full run: the difference is
what the class costs on the critical path of the real, overlapped schedule -- unlike the
single-stream per-class times of bench.py's profile pass.
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
    ap.add_argument("--sets", default="none,normals,trmm,target,mh,syrk,potrf,normals+trmm+target,potrf+mh")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    kind, d, per_gpu, n_lag, M = cfg
    lib = pkg.load()
    path = bench.make_target_file(kind, d)
    t = lib.target_load(path)
    base = None
    for s in args.sets.split(","):
        if s == "none":
            os.environ.pop("DIAM_B200_SKIP", None)
        else:
            os.environ["DIAM_B200_SKIP"] = s
        eng = lib.engine(t, **bench.run_options(cfg, per_gpu))
        eng.run_batches(2)
        ms = eng.run_batches(args.batches) / args.batches
        del eng
        if base is None:
            base = ms
        print(f"skip {s:24s} {ms:7.2f} ms/batch  (saves {base - ms:6.2f})", flush=True)
    os.environ.pop("DIAM_B200_SKIP", None)
    os.unlink(path)


if __name__ == "__main__":
    main()
