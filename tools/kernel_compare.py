"""Batch time of the d=1024 bench workload per sampler kernel (diam/am refactor every
window; pcn/rw never do): the difference is what the refactorization costs in the
grouped engine.

    python tools/kernel_compare.py [--config d1024]
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
    ap.add_argument("--batches", type=int, default=3)
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    kind, d, per_gpu, n_lag, M = cfg
    lib = pkg.load()
    path = bench.make_target_file(kind, d)
    t = lib.target_load(path)
    for kern in ("diam", "am", "pcn", "rw"):
        eng = lib.engine(t, **bench.run_options(cfg, per_gpu, kernel=kern))
        eng.run_batches(2)
        ms = eng.run_batches(args.batches) / args.batches
        print(f"{kern:5s}: {ms:7.2f} ms per batch")
        del eng
    os.unlink(path)


if __name__ == "__main__":
    main()
