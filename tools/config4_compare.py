"""AM vs DIAM on the twisted targets pi5 (b=0.3) and pi6 (b=2) at
d=2040 (d % 20 == 0), 256 chains, n_lag = d/2, DIAM inflation 1.2 (as in the reference's
acceptance test), same seeds: covariance / mean error against samples and wall time.

    python tools/config4_compare.py [--batches 40] [--out profiles/r01_config4.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1506_05741_b200 as pkg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=2040)
    ap.add_argument("--chains", type=int, default=256)
    ap.add_argument("--batches", type=int, default=40)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    lib = pkg.load()
    out = {"d": args.d, "chains": args.chains, "n_lag": args.d // 2, "runs": []}
    for kind in ("pi5", "pi6"):
        t0 = time.perf_counter()
        t = lib.target_build(kind, args.d, 1)  # GPU target builder at this size
        build_s = time.perf_counter() - t0
        for kern in ("am", "diam"):
            kw = dict(kernel=kern, chains=args.chains, intervals_per_batch=1, max_batches=args.batches, n0=0,
                      master_seed=7, record_traces=0, trace_eigen_projections=0)
            if kern == "diam":
                kw["inflation"] = 1.2
            t0 = time.perf_counter()
            r = lib.sample(t, **kw)
            wall = time.perf_counter() - t0
            ce = [float(x) for x in r.history("cov_error")]
            me = [float(x) for x in r.history("mean_error")]
            bs = [float(x) for x in r.history("batch_seconds")]
            acc = sum(r.chain_history(c, "acceptance")[-1] for c in range(args.chains)) / args.chains
            run = {"target": kind, "kernel": kern, "wall_seconds": wall, "target_build_seconds": build_s,
                   "samples": r.total_samples, "samples_per_second": r.total_samples / wall,
                   "final_cov_error": ce[-1], "final_mean_error": me[-1], "final_acceptance": float(acc),
                   "cov_error_history": ce, "mean_error_history": me, "batch_seconds": bs}
            out["runs"].append(run)
            print(f"{kind} {kern:4s}: {r.total_samples} samples in {wall:.1f} s "
                  f"({r.total_samples / wall / 1e6:.2f} M/s), cov_error {ce[0]:.3f} -> {ce[-1]:.3f}, "
                  f"mean_error {me[0]:.3f} -> {me[-1]:.3f}, acceptance {acc:.3f}", flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
