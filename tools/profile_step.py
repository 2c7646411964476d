"""One warm-up batch + N profiled batches of the bench workload (for ncu / nsys-less timing).

    python tools/profile_step.py [--config d1024] [--batches 1]
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
    ap.add_argument("--batches", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=1, help="batches before the timed ones (the chains adapt: "
                    "the per-batch cost settles after ~10)")
    ap.add_argument("--chains", type=int, default=0)
    ap.add_argument("--classes", action="store_true", help="per-kernel-class CUDA-event times of one more batch")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    kind, d, per_gpu, n_lag, M = cfg
    lib = pkg.load()
    path = bench.make_target_file(kind, d)
    t = lib.target_load(path)
    eng = lib.engine(t, **bench.run_options(cfg, args.chains or per_gpu))
    print(f"layout {eng.layout}", flush=True)
    eng.run_batches(args.warmup)
    ms = eng.run_batches(args.batches)
    os.unlink(path)
    n = (args.chains or per_gpu) * M * n_lag * args.batches
    print(f"{args.config}: {args.batches} batch(es) {ms:.2f} ms -> {n / ms * 1e3:.0f} chain-samples/s")
    if args.classes:
        eng.set_profiling(True)
        eng.run_batches(1)
        for c in ["gemm_target", "trmm_noise", "syrk_moments", "potrf", "mh_window", "normals", "blend_cov",
                  "gemv_state", "trsv", "merge", "xi_accepted", "reconstruct"]:
            t, fl, k = eng.stat(c)
            print(f"  {c:14s} {t:8.3f} ms {k:5d} launches" + (f" {fl / t / 1e9:6.2f} TFLOP/s" if fl and t else ""))


if __name__ == "__main__":
    main()
