"""Is the engine host-bound? Host time to enqueue K batches vs their device time.

    python tools/host_bound.py [--config d1024] [--batches 5]

run_batches returns once the host has enqueued every kernel and the GPU has finished; the
engine records how long the host took to enqueue (host_enqueue) and how much of that it
spent blocked on the GPU (host_wait: the POTRF statuses of the jitter ladder). Enqueue time
minus wait time close to the device time means the launch rate bounds the batch.
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
    ap.add_argument("--groups", default="")
    ap.add_argument("--warmup", type=int, default=2)
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    kind, d, per_gpu, n_lag, M = cfg
    lib = pkg.load()
    path = bench.make_target_file(kind, d)
    t = lib.target_load(path)
    for g in (args.groups.split(",") if args.groups else [""]):
        if g:
            os.environ["DIAM_B200_GROUPS"] = g
        eng = lib.engine(t, **bench.run_options(cfg, per_gpu))
        eng.run_batches(args.warmup)
        l0 = lib.launch_count()
        e0 = eng.stat("host_enqueue")[0]
        w0 = eng.stat("host_wait")[0]
        ms = eng.run_batches(args.batches)
        enq = eng.stat("host_enqueue")[0] - e0
        wait = eng.stat("host_wait")[0] - w0
        n = lib.launch_count() - l0
        print(f"groups={eng.layout['groups']}: device {ms / args.batches:.2f} ms/batch, host enqueue "
              f"{enq / args.batches:.2f} ms/batch of which waiting {wait / args.batches:.2f} -> busy "
              f"{(enq - wait) / args.batches:.2f} ms; {n / args.batches:.0f} launches/batch "
              f"({1e3 * (enq - wait) / max(n, 1):.2f} us each)", flush=True)
        del eng
    os.unlink(path)


if __name__ == "__main__":
    main()
