"""Where does the end-to-end diam_sample time go? (engine init vs batches)"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1506_05741_b200 as pkg  # noqa: E402


def main():
    cfg_name = sys.argv[1] if len(sys.argv) > 1 else "d1024"
    cfg = bench.CONFIGS[cfg_name]
    kind, d, per_gpu, n_lag, M = cfg
    lib = pkg.load()
    path = bench.make_target_file(kind, d)
    t = lib.target_load(path)
    lib.sample(t, **bench.run_options(cfg, per_gpu, max_batches=1))
    for K in (1, 2, 4, 8):
        t0 = time.perf_counter()
        r = lib.sample(t, **bench.run_options(cfg, per_gpu, max_batches=K))
        wall = time.perf_counter() - t0
        bs = r.history("batch_seconds")
        print(f"K={K}: wall {wall:.3f}s  batches {[round(x, 4) for x in bs]}  init+rest {wall - bs.sum():.3f}s "
              f"-> {r.total_samples / wall:.0f} chain-samples/s")
    t0 = time.perf_counter()
    e = lib.engine(t, **bench.run_options(cfg, per_gpu))
    print(f"engine create {time.perf_counter() - t0:.3f}s")
    for i in range(4):
        print(f"batch {i}: {e.run_batches(1):.2f} ms")
    os.unlink(path)


if __name__ == "__main__":
    main()
