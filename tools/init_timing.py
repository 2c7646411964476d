"""Fixed costs of one diam_sample call (engine construction, result, teardown).

    DIAM_B200_INIT_TIMING=1 python tools/init_timing.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1506_05741_b200 as p  # noqa: E402

lib = p.load()
cfg = bench.CONFIGS["d1024"]
path = bench.make_target_file("pi1", 1024)
t = lib.target_load(path)
for i in range(6):
    t0 = time.perf_counter()
    r = lib.sample(t, **bench.run_options(cfg, 64, max_batches=0))
    print("diam_sample, 0 batches:", round((time.perf_counter() - t0) * 1e3, 2), "ms", flush=True)
for i in range(3):
    t0 = time.perf_counter()
    r = lib.sample(t, **bench.run_options(cfg, 64, max_batches=4))
    print("diam_sample, 4 batches:", round((time.perf_counter() - t0) * 1e3, 2), "ms; batches",
          [round(x * 1e3, 2) for x in r.history("batch_seconds")], flush=True)
os.unlink(path)
