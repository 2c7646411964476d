"""Per-batch device time over a long run of the bench workload (does the cost drift as the
chains adapt?): ms of each batch and the mean acceptance of its windows."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1506_05741_b200 as pkg  # noqa: E402

lib = pkg.load()
cfg = bench.CONFIGS["d1024"]
path = bench.make_target_file("pi1", 1024)
t = lib.target_load(path)
eng = lib.engine(t, **bench.run_options(cfg, 64))
for b in range(40):
    ms = eng.run_batches(1)
    print(f"batch {b:2d}: {ms:6.2f} ms", flush=True)
os.unlink(path)
