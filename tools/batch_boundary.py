"""Cost of the batch boundary: ms per window at d=1024, 64 chains for M windows per batch.

    python tools/batch_boundary.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1506_05741_b200 as p  # noqa: E402

lib = p.load()
path = bench.make_target_file("pi1", 1024)
t = lib.target_load(path)
for M in (1, 2, 4, 8, 16):
    eng = lib.engine(t, **bench.run_options(("pi1", 1024, 64, 512, M), 64))
    eng.run_batches(3)
    k = max(2, 40 // M)
    ms = min(eng.run_batches(k) for _ in range(2))
    print(f"M={M:2d}: {ms / k:7.2f} ms/batch, {ms / k / M:6.2f} ms/window", flush=True)
    del eng
os.unlink(path)
