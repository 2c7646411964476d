import time, sys, os
sys.path.insert(0, '.')
import bench, paper_1506_05741_b200 as p
lib = p.load()
cfg = bench.CONFIGS["d1024"]
path = bench.make_target_file("pi1", 1024)
t = lib.target_load(path)
for steps in (1, 20, 20, 10, 20):
    t0 = time.perf_counter(); r = lib.sample(t, **bench.run_options(cfg, 64, max_batches=steps)); t1 = time.perf_counter()
    b = r.history("batch_seconds")
    print(f"steps {steps}: wall {1e3*(t1-t0):.1f} ms, batches {1e3*b.sum():.1f} ms, fixed {1e3*(t1-t0-b.sum()):.1f} ms", flush=True)
