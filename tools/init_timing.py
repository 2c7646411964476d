import time, sys
sys.path.insert(0, '.')
import bench, paper_1506_05741_b200 as p
lib = p.load()
cfg = bench.CONFIGS["d1024"]
path = bench.make_target_file("pi1", 1024)
t = lib.target_load(path)
for i in range(4):
    t0 = time.perf_counter(); r = lib.sample(t, **bench.run_options(cfg, 64, max_batches=0)); t1 = time.perf_counter()
    print("max_batches=0:", round((t1 - t0) * 1e3, 2), "ms", r.stop_reason)
for i in range(3):
    t0 = time.perf_counter(); e = lib.engine(t, **bench.run_options(cfg, 64)); t1 = time.perf_counter(); del e; t2 = time.perf_counter()
    print("engine create", round((t1 - t0) * 1e3, 2), "ms, free", round((t2 - t1) * 1e3, 2), "ms")
