import time, sys
sys.path.insert(0, '.')
import bench, paper_1506_05741_b200 as p
lib = p.load()
print(bench.time_to_cov_error(lib, with_reference=False))
print(bench.time_to_cov_error(lib, with_reference=False))
kw = dict(kernel="diam", chains=8, intervals_per_batch=2, max_batches=200, n0=0, master_seed=3, record_traces=0, trace_eigen_projections=0)
t = lib.target_build("pi2", 100, 1)
for i in range(2):
    t0 = time.perf_counter(); r = lib.sample(t, **kw); print("200 batches", time.perf_counter() - t0)
eng = lib.engine(t, **kw)
eng.run_batches(5)
ms = eng.run_batches(200); print("engine 200 batches device ms", ms)
