import time, sys, os
sys.path.insert(0, '.')
import bench, paper_1506_05741_b200 as p
lib = p.load()
path = bench.make_target_file("pi1", 1024)
t = lib.target_load(path)
for tol in (0.5, 0.3, 0.2):
    kw = dict(kernel="diam", chains=64, intervals_per_batch=4, max_batches=3000, n0=0, cov_tol=tol, master_seed=3, record_traces=0, trace_eigen_projections=0)
    t0 = time.perf_counter(); r = lib.sample(t, **kw); dt = time.perf_counter() - t0
    print(f"d=1024 pi1 64 chains tol {tol}: {dt:.2f} s, {r.total_samples} samples, batches {r.batches}, stop {r.stop_reason}, final cov err {r.final_cov_error:.4f}", flush=True)
