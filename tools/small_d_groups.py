import time, sys, os
sys.path.insert(0, '.')
import bench, paper_1506_05741_b200 as p
lib = p.load()
kw = dict(kernel="diam", chains=8, intervals_per_batch=2, max_batches=5000, n0=0, cov_tol=0.3, master_seed=3, record_traces=0, trace_eigen_projections=0)
t = lib.target_build("pi2", 100, 1)
lib.sample(t, **dict(kw, max_batches=1))
for g in ["", "1", "2", "4", "8"]:
    if g: os.environ["DIAM_B200_GROUPS"] = g
    secs = []
    for _ in range(2):
        t0 = time.perf_counter(); r = lib.sample(t, **kw); secs.append(time.perf_counter() - t0)
    eng = lib.engine(t, **dict(kw, cov_tol=-1.0, max_batches=1000))
    eng.run_batches(5)
    e0 = eng.stat("host_enqueue")[0]; w0 = eng.stat("host_wait")[0]
    ms = eng.run_batches(100)
    print(f"groups={g or 'default'} layout={eng.layout}: time_to_cov {min(secs):.3f}s ({r.total_samples} samples); "
          f"100 batches {ms:.1f} ms device, host {eng.stat('host_enqueue')[0]-e0:.1f} ms (wait {eng.stat('host_wait')[0]-w0:.1f})", flush=True)
    del eng
