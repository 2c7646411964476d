"""Small-d window anatomy (d=100 pi2, 8 chains, the time-to-cov-error workload): engine
batches for an ncu launch list, and the device time per batch."""
import sys
sys.path.insert(0, '.')
import paper_1506_05741_b200 as p
lib = p.load()
kw = dict(kernel="diam", chains=8, intervals_per_batch=2, max_batches=1000, n0=0, master_seed=3, record_traces=0,
          trace_eigen_projections=0)
t = lib.target_build("pi2", 100, 1)
eng = lib.engine(t, **kw)
eng.run_batches(20)
ms = eng.run_batches(50)
print(f"d=100: {ms / 50:.3f} ms per batch of 2 windows", flush=True)
