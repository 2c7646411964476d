"""AM on the time-to-cov-error workload, GPU vs the reference library: where the two
trajectories part (relative cov-error difference per batch, first beta-history difference per
chain)."""
import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_1506_05741_b200 as pkg, _oracle as O
from paper_1506_05741_b200.abi import DiamABI
b = pkg.load(); ref = DiamABI(O.REF_SO)
kw = dict(kernel="am", chains=8, intervals_per_batch=2, max_batches=3000, n0=0, cov_tol=0.3, master_seed=3, record_traces=0, trace_eigen_projections=0)
g = b.sample(b.target_build("pi2", 100, 1), **kw); r = ref.sample(ref.target_build("pi2", 100, 1), threads=8, **kw)
hg, hr = g.history("cov_error"), r.history("cov_error")
n = min(len(hg), len(hr)); rel = np.abs(hg[:n]-hr[:n])/np.abs(hr[:n])
idx = np.nonzero(rel > 1e-8)[0]
print("batches", g.batches, r.batches, "first >1e-8 at", idx[:5], "rel there", rel[idx[:5]] if len(idx) else None)
for i in range(0, n, max(1, n//20)): print(i, hg[i], hr[i], rel[i])
bg = [g.chain_history(p, "beta") for p in range(8)]; br = [r.chain_history(p, "beta") for p in range(8)]
for p in range(8):
    m = min(len(bg[p]), len(br[p]))
    d = np.nonzero(bg[p][:m] != br[p][:m])[0]
    print("chain", p, "beta hist len", len(bg[p]), len(br[p]), "first diff", d[:3])
