"""The per-group factorization graph (Engine::factor) replays exactly the launches it
captured: a run with the graphs and one with direct launches (DIAM_B200_GRAPHS=0, read once
per process, hence subprocesses) give bit-identical results -- moments, histories and the
final factors' effect on every decision -- on the bench's d=1024 shape (16 chain groups,
the first batch's jitter ladder) and on a small DIAM run with the adaptive reference."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
sys.path.insert(0, {root!r})
import numpy as np
import paper_1506_05741_b200 as pkg
from paper_1506_05741_b200 import fixtures
lib = pkg.load()
case = {case!r}
if case == "d1024":
    fixtures.make("/tmp/graph_pi1_1024.bin", "pi1", 1024, 1)
    t = lib.target_load("/tmp/graph_pi1_1024.bin")
    r = lib.sample(t, kernel="diam", chains=64, intervals_per_batch=4, max_batches=3, n0=0, master_seed=11,
                   record_traces=0, trace_eigen_projections=0)
else:
    t = lib.target_build("pi1", 96, 2)
    r = lib.sample(t, kernel="diam", chains=12, intervals_per_batch=3, max_batches=4, n0=0, master_seed=5,
                   adaptive_ref=1, n_ref_start=96, record_traces=1, trace_thin=3)
out = dict(mean=r.mean().tolist(), cov=np.asarray(r.cov()).ravel()[::97].tolist(),
           beta=[r.chain_history(p, "beta").tolist() for p in range(r.chains)],
           acc=[r.chain_history(p, "acceptance").tolist() for p in range(r.chains)],
           samples=int(r.total_samples))
print(json.dumps(out))
"""


def run_case(case, graphs):
    env = dict(os.environ, DIAM_B200_GRAPHS=graphs)
    p = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, case=case)], capture_output=True, text=True,
                       env=env, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("case", ["d1024", "small_diam_adaptive"])
def test_factorization_graph_is_bit_identical(case):
    a = run_case(case, "1")
    b = run_case(case, "0")
    assert a == b
