"""A/B of engine configurations on the d=1024 bench workload (device time per batch).

    python tools/engine_ab.py "DIAM_B200_GEMM_CFG=2" "" "DIAM_B200_POTRF=wide" ...
Each argument is a space-separated list of VAR=value settings ("" = defaults); the
configurations are run round-robin twice, min of two 10-batch timings each.
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys
sys.path.insert(0, %r)
import bench, paper_1506_05741_b200 as p
lib = p.load()
path = bench.make_target_file("pi1", 1024)
t = lib.target_load(path)
eng = lib.engine(t, **bench.run_options(bench.CONFIGS["d1024"], 64))
eng.run_batches(3)
print(min(eng.run_batches(10) for _ in range(2)) / 10)
os.unlink(path)
''' % ROOT

res = {a: [] for a in sys.argv[1:]}
for rnd in range(2):
    for a in sys.argv[1:]:
        env = dict(os.environ)
        for kv in a.split():
            k, v = kv.split("=", 1)
            env[k] = v
        out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        try:
            res[a].append(float(out.stdout.strip().splitlines()[-1]))
        except Exception:
            res[a].append(float("nan"))
            print(out.stderr[-500:], file=sys.stderr)
for a, v in res.items():
    print(f"{a or '(defaults)':40s} " + "  ".join(f"{x:6.2f}" for x in v) + " ms/batch")
