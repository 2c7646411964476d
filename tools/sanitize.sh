#!/bin/bash
# compute-sanitizer over a small DIAM run through the C ABI (d=133: a ragged last block
# column, two 128-wide block columns, the augmented row), one tool per invocation:
#   gpurun -- 'bash tools/sanitize.sh memcheck'   (racecheck, synccheck, initcheck)
tool=${1:-memcheck}
mkdir -p gpurun_out
cat > /tmp/san_run.py <<'PY'
import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_1506_05741_b200 as pkg
lib = pkg.load()
t = lib.target_build("pi1", 133, 3)
for kern, extra in (("diam", {}), ("am", {}), ("pcn", {"use_explicit_inverse": 1}),
                    ("diam", {"adaptive_ref": 1, "n_ref_start": 200})):
    r = lib.sample(t, kernel=kern, chains=5, intervals_per_batch=2, max_batches=2, n_lag=70, n0=0, master_seed=4,
                   **extra)
    print(kern, extra, r.batches, r.final_cov_error)
t5 = lib.target_build("pi5", 40, 2)
r = lib.sample(t5, kernel="diam", chains=3, intervals_per_batch=2, max_batches=2, n_lag=30, n0=0, inflation=1.2)
print("pi5", r.batches)
PY
DIAM_B200_GROUPS=2 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python /tmp/san_run.py \
    > gpurun_out/sanitize_${tool}.log 2>&1
echo "exit $?" >> gpurun_out/sanitize_${tool}.log
tail -5 gpurun_out/sanitize_${tool}.log
