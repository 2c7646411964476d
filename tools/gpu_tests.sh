#!/bin/bash
# One gpurun call: selected GPU tests (pytest -k expression, default all), durations shown.
#   /usr/local/graft/bin/gpurun --timeout 1800 -- 'bash tools/gpu_tests.sh "bench_parity or golden"'
nproc
if [ -n "$1" ]; then
  python -m pytest tests -q -m gpu -k "$1" --durations=8 2>&1 | tail -40
else
  python -m pytest tests -q -m gpu --durations=8 2>&1 | tail -40
fi
