#!/bin/bash
# One gpurun call: the GPU test suite, then a short bench (no CPU baseline).
#   /usr/local/graft/bin/gpurun --timeout 1200 -- 'bash tools/gpu_check.sh TAG'
tag=${1:-check}
python -m pytest tests -x -q -m gpu 2>&1 | tail -15
python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2> gpurun_out/bench_${tag}.err | tee gpurun_out/bench_${tag}.json | cut -c1-400
tail -3 gpurun_out/bench_${tag}.err
