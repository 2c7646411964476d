#!/usr/bin/env bash
# Round-2 measurement pass on one B200 (gpurun): bench lines of every config, the reference
# arm, the bench's launch list and the per-kernel ncu captures. Outputs in gpurun_out/.
set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/r02_bench_d1024.json 2> gpurun_out/r02_bench_d1024.err
DIAM_B200_GROUPS=1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_g1.json 2>/dev/null
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02_bench_reference_arm.json 2> gpurun_out/r02_bench_ref.err
for c in d2040 d4096 d8192; do
    timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.err
done
DIAM_B200_GROUPS=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/r02_launches_d1024.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02_launches.log 2>&1
bash tools/ncu_capture.sh r02c > gpurun_out/r02b_capture.log 2>&1
echo done
