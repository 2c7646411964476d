#!/usr/bin/env bash
# One `ncu --set full` capture per hot kernel of the d=1024 bench batch, on a single
# stream (DIAM_B200_GROUPS=1: nothing overlaps, so each launch is the kernel alone).
#   gpurun -- 'bash tools/ncu_capture.sh <tag>'   -> gpurun_out/<tag>_<kernel>.ncu-rep
# then, locally: python tools/ncu_summary.py <tag>  -> profiles/<tag>_ncu_<kernel>.csv
set -euo pipefail
tag=${1:-r01}
only=${2:-all}   # "potrf": just the two POTRF captures
export DIAM_B200_GROUPS=1
mkdir -p gpurun_out
cmd="python tools/profile_step.py --batches 1"
full="ncu --set full --clock-control none --import-source on -f -c 1"
if [ "$only" = all ]; then
# the plain run first (ncu only after the same command exited 0 without it)
$cmd > gpurun_out/${tag}_plain.log 2>&1
for cls in trmm_noise syrk_moments xi_accepted; do
    # skip the warm-up batch's launches of the class (4 windows; TRMM: 3, window 0 is the identity)
    $full --nvtx --nvtx-include "$cls/" -k regex:gemm_f64 -s 3 -o gpurun_out/${tag}_${cls} $cmd \
        > gpurun_out/${tag}_${cls}.log 2>&1
done
for k in mh_window normals blend_cov reconstruct; do
    $full -k regex:$k -s 4 -o gpurun_out/${tag}_${k} $cmd > gpurun_out/${tag}_${k}.log 2>&1
done
fi
# the POTRF kernels from the third batch (the first batch's adaptations are rank-deficient:
# jitter ladder, chains that fail early skip the remaining launches): a long-K update GEMM,
# a diagonal block and the below-diagonal solve kernel
cmd3="python tools/profile_step.py --batches 2"
$cmd3 > gpurun_out/${tag}_plain3.log 2>&1
$full --nvtx --nvtx-include "potrf/" -k regex:gemm_f64 -s 45 -o gpurun_out/${tag}_potrf_update $cmd3 \
    > gpurun_out/${tag}_potrf_update.log 2>&1
$full -k regex:potrf_diag -s 20 -o gpurun_out/${tag}_potrf_diag $cmd3 > gpurun_out/${tag}_potrf_diag.log 2>&1
$full -k regex:potrf_trsm -s 100 -o gpurun_out/${tag}_potrf_trsm $cmd3 > gpurun_out/${tag}_potrf_trsm.log 2>&1
echo captured
