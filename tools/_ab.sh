python -m pytest tests -q -m gpu -x 2>&1 | tail -4
python tools/host_bound.py --batches 8
DIAM_B200_GROUPS=1 python tools/profile_step.py --classes 2>&1 | grep -E "gemm_target|trmm|batch"
