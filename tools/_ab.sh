DIAM_B200_NOISE=fused python -m pytest tests -q -m gpu -x -k "lockstep or bench_parity or smoke or golden" 2>&1 | tail -3
for v in split fused split fused; do echo "== $v"; DIAM_B200_NOISE=$v python tools/host_bound.py --batches 8; DIAM_B200_NOISE=$v DIAM_B200_GROUPS=1 python tools/profile_step.py --classes 2>&1 | grep -E "normals|trmm|batch"; done
