python -m pytest tests -q -m gpu -x -k "lockstep or bench_parity or smoke or golden or pipelined or sharded or explicit or checkpoint" 2>&1 | tail -2
tools/mh_lat 1024 64
python tools/host_bound.py --batches 8
DIAM_B200_GROUPS=1 python tools/profile_step.py --classes 2>&1 | grep -E "mh_window|batch"
