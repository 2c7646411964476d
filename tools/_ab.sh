for g in 16 8 12 24 32 16; do DIAM_B200_GROUPS=$g python tools/host_bound.py --batches 8; done
