"""Throughput of the batched Cholesky in the engine's shape (timing tool).

    python tools/potrf_bench.py [--d 1024] [--groups 16] [--chains 4] [--rounds 8] [--aug 1]

`groups` concurrent streams each refactor `chains` matrices `rounds` times (a D2D copy of a
pristine SPD matrix, then potrf_batched with the augmented row of the usable guard), as the
d=1024 bench's 16 chain groups do once per window. Reports the achieved FP64 rate of the
d^3/3 flops per factorization against the DMMA peak.
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_05741_b200 as pkg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=1024)
    ap.add_argument("--groups", default="16,1")
    ap.add_argument("--chains", default="4,64")
    ap.add_argument("--rounds", type=int, default=8)
    ap.add_argument("--aug", type=int, default=1)
    args = ap.parse_args()
    lib = pkg.load()
    d = args.d
    ld = (d + 7) // 8 * 8
    rng = np.random.default_rng(1)
    a = rng.normal(size=(d, d + 8))
    m = a @ a.T / d + np.eye(d)
    host = np.zeros((d + args.aug, ld))
    host[:d, :d] = np.tril(m)
    if args.aug:
        host[d, :d] = rng.normal(size=d)
    src = torch.from_numpy(host).cuda()
    peak = C.c_double()
    lib.check(lib.lib.diamx_fp64_peak(C.byref(peak)))
    for g, c in zip([int(x) for x in args.groups.split(",")], [int(x) for x in args.chains.split(",")]):
        ms = C.c_double()
        lib.check(lib.lib.diamx_potrf_bench(C.c_void_p(src.data_ptr()), ld, d, args.aug, g, c, args.rounds,
                                             C.byref(ms)))
        n = g * c * args.rounds
        fl = n * d ** 3 / 3.0
        tf = fl / (ms.value / 1e3) / 1e12
        print(f"d={d} groups={g} chains={c} rounds={args.rounds}: {ms.value:.2f} ms, "
              f"{ms.value / args.rounds:.3f} ms per round of {g * c} factorizations, {tf:.1f} TFLOP/s "
              f"({100 * tf / peak.value:.0f}% of DMMA peak {peak.value:.1f})", flush=True)


if __name__ == "__main__":
    main()
