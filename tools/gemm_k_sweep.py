"""Per-tile fixed cost of the DMMA GEMM: time of C(MxN) = A B over K, fit t = a + b K.

    python tools/gemm_k_sweep.py
"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_05741_b200 as p  # noqa: E402

lib = p.load()
dev = torch.device("cuda:0")
M, N = 32768, 1024
s = torch.cuda.current_stream()
peak = C.c_double()
lib.check(lib.lib.diamx_fp64_peak(C.byref(peak)))
print(f"DMMA peak {peak.value:.2f} TFLOP/s")
for ak in (1, 0):
    for beta in (0.0, 1.0):
        rows = []
        for K in (128, 256, 512, 1024, 2048):
            a = torch.randn(M * K, dtype=torch.float64, device=dev)
            b = torch.randn(N * K, dtype=torch.float64, device=dev)
            c = torch.zeros(M * N, dtype=torch.float64, device=dev)
            lda = K if ak else M
            args = (C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), C.c_void_p(c.data_ptr()), M, N, K, lda, K, N,
                    ak, 1, 1.0, beta, 0, 0, C.c_void_p(s.cuda_stream))
            for _ in range(2):
                lib.check(lib.lib.diamx_gemm(*args))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            best = 1e9
            for _ in range(3):
                e0.record(s)
                for _ in range(5):
                    lib.check(lib.lib.diamx_gemm(*args))
                e1.record(s)
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1) / 5)
            tf = 2.0 * M * N * K / (best / 1e3) / 1e12
            rows.append((K, best))
            print(f"a_kmajor={ak} beta={beta:.0f} K={K:5d}: {best * 1e3:8.1f} us  {tf:6.2f} TFLOP/s "
                  f"({tf / peak.value * 100:5.1f}%)", flush=True)
            del a, b, c
        # least squares t = a + b K
        import numpy as np
        k = np.array([r[0] for r in rows], float)
        t = np.array([r[1] for r in rows], float)
        bb, aa = np.polyfit(k, t, 1)
        print(f"  fit: fixed {aa * 1e3:.1f} us per launch, {bb * 1e3 * 1024:.1f} us per 1024 of K "
              f"(fixed = {aa / bb:.0f} K-units)")
