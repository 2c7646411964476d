"""Time the batched POTRF alone (diamx_potrf) on random SPD matrices.

    python tools/bench_diag.py [d ...]
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_05741_b200 as pkg  # noqa: E402


def main():
    lib = pkg.load()
    ds = [int(a) for a in sys.argv[1:]] or [64, 1024]
    batch = 64
    for d in ds:
        ld = (d + 7) // 8 * 8
        rng = np.random.default_rng(1)
        a = rng.normal(size=(d, d + 8))
        m = a @ a.T / d + np.eye(d)
        host = np.zeros((batch, d, ld))
        host[:, :, :d] = np.tril(m)
        src = torch.from_numpy(host).cuda()
        A = src.clone()
        st = torch.zeros(batch, dtype=torch.int32, device="cuda")
        p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
        for _ in range(3):
            A.copy_(src)
            lib.check(lib.lib.diamx_potrf(p(A), d * ld, ld, d, batch, p(st), None))
        torch.cuda.synchronize()
        reps = 20
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tot = 0.0
        for _ in range(reps):
            A.copy_(src)
            torch.cuda.synchronize()
            e0.record()
            lib.check(lib.lib.diamx_potrf(p(A), d * ld, ld, d, batch, p(st), None))
            e1.record()
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        ms = tot / reps
        fl = batch * d ** 3 / 3
        print(f"d={d} batch={batch}: {ms * 1e3:.1f} us per batched POTRF, {fl / ms / 1e9:.2f} TFLOP/s, "
              f"status {int(st.sum())}")


if __name__ == "__main__":
    main()
