"""One batched POTRF (diamx_potrf) of `batch` random SPD d x d matrices, for ncu launch lists:

    ncu --metrics gpu__time_duration.sum --csv python tools/potrf_once.py 1024 64
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_05741_b200 as pkg  # noqa: E402

lib = pkg.load()
d, batch = int(sys.argv[1]), int(sys.argv[2])
ld = (d + 7) // 8 * 8
rng = np.random.default_rng(1)
a = rng.normal(size=(d, d + 8))
m = a @ a.T / d + np.eye(d)
host = np.zeros((batch, d, ld))
host[:, :, :d] = np.tril(m)
A = torch.from_numpy(host).cuda()
st = torch.zeros(batch, dtype=torch.int32, device="cuda")
lib.check(lib.lib.diamx_potrf(C.c_void_p(A.data_ptr()), d * ld, ld, d, batch, C.c_void_p(st.data_ptr()), None))
torch.cuda.synchronize()
print("status", int(st.sum()))
