"""cuBLAS DGEMM throughput (context for the FP64 roofline denominator)."""
import torch, time
torch.backends.cuda.matmul.allow_tf32 = False
for n in (1024, 2048, 4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10 if n <= 4096 else 4
    e0.record()
    for _ in range(reps):
        c = a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"dgemm n={n}: {2*n**3/ms/1e9:.2f} TFLOP/s ({ms:.3f} ms)")
