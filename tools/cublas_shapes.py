"""cuBLAS (torch.matmul, FP64) on the sampler's GEMM shapes, for comparison with the DMMA
kernel (tools/gemm_k_sweep.py): C = A B^T, A 32768 x K, B 1024 x K."""
import torch

dev = torch.device("cuda")
for K in (256, 512, 1024, 2048, 8192):
    a = torch.randn(32768, K, dtype=torch.float64, device=dev)
    b = torch.randn(1024, K, dtype=torch.float64, device=dev)
    for _ in range(2):
        c = a @ b.T
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(3):
        e0.record()
        for _ in range(5):
            c = a @ b.T
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 5)
    tf = 2 * 32768 * 1024 * K / (best / 1e3) / 1e12
    print(f"cuBLAS K={K:5d}: {best * 1e3:8.1f} us  {tf:6.2f} TFLOP/s ({tf / 37.12 * 100:5.1f}% of the DMMA peak)",
          flush=True)
