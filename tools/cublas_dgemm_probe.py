"""torch (cuBLAS) DGEMM at 8192^3, for ncu: which kernel cuBLAS runs for FP64 on this GPU and at what tensor-pipe utilisation (profiles/README.md)."""
import torch
a=torch.randn(8192,8192,dtype=torch.float64,device='cuda'); b=torch.randn(8192,8192,dtype=torch.float64,device='cuda')
for _ in range(3): c=a@b
torch.cuda.synchronize()
