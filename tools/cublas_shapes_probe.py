import torch
a=torch.randn(64,512,1024,dtype=torch.float64,device='cuda'); b=torch.randn(64,1024,1024,dtype=torch.float64,device='cuda')
b1=torch.randn(1024,1024,dtype=torch.float64,device='cuda')
for _ in range(3):
    c=torch.bmm(a,b)
    d=a.reshape(-1,1024)@b1
torch.cuda.synchronize()
s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10): c=torch.bmm(a,b)
e.record(); torch.cuda.synchronize(); ms=s.elapsed_time(e)/10
print("bmm 64x512x1024x1024: %.3f ms %.2f TF/s"%(ms, 2*64*512*1024*1024/ms/1e9))
s.record()
for _ in range(10): d=a.reshape(-1,1024)@b1
e.record(); torch.cuda.synchronize(); ms=s.elapsed_time(e)/10
print("mm 32768x1024x1024: %.3f ms %.2f TF/s"%(ms, 2*64*512*1024*1024/ms/1e9))
