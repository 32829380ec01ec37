import torch, time
a=torch.randn(10000,768,dtype=torch.float64,device='cuda'); b=torch.randn(768,256,dtype=torch.float64,device='cuda')
c=torch.randn(10000,256,dtype=torch.float64,device='cuda'); e=torch.randn(1024,256,dtype=torch.float64,device='cuda')
for _ in range(3): a@b; c@e.T
torch.cuda.synchronize()
s=torch.cuda.Event(enable_timing=True); t=torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20): a@b
t.record(); torch.cuda.synchronize(); ms=s.elapsed_time(t)/20; print("proj f64 cublas ms", ms, "TF", 2*10000*768*256/ms/1e9)
s.record()
for _ in range(20): c@e.T
t.record(); torch.cuda.synchronize(); ms=s.elapsed_time(t)/20; print("route f64 cublas ms", ms, "TF", 2*10000*1024*256/ms/1e9)
x=torch.randn(8192,8192,dtype=torch.float64,device='cuda')
for _ in range(2): x@x
torch.cuda.synchronize(); s.record(); x@x; t.record(); torch.cuda.synchronize(); ms=s.elapsed_time(t); print("big f64 TF", 2*8192**3/ms/1e9)
