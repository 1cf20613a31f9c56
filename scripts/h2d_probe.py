import torch, time
x = torch.empty(1610612736 // 2, dtype=torch.bfloat16).pin_memory()
y = torch.empty_like(x, device="cuda")
for i in range(3):
    torch.cuda.synchronize(); t=time.perf_counter(); y.copy_(x, non_blocking=True); torch.cuda.synchronize(); dt=time.perf_counter()-t
    print("h2d GB/s", x.numel()*2/dt/1e9)
z = torch.empty(1073741824//2, dtype=torch.bfloat16).pin_memory(); w = torch.empty_like(z, device="cuda")
for i in range(3):
    torch.cuda.synchronize(); t=time.perf_counter(); z.copy_(w, non_blocking=True); torch.cuda.synchronize(); dt=time.perf_counter()-t
    print("d2h GB/s", z.numel()*2/dt/1e9)
s1=torch.cuda.Stream(); s2=torch.cuda.Stream()
for i in range(3):
    torch.cuda.synchronize(); t=time.perf_counter()
    with torch.cuda.stream(s1): y.copy_(x, non_blocking=True)
    with torch.cuda.stream(s2): z.copy_(w, non_blocking=True)
    torch.cuda.synchronize(); dt=time.perf_counter()-t
    print("both ms", dt*1e3)
