"""Quick device timing of the plan build (and generic passes at small L) -- dev probe."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_22575_b200 as s2o

def timeit(fn, reps=3):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return min(ts)

for L in (32768, 131072):
    torch.manual_seed(0)
    q = torch.randn(1, 32, L, 128, device='cuda').to(torch.bfloat16)
    k = torch.randn(1, 8, L, 128, device='cuda').to(torch.bfloat16)
    ms = timeit(lambda: s2o.build_plan(q, k, 2048))
    print(f"plan L={L}: {ms:.2f} ms", flush=True)
q = torch.randn(1, 32, 32768, 128, device='cuda').to(torch.bfloat16)
k = torch.randn(1, 8, 32768, 128, device='cuda').to(torch.bfloat16)
v = torch.randn(1, 8, 32768, 128, device='cuda').to(torch.bfloat16)
cfg = s2o.KernelConfig(seg_len=2048, tau=0.005, path=s2o.PATH_GENERIC)
ms = timeit(lambda: s2o.s2o_attention(q[:, :4], k[:, :1], v[:, :1], cfg), reps=1)
print(f"generic s2o 32K 4 heads: {ms:.1f} ms", flush=True)
