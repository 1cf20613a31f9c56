"""Quick device timing of the plan builds (full permutation and truncated top-T) -- dev probe."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_22575_b200 as s2o


def timeit(fn, reps=5):
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
    full = timeit(lambda: s2o.build_plan(q, k, 2048))
    trunc = timeit(lambda: s2o.build_plan_truncated(q, k, 2048))
    print(f"plan L={L}: full {full:.2f} ms, truncated {trunc:.2f} ms", flush=True)
