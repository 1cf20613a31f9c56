"""Dev A/B: trace / output agreement of the current build vs the oracle-free full-precision
reference run at 32K (tcgen05 path vs generic exact path on 4 heads)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_22575_b200 as s2o
L = 16384
q, k, v = s2o.generate_synthetic("mixed", L // 64, 8.0, 3, 1, 8, L, 128)
qd = torch.from_numpy(q).cuda().to(torch.bfloat16)
kd = torch.from_numpy(k[:, :2]).cuda().to(torch.bfloat16)
vd = torch.from_numpy(v[:, :2]).cuda().to(torch.bfloat16)
for tau in (0.002, 0.005, 0.01):
    tc = s2o.s2o_attention(qd, kd, vd, s2o.KernelConfig(seg_len=2048, tau=tau, path=s2o.PATH_TCGEN05), want_plan=False)
    ex = s2o.s2o_attention(qd, kd, vd, s2o.KernelConfig(seg_len=2048, tau=tau, path=s2o.PATH_GENERIC), want_plan=False)
    torch.cuda.synchronize()
    a, b = tc.trace.processed.flatten(), ex.trace.processed.flatten()
    dif = (a != b)
    d = (tc.out.float() - ex.out.float()).abs()
    print(f"tau={tau}: tiles {a.numel()} differing {int(dif.sum())} max|dchunk| {int((a-b).abs().max())} "
          f"out max {d.max().item():.3e} mean {d.mean().item():.3e}", flush=True)
