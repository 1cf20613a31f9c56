"""One s2o_attention at the C3 shape with the truncated plan (want_plan=False), for ncu captures."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_22575_b200 as s2o
L = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
q, k, v = s2o.generate_synthetic("mixed", L // 64, 8.0, 0, 1, 32, L, 128)
qd = torch.from_numpy(q).cuda().to(torch.bfloat16)
kd = torch.from_numpy(k[:, :8]).cuda().to(torch.bfloat16)
vd = torch.from_numpy(v[:, :8]).cuda().to(torch.bfloat16)
res = s2o.s2o_attention(qd, kd, vd, s2o.KernelConfig(seg_len=2048, tau=0.005), want_plan=False)
torch.cuda.synchronize()
print("pairs", res.trace.pass1_pairs.sum().item(), res.trace.pass2_pairs.sum().item())
