"""Dev probe: how unevenly the two tiles of a pass-2 pair stop (trace.processed per tile at C3)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2602_22575_b200 as s2o

L = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
q, k, v = s2o.generate_synthetic("mixed", L // 64, 8.0, 0, 1, 32, L, 128)
qd = torch.from_numpy(q).cuda().to(torch.bfloat16)
kd = torch.from_numpy(k[:, :8]).cuda().to(torch.bfloat16)
vd = torch.from_numpy(v[:, :8]).cuda().to(torch.bfloat16)
del q, k, v
res = s2o.s2o_attention(qd, kd, vd, s2o.KernelConfig(seg_len=2048, tau=0.005), want_plan=False)
torch.cuda.synchronize()
pr = res.trace.processed.cpu().numpy().astype(np.int64)
print("processed shape", pr.shape, "dtype", pr.dtype)
flat = pr.reshape(-1, pr.shape[-1])
T = flat.shape[-1]
a, b = flat[:, 0:T - 1:2], flat[:, 1:T:2]
d = np.abs(a - b)
blocks = (a + b)
print(f"tiles {flat.size}, mean processed {flat.mean():.2f}, pairs {a.size}")
print(f"|diff| mean {d.mean():.2f} median {np.median(d):.0f} p90 {np.percentile(d, 90):.0f}; sum |diff| / sum(max) = {d.sum() / np.maximum(a, b).sum():.3f}")
