"""Localise tc-vs-generic differences: pass-1 states, then pass-2 traces on identical inputs."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_22575_b200 as s2o
L, S, HQ, HKV = int(sys.argv[1]), int(sys.argv[2]), 8, 2
q, k, v = s2o.generate_synthetic("mixed", L // 64, 8.0, 1, 1, HQ, L, 128)
qd = torch.from_numpy(q).cuda().to(torch.bfloat16)
kd = torch.from_numpy(k[:, :HKV].copy()).cuda().to(torch.bfloat16)
vd = torch.from_numpy(v[:, :HKV].copy()).cuda().to(torch.bfloat16)
ct = s2o.KernelConfig(seg_len=S, tau=0.005, path=2)
cg = s2o.KernelConfig(seg_len=S, tau=0.005, path=1)
bt = s2o.pass1_dense_init(qd, kd, vd, ct)
bg = s2o.pass1_dense_init(qd, kd, vd, cg)
ot = bt.acc / bt.ell[..., None]
og = bg.acc / bg.ell[..., None]
print("pass1 finalized max|diff|", (ot - og).abs().max().item())
lt = torch.log(bt.ell) + bt.m
lg = torch.log(bg.ell) + bg.m
print("pass1 logsumexp max|diff|", (lt - lg).abs().max().item())
plan, _ = s2o.build_plan(qd, kd, S)
for name, bufs in (("tc-state", bt), ("gen-state", bg)):
    o1, t1 = s2o.pass2_sparse(qd, kd, vd, bufs, plan, ct)
    o2, t2 = s2o.pass2_sparse(qd, kd, vd, bufs, plan, cg)
    torch.cuda.synchronize()
    d = (t1.processed != t2.processed)
    print(name, "pass2 trace diffs", d.sum().item(), "/", d.numel(), "tc-gen committed sum",
          (t1.processed - t2.processed).sum().item(), "out max|diff|", (o1.float() - o2.float()).abs().max().item())
    if d.any():
        idx = d.nonzero()[:5]
        for i in idx:
            i = tuple(i.tolist())
            print("   tile", i, "tc", t1.processed[i].item(), "gen", t2.processed[i].item())
