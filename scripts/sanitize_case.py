"""Small S2O runs for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool memcheck python scripts/sanitize_case.py

covers the plan kernels (full permutation and truncated top-T with plan levels), pass-1
(tc_diag_kernel), pass-2 (tc_pass_kernel, dynamic work ring), the fused variant, the generic
fp64 path and the block top-k baseline, on 2 q / 1 kv head x 2048 tokens."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2602_22575_b200 as s2o

q, k, v = s2o.generate_synthetic("mixed", 32, 8.0, 0, 1, 2, 2048, 128)
qd = torch.from_numpy(q).cuda().to(torch.bfloat16)
kd = torch.from_numpy(k[:, :1].copy()).cuda().to(torch.bfloat16)
vd = torch.from_numpy(v[:, :1].copy()).cuda().to(torch.bfloat16)
cfg = s2o.KernelConfig(seg_len=512, tau=0.005)
r = s2o.s2o_attention(qd, kd, vd, cfg)                                   # full plan, pass-1 + pass-2
r = s2o.s2o_attention(qd, kd, vd, s2o.KernelConfig(seg_len=512, tau=0.005, plan_depth=128), want_plan=False)
r = s2o.s2o_attention(qd, kd, vd, s2o.KernelConfig(seg_len=512, tau=0.005, q_reorder=False, fused=True))
r = s2o.s2o_attention(qd.float(), kd.float(), vd.float(), s2o.KernelConfig(seg_len=512, tau=0.005, tiles=s2o.TileSpec(64, 64)))
o, pc = s2o.block_topk_attention(qd, kd, vd, 128, 128, 2)
torch.cuda.synchronize()
print("sanitize case done", float(r.out.float().abs().sum()), int(pc.sum()))
