"""Dev probe: device time of one (kv head) chunk of the C3 problem (4 q heads, 1 kv head)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_22575_b200 as s2o
L = 131072
for hq, hkv in ((4, 1), (8, 2), (32, 8), (1, 1)):
    q, k, v = s2o.generate_synthetic("mixed", L // 64, 8.0, 0, 1, hq, L, 128)
    qd = torch.from_numpy(q).cuda().to(torch.bfloat16); kd = torch.from_numpy(k[:, :hkv].copy()).cuda().to(torch.bfloat16)
    vd = torch.from_numpy(v[:, :hkv].copy()).cuda().to(torch.bfloat16)
    cfg = s2o.KernelConfig(seg_len=2048, tau=0.005)
    out = torch.empty_like(qd)
    f = lambda: s2o.s2o_attention(qd, kd, vd, cfg, out=out, want_plan=False)
    f(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record(); torch.cuda.synchronize(); best = min(best, a.elapsed_time(b))
    print(f"hq={hq} hkv={hkv}: {best:.2f} ms ({best / hq:.3f} ms per q head)", flush=True)
    del qd, kd, vd, q, k, v
