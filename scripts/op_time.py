"""Dev probe: the whole operator (s2o_attention, truncated plan) at C3, CUDA events, min of 5.
Honors S2O_LIB_PATH and the A/B environment flags."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_22575_b200 as s2o

L = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
q, k, v = s2o.generate_synthetic("mixed", L // 64, 8.0, 0, 1, 32, L, 128)
qd = torch.from_numpy(q).cuda().to(torch.bfloat16)
kd = torch.from_numpy(k[:, :8]).cuda().to(torch.bfloat16)
vd = torch.from_numpy(v[:, :8]).cuda().to(torch.bfloat16)
del q, k, v
cfg = s2o.KernelConfig(seg_len=2048, tau=0.005)
f = lambda: s2o.s2o_attention(qd, kd, vd, cfg, want_plan=False)
res = f(); torch.cuda.synchronize()
best = 1e9
for _ in range(5):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); f(); b.record(); torch.cuda.synchronize(); best = min(best, a.elapsed_time(b))
o = res.out.float()
print(f"[{os.environ.get('S2O_QROWS', 'qrows')}] L={L} operator {best:.3f} ms  out checksum {o.abs().sum().item():.6e} "
      f"pairs {int(res.trace.pass2_pairs.sum())}", flush=True)
