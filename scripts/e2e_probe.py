"""Dev aid: e2e time of the host-buffer entry point at C3 (S2O_HOST_PART_HEADS selects the chunk
size of the host pipeline), and its output against the device-buffer operator."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_22575_b200 as s2o
L = 131072
q, k, v = s2o.generate_synthetic("mixed", L // 64, 8.0, 0, 1, 32, L, 128)
qd = torch.from_numpy(q).cuda().to(torch.bfloat16)
kd = torch.from_numpy(k[:, :8].copy()).cuda().to(torch.bfloat16)
vd = torch.from_numpy(v[:, :8].copy()).cuda().to(torch.bfloat16)
cfg = s2o.KernelConfig(seg_len=2048, tau=0.005)
ref = s2o.s2o_attention(qd, kd, vd, cfg, want_plan=False).out.cpu()
qh, kh, vh = qd.cpu().pin_memory(), kd.cpu().pin_memory(), vd.cpu().pin_memory()
oh = torch.empty_like(qh).pin_memory()
s2o.attention_host_ptr(qh, kh, vh, oh, cfg)
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    s2o.attention_host_ptr(qh, kh, vh, oh, cfg)
    ts.append((time.perf_counter() - t0) * 1e3)
print(f"parts={os.environ.get('S2O_HOST_PART_HEADS', 'default')} e2e ms min {min(ts):.2f} median {sorted(ts)[2]:.2f} "
      f"max|host-device| {(oh.float() - ref.float()).abs().max().item():.3e}")
