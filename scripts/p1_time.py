"""Dev probe: device time of pass-1 alone at the C3 shape (128K, 32 q / 8 kv heads), min of 7.
Honors S2O_LIB_PATH (A/B builds) and the kernel-selection env flags."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_22575_b200 as s2o

L = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
hq, hkv = (int(x) for x in (sys.argv[2:4] if len(sys.argv) > 3 else (32, 8)))
torch.manual_seed(0)
qd = torch.randn(1, hq, L, 128, device="cuda").to(torch.bfloat16)
kd = torch.randn(1, hkv, L, 128, device="cuda").to(torch.bfloat16)
vd = torch.randn(1, hkv, L, 128, device="cuda").to(torch.bfloat16)
cfg = s2o.KernelConfig(seg_len=2048, tau=0.005)
f = lambda: s2o.pass1_dense_init(qd, kd, vd, cfg)
f(); torch.cuda.synchronize()
best = 1e9
for _ in range(7):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); f(); b.record(); torch.cuda.synchronize(); best = min(best, a.elapsed_time(b))
tag = os.environ.get("S2O_LIB_PATH", "pkg").split("/")[-3] if os.environ.get("S2O_LIB_PATH") else "pkg"
print(f"[{tag} diag2={os.environ.get('S2O_DIAG2', '0')}] L={L} hq={hq} hkv={hkv} pass1 {best:.3f} ms", flush=True)
