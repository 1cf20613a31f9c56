"""C3 truncated plan (32 q / 8 kv heads, 128K, S=2048, T=6144), a few launches: for ncu launch lists."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_22575_b200 as s2o
L = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
q, k, _ = s2o.generate_synthetic("mixed", L // 64, 8.0, 0, 1, 32, L, 128)
qd = torch.from_numpy(q).cuda().to(torch.bfloat16)
kd = torch.from_numpy(k[:, :8].copy()).cuda().to(torch.bfloat16)
for _ in range(2):
    qp, kvt, flag = s2o.build_plan_truncated(qd, kd, 2048, 6144)
torch.cuda.synchronize()
print("flag", flag.item())
