"""Distribution of committed prefix chunks per query tile at the C2/C3 shapes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_22575_b200 as s2o
for L in [int(x) for x in sys.argv[1:]]:
    q, k, v = s2o.generate_synthetic("mixed", L // 64, 8.0, 0, 1, 32, L, 128)
    qd = torch.from_numpy(q).cuda().to(torch.bfloat16)
    kd = torch.from_numpy(k[:, :8].copy()).cuda().to(torch.bfloat16)
    vd = torch.from_numpy(v[:, :8].copy()).cuda().to(torch.bfloat16)
    del q, k, v
    res = s2o.s2o_attention(qd, kd, vd, s2o.KernelConfig(seg_len=2048, tau=0.005))
    p = res.trace.processed.cpu().numpy().reshape(32, -1, 16)
    n = p.shape[1]
    print(f"L={L}: mean {p[:, 1:].mean():.2f} max {p.max()} p99 {np.percentile(p[:, 1:], 99):.0f}")
    for thr in (16, 24, 32, 48, 64, 96):
        print(f"   tiles with >= {thr} chunks: {(p >= thr).sum()} / {p[:, 1:].size}")
    ex = [(p[:, m] >= (m * 2048) // 128).sum() for m in range(1, n)]
    print("   tiles exhausting their prefix per segment:", ex[:8], "...", sum(ex))
    # which segments hold deep tiles
    deep = (p >= 32).sum(axis=(0, 2))
    print("   deep (>=32) tiles per segment:", deep.tolist())
