"""Dev A/B: C2 (4 q / 1 kv head x 32K) outputs with and without the pass-1 poison check."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1:
    import torch, numpy as np
    import paper_2602_22575_b200 as s2o
    q, k, v = s2o.generate_synthetic("mixed", 512, 8.0, 0, 1, 4, 32768, 128)
    qd, kd, vd = (torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16) for x in (q, k[:, :1], v[:, :1]))
    res = s2o.s2o_attention(qd, kd, vd, s2o.KernelConfig(seg_len=2048, tau=0.005))
    torch.save(res.out.cpu(), sys.argv[1])
else:
    import torch
    for tag, env in (("on", {}), ("off", {"S2O_POISON_CHECK": "0"})):
        subprocess.run([sys.executable, __file__, f"/tmp/o_{tag}.pt"], env={**os.environ, **env}, check=True)
    a, b = torch.load("/tmp/o_on.pt").float(), torch.load("/tmp/o_off.pt").float()
    d = (a - b).abs()
    print("max", d.max().item(), "rows differing", int((d.amax(-1) > 0).sum()), "nan on/off", bool(a.isnan().any()), bool(b.isnan().any()))
