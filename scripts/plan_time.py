"""Dev probe: device time of the truncated plan (the operator's Step 1) at C2 / C3, min of 5, and a
hash of its output (for A/B builds: S2O_KV_SCORE=1 selects the previous kv scoring kernel)."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2602_22575_b200 as s2o


def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); best = min(best, a.elapsed_time(b))
    return best


for L in [int(x) for x in (sys.argv[1:] or ["131072"])]:
    q, k, v = s2o.generate_synthetic("mixed", L // 64, 8.0, 0, 1, 32, L, 128)
    qd = torch.from_numpy(q).cuda().to(torch.bfloat16)
    kd = torch.from_numpy(k[:, :8].copy()).cuda().to(torch.bfloat16)
    del q, k, v
    t = timeit(lambda: s2o.build_plan_truncated(qd, kd, 2048))
    qp, kv, flag = s2o.build_plan_truncated(qd, kd, 2048)
    torch.cuda.synchronize()
    h = hashlib.sha1(qp.cpu().numpy().tobytes() + kv.cpu().numpy().tobytes()).hexdigest()[:16]
    print(f"[{os.environ.get('S2O_KV_SCORE', 'v2')}] L={L} plan_truncated {t:.3f} ms flag {flag.item()} hash {h}",
          flush=True)
