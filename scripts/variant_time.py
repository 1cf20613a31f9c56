"""Dev probe: whole-operator device time of the two-pass, no-q-reorder and fused variants at the
C3 shape (128K, 32q/8kv heads) for a few tau, CUDA events, min of 3."""
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
out = torch.empty_like(qd)


def timeit(fn, reps=3):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); best = min(best, a.elapsed_time(b))
    return best


for tau in (0.005, 0.001):
    for name, qr, fu in (("two-pass", True, False), ("no-q-reorder", False, False), ("fused", False, True)):
        cfg = s2o.KernelConfig(seg_len=2048, tau=tau, q_reorder=qr, fused=fu)
        ms = timeit(lambda: s2o.s2o_attention(qd, kd, vd, cfg, out=out, want_plan=False))
        res = s2o.s2o_attention(qd, kd, vd, cfg, want_plan=False)
        torch.cuda.synchronize()
        p = int(res.trace.pass1_pairs.sum().item() + res.trace.pass2_pairs.sum().item())
        print(f"L={L} tau={tau} {name:13s} {ms:8.3f} ms  sparsity {1 - p / (32 * L * (L + 1) / 2):.5f}", flush=True)
