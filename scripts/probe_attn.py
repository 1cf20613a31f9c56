"""Dev probe: time plan / pass-1 / pass-2 / whole op at the C2/C3 shapes on the tcgen05 path."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_22575_b200 as s2o

def timeit(fn, reps=3):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return min(ts)

for L in [int(x) for x in (sys.argv[1:] or ["32768", "131072"])]:
    q, k, v = s2o.generate_synthetic("mixed", L // 64, 8.0, 0, 1, 32, L, 128)
    qd = torch.from_numpy(q).cuda().to(torch.bfloat16)
    kd = torch.from_numpy(k[:, :8]).cuda().to(torch.bfloat16)
    vd = torch.from_numpy(v[:, :8]).cuda().to(torch.bfloat16)
    del q, k, v
    cfg = s2o.KernelConfig(seg_len=2048, tau=0.005)
    plan, _ = s2o.build_plan(qd, kd, 2048)
    t_plan = timeit(lambda: s2o.build_plan(qd, kd, 2048))
    t_p1 = timeit(lambda: s2o.pass1_dense_init(qd, kd, vd, cfg))
    bufs = s2o.pass1_dense_init(qd, kd, vd, cfg)
    t_p2 = timeit(lambda: s2o.pass2_sparse(qd, kd, vd, bufs, plan, cfg))
    t_all = timeit(lambda: s2o.s2o_attention(qd, kd, vd, cfg, want_plan=False))
    res = s2o.s2o_attention(qd, kd, vd, cfg)
    torch.cuda.synchronize()
    p1 = res.trace.pass1_pairs.sum().item(); p2 = res.trace.pass2_pairs.sum().item()
    tot = 32 * L * (L + 1) / 2
    t_dense = timeit(lambda: torch.nn.functional.scaled_dot_product_attention(qd, kd.repeat_interleave(4, 1), vd.repeat_interleave(4, 1), is_causal=True), reps=2)
    fl = 4 * 128 * (p1 + p2)
    print(f"L={L}: plan {t_plan:.2f} ms, pass1 {t_p1:.2f} ms, pass2 {t_p2:.2f} ms, total {t_all:.2f} ms; "
          f"sparsity {1 - (p1 + p2) / tot:.4f}; alg TFLOP/s (passes) {fl / ((t_p1 + t_p2) * 1e-3) / 1e12:.1f}; "
          f"dense sdpa {t_dense:.2f} ms", flush=True)
