"""Dev probe: device time of pass-1 and pass-2 alone at 128K (C3 shape), min of 5. Honors
S2O_VARIANT_DIR (A/B builds, paper_2602_22575_b200/build.py)."""
import os, sys
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


L = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
q, k, v = s2o.generate_synthetic("mixed", L // 64, 8.0, 0, 1, 32, L, 128)
qd = torch.from_numpy(q).cuda().to(torch.bfloat16)
kd = torch.from_numpy(k[:, :8]).cuda().to(torch.bfloat16)
vd = torch.from_numpy(v[:, :8]).cuda().to(torch.bfloat16)
del q, k, v
cfg = s2o.KernelConfig(seg_len=2048, tau=0.005)
plan, _ = s2o.build_plan(qd, kd, 2048)
t1 = timeit(lambda: s2o.pass1_dense_init(qd, kd, vd, cfg))
bufs = s2o.pass1_dense_init(qd, kd, vd, cfg)
t2 = timeit(lambda: s2o.pass2_sparse(qd, kd, vd, bufs, plan, cfg, check=False))
o, tr = s2o.pass2_sparse(qd, kd, vd, bufs, plan, cfg)
torch.cuda.synchronize()
pairs = int(tr.pass2_pairs.sum().item())
print(f"[{os.environ.get('S2O_VARIANT_DIR', 'pkg')} {os.environ.get('S2O_NVCC_FLAGS', '')}] L={L} pass1 {t1:.3f} ms "
      f"pass2 {t2:.3f} ms  pass2 pairs {pairs}  ({pairs * 512 / t2 / 1e9:.1f} TFLOP/s)", flush=True)
