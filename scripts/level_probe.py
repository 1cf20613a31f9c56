"""Dev probe: plan levels and stage times at C3 for a small tau (set S2O_LEVEL_LOG=1)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_22575_b200 as s2o
L = 131072
tau = float(sys.argv[1]) if len(sys.argv) > 1 else 0.001
q, k, v = s2o.generate_synthetic("mixed", L // 64, 8.0, 0, 1, 32, L, 128)
qd = torch.from_numpy(q).cuda().to(torch.bfloat16)
kd = torch.from_numpy(k[:, :8]).cuda().to(torch.bfloat16)
vd = torch.from_numpy(v[:, :8]).cuda().to(torch.bfloat16)
cfg = s2o.KernelConfig(seg_len=2048, tau=tau)
s2o.s2o_attention(qd, kd, vd, cfg, want_plan=False); torch.cuda.synchronize()
t0 = time.perf_counter(); res = s2o.s2o_attention(qd, kd, vd, cfg, want_plan=False); torch.cuda.synchronize()
print("total ms", (time.perf_counter() - t0) * 1e3)
p = res.trace.processed.cpu().numpy()
print("walk chunks: mean %.1f p99 %.0f max %d" % (p[:, :, 1:].mean(), __import__('numpy').percentile(p[:, :, 1:], 99), p.max()))
plan, _ = s2o.build_plan(qd, kd, 2048)
bufs = s2o.pass1_dense_init(qd, kd, vd, cfg)
def timeit(fn):
    fn(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); fn(); b.record(); torch.cuda.synchronize(); return a.elapsed_time(b)
print("pass2 on the full plan ms", timeit(lambda: s2o.pass2_sparse(qd, kd, vd, bufs, plan, cfg)))
print("full plan ms", timeit(lambda: s2o.build_plan(qd, kd, 2048)))
