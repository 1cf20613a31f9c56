import sys, time, torch, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2602_22575_b200 as s2o
torch.cuda.set_device(0)
def bf(x): return torch.from_numpy(x).cuda().to(torch.bfloat16)
for (hq, hkv, L, S, seed) in [(4, 2, 16384, 1024, 2), (8, 2, 32768, 2048, 1), (4, 1, 65536, 2048, 3)]:
    q, k, _ = s2o.generate_synthetic("mixed", L // 64, 8.0, seed, 1, hq, L, 128)
    qd, kd = bf(q), bf(k[:, :hkv].copy())
    plan, _ = s2o.build_plan(qd, kd, S)
    for depth in (128, 1000, 4096, 6144):
        qp, kvt, flag = s2o.build_plan_truncated(qd, kd, S, depth)
        torch.cuda.synchronize()
        bad = 0
        for n in range(1, L // S):
            t = min(n * S, depth)
            off = plan.seg.kv_offset(n)
            if not torch.equal(kvt[:, :, n, :t], plan.kv_perm[:, :, off: off + t]): bad += 1
        print(hq, hkv, L, S, depth, "flag", flag.item(), "bad segs", bad, "qperm", torch.equal(qp, plan.q_perm), flush=True)
# gaussian, ties
L, S = 16384, 2048
q = np.random.default_rng(0).standard_normal((1, 4, L, 128)).astype(np.float32)
k = np.random.default_rng(1).standard_normal((1, 2, L, 128)).astype(np.float32)
for name, kk in [("gauss", k), ("ties", np.full_like(k, 0.5)), ("quant", np.round(k))]:
    qd, kd = bf(q), bf(kk)
    plan, _ = s2o.build_plan(qd, kd, S)
    qp, kvt, flag = s2o.build_plan_truncated(qd, kd, S, 6144)
    torch.cuda.synchronize()
    bad = sum(not torch.equal(kvt[:, :, n, :min(n*S, 6144)], plan.kv_perm[:, :, plan.seg.kv_offset(n): plan.seg.kv_offset(n) + min(n*S, 6144)]) for n in range(1, L // S))
    print(name, "flag", flag.item(), "bad", bad, flush=True)
# timing at C3
L = 131072
q, k, _ = s2o.generate_synthetic("mixed", L // 64, 8.0, 0, 1, 32, L, 128)
qd, kd = bf(q), bf(k[:, :8].copy())
for _ in range(3): s2o.build_plan_truncated(qd, kd, 2048, 6144)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): qp, kvt, flag = s2o.build_plan_truncated(qd, kd, 2048, 6144)
e1.record(); torch.cuda.synchronize()
print("C3 truncated plan ms", e0.elapsed_time(e1) / 10, "flag", flag.item())
