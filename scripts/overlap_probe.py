"""Dev probe: does running the truncated plan and pass-1 on two streams (they are independent)
shorten the pair? C3, CUDA events, min of 5."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_22575_b200 as s2o

L = 131072
q, k, v = s2o.generate_synthetic("mixed", L // 64, 8.0, 0, 1, 32, L, 128)
qd = torch.from_numpy(q).cuda().to(torch.bfloat16)
kd = torch.from_numpy(k[:, :8]).cuda().to(torch.bfloat16)
vd = torch.from_numpy(v[:, :8]).cuda().to(torch.bfloat16)
del q, k, v
cfg = s2o.KernelConfig(seg_len=2048, tau=0.005)
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()


def seq():
    s2o.build_plan_truncated(qd, kd, 2048)
    s2o.pass1_dense_init(qd, kd, vd, cfg)


def par():
    cur = torch.cuda.current_stream()
    e0 = torch.cuda.Event()
    e0.record(cur)
    sa.wait_event(e0)
    sb.wait_event(e0)
    with torch.cuda.stream(sa):
        s2o.build_plan_truncated(qd, kd, 2048)
    with torch.cuda.stream(sb):
        s2o.pass1_dense_init(qd, kd, vd, cfg)
    ea, eb = torch.cuda.Event(), torch.cuda.Event()
    ea.record(sa)
    eb.record(sb)
    cur.wait_event(ea)
    cur.wait_event(eb)


def t(fn):
    fn(); fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); best = min(best, a.elapsed_time(b))
    return best


print(f"sequential {t(seq):.3f} ms, two streams {t(par):.3f} ms", flush=True)
