"""Dev probe: clock64 timeline of the first CTA pair of the cta_group::2 pass kernel
(build with S2O_NVCC_FLAGS=-DS2O_TIMELINE). Leader events e, peer events e + 16:
1 s_full seen, 2 P stored, 3 p_full arrived, 4 d_full seen (softmax slot 0, row 0);
5 p_full seen, 6 PV issued, 7 S(j+1) issued, 8 k_full seen (MMA); 9/10 K/V expect_tx."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np, torch
import paper_2602_22575_b200 as s2o
CAP = 1024
L = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
lib = s2o.lib()
lib.s2o_debug_timeline.argtypes = [C.c_void_p]
q, k, v = s2o.generate_synthetic("mixed", L // 64, 8.0, 0, 1, 32, L, 128)
qd = torch.from_numpy(q).cuda().to(torch.bfloat16); kd = torch.from_numpy(k[:, :8]).cuda().to(torch.bfloat16)
vd = torch.from_numpy(v[:, :8]).cuda().to(torch.bfloat16)
del q, k, v
cfg = s2o.KernelConfig(seg_len=2048, tau=0.005)
plan, _ = s2o.build_plan(qd, kd, 2048)
bufs = s2o.pass1_dense_init(qd, kd, vd, cfg)
s2o.pass2_sparse(qd, kd, vd, bufs, plan, cfg); torch.cuda.synchronize()
buf = torch.zeros(32 * CAP, dtype=torch.int64, device="cuda")
names = {1: "sfull", 2: "Pdone", 3: "arrive", 4: "dfull", 5: "m_pfull", 6: "m_PV", 7: "m_S", 8: "m_kfull", 9: "ld_K", 10: "ld_V"}
for tag, fn in (("pass1", lambda: s2o.pass1_dense_init(qd, kd, vd, cfg)), ("pass2", lambda: s2o.pass2_sparse(qd, kd, vd, bufs, plan, cfg))):
    buf.zero_()
    lib.s2o_debug_timeline(C.c_void_p(buf.data_ptr()))
    fn(); torch.cuda.synchronize()
    lib.s2o_debug_timeline(C.c_void_p(0))
    t = buf.cpu().numpy().reshape(32, CAP).astype(np.int64)
    t0 = t[t > 0].min()
    rel = np.where(t > 0, t - t0, -1)
    print("==", tag)
    for ev in (9, 10, 8, 1, 17, 2, 18, 3, 19, 5, 6, 7, 4, 20):
        row = rel[ev]
        nm = names.get(ev if ev < 16 else ev - 16, "?") + ("(peer)" if ev >= 16 else "")
        print(f"{nm:>14} " + " ".join(f"{x:7d}" for x in row[2:22]))
