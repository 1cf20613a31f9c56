"""Dev probe: clock64 pipeline timeline of CTA 0 of the tcgen05 pass kernel (pass-1, pass-2).

    python scripts/timeline.py [L]

Events (attn_sm100.cu tl_mark): 5 k_full seen by MMA, 6/7 p_full[x] seen by MMA, 8 kv_empty
committed, 9 loader acquired stage, 10 loader issued block, 11/15 pair start (slot 0/1),
12/16 state init done, 13/17 o_done seen, 14/18 epilogue done, 19/22 s_full seen,
20/23 exps done, 21/24 p_full arrived.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C

import numpy as np
import torch

import paper_2602_22575_b200 as s2o

CAP = 1024
NAMES = {5: "k_full", 6: "p0_seen", 7: "p1_seen", 8: "kv_empty", 9: "ld_acq", 10: "ld_iss",
         11: "s0_pair", 12: "s0_init", 13: "s0_odone", 14: "s0_epi", 15: "s1_pair", 16: "s1_init",
         17: "s1_odone", 18: "s1_epi", 19: "s0_sfull", 20: "s0_exps", 21: "s0_arrive",
         22: "s1_sfull", 23: "s1_exps", 24: "s1_arrive", 25: "s0_ldwait", 26: "mma_qfull", 27: "mma_s0iss",
         28: "v_full", 29: "kq_issued", 30: "kq_start", 1: "v_acq", 2: "v_iss", 31: "s0_issued"}


def dump(tag, buf):
    t = buf.cpu().numpy().reshape(32, CAP).astype(np.int64)
    t0 = t[t > 0].min()
    rel = np.where(t > 0, t - t0, -1)
    np.save(os.path.join("gpurun_out", f"timeline_{tag}.npy"), rel)
    st, en = t[0][:148], t[3][:148]
    if (st > 0).all() and (en > 0).all():  # per-CTA spans (global timer, ns)
        d = (en - st) / 1e3
        print(f"   CTA spans us: min {d.min():.0f} median {np.median(d):.0f} max {d.max():.0f}; "
              f"starts spread {(st.max() - st.min()) / 1e3:.1f} us; kernel {(en.max() - st.min()) / 1e3:.0f} us; "
              f"slowest CTAs {np.argsort(d)[-5:].tolist()}")
    print(f"== {tag}: total span {rel.max()} clk")
    for ev in (9, 10, 1, 2, 5, 28, 31, 19, 25, 20, 21, 6, 22, 23, 24, 7, 8):
        row = rel[ev]
        n = int((row >= 0).sum())
        first = row[:24]
        print(f"{NAMES[ev]:>10} n={n:4d} " + " ".join(f"{v:7d}" for v in first))
    for ev in (30, 29, 26, 27, 11, 12, 13, 14, 15, 16, 17, 18):
        row = rel[ev]
        print(f"{NAMES[ev]:>10} " + " ".join(f"{v:7d}" for v in row[:12]))


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
    lib = s2o.lib()
    lib.s2o_debug_timeline.argtypes = [C.c_void_p]
    q, k, v = s2o.generate_synthetic("mixed", L // 64, 8.0, 0, 1, 32, L, 128)
    qd = torch.from_numpy(q).cuda().to(torch.bfloat16)
    kd = torch.from_numpy(k[:, :8]).cuda().to(torch.bfloat16)
    vd = torch.from_numpy(v[:, :8]).cuda().to(torch.bfloat16)
    del q, k, v
    cfg = s2o.KernelConfig(seg_len=2048, tau=0.005)
    plan, _ = s2o.build_plan(qd, kd, 2048)
    bufs = s2o.pass1_dense_init(qd, kd, vd, cfg)
    s2o.pass2_sparse(qd, kd, vd, bufs, plan, cfg)
    torch.cuda.synchronize()
    buf = torch.zeros(32 * CAP, dtype=torch.int64, device="cuda")
    lib.s2o_debug_timeline(C.c_void_p(buf.data_ptr()))
    bufs = s2o.pass1_dense_init(qd, kd, vd, cfg)
    torch.cuda.synchronize()
    dump("pass1", buf)
    buf.zero_()
    s2o.pass2_sparse(qd, kd, vd, bufs, plan, cfg)
    torch.cuda.synchronize()
    dump("pass2", buf)
    lib.s2o_debug_timeline(C.c_void_p(0))


if __name__ == "__main__":
    main()
