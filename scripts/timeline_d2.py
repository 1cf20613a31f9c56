"""Dev probe: clock64 timeline of CTA 0 of tc_diag2_kernel (build with S2O_NVCC_FLAGS=-DS2O_TIMELINE,
run with S2O_DIAG2=1). Events: MMA (seq = block) 1 iteration start, 2/5 p_full[x] seen, 4/7 P V_x
issued, 8/9 S_x issued; softmax x (seq = block of slot x) 10+4x s_full seen, 11+4x S loaded,
12+4x exps done, 13+4x p_full arrived; epilogue 18+2x o_done seen, 19+2x o_free; loaders 22 K /
23 V slot acquired, 24 Q slot acquired, 25 Q seen by MMA."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import torch
import paper_2602_22575_b200 as s2o

CAP = 1024
L = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
lib = s2o.lib()
lib.s2o_debug_timeline.argtypes = [C.c_void_p]
torch.manual_seed(0)
qd = torch.randn(1, 32, L, 128, device="cuda").to(torch.bfloat16)
kd = torch.randn(1, 8, L, 128, device="cuda").to(torch.bfloat16)
vd = torch.randn(1, 8, L, 128, device="cuda").to(torch.bfloat16)
cfg = s2o.KernelConfig(seg_len=2048, tau=0.005)
s2o.pass1_dense_init(qd, kd, vd, cfg)
buf = torch.zeros(32 * CAP, dtype=torch.int64, device="cuda")
lib.s2o_debug_timeline(buf.data_ptr())
s2o.pass1_dense_init(qd, kd, vd, cfg)
torch.cuda.synchronize()
lib.s2o_debug_timeline(None)
t = buf.cpu().numpy().reshape(32, CAP)
st, en = t[0][:148], t[3][:148]
if (st > 0).all() and (en > 0).all():  # per-CTA spans (global timer, ns)
    d = (en - st) / 1e3
    print(f"CTA spans us: min {d.min():.0f} median {np.median(d):.0f} max {d.max():.0f}; kernel "
          f"{(en.max() - st.min()) / 1e3:.0f} us; end spread {(en.max() - en.min()) / 1e3:.0f} us")
    np.save("gpurun_out/cta_spans_d2.npy", np.stack([st, en]))
t[0] = 0
t[3] = 0
t0 = t[t > 0].min()
rel = np.where(t > 0, t - t0, -1)
np.save("gpurun_out/timeline_d2.npy", rel)
names = {1: "it", 2: "p0seen", 4: "pv0iss", 8: "s0iss", 5: "p1seen", 7: "pv1iss", 9: "s1iss",
         10: "sm0_sf", 11: "sm0_ld", 12: "sm0_ex", 13: "sm0_arr", 14: "sm1_sf", 15: "sm1_ld", 16: "sm1_ex",
         17: "sm1_arr", 18: "ep0_od", 19: "ep0_free", 20: "ep1_od", 21: "ep1_free", 22: "k_acq", 23: "v_acq",
         24: "q_acq", 25: "q_seen"}
lo = int(sys.argv[2]) if len(sys.argv) > 2 else 100
for ev, nm in names.items():
    row = rel[ev]
    print(f"{nm:>9} " + " ".join(f"{v:7d}" for v in row[lo:lo + 16]))
it = rel[1]
ok = it > 0
d = np.diff(it[ok])
print("iteration period clk: median", np.median(d), "mean", d.mean())
for a, b, nm in ((1, 2, "it->p0seen"), (2, 4, "p0seen->pv0iss"), (4, 8, "pv0->s0iss"), (8, 5, "s0iss->p1seen"),
                 (5, 7, "p1seen->pv1iss"), (7, 9, "pv1->s1iss")):
    x = rel[b] - rel[a]
    m = (rel[a] > 0) & (rel[b] > 0)
    print(f"{nm:>16}: median {np.median(x[m]):7.0f} mean {x[m].mean():7.0f}")
for x in (0, 1):
    b = 10 + 4 * x
    for a2, b2, nm in ((b, b + 1, "sf->ld"), (b + 1, b + 2, "ld->exps"), (b + 2, b + 3, "exps->arr")):
        v = rel[b2] - rel[a2]
        m = (rel[a2] > 0) & (rel[b2] > 0)
        print(f"softmax{x} {nm:>10}: median {np.median(v[m]):7.0f} mean {v[m].mean():7.0f}")
    # arrival -> next s_full seen
    v = rel[b][1:] - rel[b + 3][:-1]
    m = (rel[b][1:] > 0) & (rel[b + 3][:-1] > 0)
    print(f"softmax{x} arr->next sf: median {np.median(v[m]):7.0f} mean {v[m].mean():7.0f}")
