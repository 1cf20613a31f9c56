"""Dev aid: candidate statistics of the candidate-pruned selection at C3 (torch emulation, fp32)."""
import sys, os, math, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_22575_b200 as s2o
L, S, T = 131072, 2048, 6144
q, k, _ = s2o.generate_synthetic("mixed", L // 64, 8.0, 0, 1, 4, L, 128)
qd = torch.from_numpy(q).cuda().to(torch.bfloat16).float()[0]
kd = torch.from_numpy(k[:, :1].copy()).cuda().to(torch.bfloat16).float()[0, 0]
N = L // S
kn = kd.norm(dim=1)
print("||k|| median %.3f max %.3f" % (kn.median().item(), kn.max().item()))
for h in range(1):
    qm = qd[h].view(N, S, 128).double().mean(1).float()
    for n in (5, 6, 8, 12, 16, 32, 48, 63):
        s = (kd[: n * S].double() @ qm[n].double()).float()
        samp = s[7::16][: n * 128]
        m = samp.numel(); x = min(T, n * S) * m / (n * S)
        r = min(m, max(1, math.ceil(x + 6 * math.sqrt(x) + 18)))
        theta = samp.sort(descending=True).values[r - 1]
        e = qm[n].norm() / 4096
        cand = ((s + e * kn[: n * S]) >= theta).sum().item()
        above = (s >= theta).sum().item()
        print(f"n={n:2d} nS={n*S:6d} ||q||={qm[n].norm().item():.4f} theta={theta.item():.4f} e*|k|med={(e*kn.median()).item():.2e} above={above} cand={cand}")
