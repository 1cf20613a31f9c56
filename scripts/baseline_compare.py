"""Matched-sparsity comparison (PAPER.md C7 direction): S2O at tau against
the block top-k baseline with the k whose sparsity is closest, both against dense causal
attention on the same GPU (torch SDPA, fp32 comparison), on the stripe-structured synthetic.

    python scripts/baseline_compare.py [L] [heads] [--out profiles/baseline_compare.json]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2602_22575_b200 as s2o


def timed(fn):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, time.perf_counter() - t0


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    L = int(args[0]) if args else 16384
    H = int(args[1]) if len(args) > 1 else 4
    out_path = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    S, B = 2048, 128
    q, k, v = s2o.generate_synthetic("mixed", L // 64, 8.0, 0, 1, H, L, 128)
    dq, dk, dv = (torch.from_numpy(x).cuda().to(torch.bfloat16) for x in (q, k, v))
    dense = torch.nn.functional.scaled_dot_product_attention(dq, dk, dv, is_causal=True).float()
    total = H * L * (L + 1) / 2
    rows = []
    for tau in (0.005, 0.02):
        cfg = s2o.KernelConfig(seg_len=S, tau=tau)
        res, secs = timed(lambda: s2o.s2o_attention(dq, dk, dv, cfg, want_plan=False))
        pairs = int(res.trace.pass1_pairs.sum().item() + res.trace.pass2_pairs.sum().item())
        sp = 1 - pairs / total
        mse = float(((res.out.float() - dense) ** 2).mean().item())
        # block top-k: pairs per head = self triangles + rows x kept prefix tokens (nested in k)
        nqb = L // B
        best = None
        for kk in range(0, nqb):
            kept = sum(min(kk, qb) for qb in range(nqb)) * B * B + nqb * B * (B + 1) // 2
            if best is None or abs(kept * H - pairs) < abs(best[1] * H - pairs):
                best = (kk, kept)
            if kept * H > pairs:
                break
        kk = best[0]
        (bo, bp), bsecs = timed(lambda: s2o.block_topk_attention(dq, dk, dv, B, B, kk))
        bpairs = int(bp.sum().item())
        bmse = float(((bo.float() - dense) ** 2).mean().item())
        row = {"tau": tau, "s2o": {"sparsity": round(sp, 5), "mse": mse, "ms": round(secs * 1e3, 3)},
               "block_topk": {"k": kk, "block": B, "sparsity": round(1 - bpairs / total, 5), "mse": bmse,
                              "ms": round(bsecs * 1e3, 1)},
               "mse_ratio_topk_over_s2o": bmse / mse if mse > 0 else None}
        rows.append(row)
        print(json.dumps(row), flush=True)
    if out_path:
        with open(out_path, "w") as f:
            json.dump({"config": {"L": L, "heads": H, "d": 128, "seg_len": S, "block": B, "dtype": "bf16",
                                  "data": "synthetic mixed stripes (L/64, gain 8, seed 0)",
                                  "dense": "torch SDPA bf16 causal (fp32 difference)"},
                       "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
