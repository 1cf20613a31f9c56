"""Dev probe: per-pair depth statistics of the pass-2 trace at the C3 shape (pairs = tiles 2p, 2p+1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_22575_b200 as s2o
L = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
q, k, v = s2o.generate_synthetic("mixed", L // 64, 8.0, 0, 1, 32, L, 128)
qd = torch.from_numpy(q).cuda().to(torch.bfloat16); kd = torch.from_numpy(k[:, :8]).cuda().to(torch.bfloat16)
vd = torch.from_numpy(v[:, :8]).cuda().to(torch.bfloat16)
res = s2o.s2o_attention(qd, kd, vd, s2o.KernelConfig(seg_len=2048, tau=0.005))
torch.cuda.synchronize()
pt = res.trace.processed.reshape(32, L // 2048, 16).cpu().numpy()[:, 1:, :]  # skip segment 0
c0, c1 = pt[..., 0::2], pt[..., 1::2]
blocks = np.maximum(c0, c1) + 1
both = np.minimum(c0, c1) + 1
print("tile depth mean %.2f max %d" % (pt.mean(), pt.max()))
print("pair blocks mean %.2f; both-active mean %.2f; single-slot fraction of pair-blocks %.3f"
      % (blocks.mean(), both.mean(), 1 - both.sum() / blocks.sum()))
print("tile-chunks (committed+stop) %d, pair-blocks %d" % ((pt + 1).sum(), blocks.sum()))
np.save("gpurun_out/trace_c3.npy", pt)
