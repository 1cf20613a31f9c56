"""Head sharding through the real operator: for N = 2/4/8 every rank's shard --
whole GQA groups, kv heads [r*Hkv/N, (r+1)*Hkv/N) and their q heads -- run alone on one GPU gives
bit for bit the outputs, traces and pair counts of the same heads in the unsharded run (heads are
independent; no kernel result depends on which other heads share the launch)."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import bf16_round

pytestmark = pytest.mark.gpu


def test_every_shard_equals_the_full_run(cuda):
    import paper_2602_22575_b200 as s2o
    from paper_2602_22575_b200.shard import head_shard, shard_inputs
    torch = cuda
    hq, hkv, l = 32, 8, 8192
    q, k, v = s2o.generate_synthetic("mixed", l // 64, 8.0, 0, 1, hq, l, 128)
    qd, kd, vd = (torch.from_numpy(np.ascontiguousarray(bf16_round(x))).cuda().to(torch.bfloat16)
                  for x in (q, k[:, :hkv], v[:, :hkv]))
    cfg = s2o.KernelConfig(seg_len=1024, tau=0.005)
    full = s2o.s2o_attention(qd, kd, vd, cfg, want_plan=False)
    torch.cuda.synchronize()
    for world in (2, 4, 8):
        for rank in range(world):
            sh = head_shard(hq, hkv, world, rank)
            qs, ks, vs = (t.contiguous() for t in shard_inputs(qd, kd, vd, sh))
            part = s2o.s2o_attention(qs, ks, vs, cfg, want_plan=False)
            torch.cuda.synchronize()
            assert torch.equal(part.out, full.out[:, sh.q_lo:sh.q_hi]), (world, rank)
            assert torch.equal(part.trace.processed, full.trace.processed[:, sh.q_lo:sh.q_hi]), (world, rank)
            assert torch.equal(part.trace.pass2_pairs, full.trace.pass2_pairs[:, sh.q_lo:sh.q_hi]), (world, rank)
