"""The candidate-pruned top-T selection (csrc/plan_tc.cuh) is an exact replacement for scoring
every prefix key: its truncated plan must equal the first min(nS, T) entries of every segment of
the full permutation (build_plan, which is itself bit-identical to the oracle), for the shapes the
operator sees, for inputs without structure, with heavy score ties and with quantised keys.
A row whose candidates cannot be certified raises the flag (the operator then builds the full
plan); every listed index stays in bounds. Needs a B200."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _dev(torch, x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16)


def _check_prefix(torch, s2o, qd, kd, seg, depth, expect_flag=None):
    plan, _ = s2o.build_plan(qd, kd, seg)
    qp, kvt, flag = s2o.build_plan_truncated(qd, kd, seg, depth)
    torch.cuda.synchronize()
    if expect_flag is not None:
        assert flag.item() == expect_flag
    n_seg = plan.seg.seg_count
    last = plan.seg.last_len  # q_perm of the (ragged) last segment: its first last_len entries
    assert torch.equal(qp[:, :, : n_seg - 1], plan.q_perm[:, :, : n_seg - 1])
    assert torch.equal(qp[:, :, n_seg - 1, :last], plan.q_perm[:, :, n_seg - 1, :last])
    bad = []
    for n in range(1, n_seg):
        t = min(n * seg, depth)
        off = plan.seg.kv_offset(n)
        got = kvt[:, :, n, :t]
        assert int(got.min()) >= 0 and int(got.max()) < n * seg  # in bounds even when flagged
        if flag.item() == 0 and not torch.equal(got, plan.kv_perm[:, :, off: off + t]):
            bad.append(n)
    assert not bad, f"segments whose truncated list differs from the full plan: {bad}"
    return flag.item()


@pytest.mark.parametrize("hq,hkv,l,seg,seed", [(4, 2, 16384, 1024, 2), (8, 2, 32768, 2048, 1),
                                               (4, 1, 65536, 2048, 3)])
@pytest.mark.parametrize("depth", [128, 1000, 6144])
def test_candidate_plan_is_prefix_of_full_plan(cuda, hq, hkv, l, seg, seed, depth):
    import paper_2602_22575_b200 as s2o
    torch = cuda
    q, k, _ = s2o.generate_synthetic("mixed", l // 64, 8.0, seed, 1, hq, l, 128)
    assert _check_prefix(torch, s2o, _dev(torch, q), _dev(torch, k[:, :hkv]), seg, depth) == 0


def test_candidate_plan_unstructured_and_quantised(cuda):
    """Gaussian inputs (no stripes: the score distribution has no gap at the threshold) and keys
    rounded to integers (many exactly equal scores, resolved by index) select exactly."""
    import paper_2602_22575_b200 as s2o
    torch = cuda
    rng = np.random.default_rng(0)
    q = rng.standard_normal((1, 4, 16384, 128)).astype(np.float32)
    k = rng.standard_normal((1, 2, 16384, 128)).astype(np.float32)
    for kk in (k, np.round(k)):
        assert _check_prefix(torch, s2o, _dev(torch, q), _dev(torch, kk), 2048, 6144) == 0


def test_candidate_plan_all_ties_flags_and_falls_back(cuda):
    """Every key equal: every key is a candidate, more than a row can hold, so the selection
    flags itself; the operator's result still equals the full-plan operator's."""
    import paper_2602_22575_b200 as s2o
    torch = cuda
    rng = np.random.default_rng(1)
    q = rng.standard_normal((1, 4, 16384, 128)).astype(np.float32)
    k = np.full((1, 2, 16384, 128), 0.5, np.float32)
    v = rng.standard_normal((1, 2, 16384, 128)).astype(np.float32)
    assert _check_prefix(torch, s2o, _dev(torch, q), _dev(torch, k), 2048, 6144, expect_flag=1) == 1
    qd, kd, vd = _dev(torch, q), _dev(torch, k), _dev(torch, v)
    cfg = s2o.KernelConfig(seg_len=2048, tau=0.005)
    full = s2o.s2o_attention(qd, kd, vd, cfg)  # full plan (want_plan)
    trunc = s2o.s2o_attention(qd, kd, vd, cfg, want_plan=False)  # truncated plan -> fallback
    torch.cuda.synchronize()
    assert torch.equal(full.trace.processed, trunc.trace.processed)
    assert torch.equal(full.out, trunc.out)


@pytest.mark.parametrize("z,hq,hkv,l,seg", [(2, 4, 2, 20480 + 640, 2048),   # batch 2, ragged last segment
                                            (1, 2, 2, 24576, 2048),         # group 1
                                            (1, 8, 1, 24576, 2048)])        # group 8
def test_candidate_plan_batches_ragged_groups(cuda, z, hq, hkv, l, seg):
    """The candidate path for Z > 1, a ragged last segment and GQA groups 1 and 8 (row tiles and
    replication depend on the group) still gives the prefix of the full plan."""
    import paper_2602_22575_b200 as s2o
    torch = cuda
    q, k, _ = s2o.generate_synthetic("mixed", l // 64, 8.0, 7, z, hq, l, 128)
    qd = _dev(torch, q)
    kd = _dev(torch, k[:, :hkv])
    assert _check_prefix(torch, s2o, qd, kd, seg, 6144) == 0
    assert _check_prefix(torch, s2o, qd, kd, seg, 1000) == 0
