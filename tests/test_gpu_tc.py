"""tcgen05 path (bf16, D=128, 128x128 tiles) vs the oracle and the exact generic path.

Tolerances (bf16 operands, fp32 accumulation, bf16 output):
  * outputs: max |O_tc - O_ref| <= 2.5e-2 and mean |O_tc - O_ref| <= 2e-3, O_ref = the
    oracle's fp64 result on the same bf16-rounded inputs (rows with identical traces);
  * traces: identical, except threshold ties: every differing tile must have
    the reference's gain at its first differing chunk within |gain - tau| / tau <= 1e-4
    (conftest.assert_trace_ties replays the tile in the reference arithmetic);
  * plans: bit-identical (the plan kernels do not depend on the attention path).
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import GOLDEN, Cfg, assert_trace_ties, bf16_round

pytestmark = pytest.mark.gpu

TC, GEN = 2, 1


def dev_bf16(torch, x):
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda().to(torch.bfloat16)


def kcfg(s2o, c: Cfg, path):
    return s2o.KernelConfig(seg_len=c.seg_len, tau=c.tau, tiles=s2o.TileSpec(c.b_m, c.b_n),
                            q_reorder=c.q_reorder, fused=c.fused, path=path)


def inputs(s2o, hq, hkv, l, seed=0):
    q, k, v = s2o.generate_synthetic("mixed", max(1, l // 64), 8.0, seed, 1, hq, l, 128)
    return bf16_round(q), bf16_round(k[:, :hkv]), bf16_round(v[:, :hkv])


def run(torch, s2o, q, k, v, c, path):
    res = s2o.s2o_attention(dev_bf16(torch, q), dev_bf16(torch, k), dev_bf16(torch, v), kcfg(s2o, c, path))
    torch.cuda.synchronize()
    return res


def trace_diff(a, b):
    a = a.reshape(-1)
    b = b.reshape(-1)
    diff = a != b
    return int(diff.sum()), (int(np.abs(a - b).max()) if diff.any() else 0)


def test_tc_path_selected(cuda):
    import paper_2602_22575_b200 as s2o
    torch = cuda
    q, k, v = inputs(s2o, 2, 1, 256)
    qd, kd, vd = dev_bf16(torch, q), dev_bf16(torch, k), dev_bf16(torch, v)
    assert s2o.select_path(qd, kd, vd, s2o.KernelConfig(seg_len=128)) == TC
    assert s2o.select_path(qd.float(), kd.float(), vd.float(), s2o.KernelConfig(seg_len=128)) == GEN


def test_tc_gqa_golden(cuda, port):
    """Reference golden (Hq=4, Hkv=2, L=4096, S=512, 128x128, tau=0.005)."""
    import paper_2602_22575_b200 as s2o
    torch = cuda
    g = np.load(os.path.join(GOLDEN, "gqa_golden.npz"))
    q, k, v = s2o.generate_synthetic("mixed", 64, 8.0, 7, 1, 4, 4096, 128)
    q, k, v = bf16_round(q), bf16_round(k[:, :2]), bf16_round(v[:, :2])
    res = run(torch, s2o, q, k, v, Cfg(512, 0.005, 128, 128), TC)
    np.testing.assert_array_equal(res.plan.q_perm.reshape(4, 8, 512).cpu().numpy(), g["q_perm"])
    np.testing.assert_array_equal(res.plan.kv_perm.reshape(4, -1).cpu().numpy(), g["kv_perm"])
    got = res.trace.processed.reshape(4, 8, -1).cpu().numpy()
    assert_trace_ties(port, q, np.repeat(k, 2, 1), np.repeat(v, 2, 1), Cfg(512, 0.005, 128, 128), g["q_perm"],
                      g["kv_perm"], got, g["processed"])
    out = res.out.float().cpu().numpy()[:, :, ::8]
    err = np.abs(out - g["out_rows"])
    assert err.max() <= 2.5e-2 and err.mean() <= 2e-3, (err.max(), err.mean())


@pytest.mark.parametrize("l,s,reorder,fused", [
    (1024, 256, True, False), (1024, 256, False, False), (1024, 256, False, True),
    (1000, 300, True, False), (1000, 300, False, True), (2048, 2048, True, False),
    (384, 100, True, False),
])
def test_tc_matches_oracle(cuda, port, l, s, reorder, fused):
    import paper_2602_22575_b200 as s2o
    torch = cuda
    hq, hkv = 2, 1
    q, k, v = inputs(s2o, hq, hkv, l, seed=l + s)
    for tau in (0.005, 0.0, 1e9):
        c = Cfg(s, tau, 128, 128, reorder, fused)
        res = run(torch, s2o, q, k, v, c, TC)
        want_o, want_t, want_p = port.attention(q, np.repeat(k, hq // hkv, 1), np.repeat(v, hq // hkv, 1), c)
        got_t = res.trace.processed.reshape(hq, -1).cpu().numpy()
        ndiff, _ = trace_diff(got_t, want_t.processed.reshape(hq, -1))
        assert_trace_ties(port, q, np.repeat(k, hq // hkv, 1), np.repeat(v, hq // hkv, 1), c, want_p.q_perm,
                          want_p.kv_perm, got_t, want_t.processed)
        if tau >= 1e9:
            assert (got_t == 0).all()
        out = res.out.float().cpu().numpy()
        err = np.abs(out - want_o)
        assert err.max() <= 2.5e-2 and err.mean() <= 2e-3, (tau, err.max(), err.mean())
        if ndiff == 0:
            np.testing.assert_array_equal(res.trace.pass2_pairs.reshape(-1).cpu().numpy(), want_t.pass2_pairs)


def test_tc_pass1_states(cuda, port):
    import paper_2602_22575_b200 as s2o
    torch = cuda
    q, k, v = inputs(s2o, 2, 2, 1000, seed=3)
    c = Cfg(300, 0.005, 128, 128)
    bufs = s2o.pass1_dense_init(dev_bf16(torch, q), dev_bf16(torch, k), dev_bf16(torch, v), kcfg(s2o, c, TC))
    acc, ell, m = port.pass1(q, k, v, c)
    # compare the finalized partial outputs and the maxima
    got = (bufs.acc / bufs.ell[..., None]).cpu().numpy()
    want = acc / ell[..., None]
    assert np.abs(got - want).max() <= 2e-2
    # The kernel rescales lazily: the stored m is a reference max within 8 log2-units below the
    # true running max (never above); ell and acc are relative to it, so ell * e^m is invariant.
    mg = bufs.m.cpu().numpy().astype(np.float64)
    assert (mg <= m + 1e-3).all() and (mg >= m - 8.0 * np.log(2.0) - 1e-3).all()
    lg = bufs.ell.cpu().numpy() * np.exp(mg - m)
    np.testing.assert_allclose(lg, ell, rtol=2e-3)


@pytest.mark.parametrize("hq,hkv", [(4, 2), (3, 1)])
def test_tc_pass1_states_batched_gqa(cuda, port, hq, hkv):
    """The two-tile pass-1 kernel against the oracle for Z = 2, an odd number of tiles per segment
    (S = 384: 3 tiles) and a ragged last segment: q-head pairs (group 2) and adjacent-tile pairs
    (group 3, whose last pair of a segment has one tile)."""
    import paper_2602_22575_b200 as s2o
    torch = cuda
    parts = [inputs(s2o, hq, hkv, 1000, seed=s) for s in (11, 12)]
    q, k, v = (np.concatenate([pp[i] for pp in parts], axis=0) for i in range(3))
    c = Cfg(384, 0.005, 128, 128)
    bufs = s2o.pass1_dense_init(dev_bf16(torch, q), dev_bf16(torch, k), dev_bf16(torch, v), kcfg(s2o, c, TC))
    rep = hq // hkv
    acc, ell, m = port.pass1(q, np.repeat(k, rep, 1), np.repeat(v, rep, 1), c)
    got = (bufs.acc / bufs.ell[..., None]).cpu().numpy()
    assert np.abs(got - acc / ell[..., None]).max() <= 2e-2
    mg = bufs.m.cpu().numpy().astype(np.float64)
    assert (mg <= m + 1e-3).all() and (mg >= m - 8.0 * np.log(2.0) - 1e-3).all()
    np.testing.assert_allclose(bufs.ell.cpu().numpy() * np.exp(mg - m), ell, rtol=2e-3)


def test_tc_dense_vs_sdpa(cuda):
    import paper_2602_22575_b200 as s2o
    torch = cuda
    torch.manual_seed(0)
    q = torch.randn(1, 4, 2048, 128, device="cuda").to(torch.bfloat16)
    k = torch.randn(1, 2, 2048, 128, device="cuda").to(torch.bfloat16)
    v = torch.randn(1, 2, 2048, 128, device="cuda").to(torch.bfloat16)
    o = s2o.dense_causal_attention(q, k, v, path=TC)
    ref = torch.nn.functional.scaled_dot_product_attention(
        q.float(), k.float().repeat_interleave(2, 1), v.float().repeat_interleave(2, 1), is_causal=True)
    assert (o - ref).abs().max().item() <= 2e-2


def test_tc_generic_agree_at_scale(cuda, ref):
    """L=8192, 8 q / 2 kv heads, S=1024: tcgen05 and the exact generic path see the same plan;
    the exact path's trace equals the compiled reference's, the tcgen05 trace equals it up to
    threshold ties; outputs agree to the bf16 tolerance."""
    import paper_2602_22575_b200 as s2o
    torch = cuda
    q, k, v = inputs(s2o, 8, 2, 8192, seed=1)
    c = Cfg(1024, 0.005, 128, 128)
    a = run(torch, s2o, q, k, v, c, TC)
    b = run(torch, s2o, q, k, v, c, GEN)
    assert torch.equal(a.plan.kv_perm, b.plan.kv_perm)
    kx, vx = np.repeat(k, 4, 1), np.repeat(v, 4, 1)
    _, want_t, want_p = ref.attention(q, kx, vx, c)
    np.testing.assert_array_equal(b.trace.processed.reshape(8, 8, -1).cpu().numpy(), want_t.processed)
    np.testing.assert_array_equal(a.plan.kv_perm.reshape(8, -1).cpu().numpy(), want_p.kv_perm)
    assert_trace_ties(ref, q, kx, vx, c, want_p.q_perm, want_p.kv_perm, a.trace.processed.cpu().numpy(),
                      want_t.processed)
    err = (a.out.float() - b.out.float()).abs()
    assert err.max().item() <= 2.5e-2 and err.mean().item() <= 2e-3


@pytest.mark.parametrize("path,fused", [(TC, False), (GEN, False), (TC, True)])
def test_truncated_plan_matches_full_plan(cuda, path, fused):
    """s2o_attention without a kv_perm output keeps only the exact top-T of each kv_perm
    segment; a tile that exhausts it saves its state and resumes on the next level (entries
    [T, 2T), ... of the same order), so traces equal the full-plan run for any depth (tiny
    depths force many levels). Outputs agree to state-round-trip rounding (the fp32 state is
    re-based at every level boundary): |dO| <= 1e-2 |O| + 1e-3 elementwise (one bf16 ulp is
    2^-8 relative) and mean |dO| <= 1e-4."""
    import paper_2602_22575_b200 as s2o
    torch = cuda
    hq, hkv, l, s = 4, 2, 8192, 1024
    q, k, v = inputs(s2o, hq, hkv, l, seed=5)
    qd, kd, vd = dev_bf16(torch, q), dev_bf16(torch, k), dev_bf16(torch, v)
    base = s2o.KernelConfig(seg_len=s, tau=0.005, path=path, q_reorder=not fused, fused=fused)
    full = s2o.s2o_attention(qd, kd, vd, base)  # kv_perm requested -> full plan
    torch.cuda.synchronize()
    for depth in (0, 128, 512, 2048):
        cfg = s2o.KernelConfig(seg_len=s, tau=0.005, path=path, plan_depth=depth, q_reorder=not fused, fused=fused)
        res = s2o.s2o_attention(qd, kd, vd, cfg, want_plan=False)
        torch.cuda.synchronize()
        assert torch.equal(res.trace.processed, full.trace.processed), depth
        assert torch.equal(res.trace.pass2_pairs, full.trace.pass2_pairs), depth
        d = (res.out.float() - full.out.float()).abs()
        excess = (d - (1e-2 * full.out.float().abs() + 1e-3)).max().item()
        assert excess <= 0 and d.mean().item() <= 1e-4, (depth, d.max().item(), d.mean().item())


def test_truncated_plan_gaussian_fallback(cuda):
    """Pure gaussian inputs never stop early: every tile exhausts every truncated level and walks
    the whole prefix level by level, in the two-pass and the fused variant (whose tiles save
    their state at a level boundary like pass-2's)."""
    import paper_2602_22575_b200 as s2o
    torch = cuda
    torch.manual_seed(0)
    q = torch.randn(1, 2, 4096, 128, device="cuda").to(torch.bfloat16)
    k = torch.randn(1, 1, 4096, 128, device="cuda").to(torch.bfloat16)
    v = torch.randn(1, 1, 4096, 128, device="cuda").to(torch.bfloat16)
    full = s2o.s2o_attention(q, k, v, s2o.KernelConfig(seg_len=512, tau=0.005))
    res = s2o.s2o_attention(q, k, v, s2o.KernelConfig(seg_len=512, tau=0.005, plan_depth=256), want_plan=False)
    torch.cuda.synchronize()
    assert torch.equal(res.trace.processed, full.trace.processed)
    d = (res.out.float() - full.out.float()).abs()
    excess = (d - (1e-2 * full.out.float().abs() + 1e-3)).max().item()
    assert excess <= 0 and d.mean().item() <= 1e-4, (d.max().item(), d.mean().item())
    fcfg = s2o.KernelConfig(seg_len=512, tau=0.005, q_reorder=False, fused=True)
    ffull = s2o.s2o_attention(q, k, v, fcfg)
    fcfg.plan_depth = 256
    fres = s2o.s2o_attention(q, k, v, fcfg, want_plan=False)
    torch.cuda.synchronize()
    assert torch.equal(fres.trace.processed, ffull.trace.processed)
    assert torch.equal(fres.trace.pass2_pairs, ffull.trace.pass2_pairs)
    d = (fres.out.float() - ffull.out.float()).abs()
    excess = (d - (1e-2 * ffull.out.float().abs() + 1e-3)).max().item()
    assert excess <= 0 and d.mean().item() <= 1e-4, (d.max().item(), d.mean().item())


@pytest.mark.parametrize("z,hq,hkv,pinned", [(2, 4, 2, True), (1, 8, 4, False), (1, 2, 1, True)])
def test_host_pipelined_equals_device(cuda, z, hq, hkv, pinned):
    """s2o_attention_host pipelines (batch, kv head) chunks over copy-in / compute / copy-out
    streams; the result must equal the one-shot device call bit for bit (same kernels, same
    per-head work), for pinned and pageable host buffers and Z > 1."""
    import paper_2602_22575_b200 as s2o
    torch = cuda
    l = 4096
    q, k, v = s2o.generate_synthetic("mixed", l // 64, 8.0, 4, z, hq, l, 128)
    qd = torch.from_numpy(q).cuda().to(torch.bfloat16)
    kd = torch.from_numpy(k[:, :hkv].copy()).cuda().to(torch.bfloat16)
    vd = torch.from_numpy(v[:, :hkv].copy()).cuda().to(torch.bfloat16)
    cfg = s2o.KernelConfig(seg_len=512, tau=0.005)
    want = s2o.s2o_attention(qd, kd, vd, cfg, want_plan=False).out
    torch.cuda.synchronize()
    qh, kh, vh = qd.cpu(), kd.cpu(), vd.cpu()
    oh = torch.empty_like(qh)
    if pinned:
        qh, kh, vh, oh = qh.pin_memory(), kh.pin_memory(), vh.pin_memory(), oh.pin_memory()
    s2o.attention_host_ptr(qh, kh, vh, oh, cfg)
    assert torch.equal(oh, want.cpu())


_PASS1_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2602_22575_b200 as s2o
hq, hkv, l, s = (int(x) for x in sys.argv[3:7])
q, k, v = s2o.generate_synthetic("mixed", l // 64, 8.0, 5, 1, hq, l, 128)
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16)
cfg = s2o.KernelConfig(seg_len=s, tau=0.005, tiles=s2o.TileSpec(128, 128), path=2)
b = s2o.pass1_dense_init(dev(q), dev(k[:, :hkv]), dev(v[:, :hkv]), cfg)
torch.cuda.synchronize()
np.savez(sys.argv[2], acc=b.acc.cpu().numpy(), ell=b.ell.cpu().numpy(), m=b.m.cpu().numpy())
"""


@pytest.mark.parametrize("var,hq,hkv,l,seg", [
    ("S2O_DIAG_KERNEL=0", 4, 2, 3000, 700),  # the pair kernel
    ("S2O_DIAG2=0", 4, 2, 3000, 700),        # the single-tile kernel vs the two-tile default:
    ("S2O_DIAG2=0", 8, 1, 5000, 2048),       #   q heads 2i, 2i+1 of a group,
    ("S2O_DIAG2=0", 6, 2, 3000, 700),        #   odd group: adjacent tiles of one head
    ("S2O_DIAG2=0", 3, 3, 4200, 1000)])
def test_diag_kernel_equals_variant(cuda, tmp_path, var, hq, hkv, l, seg):
    """Pass-1 on the default diagonal kernel (two tiles per item) and on a variant kernel (env
    flag, read once per process, hence the subprocesses): the same state up to fp32 summation
    order (ragged segments, GQA groups even, odd and 1)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    name, val = var.split("=")
    out = {}
    for tag, extra in (("base", {}), ("var", {name: val})):
        f = str(tmp_path / f"p1_{tag}.npz")
        env = dict(os.environ, **extra)
        subprocess.run([sys.executable, "-c", _PASS1_SCRIPT, root, f, str(hq), str(hkv), str(l), str(seg)],
                       check=True, env=env, timeout=600)
        out[tag] = np.load(f)
    a, b = out["base"], out["var"]
    # invariant under the lazy reference: O = acc / ell and ell * e^m
    oa = a["acc"] / a["ell"][..., None]
    ob = b["acc"] / b["ell"][..., None]
    assert np.isfinite(ob).all()
    assert np.abs(oa - ob).max() <= 2e-2 and np.abs(oa - ob).mean() <= 1e-3
    np.testing.assert_allclose(a["ell"] * np.exp(a["m"] - b["m"]), b["ell"], rtol=2e-3)


def test_diag_dense_ragged_gqa_vs_sdpa(cuda):
    """The dense reference (one segment = L) on the diagonal kernel with a ragged last tile."""
    import paper_2602_22575_b200 as s2o
    torch = cuda
    torch.manual_seed(1)
    q = torch.randn(1, 8, 3000, 128, device="cuda").to(torch.bfloat16)
    k = torch.randn(1, 2, 3000, 128, device="cuda").to(torch.bfloat16)
    v = torch.randn(1, 2, 3000, 128, device="cuda").to(torch.bfloat16)
    o = s2o.dense_causal_attention(q, k, v, path=TC)
    ref = torch.nn.functional.scaled_dot_product_attention(
        q.float(), k.float().repeat_interleave(4, 1), v.float().repeat_interleave(4, 1), is_causal=True)
    assert (o.float() - ref).abs().max().item() <= 2e-2


def test_tc_pass1_states_short_tiles(cuda, port):
    """Segments of one tile (S = 128: every tile has a single block), many heads: the diagonal
    kernel's softmax finishes tiles back to back, ahead of the epilogue; the per-row (m, ell)
    hand-off must still reach the right tile (ml_free ordering)."""
    import paper_2602_22575_b200 as s2o
    torch = cuda
    q, k, v = inputs(s2o, 8, 8, 4096, seed=7)
    c = Cfg(128, 0.005, 128, 128)
    bufs = s2o.pass1_dense_init(dev_bf16(torch, q), dev_bf16(torch, k), dev_bf16(torch, v), kcfg(s2o, c, TC))
    acc, ell, m = port.pass1(q, k, v, c)
    got = (bufs.acc / bufs.ell[..., None]).cpu().numpy()
    assert np.abs(got - acc / ell[..., None]).max() <= 2e-2
    mg = bufs.m.cpu().numpy().astype(np.float64)
    assert (mg <= m + 1e-3).all() and (mg >= m - 8.0 * np.log(2.0) - 1e-3).all()
    np.testing.assert_allclose(bufs.ell.cpu().numpy() * np.exp(mg - m), ell, rtol=2e-3)


@pytest.mark.parametrize("depth", [0, 128])
def test_cuda_graph_capture_and_replay(cuda, depth):
    """s2o_attention_fwd is stream-ordered (no host synchronisation, the plan-level loop is a graph
    WHILE node): captured into a CUDA graph and replayed it reproduces the eager call bit for bit,
    also when tiles overflow a tiny truncated plan (depth 128 -> several device-side levels)."""
    import paper_2602_22575_b200 as s2o
    torch = cuda
    q, k, v = inputs(s2o, 4, 2, 4096, seed=5)
    qd, kd, vd = dev_bf16(torch, q), dev_bf16(torch, k), dev_bf16(torch, v)
    cfg = s2o.KernelConfig(seg_len=512, tau=0.005, plan_depth=depth)
    eager = s2o.s2o_attention(qd, kd, vd, cfg, want_plan=False)
    torch.cuda.synchronize()
    out = torch.empty_like(qd)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        s2o.s2o_attention(qd, kd, vd, cfg, out=out, want_plan=False, check=False)  # warm-up (workspace)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        res = s2o.s2o_attention(qd, kd, vd, cfg, out=out, want_plan=False, check=False)
    out.zero_()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, eager.out)
    assert torch.equal(res.trace.processed, eager.trace.processed)
    assert torch.equal(res.trace.pass2_pairs, eager.trace.pass2_pairs)
    out.zero_()
    graph.replay()  # replays are repeatable (level state re-initialised inside the graph)
    torch.cuda.synchronize()
    assert torch.equal(out, eager.out)
