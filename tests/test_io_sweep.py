"""S2OT tensor files and the sweep report format against the compiled reference (SURVEY.md §8f
rank 2): tensor_io.cpp:32-83, sweep.cpp:66-302. CPU tests use the reference lib as the checker;
the GPU test runs a small sweep end to end on the device."""
import json
import struct

import numpy as np
import pytest

from paper_2602_22575_b200.io import load_tensor_file, load_trio, save_tensor_file
from paper_2602_22575_b200 import sweep as sw


@pytest.fixture(scope="module")
def ref():
    from oracle.oracle import Ref, build

    build()
    return Ref()


def test_s2ot_roundtrip_and_reference_bytes(tmp_path, ref):
    rng = np.random.default_rng(0)
    x = rng.standard_normal((2, 3, 5, 7)).astype(np.float32)
    ours, theirs = tmp_path / "ours.s2ot", tmp_path / "theirs.s2ot"
    save_tensor_file(x, ours)
    ref.save_tensor(str(theirs), x)
    assert ours.read_bytes() == theirs.read_bytes()  # byte-identical writers
    assert np.array_equal(load_tensor_file(theirs), x)
    assert np.array_equal(ref.load_tensor(str(ours)), x)
    hdr = ours.read_bytes()[:24]
    assert struct.unpack("<4s5I", hdr) == (b"S2OT", 1, 2, 3, 5, 7)


@pytest.mark.parametrize("mutate,msg", [
    (lambda b: b"XXXX" + b[4:], "not an S2OT file"),
    (lambda b: b[:4] + struct.pack("<I", 2) + b[8:], "unsupported version"),
    (lambda b: b[:-4], "size mismatch"),
    (lambda b: b + b"\0", "size mismatch"),
    (lambda b: b[:8] + struct.pack("<I", 0) + b[12:], "size mismatch"),
    (lambda b: b[:2], "not an S2OT file"),
])
def test_s2ot_errors_match_reference(tmp_path, ref, mutate, msg):
    good = tmp_path / "good.s2ot"
    save_tensor_file(np.ones((1, 1, 4, 2), np.float32), good)
    bad = tmp_path / "bad.s2ot"
    bad.write_bytes(mutate(good.read_bytes()))
    with pytest.raises(RuntimeError, match=msg):
        load_tensor_file(bad)
    from oracle.oracle import OracleError

    with pytest.raises(OracleError) as e:
        ref.load_tensor(str(bad))
    assert e.value.msg == msg


def test_s2ot_open_errors(tmp_path):
    missing = tmp_path / "nope.s2ot"
    with pytest.raises(RuntimeError, match="cannot open: "):
        load_tensor_file(missing)
    with pytest.raises(RuntimeError, match="cannot open for writing: "):
        save_tensor_file(np.ones((1, 1, 1, 1)), tmp_path / "no_dir" / "x.s2ot")


def test_trio_dims(tmp_path):
    save_tensor_file(np.ones((1, 2, 4, 2)), tmp_path / "t.q.s2ot")
    save_tensor_file(np.ones((1, 2, 4, 2)), tmp_path / "t.k.s2ot")
    save_tensor_file(np.ones((1, 1, 4, 2)), tmp_path / "t.v.s2ot")
    with pytest.raises(RuntimeError, match="input tensor trio has mismatched dims"):
        load_trio(tmp_path / "t")


GRID = dict(pattern="mixed", stripe_count=4, gain=8.0, seed=0, dims=(1, 2, 256, 32),
            variants=["two-pass", "fused", "no-q-reorder", "baseline-topk"], seg_lens=[64, 128],
            taus=[0.005, 0.02], tiles=(16, 16), topk=[1, 3], block=(16, 16))


def _ref_sweep(ref, tmp_path, **over):
    g = dict(GRID, **over)
    base = str(tmp_path / "ref")
    ref.run_sweep(g["pattern"], g["stripe_count"], g["gain"], g["seed"], g["dims"], g["variants"], g["seg_lens"],
                  g["taus"], g["tiles"], g["topk"], g["block"], True, base)
    return base


def _cfg(out_base, **over):
    g = dict(GRID, **over)
    z, h, l, d = g["dims"]
    return sw.RunConfig(synthetic=sw.SyntheticSpec(g["pattern"], g["stripe_count"], g["gain"], g["seed"]),
                        z=z, h=h, l=l, d=d, variants=list(g["variants"]), seg_lens=list(g["seg_lens"]),
                        taus=list(g["taus"]), tiles=tuple(g["tiles"]), topk=list(g["topk"]),
                        block_shape=tuple(g["block"]), dump_plan=True, out_base=out_base)


class _Replay:
    """A runner that replays the reference's own points: our writer must then reproduce its files."""

    def __init__(self, doc):
        self.points = list(doc["points"])
        self.plan = doc.get("plan")

    def _next(self):
        p = self.points.pop(0)
        return p["report"], p["seconds"]

    def kernel_point(self, variant, seg, tau):
        report, secs = self._next()
        return report, secs, None

    def baseline_point(self, k):
        return self._next()


def test_sweep_files_match_reference_format(tmp_path, ref):
    base = _ref_sweep(ref, tmp_path)
    doc = json.load(open(base + ".json"))
    ours = str(tmp_path / "ours")
    res = sw.run_sweep(_cfg(ours), runner_factory=lambda cfg: _Replay(doc))
    assert not res.partial, res.error
    # CSV: byte-identical (same numbers in, %.17g formatting, empty columns)
    assert open(ours + ".csv").read() == open(base + ".csv").read()
    mine = json.load(open(ours + ".json"))
    assert "plan" in doc and "plan" not in mine  # the replay runner has no plan to dump
    doc.pop("plan")
    assert mine == doc  # same keys, values, NaN -> null for baseline taus


def test_sweep_partial_on_error(tmp_path):
    class Boom:
        def kernel_point(self, *a):
            raise RuntimeError("uncovered query row")

    out = str(tmp_path / "p")
    res = sw.run_sweep(_cfg(out, variants=["two-pass"]), runner_factory=lambda cfg: Boom())
    assert res.partial and res.error == "uncovered query row"
    doc = json.load(open(out + ".json"))
    assert doc["partial"] is True and doc["error"] == "uncovered query row" and doc["points"] == []
    assert open(out + ".csv").read() == sw.CSV_HEADER + "\n"


def test_sweep_config_errors(tmp_path):
    with pytest.raises(ValueError, match="sweep grids must be non-empty"):
        sw.run_sweep(_cfg(str(tmp_path / "e"), taus=[]))
    with pytest.raises(ValueError, match="unknown variant: warp"):
        sw.run_sweep(_cfg(str(tmp_path / "e"), variants=["warp"]))


@pytest.mark.gpu
def test_device_sweep_matches_reference(tmp_path, ref):
    """The same grid on the device (fp32 inputs: the exact generic path): identical plans, traces
    and pair counts; MSE / MAE equal to the reference's to fp32-output rounding."""
    kernel_variants = ["two-pass", "fused", "no-q-reorder"]
    base = _ref_sweep(ref, tmp_path, variants=kernel_variants)
    doc = json.load(open(base + ".json"))
    ours = str(tmp_path / "dev")
    res = sw.run_sweep(_cfg(ours, variants=kernel_variants))
    assert not res.partial, res.error
    mine = json.load(open(ours + ".json"))
    assert mine["config"] == doc["config"]
    assert mine["plan"] == doc["plan"]
    assert len(mine["points"]) == len(doc["points"]) == 12
    for a, b in zip(mine["points"], doc["points"]):
        assert (a["variant"], a["S"], a["tau"], a["tiles"]) == (b["variant"], b["S"], b["tau"], b["tiles"])
        assert a["report"]["ranking_cost"] == b["report"]["ranking_cost"]
        for ha, hb in zip(a["report"]["per_head"], b["report"]["per_head"]):
            assert (ha["z"], ha["h"], ha["computed_pairs"], ha["total_causal_pairs"], ha["sparsity"]) == \
                (hb["z"], hb["h"], hb["computed_pairs"], hb["total_causal_pairs"], hb["sparsity"])
            assert ha["mse"] == pytest.approx(hb["mse"], rel=2e-3, abs=1e-12)
            assert ha["mae"] == pytest.approx(hb["mae"], rel=2e-3, abs=1e-9)
    rows = open(ours + ".csv").read().splitlines()
    assert rows[0] == sw.CSV_HEADER and len(rows) == 13
    assert [r.split(",")[:3] for r in rows[1:]] == [r.split(",")[:3] for r in open(base + ".csv").read().splitlines()[1:]]


# ------------------------------------------------------------------ block top-k baseline (§8f rank 3)
def test_block_topk_budget_errors():
    """The C-ABI validates the budget before touching device memory (no GPU needed)."""
    import ctypes as C

    from paper_2602_22575_b200 import s2o as ops

    p = ops._Problem()
    ops.lib().s2o_problem_init(C.byref(p), C.c_int64(1), C.c_int64(1), C.c_int64(1), C.c_int64(64),
                               C.c_int64(16), C.c_int32(ops.S2O_F32), C.c_int32(ops.S2O_F32))
    nbytes = C.c_size_t(0)
    for rows, cols, k in ((16, 16, -1), (0, 16, 1), (16, 0, 1)):
        rc = ops.lib().s2o_block_topk_workspace_size(C.byref(p), C.c_int64(rows), C.c_int64(cols), C.c_int64(k),
                                                     C.byref(nbytes))
        assert rc == 19
        assert ops.lib().s2o_last_error().decode() == "block budget must have positive shape and k >= 0"
    rc = ops.lib().s2o_block_topk_workspace_size(C.byref(p), C.c_int64(16), C.c_int64(8), C.c_int64(1),
                                                 C.byref(nbytes))
    assert rc == 15  # unsupported: square blocks only
    assert ops.lib().s2o_block_topk_workspace_size(C.byref(p), C.c_int64(16), C.c_int64(16), C.c_int64(2),
                                                   C.byref(nbytes)) == 0 and nbytes.value > 0


@pytest.mark.gpu
@pytest.mark.parametrize("topk", [0, 1, 3, 100])
def test_block_topk_matches_reference_fp32(ref, topk):
    """fp32 inputs (exact fp64 generic path): identical pair counts, outputs to fp32 rounding."""
    import torch

    import paper_2602_22575_b200 as s2o

    q, k, v = ref.generate_synthetic("mixed", 4, 8.0, 3, 1, 2, 256, 32)
    want, want_pairs = ref.block_topk(q, k, v, 16, 16, topk)
    dq, dk, dv = (torch.from_numpy(x).cuda() for x in (q, k, v))
    got, pairs = s2o.block_topk_attention(dq, dk, dv, 16, 16, topk)
    assert pairs.cpu().numpy().reshape(-1).tolist() == want_pairs.tolist()
    np.testing.assert_allclose(got.cpu().numpy(), want, rtol=0, atol=2e-6)


@pytest.mark.gpu
def test_block_topk_tcgen05_matches_reference(ref):
    """bf16, D = 128, 128-token blocks: the masked attention runs on the tcgen05 path; the
    selection is still exact, so the kept sets (pair counts) equal the reference's on the same
    bf16-rounded inputs; outputs within bf16 tolerance."""
    import torch

    import paper_2602_22575_b200 as s2o

    q, k, v = ref.generate_synthetic("mixed", 16, 8.0, 1, 1, 2, 1024, 128)
    dq, dk, dv = (torch.from_numpy(x).cuda().to(torch.bfloat16) for x in (q, k, v))
    qr, kr, vr = (x.float().cpu().numpy() for x in (dq, dk, dv))
    want, want_pairs = ref.block_topk(qr, kr, vr, 128, 128, 2)
    got, pairs = s2o.block_topk_attention(dq, dk, dv, 128, 128, 2, path=s2o.PATH_TCGEN05)
    assert pairs.cpu().numpy().reshape(-1).tolist() == want_pairs.tolist()
    err = np.abs(got.float().cpu().numpy() - want)
    assert err.max() <= 2e-2 and err.mean() <= 2e-3


@pytest.mark.gpu
def test_device_sweep_baseline_matches_reference(tmp_path, ref):
    base = _ref_sweep(ref, tmp_path, variants=["baseline-topk"], topk=[0, 1, 3])
    doc = json.load(open(base + ".json"))
    ours = str(tmp_path / "devb")
    res = sw.run_sweep(_cfg(ours, variants=["baseline-topk"], topk=[0, 1, 3]))
    assert not res.partial, res.error
    mine = json.load(open(ours + ".json"))
    assert mine["config"] == doc["config"] and len(mine["points"]) == 3
    for a, b in zip(mine["points"], doc["points"]):
        assert a["k"] == b["k"] and a["report"]["ranking_cost"] == b["report"]["ranking_cost"]
        for ha, hb in zip(a["report"]["per_head"], b["report"]["per_head"]):
            assert ha["computed_pairs"] == hb["computed_pairs"] and ha["sparsity"] == hb["sparsity"]
            assert ha["mse"] == pytest.approx(hb["mse"], rel=2e-3, abs=1e-12)


@pytest.mark.gpu
def test_block_topk_ragged_gqa(ref):
    """L not a multiple of the block (ragged last block) and GQA (K/V expanded for the reference)."""
    import torch

    import paper_2602_22575_b200 as s2o

    q, k, v = ref.generate_synthetic("mixed", 3, 8.0, 7, 2, 4, 200, 16)
    kk, vv = k[:, ::2].copy(), v[:, ::2].copy()  # hkv = 2: q head h reads kv head h // 2
    want, want_pairs = ref.block_topk(q, np.repeat(kk, 2, axis=1), np.repeat(vv, 2, axis=1), 16, 16, 2)
    dq, dk, dv = (torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (q, kk, vv))
    got, pairs = s2o.block_topk_attention(dq, dk, dv, 16, 16, 2)
    assert pairs.cpu().numpy().reshape(-1).tolist() == want_pairs.tolist()
    np.testing.assert_allclose(got.cpu().numpy(), want, rtol=0, atol=2e-6)


@pytest.mark.gpu
def test_sweep_from_s2ot_trio_equals_synthetic(tmp_path):
    """The file input source (<base>.{q,k,v}.s2ot) gives the same report as the generator."""
    import paper_2602_22575_b200 as s2o

    q, k, v = s2o.generate_synthetic("mixed", 4, 8.0, 0, 1, 2, 256, 32)
    base = str(tmp_path / "in")
    for name, x in (("q", q), ("k", k), ("v", v)):
        save_tensor_file(x, f"{base}.{name}.s2ot")
    grid = dict(variants=["two-pass", "baseline-topk"], taus=[0.02], seg_lens=[64], topk=[2])
    syn = sw.run_sweep(_cfg(str(tmp_path / "syn"), **grid))
    cfg = _cfg(str(tmp_path / "file"), **grid)
    cfg.synthetic, cfg.input_base = None, base
    fil = sw.run_sweep(cfg)
    assert not syn.partial and not fil.partial, (syn.error, fil.error)
    a, b = json.load(open(syn.json_path)), json.load(open(fil.json_path))
    assert b["config"]["input"] == base
    for pa, pb in zip(a["points"], b["points"]):
        assert pa["report"] == pb["report"]
