"""Benchmark sweep with the reference's report format (sweep.cpp:66-302, sweep.hpp:28-64).

`run_sweep(cfg)` runs the dense reference once and then every grid point (variant x S x tau,
or baseline-topk x k) on the GPU, and writes <out_base>.json and <out_base>.csv with the same
schema, key order and number formatting as the reference's run_sweep, so GPU results drop into
its report pipeline:

* CSV header ``variant,S,tau,k,sparsity,mse,mae,pairs,dot_products,seconds``; floats as %.17g;
  kernel points leave ``k`` empty, baseline points leave ``S``, ``tau`` and ``dot_products``.
* JSON ``{"config", "points": [{"variant", "S", "tau" | "k", "tiles", "report", "seconds"}],
  "partial", ["error"], ["plan"]}`` with nlohmann's key order (sorted), NaN as null and a
  two-space indent; ``report`` = make_sparsity_report (metrics.cpp:59-90).

Inputs: exactly one of an S2OT trio (<base>.{q,k,v}.s2ot, io.py) or the synthetic generator.
The dense reference is the device's exact fp64 generic path (dense_causal_attention), the
kernels run on the device (fp32 inputs take the fp64 generic path like the reference's numerics;
``dtype="bf16"`` rounds the inputs to bf16 and runs the tcgen05 path). ``seconds`` is the median
of three timed calls after a warm-up, synchronised wall clock around the whole operator, as in
sweep.cpp:252-258. A failing point stops the sweep, marks the report partial and records the
error; run_sweep returns (callers exit nonzero).
"""
from __future__ import annotations

import json
import math
import time
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

VARIANTS = ("two-pass", "fused", "no-q-reorder", "baseline-topk")
CSV_HEADER = "variant,S,tau,k,sparsity,mse,mae,pairs,dot_products,seconds"


@dataclass
class SyntheticSpec:
    """SyntheticSpec (synthetic.hpp:27-32)."""
    pattern: str = "gaussian"
    stripe_count: int = 0
    stripe_gain: float = 0.0
    seed: int = 0


@dataclass
class RunConfig:
    """RunConfig (sweep.hpp:28-46); `dtype` selects the device compute precision."""
    input_base: Optional[str] = None
    synthetic: Optional[SyntheticSpec] = None
    z: int = 1
    h: int = 1
    l: int = 256
    d: int = 32
    variants: list = field(default_factory=lambda: ["two-pass"])
    seg_lens: list = field(default_factory=lambda: [128])
    taus: list = field(default_factory=lambda: [0.005])
    tiles: tuple = (16, 16)
    topk: list = field(default_factory=list)
    block_shape: tuple = (16, 16)
    dump_plan: bool = False
    out_base: str = "s2o_report"
    dtype: str = "fp32"


@dataclass
class SweepPoint:
    variant: str
    seg_len: int       # -1 for baseline points
    tau: float         # NaN for baseline points
    k: int             # -1 for kernel points
    report: dict
    seconds: float


@dataclass
class SweepResult:
    points: list = field(default_factory=list)
    partial: bool = False
    error: str = ""
    json_path: str = ""
    csv_path: str = ""


def parse_variant(name: str) -> str:
    if name not in VARIANTS:
        raise ValueError("unknown variant: " + name)
    return name


def fmt_double(v: float) -> str:
    """%.17g, sweep.cpp:60-64 (nan / inf spelled like glibc's printf)."""
    return "%.17g" % v


def median3(a: float, b: float, c: float) -> float:
    return max(min(a, b), min(max(a, b), c))


def _jsonable(x):
    """nlohmann writes NaN / inf as null."""
    if isinstance(x, float) and not math.isfinite(x):
        return None
    if isinstance(x, dict):
        return {k: _jsonable(v) for k, v in x.items()}
    if isinstance(x, list):
        return [_jsonable(v) for v in x]
    return x


def dump_json(obj) -> str:
    return json.dumps(_jsonable(obj), indent=2, sort_keys=True, allow_nan=False)


def make_sparsity_report(errors, sparsity, dots: int, sort_items: int) -> dict:
    """make_sparsity_report (metrics.cpp:59-90) as report_json (sweep.cpp:66-84).

    errors: [(z, h, mse, mae)], sparsity: [(z, h, computed_pairs, total_causal_pairs)]."""
    if len(errors) != len(sparsity) or not errors:
        raise ValueError("error and sparsity head lists must align")
    heads = []
    s_mse = s_mae = s_sp = 0.0
    for (z, h, mse, mae), (z2, h2, pairs, total) in zip(errors, sparsity):
        if (z, h) != (z2, h2):
            raise ValueError("error and sparsity head order must align")
        sp = 1.0 - float(pairs) / float(total)
        heads.append({"z": int(z), "h": int(h), "mse": float(mse), "mae": float(mae),
                      "computed_pairs": int(pairs), "total_causal_pairs": int(total), "sparsity": sp})
        s_mse += float(mse)
        s_mae += float(mae)
        s_sp += sp
    inv = 1.0 / len(heads)
    return {"per_head": heads,
            "aggregate": {"mean_mse": s_mse * inv, "mean_mae": s_mae * inv, "mean_sparsity": s_sp * inv},
            "ranking_cost": {"dot_products": int(dots), "sort_items": int(sort_items)}}


def config_json(cfg: RunConfig) -> dict:
    """config_json (sweep.cpp:102-127)."""
    j = {}
    if cfg.input_base is not None:
        j["input"] = cfg.input_base
    else:
        s = cfg.synthetic
        j["synthetic"] = {"pattern": s.pattern, "stripe_count": int(s.stripe_count),
                          "stripe_gain": float(s.stripe_gain), "seed": int(s.seed),
                          "dims": [cfg.z, cfg.h, cfg.l, cfg.d]}
    j["variants"] = list(cfg.variants)
    j["segment_lens"] = [int(x) for x in cfg.seg_lens]
    j["taus"] = [float(x) for x in cfg.taus]
    j["tiles"] = [int(cfg.tiles[0]), int(cfg.tiles[1])]
    if cfg.topk:
        j["topk"] = [int(x) for x in cfg.topk]
        j["block"] = [int(cfg.block_shape[0]), int(cfg.block_shape[1])]
    return j


def csv_row(point: SweepPoint) -> str:
    """One CSV line (sweep.cpp:189-200)."""
    r = point.report
    pairs = sum(e["computed_pairs"] for e in r["per_head"])
    agg = r["aggregate"]
    if point.variant != "baseline-topk":
        head = f"{point.variant},{point.seg_len},{fmt_double(point.tau)},,"
        dots = str(r["ranking_cost"]["dot_products"])
    else:
        head = f"{point.variant},,,{point.k},"
        dots = ""
    return (head + f"{fmt_double(agg['mean_sparsity'])},{fmt_double(agg['mean_mse'])},"
            f"{fmt_double(agg['mean_mae'])},{pairs},{dots},{fmt_double(point.seconds)}")


def point_json(point: SweepPoint, tiles) -> dict:
    pj = {"variant": point.variant}
    if point.variant != "baseline-topk":
        pj["S"] = int(point.seg_len)
        pj["tau"] = float(point.tau)
    else:
        pj["k"] = int(point.k)
    pj["tiles"] = [int(tiles[0]), int(tiles[1])]
    pj["report"] = point.report
    pj["seconds"] = float(point.seconds)
    return pj


def plan_json(plan_segments) -> dict:
    """plan_json (sweep.cpp:86-100) from [(z, h, n, q_perm list, kv_perm list)]."""
    return {"guide_source": "k_mean[segment 0]",
            "segments": [{"z": z, "h": h, "segment": n, "q_perm": qp, "kv_perm": kv}
                         for z, h, n, qp, kv in plan_segments]}


# ----------------------------------------------------------------------------- device runner
class DeviceRunner:
    """Runs the grid points on the GPU through the product (libs2o_cuda.so)."""

    def __init__(self, cfg: RunConfig):
        import torch

        from . import s2o as ops
        from .io import load_trio

        self.torch, self.ops, self.cfg = torch, ops, cfg
        if (cfg.input_base is None) == (cfg.synthetic is None):
            raise ValueError("exactly one input source required (file or synthetic)")
        if cfg.input_base is not None:
            q, k, v = load_trio(cfg.input_base)
        else:
            s = cfg.synthetic
            q, k, v = ops.generate_synthetic(s.pattern, s.stripe_count, s.stripe_gain, s.seed, cfg.z, cfg.h,
                                             cfg.l, cfg.d)
        dev = torch.device("cuda")
        self.q32, self.k32, self.v32 = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (q, k, v))
        if cfg.dtype == "bf16":
            self.q, self.k, self.v = (x.to(torch.bfloat16) for x in (self.q32, self.k32, self.v32))
        elif cfg.dtype == "fp32":
            self.q, self.k, self.v = self.q32, self.k32, self.v32
        else:
            raise ValueError("dtype must be fp32 or bf16")
        self.z, self.h, self.l = self.q.shape[0], self.q.shape[1], self.q.shape[2]
        # dense reference: exact fp64 accumulation on the same (possibly bf16-rounded) values
        self.ref = ops.dense_causal_attention(self.q.float(), self.k.float(), self.v.float(),
                                              ops.S2O_F32, ops.PATH_GENERIC).double()

    def _errors(self, out):
        diff = out.double() - self.ref
        n = float(diff.shape[2] * diff.shape[3])
        mse = (diff * diff).sum(dim=(2, 3)) / n
        mae = diff.abs().sum(dim=(2, 3)) / n
        mse, mae = mse.cpu().numpy(), mae.cpu().numpy()
        return [(z, h, float(mse[z, h]), float(mae[z, h])) for z in range(self.z) for h in range(self.h)]

    def _timed(self, fn):
        torch = self.torch
        res = fn()  # warm-up
        times = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = fn()
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
        return res, median3(*times)

    def kernel_point(self, variant: str, seg: int, tau: float):
        ops, cfg = self.ops, self.cfg
        kc = ops.KernelConfig(seg_len=int(seg), tau=float(tau), tiles=ops.TileSpec(*cfg.tiles),
                              q_reorder=variant == "two-pass", fused=variant == "fused")
        kc.validate(self.l)
        res, secs = self._timed(lambda: ops.s2o_attention(self.q, self.k, self.v, kc, want_plan=cfg.dump_plan))
        total = self.l * (self.l + 1) // 2
        p1 = res.trace.pass1_pairs.cpu().numpy().reshape(self.z, self.h)
        p2 = res.trace.pass2_pairs.cpu().numpy().reshape(self.z, self.h)
        sp = [(z, h, int(p1[z, h]) + int(p2[z, h]), total) for z in range(self.z) for h in range(self.h)]
        report = make_sparsity_report(self._errors(res.out), sp, res.cost.dot_products, res.cost.sort_items)
        return report, secs, res.plan

    def plan_segments(self, plan):
        seg = plan.seg
        qp = plan.q_perm.cpu().numpy()
        kv = plan.kv_perm.cpu().numpy()
        out = []
        for z in range(plan.z):
            for h in range(plan.h):
                for n in range(seg.seg_count):
                    rows = seg.seg_len if n + 1 < seg.seg_count else seg.last_len
                    off = seg.seg_len * n * (n - 1) // 2
                    out.append((z, h, n, qp[z, h, n, :rows].tolist(), kv[z, h, off:off + n * seg.seg_len].tolist()))
        return out

    def baseline_point(self, k: int):
        """One baseline-topk point (sweep.cpp:210-246): block_topk_attention, median of 3."""
        ops, cfg = self.ops, self.cfg
        rows, cols = cfg.block_shape
        (out, pairs), secs = self._timed(lambda: ops.block_topk_attention(self.q, self.k, self.v, rows, cols, k))
        total = self.l * (self.l + 1) // 2
        pc = pairs.cpu().numpy().reshape(self.z, self.h)
        sp = [(z, h, int(pc[z, h]), total) for z in range(self.z) for h in range(self.h)]
        return make_sparsity_report(self._errors(out), sp, 0, 0), secs


def run_sweep(cfg: RunConfig, runner_factory: Callable[[RunConfig], object] = DeviceRunner) -> SweepResult:
    """run_sweep (sweep.cpp:141-302). `runner_factory` is injectable for host-only tests."""
    if not cfg.variants or not cfg.seg_lens or not cfg.taus:
        raise ValueError("sweep grids must be non-empty")
    for v in cfg.variants:
        parse_variant(v)
    result = SweepResult(json_path=cfg.out_base + ".json", csv_path=cfg.out_base + ".csv")
    root = {"config": config_json(cfg), "points": [], "partial": False}
    try:
        csv = open(result.csv_path, "w")
    except OSError:
        raise RuntimeError("cannot open for writing: " + result.csv_path) from None

    def flush_json(err: str) -> None:
        if err:
            root["partial"] = True
            root["error"] = err
        with open(result.json_path, "w") as f:
            f.write(dump_json(root) + "\n")

    with csv:
        csv.write(CSV_HEADER + "\n")
        try:
            runner = runner_factory(cfg)

            def emit(point: SweepPoint) -> None:
                result.points.append(point)
                root["points"].append(point_json(point, cfg.tiles))
                csv.write(csv_row(point) + "\n")
                csv.flush()

            for variant in cfg.variants:
                if variant == "baseline-topk":
                    if not cfg.topk:
                        raise ValueError("baseline-topk variant needs a k grid")
                    for k in cfg.topk:
                        report, secs = runner.baseline_point(int(k))
                        emit(SweepPoint(variant, -1, float("nan"), int(k), report, secs))
                    continue
                for seg in cfg.seg_lens:
                    for tau in cfg.taus:
                        report, secs, plan = runner.kernel_point(variant, int(seg), float(tau))
                        emit(SweepPoint(variant, int(seg), float(tau), -1, report, secs))
                        if cfg.dump_plan and "plan" not in root and plan is not None and plan.q_perm is not None:
                            root["plan"] = plan_json(runner.plan_segments(plan))
        except Exception as e:  # noqa: BLE001 -- the reference records any failure and stops
            result.partial = True
            result.error = str(e)
            flush_json(str(e))
            return result
    flush_json("")
    return result
