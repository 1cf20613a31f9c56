"""bench.py -- S2O sparse prefill attention on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[2]): one Llama-3.1-8B attention layer,
32 q heads / 8 kv heads (GQA), d=128, bf16, L=131072, S=2048, tiles 128x128, tau=0.005, on
the reference's stripe-structured synthetic input (generate_synthetic mixed, L/64 stripes,
gain 8, seed = layer = rank). A step = the whole operator: plan (block scoring +
permutation build) + pass-1 + pass-2 for all 32 heads.

Multi-GPU: every rank runs its own layer (seed = rank) with no
collective on the data path; `value` = max-over-ranks step time / N = ms per layer of the
whole job ("scaling": "weak").

Timing: W warm-up steps, then K steps bracketed by barrier + synchronize, CUDA events on the
launching stream; inputs (1.6 GB) exceed L2 (126 MB). `e2e` runs the same operator through
the host-buffer C-ABI entry point (s2o_attention_host) from pinned host memory, H2D of Q/K/V
and D2H of O inside the timed region. `cpu_baseline` (rank 0, N=1) times the compiled
reference (oracle/_ref) on a bounded prefix sample of the same input and extrapolates by the
algorithmic pair count (see `cpu_baseline.sample`).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HQ, HKV, D = 32, 8, 128
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
METRIC = "S2O prefill attn ms @128K Llama-3.1-8B shape; speedup vs dense; MSE @sparsity"
PAIRS_FILE = os.path.join(ROOT, "profiles", "c3_pairs.json")


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        d["_source"] = "measured"
        return d
    d = dict(PEAKS_FALLBACK)
    d["_source"] = "fallback"
    return d


class ClockSampler:
    """SM clocks + throttle reasons sampled every 5 ms (NVML); started before the warm-up so the
    first (slow) NVML queries are done, and only the samples taken inside the timed region
    (mark_start .. mark_end) are reported."""

    def __init__(self, index: int):
        self.index = index
        self.samples: list[tuple[float, float, int, float]] = []
        self._stop = threading.Event()
        self.ok = False
        self.t0 = None
        self.t1 = None

    def mark_start(self):
        self.t0 = time.perf_counter()

    def mark_end(self):
        self.t1 = time.perf_counter()

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.ok = True
        except Exception:  # noqa: BLE001
            return
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def _run(self):
        n = self.nvml
        while not self._stop.is_set():
            try:
                sm = float(n.nvmlDeviceGetClockInfo(self.h, n.NVML_CLOCK_SM))
                pw = n.nvmlDeviceGetPowerUsage(self.h) / 1000.0
                rs = n.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((sm, pw, rs, time.perf_counter()))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.005)

    def stop(self) -> dict:
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        self._stop.set()
        self.thread.join(timeout=2)
        n = self.nvml
        names = {
            "hw_slowdown": getattr(n, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(n, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(n, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_power_cap": getattr(n, "nvmlClocksEventReasonSwPowerCap", 0x4),
        }
        if self.t0 is not None and self.t1 is not None:
            inside = [x for x in self.samples if self.t0 <= x[3] <= self.t1]
            self.samples = inside or sorted(self.samples, key=lambda x: abs(x[3] - self.t1))[:1]
        reasons = set()
        for _, _, rs, _ in self.samples:
            for name, bit in names.items():
                if rs & bit:
                    reasons.add(name)
        sms = sorted(x[0] for x in self.samples)
        med = sms[len(sms) // 2] if sms else None
        pmax = max((x[1] for x in self.samples), default=None)
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(reasons),
                "samples": len(sms), "power_w_max": pmax}


def make_inputs(torch, s2o, l: int, seed: int, device):
    """Synthetic stripe-structured layer: Q = 32 heads, K/V = heads 0..7 of the same
    generation (== an H=8 generation), rounded to bf16."""
    q, k, v = s2o.generate_synthetic("mixed", l // 64, 8.0, seed, 1, HQ, l, D)
    qd = torch.from_numpy(q).to(device).to(torch.bfloat16)
    kd = torch.from_numpy(k[:, :HKV].copy()).to(device).to(torch.bfloat16)
    vd = torch.from_numpy(v[:, :HKV].copy()).to(device).to(torch.bfloat16)
    del q, k, v
    return qd, kd, vd


def cuda_time(torch, fn, reps: int, stream=None) -> float:
    """Min ms of fn() over reps (after one untimed call that absorbs allocator / first-touch
    effects), CUDA events on the current stream, synchronized around each call."""
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def plan_sort_passes(l: int, s: int) -> int:
    n = -(-l // s)
    max_len = (n - 1) * s
    passes, w = 0, 2048
    while w < max_len:
        passes += 1
        w *= 2
    return passes


def plan_hbm(l: int, s: int, t_ms: float, pk: dict) -> dict:
    """SURVEY.md §8(d) algorithmic preprocessing bytes and the achieved fraction of HBM."""
    n = -(-l // s)
    b_alg = HQ * l * D * 2 + HKV * l * D * 2 + HQ * s * n * (n - 1) // 2 * 4 + HQ * l * 4
    gbs = b_alg / (t_ms * 1e-3) / 1e9
    peak = float(pk.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"]))
    return {"alg_bytes": b_alg, "achieved_gbs": round(gbs, 1), "peak_gbs": peak, "frac": round(gbs / peak, 4),
            "bound": "fp64 (exact scoring) and sort, not HBM"}


def launches_per_step(l: int, s: int) -> int:
    """Our kernels per s2o_attention_fwd call with the truncated plan (no overflow rerun):
    guide means, q ranking (+ q sort when S > 2048), kv scoring, top-T selection (scan + sort
    kernels), trace init, pass-1 (tc_diag_kernel), pass-2 (tc_pass_kernel)."""
    n = -(-l // s)
    count = 2
    if s > 2048:
        count += 2 + plan_sort_passes(l, s)
    if n > 1:
        count += 3
    return count + 3


# ------------------------------------------------------------------ reference (CPU) arm
def reference_sample(l_full: int, s: int, tau: float, seg_sample: int, threads: int):
    """Run the compiled reference on `threads` heads of the first `seg_sample` segments of the
    benchmark input (causality: segments 0..m-1 of the full problem are exactly the problem
    on the first m*S tokens). Returns (seconds, pairs_sample_per_head)."""
    import numpy as np

    import paper_2602_22575_b200 as s2o
    from oracle.oracle import Ref, build

    build()
    ref = Ref()
    lp = min(l_full, seg_sample * s)
    q, k, v = s2o.generate_synthetic("mixed", l_full // 64, 8.0, 0, 1, HQ, l_full, D)
    hs = list(range(threads))
    # bf16-rounded inputs, K/V expanded h -> h/4 (the reference has no GQA)
    def bf(x):
        u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
        return (((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16).astype(np.uint32).view(np.float32)
    qs = bf(q[:, hs, :lp])
    ks = bf(k[:, [h // (HQ // HKV) for h in hs], :lp])
    vs = bf(v[:, [h // (HQ // HKV) for h in hs], :lp])
    del q, k, v

    class Cfg:
        pass
    cfg = Cfg()
    cfg.seg_len, cfg.tau, cfg.b_m, cfg.b_n = s, tau, 128, 128
    cfg.q_reorder, cfg.fused, cfg.local_window = True, False, -1
    os.environ["S2O_THREADS"] = str(threads)
    t0 = time.perf_counter()
    _, tr, _ = ref.attention(qs, ks, vs, cfg)
    secs = time.perf_counter() - t0
    pairs = float((tr.pass1_pairs + tr.pass2_pairs).mean())
    return secs, pairs


def full_pairs_per_head(l: int) -> float | None:
    if os.path.exists(PAIRS_FILE):
        with open(PAIRS_FILE) as f:
            d = json.load(f)
        if int(d.get("L", 0)) == l:
            return float(d["pairs_per_head"])
    return None


def cpu_extrapolate(secs: float, pairs_sample: float, pairs_full: float, threads: int) -> float:
    """ms per layer (32 heads) on `threads` cores, heads in parallel (parallel.cpp:25-66)."""
    per_head = secs * pairs_full / pairs_sample  # each thread ran one head's sample
    waves = math.ceil(HQ / threads)
    return per_head * waves * 1e3


def run_reference_arm(args, rank: int):
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    threads = min(cores, HQ)
    pairs_full = full_pairs_per_head(args.L)
    vals = []
    for i in range(args.warmup + args.steps):
        secs, pairs = reference_sample(args.L, args.seg, args.tau, args.ref_segments, threads)
        if pairs_full is None:
            pairs_full = pairs * (args.L / (args.ref_segments * args.seg)) ** 1.2  # crude guess
        if i >= args.warmup:
            vals.append(cpu_extrapolate(secs, pairs, pairs_full, threads))
    value = sum(vals) / len(vals)
    out = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "ms",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(value, 3),
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generate_synthetic mixed, bf16-rounded)",
        "config": {"workload": "C3: 1 layer, 32q/8kv heads, d=128, L=%d, S=%d, tau=%g" % (args.L, args.seg, args.tau)},
        "cpu_baseline": {"value": round(value, 3), "unit": "ms", "cores": threads, "kind": "reference",
                         "sample": f"compiled reference s2o_attention on {threads} heads x first "
                                   f"{args.ref_segments} segments ({args.ref_segments * args.seg} tokens), "
                                   f"extrapolated by pass1+pass2 pair count to {HQ} heads x L={args.L}"},
        "e2e": {"value": round(value, 3), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------ our arm
def run_ours(args, rank: int, world: int):
    import torch

    import paper_2602_22575_b200 as s2o

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    s2o.lib()
    L, S = args.L, args.seg
    cfg = s2o.KernelConfig(seg_len=S, tau=args.tau, tiles=s2o.TileSpec(128, 128), q_reorder=True)
    q, k, v = make_inputs(torch, s2o, L, seed=rank, device=dev)
    out = torch.empty_like(q)
    path = s2o.select_path(q, k, v, cfg)

    def step():
        s2o.s2o_attention(q, k, v, cfg, out=out, want_plan=False)

    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark_start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        step()
    ev1.record()
    torch.cuda.synchronize()
    clocks.mark_end()
    elapsed = ev0.elapsed_time(ev1)
    clk = clocks.stop()
    if dist:
        t = torch.tensor([elapsed], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = t.item()
        dist.barrier()
    ms_step = elapsed / args.steps
    value = ms_step / world

    # ---- stage breakdown, trace, roofline (device-resident inputs)
    res = s2o.s2o_attention(q, k, v, cfg)
    torch.cuda.synchronize()
    p1 = int(res.trace.pass1_pairs.sum().item())
    p2 = int(res.trace.pass2_pairs.sum().item())
    total_pairs = HQ * L * (L + 1) // 2
    sparsity = 1.0 - (p1 + p2) / total_pairs
    plan, _ = s2o.build_plan(q, k, S)
    t_plan_full = cuda_time(torch, lambda: s2o.build_plan(q, k, S), 2)
    t_plan = cuda_time(torch, lambda: s2o.build_plan_truncated(q, k, S), 3)
    t_p1 = cuda_time(torch, lambda: s2o.pass1_dense_init(q, k, v, cfg), 3)
    bufs = s2o.pass1_dense_init(q, k, v, cfg)
    t_p2 = cuda_time(torch, lambda: s2o.pass2_sparse(q, k, v, bufs, plan, cfg, out=out), 3)
    del bufs
    pk = peaks()
    f_p1, f_p2 = 4.0 * D * p1, 4.0 * D * p2
    if t_p2 >= t_p1:
        dom, f_dom, t_dom = "tc_pass_kernel (pass-2)", f_p2, t_p2
    else:
        dom, f_dom, t_dom = "tc_pass_kernel (pass-1)", f_p1, t_p1
    achieved = f_dom / (t_dom * 1e-3) / 1e12
    peak = float(pk.get("bf16_tflops", PEAKS_FALLBACK["bf16_tflops"]))
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        with open(prof) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    roofline = {"bound": "tensor", "kernel": dom, "achieved": round(achieved, 2), "peak": peak,
                "unit": "TFLOP/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                "peak_source": pk["_source"] + " burst bf16",
                "work": "4*D*(committed pairs) per launch, from the kernel's own trace"}
    # dense comparator on the same GPU (cuDNN/flash SDPA, bf16, causal, GQA)
    dense_ms = None
    mse = None
    if rank == 0 and not args.no_dense:
        try:
            def dense():
                return torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
            dense()
            dense_ms = cuda_time(torch, dense, 2)
            od = dense().float()
            diff = (res.out.float() - od)
            mse = float((diff * diff).mean().item())
            del od, diff
        except Exception as e:  # noqa: BLE001
            dense_ms = f"unavailable: {type(e).__name__}"

    # ---- e2e through the host-buffer C-ABI entry point
    e2e = None
    if not args.no_e2e:
        qh = q.cpu().pin_memory()
        kh = k.cpu().pin_memory()
        vh = v.cpu().pin_memory()
        oh = torch.empty_like(qh).pin_memory()
        s2o.attention_host_ptr(qh, kh, vh, oh, cfg)
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            s2o.attention_host_ptr(qh, kh, vh, oh, cfg)
        e_ms = (time.perf_counter() - t0) * 1e3 / args.e2e_steps
        if dist:
            t = torch.tensor([e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = t.item()
        s2o.lib().s2o_host_release()
        hb = (qh.numel() + kh.numel() + vh.numel()) * qh.element_size()
        db = oh.numel() * oh.element_size()
        e2e = {"value": round(e_ms / world, 3), "unit": "ms", "h2d_bytes_per_step": hb, "d2h_bytes_per_step": db,
               "timer": "host wall clock around the synchronous C-ABI call"}

    # ---- CPU baseline: compiled reference on a bounded sample (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            os.makedirs(os.path.dirname(PAIRS_FILE), exist_ok=True)
            with open(PAIRS_FILE, "w") as f:
                json.dump({"L": L, "S": S, "tau": args.tau, "pairs_per_head": (p1 + p2) / HQ,
                           "pass1_pairs": p1, "pass2_pairs": p2}, f)
            cores = os.cpu_count() or 1
            threads = min(cores, HQ)
            secs, pairs = reference_sample(L, S, args.tau, args.ref_segments, threads)
            val = cpu_extrapolate(secs, pairs, (p1 + p2) / HQ, threads)
            cpu = {"value": round(val, 1), "unit": "ms", "cores": threads, "kind": "reference",
                   "sample": f"compiled reference s2o_attention on {threads} heads x first {args.ref_segments} "
                             f"segments ({args.ref_segments * S} tokens) took {secs:.2f} s; extrapolated by "
                             f"pass1+pass2 pair count to {HQ} heads x L={L}"}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "ms", "cores": 0, "kind": "reference", "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 4), "unit": "ms", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (reference generate_synthetic mixed stripes, L/64 stripes, gain 8, seed=rank)",
            "config": {"workload": "C3: one Llama-3.1-8B attention layer per rank (32 q / 8 kv heads GQA, d=128)",
                       "seq_len": L, "seg_len": S, "tiles": [128, 128], "tau": args.tau,
                       "parallelism": f"layer-per-rank x{world}, no collective",
                       "l2": "inputs 1.6 GB > 126 MB L2 (no flush needed)", "path": {1: "generic", 2: "tcgen05"}[path]},
            "breakdown_ms": {"plan_truncated": round(t_plan, 3), "pass1": round(t_p1, 3), "pass2": round(t_p2, 3),
                             "plan_full_permutation": round(t_plan_full, 3)},
            # preprocessing against HBM (SURVEY.md §8(d) B_alg: Q + K read, full kv_perm + q_perm
            # written; the truncated plan writes only the top-T lists, so this overstates its bytes)
            "plan_hbm": plan_hbm(L, S, t_plan, peaks()),
            "sparsity": round(sparsity, 5), "pairs": {"pass1": p1, "pass2": p2},
            "dense_ms": round(dense_ms, 3) if isinstance(dense_ms, float) else dense_ms,
            "speedup_vs_dense": round(dense_ms / ms_step, 2) if isinstance(dense_ms, float) else None,
            "mse_vs_dense": mse,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches_per_step(L, S) * args.steps,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def run_heads(args, rank: int, world: int):
    """--shard heads: one layer's heads partitioned over the ranks in whole GQA
    groups (rank r: kv heads [r*8/N, (r+1)*8/N) and their q heads), no collective on the data
    path; with --allgather every step ends with an NCCL all-gather of the output shards over
    NVLink (reported separately as allgather_ms). value = max-over-ranks ms per layer."""
    import torch

    import paper_2602_22575_b200 as s2o
    from paper_2602_22575_b200.shard import gather_heads, head_shard

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    s2o.lib()
    L, S = args.L, args.seg
    cfg = s2o.KernelConfig(seg_len=S, tau=args.tau, tiles=s2o.TileSpec(128, 128), q_reorder=True)
    sh = head_shard(HQ, HKV, world, rank)
    qh, kh, vh = s2o.generate_synthetic("mixed", L // 64, 8.0, 0, 1, sh.q_hi, L, D)  # heads < q_hi
    q = torch.from_numpy(qh[:, sh.q_lo:sh.q_hi].copy()).to(dev).to(torch.bfloat16)
    k = torch.from_numpy(kh[:, sh.kv_lo:sh.kv_hi].copy()).to(dev).to(torch.bfloat16)
    v = torch.from_numpy(vh[:, sh.kv_lo:sh.kv_hi].copy()).to(dev).to(torch.bfloat16)
    del qh, kh, vh
    out = torch.empty_like(q)

    def step():
        s2o.s2o_attention(q, k, v, cfg, out=out, want_plan=False)
        if args.allgather and dist:
            gather_heads(out, world)

    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark_start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        step()
    ev1.record()
    torch.cuda.synchronize()
    clocks.mark_end()
    elapsed = ev0.elapsed_time(ev1)
    clk = clocks.stop()
    ag_ms = None
    if dist:
        t = torch.tensor([elapsed], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = t.item()
        if args.allgather:
            ag_ms = cuda_time(torch, lambda: gather_heads(out, world), 3)
            t = torch.tensor([ag_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ag_ms = t.item()
    ms_step = elapsed / args.steps
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(ms_step, 4), "unit": "ms", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (reference generate_synthetic mixed stripes, L/64 stripes, gain 8, seed 0)",
            "config": {"workload": "C4: one Llama-3.1-8B attention layer, heads sharded in whole GQA groups",
                       "seq_len": L, "seg_len": S, "tau": args.tau,
                       "parallelism": f"heads/{world} ({sh.hq} q / {sh.hkv} kv heads per rank)",
                       "allgather": bool(args.allgather)},
            "allgather_ms": round(ag_ms, 3) if ag_ms is not None else None,
            "gpu_launches": launches_per_step(L, S) * args.steps, "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--L", type=int, default=131072)
    ap.add_argument("--seg", type=int, default=2048)
    ap.add_argument("--tau", type=float, default=0.005)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--ref-segments", type=int, default=8)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--shard", default="layers", choices=["layers", "heads"],
                    help="multi-GPU: a full layer per rank (weak) or one layer's heads split (strong)")
    ap.add_argument("--allgather", action="store_true", help="--shard heads: NCCL all-gather of O")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference_arm(args, rank)
        return
    if args.shard == "heads":
        run_heads(args, rank, world)
        return
    run_ours(args, rank, world)


if __name__ == "__main__":
    main()
