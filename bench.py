"""bench.py -- S2O sparse prefill attention on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[2]): one Llama-3.1-8B attention layer,
32 q heads / 8 kv heads (GQA), d=128, bf16, L=131072, S=2048, tiles 128x128, tau=0.005, on
the reference's stripe-structured synthetic input (generate_synthetic mixed, L/64 stripes,
gain 8, seed = layer = rank). A step = the whole operator: plan (block scoring +
permutation build) + pass-1 + pass-2 for all 32 heads.

Multi-GPU: the layer's heads are partitioned over the ranks in whole GQA
groups (rank r: kv heads [r*8/N, (r+1)*8/N) and their q heads), no collective on the data
path; `value` = max-over-ranks ms per layer ("scaling": "strong"); --allgather adds an NCCL
all-gather of O (timed inside the step, and alone as breakdown_ms.allgather). --shard layers
(opt-in) runs a whole layer per rank instead (weak scaling, value = ms per layer of the job).

Timing: W warm-up steps, then K steps bracketed by barrier + synchronize, CUDA events on the
launching stream; inputs (1.6 GB) exceed L2 (126 MB). `e2e` runs the same operator through
the host-buffer C-ABI entry point (s2o_attention_host) from pinned host memory, H2D of Q/K/V
and D2H of O inside the timed region. `cpu_baseline` (rank 0, N=1) times the compiled
reference (oracle/_ref, its own input generator) on a bounded prefix sample of the same layer
and scales it by the reference's own full-length/sample time ratio recorded in
profiles/ref_c3_calibration.json (scripts/ref_calibrate.py); the sample is also diffed against
the device operator on the same heads and tokens (`cpu_baseline.sample_parity`).
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
CALIB_FILE_REL = "profiles/ref_c3_calibration.json"
CALIB_FILE = os.path.join(ROOT, CALIB_FILE_REL)


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
    """Our kernels per s2o_attention_fwd call with the truncated plan (no overflow rerun), as the
    ncu launch list of a bench run shows them: guide means and q ranking (+ the q sort when
    S > 2048); for N > 1 segments the candidate top-T selection (dense kv scoring of the first
    segments, sample scoring, threshold, kv_cand, two pack kernels, sel_scan, sel_sort); then trace
    init, the masked-key poison scan, pass-1 (tc_diag2_kernel), the (empty) poison rerun and
    pass-2 (tc_pass_kernel)."""
    n = -(-l // s)
    count = 2
    if s > 2048:
        count += 2 + plan_sort_passes(l, s)
    if n > 1:
        count += 8
    return count + 5


# ------------------------------------------------------------------ shared description
def cpu_info() -> dict:
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def workload_config(args, world: int) -> dict:
    """The `config` of BOTH arms (identical dicts: the same workload, whoever computes it)."""
    return {"workload": "C3: one Llama-3.1-8B attention layer (32 q / 8 kv heads GQA, d=128), S2O prefill",
            "seq_len": args.L, "seg_len": args.seg, "tiles": [128, 128], "tau": args.tau,
            "inputs": "generate_synthetic mixed, L/64 stripes, gain 8, seed 0, bf16-rounded",
            "parallelism": (f"heads/{world} (whole GQA groups, no collective)" if args.shard == "heads"
                            else f"layer-per-rank x{world} (seed = rank, no collective)"),
            "l2": "inputs 1.6 GB > 126 MB L2 (no flush needed)"}


# ------------------------------------------------------------------ reference (CPU) arm
def bf16_round_np(x):
    import numpy as np
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    return (((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16).astype(np.uint32).view(np.float32)


class _Cfg:
    def __init__(self, seg_len, tau):
        self.seg_len, self.tau, self.b_m, self.b_n = seg_len, tau, 128, 128
        self.q_reorder, self.fused, self.local_window = True, False, -1


_REF_INPUTS: dict = {}


def reference_sample(l_full: int, s: int, tau: float, seg_sample: int, heads: list[int], want_out: bool = False):
    """The compiled reference (oracle/_ref, its own generate_synthetic and s2o_attention) on q
    heads `heads` (one host thread each) of the first `seg_sample` segments of the benchmark
    layer: by causality exactly segments 0..m-1 of the full problem. K/V of kv head h // 4 are
    expanded per q head (the reference has no GQA); inputs bf16-rounded as on the device.
    Returns (seconds, mean pairs per head, (q, out, trace, plan) if want_out)."""
    from oracle.oracle import Ref, build

    build()
    ref = Ref()
    lp = min(l_full, seg_sample * s)
    nh = max(heads) + 1
    key = (l_full, nh)
    if key not in _REF_INPUTS:  # the full-length layer once per process (stripe geometry depends on L)
        _REF_INPUTS.clear()
        os.environ["S2O_THREADS"] = str(os.cpu_count() or 1)
        _REF_INPUTS[key] = ref.generate_synthetic("mixed", l_full // 64, 8.0, 0, 1, nh, l_full, D)
    q, k, v = _REF_INPUTS[key]
    qs = bf16_round_np(q[:, heads, :lp])
    ks = bf16_round_np(k[:, [h // (HQ // HKV) for h in heads], :lp])
    vs = bf16_round_np(v[:, [h // (HQ // HKV) for h in heads], :lp])
    os.environ["S2O_THREADS"] = str(len(heads))
    t0 = time.perf_counter()
    out, tr, plan = ref.attention(qs, ks, vs, _Cfg(s, tau))
    secs = time.perf_counter() - t0
    pairs = float((tr.pass1_pairs + tr.pass2_pairs).mean())
    return secs, pairs, ((qs, ks, vs, out, tr, plan) if want_out else None)


def load_calibration(args, threads: int):
    """profiles/ref_c3_calibration.json (scripts/ref_calibrate.py, run on the GPU box host): the
    compiled reference's own seconds for the sample and for the FULL-length layer on the same heads
    and thread count."""
    if not os.path.exists(CALIB_FILE):
        return None
    with open(CALIB_FILE) as f:
        c = json.load(f)
    if (int(c.get("L", 0)) != args.L or int(c.get("S", 0)) != args.seg or float(c.get("tau", -1)) != args.tau
            or int(c.get("sample_segments", 0)) != args.ref_segments):
        return None
    return c


def reference_step(args, threads: int, calib):
    """One reference-arm step: the bounded sample, scaled to the layer by the calibration's
    measured full/sample time ratio and by head waves (heads run one per thread)."""
    heads = list(range(threads))
    secs, pairs, _ = reference_sample(args.L, args.seg, args.tau, args.ref_segments, heads)
    waves = math.ceil(HQ / threads)
    if calib is not None:
        ratio = float(calib["full_seconds"]) / float(calib["sample_seconds"])
        how = (f"x {ratio:.2f} = the reference's own full-length/sample time ratio on {calib['threads']} heads "
               f"({calib['full_seconds']:.1f} s / {calib['sample_seconds']:.2f} s, {CALIB_FILE_REL}, "
               f"{calib.get('cpu_model')}), x {waves} head wave(s)")
    else:
        ratio = None
        how = "no calibration for this config: value is the sample time x head waves (a lower bound)"
    value_ms = secs * (ratio if ratio else 1.0) * waves * 1e3
    return value_ms, secs, pairs, how


def run_reference_arm(args, rank: int, world: int):
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    threads = min(cores, HQ)
    calib = load_calibration(args, threads)
    vals, how, secs_all = [], "", []
    for i in range(args.warmup + args.steps):
        v_ms, secs, _, how = reference_step(args, threads, calib)
        if i >= args.warmup:
            vals.append(v_ms)
            secs_all.append(secs)
    value = sum(vals) / len(vals)
    sample = (f"compiled reference (oracle/_ref: unmodified proj/src, its own generate_synthetic) s2o_attention on "
              f"{threads} q heads x the first {args.ref_segments} segments ({args.ref_segments * args.seg} tokens), "
              f"{threads} host threads, {sum(secs_all) / len(secs_all):.2f} s per sample; {how}")
    out = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "ms",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(value, 3),
        "higher_is_better": False, "scaling": "strong" if args.shard == "heads" else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generate_synthetic mixed stripes, bf16-rounded)",
        "config": workload_config(args, world),
        "cpu_baseline": {"value": round(value, 3), "unit": "ms", "cores": threads, "kind": "reference",
                         "sample": sample, **cpu_info(),
                         "extrapolated": calib is not None, "calibration": calib},
        "e2e": {"value": round(value, 3), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(out), flush=True)


def sample_parity(torch, s2o, args, dev, ref_data):
    """The cpu_baseline sample, diffed: the device operator on the same heads x tokens as the
    reference sample. Reports differing trace tiles (with their threshold-tie status, SURVEY.md
    §8c P2), the max |dO| and the ratio of the two outputs' MSE against the same fp32 dense
    reference (device, SDPA in fp32 on the bf16-rounded inputs)."""
    import numpy as np
    from oracle.oracle import Ref, trace_ties

    qs, ks, vs, ref_out, ref_tr, ref_plan = ref_data
    g = HQ // HKV
    qd = torch.from_numpy(qs).to(dev).to(torch.bfloat16)
    # one kv head per q head (the reference's expanded K/V): Hq = Hkv = len(heads)
    kd = torch.from_numpy(ks).to(dev).to(torch.bfloat16)
    vd = torch.from_numpy(vs).to(dev).to(torch.bfloat16)
    cfg = s2o.KernelConfig(seg_len=args.seg, tau=args.tau, tiles=s2o.TileSpec(128, 128))
    res = s2o.s2o_attention(qd, kd, vd, cfg, want_plan=False)
    got_t = res.trace.processed.reshape(qs.shape[1], -1, res.trace.processed.shape[-1]).cpu().numpy()
    ties = trace_ties(Ref(), qs, ks, vs, cfg, ref_plan.q_perm, ref_plan.kv_perm, got_t, ref_tr.processed)
    out = res.out.float()
    dense = torch.nn.functional.scaled_dot_product_attention(qd.float(), kd.float(), vd.float(), is_causal=True)
    ro = torch.from_numpy(ref_out).to(dev)
    mse_gpu = float(((out - dense) ** 2).mean().item())
    mse_ref = float(((ro - dense) ** 2).mean().item())
    return {"heads": int(qs.shape[1]), "tokens": int(qs.shape[2]),
            "trace_tiles": int(got_t.size), "trace_tiles_differing": len(ties),
            "trace_differences_all_ties": all(t["tie"] for t in ties),
            "max_rel_gap_to_tau": max((t["rel_to_tau"] for t in ties), default=None),
            "max_abs_out_diff": float((out - ro).abs().max().item()),
            "mse_vs_dense_fp32": {"device": mse_gpu, "reference": mse_ref,
                                  "ratio": (mse_gpu / mse_ref) if mse_ref > 0 else None}}


# ------------------------------------------------------------------ our arm
def time_steps(torch, dist, step, steps: int, warmup: int, clocks) -> float:
    """W warm-up steps, then K steps between barrier + synchronize, CUDA events on the launching
    stream; returns the max over ranks of the timed region in ms."""
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark_start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(steps):
        step()
    ev1.record()
    torch.cuda.synchronize()
    clocks.mark_end()
    elapsed = ev0.elapsed_time(ev1)
    if dist:
        t = torch.tensor([elapsed], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = t.item()
        dist.barrier()
    return elapsed


def run_ours(args, rank: int, world: int):
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
    if args.shard == "heads":
        # C4: one layer (seed 0), rank r owns whole GQA groups: kv heads
        # [r*8/N, (r+1)*8/N) and their q heads; no collective on the data path (strong scaling)
        sh = head_shard(HQ, HKV, world, rank)
        qh, kh, vh = s2o.generate_synthetic("mixed", L // 64, 8.0, 0, 1, sh.q_hi, L, D)
        q = torch.from_numpy(qh[:, sh.q_lo:sh.q_hi].copy()).to(dev).to(torch.bfloat16)
        k = torch.from_numpy(kh[:, sh.kv_lo:sh.kv_hi].copy()).to(dev).to(torch.bfloat16)
        v = torch.from_numpy(vh[:, sh.kv_lo:sh.kv_hi].copy()).to(dev).to(torch.bfloat16)
        del qh, kh, vh
        hq_local, hkv_local = sh.hq, sh.hkv
    else:  # opt-in weak scaling: a whole layer per rank (seed = rank)
        q, k, v = make_inputs(torch, s2o, L, seed=rank, device=dev)
        hq_local, hkv_local = HQ, HKV
    out = torch.empty_like(q)
    path = s2o.select_path(q, k, v, cfg)
    gather = args.allgather and dist is not None and args.shard == "heads"

    def step():
        s2o.s2o_attention(q, k, v, cfg, out=out, want_plan=False, check=False)
        if gather:
            gather_heads(out, world)

    clocks = ClockSampler(local)
    clocks.start()
    elapsed = time_steps(torch, dist, step, args.steps, args.warmup, clocks)
    clk = clocks.stop()
    ms_step = elapsed / args.steps
    # heads: a step is one layer over all ranks (max over ranks); layers: N layers per step
    value = ms_step if args.shard == "heads" else ms_step / world
    ag_ms = None
    if gather:
        ag_ms = cuda_time(torch, lambda: gather_heads(out, world), 3)

    # ---- stage breakdown, trace, roofline (device-resident inputs, this rank's heads)
    res = s2o.s2o_attention(q, k, v, cfg)
    torch.cuda.synchronize()
    p1 = int(res.trace.pass1_pairs.sum().item())
    p2 = int(res.trace.pass2_pairs.sum().item())
    total_pairs = hq_local * L * (L + 1) // 2
    sparsity = 1.0 - (p1 + p2) / total_pairs
    plan, _ = s2o.build_plan(q, k, S)
    t_plan_full = cuda_time(torch, lambda: s2o.build_plan(q, k, S), 2)
    t_plan = cuda_time(torch, lambda: s2o.build_plan_truncated(q, k, S), 3)
    t_p1 = cuda_time(torch, lambda: s2o.pass1_dense_init(q, k, v, cfg), 3)
    bufs = s2o.pass1_dense_init(q, k, v, cfg)
    t_p2 = cuda_time(torch, lambda: s2o.pass2_sparse(q, k, v, bufs, plan, cfg, out=out, check=False), 3)
    del bufs, plan
    pk = peaks()
    f_p1, f_p2 = 4.0 * D * p1, 4.0 * D * p2
    if t_p2 >= t_p1:
        dom, f_dom, t_dom = "tc_pass_kernel (pass-2)", f_p2, t_p2
    else:
        dom, f_dom, t_dom = "tc_diag2_kernel (pass-1)", f_p1, t_p1
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
                "work": "4*D*(committed pairs) per launch, from the kernel's own trace",
                "pass1": {"ms": round(t_p1, 3), "tflops": round(f_p1 / (t_p1 * 1e-3) / 1e12, 1),
                          "frac": round(f_p1 / (t_p1 * 1e-3) / 1e12 / peak, 4)},
                "pass2": {"ms": round(t_p2, 3), "tflops": round(f_p2 / (t_p2 * 1e-3) / 1e12, 1),
                          "frac": round(f_p2 / (t_p2 * 1e-3) / 1e12 / peak, 4)}}
    # dense comparators on the same GPU (cuDNN/flash SDPA, bf16, causal, GQA): the whole layer,
    # and pass-1's exact work (block-diagonal causal attention, segments as the batch)
    dense_ms = mse = p1_cudnn = None
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
            nseg = L // S
            if nseg * S == L:
                qs_ = q.view(hq_local, nseg, S, D).transpose(0, 1).contiguous()
                ks_ = k.view(hkv_local, nseg, S, D).transpose(0, 1).contiguous()
                vs_ = v.view(hkv_local, nseg, S, D).transpose(0, 1).contiguous()

                def blockdiag():
                    return torch.nn.functional.scaled_dot_product_attention(qs_, ks_, vs_, is_causal=True,
                                                                           enable_gqa=True)
                p1_cudnn = cuda_time(torch, blockdiag, 3)
                del qs_, ks_, vs_
        except Exception as e:  # noqa: BLE001
            dense_ms = f"unavailable: {type(e).__name__}"
    # strong-scaling predictor: the N=8 shard (4 q / 1 kv head) on this one GPU
    shard8_ms = None
    if rank == 0 and world == 1 and args.shard == "heads":
        q8, k8, v8, o8 = q[:, :4].contiguous(), k[:, :1].contiguous(), v[:, :1].contiguous(), out[:, :4].contiguous()
        shard8_ms = cuda_time(torch, lambda: s2o.s2o_attention(q8, k8, v8, cfg, out=o8, want_plan=False,
                                                               check=False), 5)
        del q8, k8, v8, o8

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
        e2e = {"value": round(e_ms if args.shard == "heads" else e_ms / world, 3), "unit": "ms",
               "h2d_bytes_per_step": hb * world, "d2h_bytes_per_step": db * world,
               "timer": "host wall clock around the synchronous C-ABI call (max over ranks)"}
        del qh, kh, vh, oh

    # ---- CPU baseline: the compiled reference on a bounded sample (rank 0, N=1), diffed
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cores = os.cpu_count() or 1
            threads = min(cores, HQ)
            calib = load_calibration(args, threads)
            val, secs, _, how = reference_step(args, threads, calib)
            _, _, ref_data = reference_sample(args.L, args.seg, args.tau, args.ref_segments,
                                              list(range(min(threads, 8))), want_out=True)
            cpu = {"value": round(val, 1), "unit": "ms", "cores": threads, "kind": "reference",
                   "sample": (f"compiled reference s2o_attention on {threads} q heads x the first {args.ref_segments} "
                              f"segments ({args.ref_segments * S} tokens) took {secs:.2f} s; {how}"),
                   **cpu_info(), "extrapolated": calib is not None,
                   "sample_parity": sample_parity(torch, s2o, args, dev, ref_data)}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "ms", "cores": 0, "kind": "reference", "sample": f"failed: {e!r}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 4), "unit": "ms", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": False, "scaling": "strong" if args.shard == "heads" else "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (reference generate_synthetic mixed stripes, L/64 stripes, gain 8)",
            "config": workload_config(args, world),
            "path": {1: "generic", 2: "tcgen05"}[path],
            "rank0_heads": {"q": hq_local, "kv": hkv_local},
            "breakdown_ms": {"plan_truncated": round(t_plan, 3), "pass1": round(t_p1, 3), "pass2": round(t_p2, 3),
                             "plan_full_permutation": round(t_plan_full, 3),
                             "allgather": round(ag_ms, 3) if ag_ms is not None else None},
            # preprocessing against HBM (SURVEY.md §8(d) B_alg: Q + K read, full kv_perm + q_perm
            # written; the truncated plan writes only the top-T lists, so this overstates its bytes)
            "plan_hbm": plan_hbm(L, S, t_plan, peaks()) if hq_local == HQ else None,
            "sparsity": round(sparsity, 5), "pairs": {"pass1": p1, "pass2": p2},
            "dense_ms": round(dense_ms, 3) if isinstance(dense_ms, float) else dense_ms,
            "speedup_vs_dense": round(dense_ms / ms_step, 2) if isinstance(dense_ms, float) else None,
            "pass1_cudnn_blockdiag_ms": round(p1_cudnn, 3) if p1_cudnn else None,
            "mse_vs_dense": mse,
            "shard_n8_on_one_gpu_ms": round(shard8_ms, 3) if shard8_ms else None,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches_per_step(L, S) * args.steps,
            "clocks": clk,
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
    ap.add_argument("--shard", default="heads", choices=["heads", "layers"],
                    help="multi-GPU: one layer's heads split in whole GQA groups (strong, default) or a full "
                         "layer per rank (weak)")
    ap.add_argument("--allgather", action="store_true", help="--shard heads: NCCL all-gather of O")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    run_ours(args, rank, world)


if __name__ == "__main__":
    main()
