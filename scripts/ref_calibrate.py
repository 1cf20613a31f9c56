"""Calibrate the reference arm of bench.py against the reference's OWN full-length run.

    python scripts/ref_calibrate.py [--L 131072] [--seg 2048] [--tau 0.005] [--ref-segments 8]

Runs the compiled reference (oracle/_ref: the unmodified proj/src behind oracle/ref_capi.cpp,
inputs from its own generate_synthetic) on min(nproc, 32) q heads -- one host thread per head,
the reference's own parallel_for -- twice: on the bench's bounded sample (the first
`ref-segments` segments) and on the FULL layer length. Writes profiles/ref_c3_calibration.json:
both wall times, the reference's pair counts, and the host CPU. bench.py's reference arm and
cpu_baseline scale each step's sample time by full_seconds / sample_seconds from this file and
by ceil(32 / threads) head waves -- no pair-count model. Run it on the GPU box host (the machine
the bench runs on); it takes about as long as one head of the full layer on one core.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=131072)
    ap.add_argument("--seg", type=int, default=2048)
    ap.add_argument("--tau", type=float, default=0.005)
    ap.add_argument("--ref-segments", type=int, default=8)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--out", default=bench.CALIB_FILE)
    args = ap.parse_args()
    threads = args.threads or min(os.cpu_count() or 1, bench.HQ)
    heads = list(range(threads))
    t0 = time.time()
    s_sec, s_pairs, _ = bench.reference_sample(args.L, args.seg, args.tau, args.ref_segments, heads)
    f_sec, f_pairs, _ = bench.reference_sample(args.L, args.seg, args.tau, args.L // args.seg + 1, heads)
    rec = {"L": args.L, "S": args.seg, "tau": args.tau, "sample_segments": args.ref_segments,
           "threads": threads, "heads": heads,
           "sample_seconds": round(s_sec, 3), "full_seconds": round(f_sec, 3),
           "sample_pairs_per_head": s_pairs, "full_pairs_per_head": f_pairs,
           "ratio": round(f_sec / s_sec, 4), **bench.cpu_info(),
           "script": "scripts/ref_calibrate.py", "wall_s": round(time.time() - t0, 1),
           "note": "compiled reference s2o_attention (oracle/_ref), one host thread per q head, bf16-rounded "
                   "inputs from the reference's generate_synthetic; full_seconds is the whole layer length for "
                   "these heads, measured, not modelled"}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(rec, f, indent=1)
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
