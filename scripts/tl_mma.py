"""Dev probe: MMA-warp event sequence of CTA 0 from gpurun_out/timeline_<pass>.npy (timeline.py)."""
import sys
import numpy as np
FINE = "--fine" in sys.argv
if FINE:
    sys.argv.remove("--fine")
tag = sys.argv[1] if len(sys.argv) > 1 else "pass1"
lo, hi = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (30, 75)
t = np.load(f"gpurun_out/timeline_{tag}.npy")
ev = {6: "p0_seen", 28: "v_full", 5: "k_full", 31: "s0_iss", 7: "p1_seen", 8: "kv_empty"}
if FINE:
    ev.update({0: "f_after_ns", 3: "f_after_sync", 4: "f_after_dec"})
rows = sorted((v, n, j) for e, n in ev.items() for j, v in enumerate(t[e][:80]) if v >= 0)
prev = None
for v, n, j in rows[lo:hi]:
    print(f"{v:8d} {n:10s} blk{j:3d} +{v - prev if prev else 0}")
    prev = v
