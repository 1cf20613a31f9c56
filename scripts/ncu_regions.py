"""Dev aid: warp-stall samples of one kernel split by code region (delimited by SASS address
ranges around landmark instructions) and by stall reason.
    python scripts/ncu_regions.py report.ncu-rep"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Address")
data = [r for r in rows if len(r) == len(hdr) and r[2].isdigit()]
reasons = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(int(r[2]) for r in data)
# regions: split at every SYNCS.PHASECHK (mbarrier wait) / BAR.SYNC so waits are their own rows
regions, cur = [], []
for r in data:
    op = r[1]
    if "PHASECHK" in op or "BAR.SYNC" in op:
        if cur: regions.append(cur)
        regions.append([r])
        cur = []
    else:
        cur.append(r)
if cur: regions.append(cur)
print("total samples", tot)
for reg in regions:
    v = sum(int(r[2]) for r in reg)
    if v < 0.01 * tot: continue
    rs = {c: sum(int(r[hdr.index(c)] or 0) for r in reg) for c in reasons}
    top = ", ".join(f"{k[6:]}:{100 * x / max(v, 1):.0f}%" for k, x in sorted(rs.items(), key=lambda x: -x[1])[:4])
    ops = {}
    for r in reg:
        o = [t for t in r[1].split() if not t.startswith("@")][0].split(".")[0]
        ops[o] = ops.get(o, 0) + 1
    lab = reg[0][1].strip()[:50] if len(reg) == 1 else f"{len(reg)} instrs, top ops " + ",".join(o for o, _ in sorted(ops.items(), key=lambda x: -x[1])[:4])
    print(f"{reg[0][0][-5:]} {v:7d} {100 * v / tot:5.1f}%  {lab}  [{top}]")
