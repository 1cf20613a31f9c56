"""Dev aid: hottest SASS instructions (warp-stall samples) per kernel of an ncu report.
    python scripts/ncu_sass.py report.ncu-rep [top] [kernel-substring]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
want = sys.argv[3] if len(sys.argv) > 3 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
kern, rows, hdr = None, {}, None
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "Kernel Name":
        kern = r[1]
        rows.setdefault(kern, [])
    elif r and r[0] == "Address":
        hdr = r
    elif kern and hdr and len(r) > 4:
        try:
            rows[kern].append((int(r[2]), r[0][-5:], r[1].strip()))
        except ValueError:
            pass
for k, lst in rows.items():
    if want not in k:
        continue
    tot = sum(v for v, _, _ in lst)
    print(f"== {k[:90]}  samples {tot}")
    for v, a, s in sorted(lst, reverse=True)[:top]:
        print(f"{v:7d} {100.0 * v / max(tot, 1):5.1f}%  {a}  {s[:90]}")

# opcode histogram of executed warp instructions (column "Instructions Executed")
if "--ops" in sys.argv:
    kern, hdr, ops = None, None, {}
    for r in csv.reader(io.StringIO(out)):
        if r and r[0] == "Kernel Name":
            kern = r[1]
        elif r and r[0] == "Address":
            hdr = r
        elif kern and hdr and len(r) > 5 and want in kern:
            try:
                n = int(r[hdr.index("Instructions Executed")])
            except (ValueError, IndexError):
                continue
            op = r[1].strip().split()
            op = [t for t in op if not t.startswith("@")]
            if op:
                o = op[0].split(".")[0]
                ops[o] = ops.get(o, 0) + n
    tot = sum(ops.values())
    print("executed warp instructions", tot)
    for o, n in sorted(ops.items(), key=lambda x: -x[1])[:25]:
        print(f"  {o:10s} {n:12d} {100.0 * n / tot:5.1f}%")
