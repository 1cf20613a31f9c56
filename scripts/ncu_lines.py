"""Dev aid: per-source-line warp-stall samples of one kernel in an ncu report (needs -lineinfo and
--import-source on).  python scripts/ncu_lines.py report.ncu-rep [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, tot = [], "", 0
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif len(r) > 4 and r[0] not in ("", "Line No"):
        try:
            v = int(r[4])
        except ValueError:
            continue
        tot += v
        rows.append((v, f"{fname}:{r[0]}", r[1].strip()[:100]))
rows.sort(reverse=True)
print("total samples", tot)
for v, loc, src in rows[:top]:
    print(f"{v:7d} {100.0 * v / max(tot, 1):5.1f}%  {loc:22s} {src}")
