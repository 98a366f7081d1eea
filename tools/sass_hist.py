"""Opcode histogram (executed instructions per launch unit) of one kernel in an
ncu report: python tools/sass_hist.py report.ncu-rep [launch index] [units]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
units = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--launch-skip",
                      str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
iS, iE, iW = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
op, st, tot = collections.Counter(), collections.Counter(), 0
for r in rows[2:]:
    try:
        n = int(r[iE])
    except (ValueError, IndexError):
        continue
    s = r[iS].strip()
    parts = s.split()
    o = (parts[1] if parts and parts[0].startswith("@") and len(parts) > 1 else (parts[0] if parts else "?")).split(".")[0]
    op[o] += n
    st[o] += int(r[iW] or 0)
    tot += n
print(rows[0][1] if len(rows[0]) > 1 else "", "total", tot, "per unit", tot / units)
for o, n in op.most_common(40):
    print(f"{o:10s} {n / units:9.1f}  stall samples {st[o]}")
