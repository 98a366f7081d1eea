"""Per-CUDA-source-line instruction and stall-sample totals of one kernel in an
ncu report (needs -lineinfo): python tools/ncu_lines.py report.ncu-rep [launch] [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--launch-skip",
                      str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[2]
iE, iW = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
lines = []
tot_e = tot_w = 0
for r in rows[3:]:
    if len(r) <= iE or not r[0]:
        continue  # SASS rows carry an empty line number
    try:
        e, w = int(r[iE] or 0), int(r[iW] or 0)
    except ValueError:
        continue
    lines.append((e, w, r[0], r[1].strip()[:90]))
    tot_e += e
    tot_w += w
print(f"total instructions {tot_e}, stall samples {tot_w}")
for e, w, ln, src in sorted(lines, key=lambda x: -x[1])[:top]:
    print(f"{ln:>5} inst {100.0 * e / max(tot_e, 1):5.1f}%  stall {100.0 * w / max(tot_w, 1):5.1f}%  {src}")
