"""Summarize an ncu report: stall ratios + hottest SASS (with sampled share)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
d = dict(zip(rows[0], rows[2]))
for k, v in d.items():
    if ("issue_stalled" in k and "ratio" in k) or k in (
            "gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "smsp__thread_inst_executed_per_inst_executed.ratio",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum"):
        try:
            if float(v) > 0.1:
                print(f"{k:70s} {v}")
        except ValueError:
            pass
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                      capture_output=True, text=True).stdout
rows = list(csv.reader(sass.splitlines()))
hdr = rows[1]
data = rows[2:]
si = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
tot = sum(float(r[si]) for r in data if len(r) > si and r[si])
top = sorted(((float(r[si]), i) for i, r in enumerate(data) if len(r) > si and r[si]), reverse=True)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for s, i in top[:n]:
    print(f"{100*s/tot:5.2f}% #{i:6d} exec={data[i][ie]:>10} {data[i][1].strip()[:90]}")
bk = {}
for i, r in enumerate(data):
    if len(r) > si and r[si]:
        bk[i // 250] = bk.get(i // 250, 0) + float(r[si])
print("by 250-instr buckets:", ", ".join(f"[{b*250}]{100*v/tot:.1f}%" for b, v in sorted(bk.items(), key=lambda x: -x[1])[:12]))
