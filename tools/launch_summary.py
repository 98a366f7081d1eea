"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
for i, r in enumerate(rows):
    if "Kernel Name" in r:
        hdr, start = r, i + 1
        break
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg, cnt, mx = {}, {}, {}
for r in rows[start:]:
    if len(r) <= vi:
        continue
    m = re.search(r"(\w+_kernel)(<\d>)?", r[ki])
    name = (m.group(1) + (m.group(2) or "")) if m else r[ki][:50]
    try:
        v = float(r[vi])
    except ValueError:
        continue
    agg[name] = agg.get(name, 0) + v
    cnt[name] = cnt.get(name, 0) + 1
    mx[name] = max(mx.get(name, 0), v)
tot = sum(agg.values())
print(f"total {tot/1e6:.2f} ms over {sum(cnt.values())} launches")
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{v/1e6:9.2f} ms {100*v/tot:5.1f}% n={cnt[k]:5d} max={mx[k]/1e3:8.1f}us avg={v/cnt[k]/1e3:8.1f}us {k}")
