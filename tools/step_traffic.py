"""Sum an ncu --csv metrics log of tools/step_probe.py by kernel class:
DRAM bytes (read + write) and duration per class -> JSON (profiles/)."""
import csv
import json
import sys
from collections import defaultdict

CLASSES = (("eval_kernel<2", "eval_order2"), ("eval_kernel<0", "eval_order0"),
           ("eval_sub_kernel<2", "eval_order2"), ("eval_sub_kernel<0", "eval_order0"), ("expand_factored", "expand"),
           ("expand_pair", "expand"), ("expand_tc", "expand"), ("expand_quad", "expand"), ("quad_volumes", "expand"), ("advance_kernel", "newton"), ("step_kernel", "newton"),
           ("build_xi", "xi_build"), ("seed_kernel", "seed"))


def main(path, out):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        rows.append(r)
    agg = defaultdict(lambda: {"launches": 0, "dram_bytes": 0.0, "ms": 0.0})
    per_launch = defaultdict(dict)
    for r in rows:
        name = r["Kernel Name"]
        cls = next((c for k, c in CLASSES if k in name), "other")
        key = (r["ID"], cls)
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3,
                 "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(unit, 1.0)
        per_launch[key][r["Metric Name"]] = v * scale
    for (lid, cls), m in per_launch.items():
        a = agg[cls]
        a["launches"] += 1
        a["dram_bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        a["ms"] += m.get("gpu__time_duration.sum", 0.0)
    agg = dict(agg)
    agg["eval"] = {k: agg.get("eval_order2", {}).get(k, 0) + agg.get("eval_order0", {}).get(k, 0)
                   for k in ("launches", "dram_bytes", "ms")}
    json.dump({"source": path, "note": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
               "gpu__time_duration.sum over one config-2 step (tools/step_probe.py, 1 lane); serialised, "
               "cold-cache per launch: use bytes, not times", "classes": agg}, open(out, "w"), indent=1)
    print(json.dumps(agg, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
