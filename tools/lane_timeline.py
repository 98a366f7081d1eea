"""GPU occupancy of a 4-lane config-2 step from CUPTI kernel records
(torch.profiler): union of kernel intervals (busy), the sum of kernel time,
and time-weighted kernel concurrency.   python tools/lane_timeline.py 1024 4"""
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2509_01180_b200 import api

P = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
lanes = int(sys.argv[2]) if len(sys.argv) > 2 else 4
ctx = api.Context(64, 16, 16 * math.pi)
tmpl = api.make_template(64, 40, 20250901)
ctx.set_template(tmpl, 60.0)
parts, _, _ = api.make_particles(tmpl, P, 1000, 3, 0.1, 60.0)
cfg = api.make_config(bands=(4, 8, 16), max_candidates=24, shift_radius=4, shift_step=2)
ctx.set_lanes(lanes, 32)
ctx.align_batch(parts, cfg)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    ctx.align_batch(parts, cfg)
    torch.cuda.synchronize()
iv = []
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and not e.name.startswith("Mem"):
        iv.append((e.time_range.start, e.time_range.end))
iv.sort()
span = iv[-1][1] - iv[0][0]
total = sum(b - a for a, b in iv)
busy, cs, ce = 0, None, None
for a, b in iv:
    if ce is None or a > ce:
        if ce is not None:
            busy += ce - cs
        cs, ce = a, b
    else:
        ce = max(ce, b)
busy += ce - cs
print(f"lanes {lanes}: span {span / 1e3:.1f} ms, busy {busy / 1e3:.1f} ms ({100 * busy / span:.1f}%), "
      f"kernel time {total / 1e3:.1f} ms, mean concurrency while busy {total / busy:.2f}, kernels {len(iv)}")
