"""One bench.py-shaped config-2 step (single lane) inside a cudaProfilerStart/Stop
range, for range-limited profilers:
  ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
      --csv --log-file gpurun_out/step_traffic.csv python tools/step_probe.py 1024"""
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2509_01180_b200 import api

P = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
ctx = api.Context(64, 16, 16 * math.pi)
tmpl = api.make_template(64, 40, 20250901)
ctx.set_template(tmpl, 60.0)
parts, _, _ = api.make_particles(tmpl, P, 1000, 3, 0.1, 60.0)
cfg = api.make_config(bands=(4, 8, 16), max_candidates=24, shift_radius=4, shift_step=2)
ctx.set_lanes(1)
ctx.align_batch(parts[:16], cfg)
torch.cuda.synchronize()
torch.cuda.profiler.start()
res = ctx.align_batch(parts, cfg)
avg = ctx.average_accumulate(parts, res)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("step done", len(res))
