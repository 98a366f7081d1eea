"""One config-2 align_batch (no warm-up) for targeted ncu captures:
  ncu -k regex:step_kernel --launch-count 1 python tools/probe_once.py 256"""
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2509_01180_b200 import api

P = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ctx = api.Context(64, 16, 16 * math.pi)
tmpl = api.make_template(64, 40, 7)
ctx.set_template(tmpl, 60.0)
parts, q, sh = api.make_particles(tmpl, P, 1000, 3, 0.1, 60.0)
ctx.set_lanes(1)
ctx.align_batch(parts, api.make_config(bands=(4, 8, 16), max_candidates=24, shift_radius=4, shift_step=2))
torch.cuda.synchronize()
