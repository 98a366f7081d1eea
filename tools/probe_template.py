"""Per-template setup cost (set_template: template expansion, tapered wedge filter,
wedge-power kernel) and context creation, 64^3 L=16 and L=20."""
import math
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2509_01180_b200 import api

for L in (16, 20):
    t0 = time.time()
    ctx = api.Context(64, L, L * math.pi)
    torch.cuda.synchronize()
    t1 = time.time()
    tmpl = api.make_template(64, 40, 1)
    ctx.set_template(tmpl, 60.0)
    torch.cuda.synchronize()
    t2 = time.time()
    for s in range(3):
        ctx.set_template(api.make_template(64, 40, 2 + s), 60.0)
    torch.cuda.synchronize()
    t3 = time.time()
    print(f"L={L}: context {1e3 * (t1 - t0):.0f} ms, first set_template {1e3 * (t2 - t1):.0f} ms, "
          f"next set_template {1e3 * (t3 - t2) / 3:.0f} ms", flush=True)
