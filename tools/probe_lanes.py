"""Config-2 step time vs concurrent lanes (1024 particles, device-resident):
  python tools/probe_lanes.py 1024 2 3 4 5 6"""
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2509_01180_b200 import api


def main():
    P = int(sys.argv[1])
    lanes = [int(x) for x in sys.argv[2:]] or [3]
    ctx = api.Context(64, 16, 16 * math.pi)
    tmpl = api.make_template(64, 40, 7)
    ctx.set_template(tmpl, 60.0)
    parts, q, sh = api.make_particles(tmpl, P, 1000, 3, 0.1, 60.0)
    cfg = api.make_config(bands=(4, 8, 16), max_candidates=24, shift_radius=4, shift_step=2)
    for n in lanes:
        ctx.set_lanes(n, 32)
        for _ in range(2):
            ctx.align_batch(parts, cfg)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            ctx.align_batch(parts, cfg)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"lanes {n}: {ms:.1f} ms/step, {P / ms * 1e3:.0f} subtomograms/s", flush=True)


if __name__ == "__main__":
    main()
