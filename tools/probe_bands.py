"""Per-band x per-kernel-class refinement times and evaluation counts of the
list-driven path at config 2 (single lane, CUDA events):
  python tools/probe_bands.py 256"""
import math
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2509_01180_b200 import api


def main():
    P = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    lanes = int(os.environ.get("LANES", "1"))
    ctx = api.Context(64, 16, 16 * math.pi)
    tmpl = api.make_template(64, 40, 7)
    ctx.set_template(tmpl, 60.0)
    parts, q, sh = api.make_particles(tmpl, P, 1000, 3, 0.1, 60.0)
    cfg = api.make_config(bands=(4, 8, 16), max_candidates=24, shift_radius=4, shift_step=2)
    ctx.set_lanes(lanes, 64)
    if not os.environ.get("BMB_NO_WARMUP"):
        ctx.align_batch(parts[:8], cfg)
    torch.cuda.synchronize()
    t0 = time.time()
    ctx.align_batch(parts, cfg)
    torch.cuda.synchronize()
    print(f"untimed: {(time.time() - t0) * 1e3:.1f} ms for {P} particles (lanes {lanes})")
    ctx.set_timing(True)
    ctx.timings(reset=True)
    ctx.eval_stats(reset=True)
    t0 = time.time()
    ctx.align_batch(parts, cfg)
    torch.cuda.synchronize()
    print(f"timed: {(time.time() - t0) * 1e3:.1f} ms")
    ms, cnt = ctx.timings()
    print({k: round(v, 2) for k, v in ms.items() if v})
    print(cnt)
    for b, d in ctx.band_timings().items():
        if d:
            print(f"band {b}: " + " ".join(f"{k}={v:.2f}" for k, v in d.items()))
    for L in (4, 8, 16):
        e2, e0 = ctx.eval_counts(L)
        print(f"L={L}: order2 {e2} order0 {e0}")


if __name__ == "__main__":
    main()
