"""Config-2 probe: 64^3, L=16, bands 4-8-16, 24 starts, wedge 60, SNR 0.1, shifts +-3."""
import math
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2509_01180_b200 import api


def geod(q1, q2):
    d = abs(float(np.dot(q1, q2)))
    return math.degrees(2 * math.acos(min(1.0, d)))


def main():
    P = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    t0 = time.time()
    ctx = api.Context(64, 16, 16 * math.pi)
    print(f"context {time.time()-t0:.1f}s coeffs {ctx.coeff_count} support {ctx.support}", flush=True)
    tmpl = api.make_template(64, 40, 7)
    t0 = time.time()
    ctx.set_template(tmpl, 60.0)
    print(f"set_template {time.time()-t0:.2f}s norm {ctx.template_norm:.4f}", flush=True)
    parts, q, sh = api.make_particles(tmpl, P, 1000, 3, 0.1, 60.0)
    torch.cuda.synchronize()
    cfg = api.make_config(bands=(4, 8, 16), max_candidates=24, shift_radius=4, shift_step=2)
    ctx.align_batch(parts[:4], cfg)  # warm-up
    ctx.set_timing(True)
    ctx.timings(reset=True)
    torch.cuda.synchronize()
    t0 = time.time()
    res = ctx.align_batch(parts, cfg)
    torch.cuda.synchronize()
    dt = time.time() - t0
    ms, cnt = ctx.timings(reset=True)
    print(f"P={P}: {dt:.3f}s  {P/dt:.1f} particles/s", flush=True)
    print("kernel ms:", {k: round(v, 2) for k, v in ms.items()}, cnt, flush=True)
    errs = [geod(r["quat"], q[i]) for i, r in enumerate(res)]
    shifts_ok = sum(tuple(r["shift"]) == tuple(sh[i]) for i, r in enumerate(res))
    print(f"shift exact {shifts_ok}/{P}; rot err median {np.median(errs):.3f} p90 {np.percentile(errs,90):.3f} "
          f"max {max(errs):.2f}; converged {sum(r['converged'] for r in res)}/{P}; "
          f"evals/particle {np.mean([r['evaluations'] for r in res]):.0f} windows {res[0]['windows']}", flush=True)


if __name__ == "__main__":
    main()
