"""Per-phase cycle profile of the fused refinement kernel (variant build with
-DBMB_FUSED_PROF):  python tools/build_variant.py prof -DBMB_FUSED_PROF
BMB_LIB=build/variants/prof.so python tools/probe_fused.py 128"""
import ctypes as C
import math
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2509_01180_b200 import _lib, api

NAMES = ["xi_build", "compose", "eval2", "step", "eval0", "accept", "final", "barrier", "iter_begin",
         "n_compose", "n_windows", "n_iters"]


def main():
    P = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    ctx = api.Context(64, 16, 16 * math.pi)
    tmpl = api.make_template(64, 40, 7)
    ctx.set_template(tmpl, 60.0)
    parts, q, sh = api.make_particles(tmpl, P, 1000, 3, 0.1, 60.0)
    cfg = api.make_config(bands=(4, 8, 16), max_candidates=24, shift_radius=4, shift_step=2)
    ctx.set_lanes(1, 64)
    ctx.align_batch(parts[:8], cfg)
    lib = _lib.lib()
    f = lib.bmb_fused_profile
    f.argtypes = [C.c_void_p, C.c_int]
    buf = (C.c_ulonglong * 16)()
    f(buf, 1)
    for mode in ("fused", "lists"):
        ctx.set_refine_mode(mode)
        ctx.set_timing(True)
        ctx.timings(reset=True)
        torch.cuda.synchronize()
        t0 = time.time()
        ctx.align_batch(parts, cfg)
        torch.cuda.synchronize()
        dt = time.time() - t0
        ms, cnt = ctx.timings(reset=True)
        print(f"{mode}: {dt*1e3:.1f} ms for {P} particles; refine {ms['refine']:.1f} ms expand {ms['expand']:.1f}"
              f" eval2 {ms['eval_order2']:.1f} eval0 {ms['eval_order0']:.1f} compose {ms['compose']:.1f}"
              f" newton {ms['newton']:.1f} xi {ms['xi_build']:.1f}", flush=True)
        ctx.set_timing(False)
        if mode == "fused":
            f(buf, 1)
            tot = sum(buf[i] for i in range(9))
            for i, n in enumerate(NAMES):
                v = buf[i]
                extra = f" ({100.0 * v / tot:.1f}%)" if i < 9 else ""
                print(f"  {n:12s} {v:16d}{extra}")
            print(f"  cycles per compose {buf[1] / max(1, buf[9]):.0f}, per window {tot / max(1, buf[10]):.0f}")


if __name__ == "__main__":
    main()
