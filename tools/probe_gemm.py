"""Timing probe for the split-precision tcgen05 GEMM at expansion shapes.

Prints one line per (fmt, block_n, kchunk): ms and dense-equivalent TFLOP/s (3 passes).
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

from paper_2509_01180_b200 import _lib


def main():
    m, n, k = 3072, int(sys.argv[1]) if len(sys.argv) > 1 else 2048, 89600
    L = _lib.lib()
    for fmt in (0, 2):
        dt = torch.float32 if fmt == 2 else torch.float16
        ahi = torch.randn(m, k, device="cuda").to(dt)
        alo = (torch.randn(m, k, device="cuda") * 1e-4).to(dt)
        bhi = torch.randn(n, k, device="cuda").to(dt)
        blo = (torch.randn(n, k, device="cuda") * 1e-4).to(dt)
        out = torch.empty(n, m, device="cuda")
        for bn in (64, 128):
            for kc in (1, 2, 4, 8, 0):
                def run():
                    rc = L.bm_split3_gemm(fmt, bn, kc, ahi.data_ptr(), alo.data_ptr(),
                                          bhi.data_ptr(), blo.data_ptr(), out.data_ptr(), m, m, n,
                                          k, m, n, None, None, None)
                    _lib.check(rc, "gemm")
                for _ in range(2):
                    run()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                reps = 4
                e0.record()
                for _ in range(reps):
                    run()
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / reps
                tf = 3 * 2.0 * m * n * k / (ms * 1e-3) / 1e12
                print(f"fmt={fmt} block_n={bn} kchunk={kc} M={m} N={n} K={k}: {ms:.3f} ms  "
                      f"{tf:.1f} TFLOP/s (3-pass)", flush=True)
        del ahi, alo, bhi, blo


if __name__ == "__main__":
    main()
