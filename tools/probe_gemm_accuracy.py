"""Accuracy probe of the split tcgen05 GEMM: separates accumulation error from split error."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

from paper_2509_01180_b200 import _lib
from paper_2509_01180_b200.splits import split_f16, split_tf32


def run(fmt, ahi, alo, bhi, blo, kchunk=4):
    m, k = ahi.shape
    n = bhi.shape[0]
    out = torch.empty(n, m, device="cuda")
    rc = _lib.lib().bm_split3_gemm(fmt, 128, kchunk, ahi.data_ptr(), alo.data_ptr(), bhi.data_ptr(),
                                   blo.data_ptr(), out.data_ptr(), m, m, n, k, m, n, None, None,
                                   None)
    _lib.check(rc)
    torch.cuda.synchronize()
    return out.double().cpu()


def main():
    m, n = 128, 128
    for k in (64, 1024, 16384, 89600):
        g = torch.Generator().manual_seed(k)
        a = torch.randn(m, k, generator=g, dtype=torch.float64)
        b = torch.randn(n, k, generator=g, dtype=torch.float64)
        for fmt, split in ((2, split_tf32), (0, split_f16)):
            ahi, alo = split(a)
            bhi, blo = split(b)
            # (1) exact hi-only inputs: pure accumulation error
            z_a = torch.zeros_like(alo)
            z_b = torch.zeros_like(blo)
            ref_hi = bhi.double() @ ahi.double().T
            o1 = run(fmt, ahi.cuda(), z_a.cuda(), bhi.cuda(), z_b.cuda(), 0)
            e1 = ((o1 - ref_hi).norm() / ref_hi.norm()).item()
            # fp32 sequential-order reference accumulation error for comparison
            ref32 = (bhi.float() @ ahi.float().T).double()
            e32 = ((ref32 - ref_hi).norm() / ref_hi.norm()).item()
            # (2) full split vs fp64
            ref = b @ a.T
            e2 = {}
            for kc in (1, 2, 4, 8, 0):
                o2 = run(fmt, ahi.cuda(), alo.cuda(), bhi.cuda(), blo.cuda(), kc)
                e2[kc] = ((o2 - ref).norm() / ref.norm()).item()
            # (3) split representation error alone (fp64 math on the parts)
            rep = (bhi.double() @ ahi.double().T + blo.double() @ ahi.double().T +
                   bhi.double() @ alo.double().T)
            e3 = ((rep - ref).norm() / ref.norm()).item()
            print(f"k={k:6d} fmt={fmt}: accum-only {e1:.2e} (torch fp32 {e32:.2e}); "
                  "split3 by kchunk " + " ".join(f"{kc}:{v:.2e}" for kc, v in e2.items()) +
                  f"; representation {e3:.2e}")


if __name__ == "__main__":
    main()
