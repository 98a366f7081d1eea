"""Does the FP16 tcgen05 path keep subnormal inputs?  Compare split errors on data
whose magnitudes span 1e-6..1 (lo parts deep in the FP16 subnormal range)."""
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
    _lib.check(_lib.lib().bm_split3_gemm(fmt, 128, kchunk, ahi.data_ptr(), alo.data_ptr(),
                                         bhi.data_ptr(), blo.data_ptr(), out.data_ptr(), m, m, n,
                                         k, m, n, None, None, None))
    torch.cuda.synchronize()
    return out.double().cpu()


g = torch.Generator().manual_seed(1)
m = n = 128
k = 4096
for span in (0, 2, 4, 6):
    a = torch.randn(m, k, generator=g, dtype=torch.float64) * 10 ** (-span * torch.rand(m, k, generator=g, dtype=torch.float64))
    b = torch.randn(n, k, generator=g, dtype=torch.float64) * 10 ** (-span * torch.rand(n, k, generator=g, dtype=torch.float64))
    a /= a.abs().max(); b /= b.abs().max()
    ref = b @ a.T
    for fmt, split in ((0, split_f16), (2, split_tf32)):
        ahi, alo = split(a); bhi, blo = split(b)
        rep = bhi.double() @ ahi.double().T + blo.double() @ ahi.double().T + bhi.double() @ alo.double().T
        o = run(fmt, ahi.cuda(), alo.cuda(), bhi.cuda(), blo.cuda())
        e = ((o - ref).norm() / ref.norm()).item()
        er = ((rep - ref).norm() / ref.norm()).item()
        if fmt == 0:
            ftz = lambda t: torch.where(t.abs() < 6.103515625e-05, torch.zeros_like(t), t)
            repf = ftz(bhi).double() @ ftz(ahi).double().T + ftz(blo).double() @ ftz(ahi).double().T + ftz(bhi).double() @ ftz(alo).double().T
            ef = ((repf - ref).norm() / ref.norm()).item()
        else:
            ef = float('nan')
        print(f"span=1e-{span} fmt={fmt}: gpu {e:.2e}  exact-parts {er:.2e}  if-FTZ {ef:.2e}")
