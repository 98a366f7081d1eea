"""Split-precision tcgen05 GEMM (kernel K2 building block) vs an FP64 matmul."""
import ctypes as C

import numpy as np
import pytest

from paper_2509_01180_b200 import _lib
from paper_2509_01180_b200.splits import split_tf32, split_f16

pytestmark = pytest.mark.gpu


def _run(fmt, block_n, m, n, k, m_valid=None, n_valid=None, seed=0):
    import torch
    g = torch.Generator().manual_seed(seed)
    a = torch.randn(m, k, generator=g, dtype=torch.float64)
    b = torch.randn(n, k, generator=g, dtype=torch.float64)
    m_valid = m if m_valid is None else m_valid
    n_valid = n if n_valid is None else n_valid
    split = split_tf32 if fmt == 2 else split_f16
    ahi, alo = split(a)
    bhi, blo = split(b)
    ahi, alo, bhi, blo = (t.cuda() for t in (ahi, alo, bhi, blo))
    out = torch.full((n, m), float("nan"), dtype=torch.float32, device="cuda")
    rc = _lib.lib().bm_split3_gemm(fmt, block_n, 4, ahi.data_ptr(), alo.data_ptr(), bhi.data_ptr(),
                                   blo.data_ptr(), out.data_ptr(), m, m, n, k, m_valid, n_valid,
                                   None, None, None)
    _lib.check(rc, "bm_split3_gemm")
    torch.cuda.synchronize()
    ref = (b @ a.T)
    return out.cpu().double(), ref, m_valid, n_valid


@pytest.mark.parametrize("fmt,block_n", [(2, 128), (2, 256), (0, 128), (0, 256)])
def test_split3_gemm_accuracy(cuda_device, fmt, block_n):
    out, ref, mv, nv = _run(fmt, block_n, 256, 512, 1024)
    err = (out - ref).norm() / ref.norm()
    assert err < 2e-6, f"rel L2 {err:.3e}"


def test_split3_gemm_ragged_valid(cuda_device):
    out, ref, mv, nv = _run(2, 128, 256, 256, 512, m_valid=200, n_valid=130)
    sub = out[:nv, :mv]
    err = (sub - ref[:nv, :mv]).norm() / ref[:nv, :mv].norm()
    assert err < 2e-6
    assert torch_isnan_all(out[nv:, :]) and torch_isnan_all(out[:, mv:])


def torch_isnan_all(t):
    import torch
    return bool(torch.isnan(t).all()) if t.numel() else True
