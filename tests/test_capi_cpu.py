"""C ABI checks that need no GPU: the library loads, exports every symbol the
header declares, and refuses to run (loudly) without a CUDA device."""
import ctypes as C
import math

import pytest

from paper_2509_01180_b200 import _lib


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    syms = _lib.declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), s
    assert L.bm_abi_version() == 3


def test_default_lambda_cut_host_metadata():
    from oracle import bmo
    for n, Lm in ((32, 8), (48, 16), (64, 24)):
        assert _lib.lib().bm_default_lambda_cut(n, Lm) == pytest.approx(
            bmo.default_lambda_cut(n, Lm), rel=1e-15)


def test_context_without_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    h = C.c_void_p()
    rc = _lib.lib().bm_context_create(0, 32, 8, 8 * math.pi, C.byref(h))
    assert rc == 2 and not h.value
    assert b"CUDA" in _lib.lib().bm_last_error()
