"""C ABI checks that need no GPU: the library loads, exports every symbol the
header declares, and refuses to run (loudly) without a CUDA device."""
import ctypes as C
import math

import numpy as np
import pytest

from oracle import bmo
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


@pytest.mark.parametrize("l_max,cut", [(8, 8 * math.pi), (16, 16 * math.pi), (20, 20 * math.pi),
                                       (24, 24 * math.pi), (42, 32 * math.pi), (42, 42 * math.pi),
                                       (1, 4.0), (0, 7.0)])
def test_host_basis_roots_match_oracle(l_max, cut):
    """The product's host basis setup (its own Bessel zeros and norms) against the
    oracle's build_spec: the same index set, roots within 5e-14 and norms within
    1e-12 (the oracle stops its Newton iteration at ~1e-14 relative, and the norm
    c = sqrt(2)/|j_{l+1}(lambda)| moves ~20x the root error); and against 40-digit
    mpmath values of the zeros and norms within 4 ulp-scale (1e-15 relative)."""
    from paper_2509_01180_b200 import api
    spec = bmo.Spec(l_max, cut)
    try:
        import mpmath
        mpmath.mp.dps = 40
    except ImportError:  # pragma: no cover
        mpmath = None
    for l in range(l_max + 1):
        r, nm = api.basis_roots(l_max, cut, l)
        assert len(r) == spec.radial_count(l), (l, len(r), spec.radial_count(l))
        for k in range(len(r)):
            assert r[k] == pytest.approx(spec.root(l, k + 1), rel=5e-14)
            assert nm[k] == pytest.approx(spec.norm(l, k + 1), rel=1e-12)
            if mpmath is not None and (k % 5 == 0 or l % 7 == 0):
                x = mpmath.findroot(lambda t: mpmath.besselj(l + 0.5, t), mpmath.mpf(r[k]))
                assert r[k] == pytest.approx(float(x), rel=1e-15, abs=0)
                j = mpmath.sqrt(mpmath.pi / (2 * x)) * mpmath.besselj(l + 1.5, x)
                assert nm[k] == pytest.approx(float(mpmath.sqrt(2) / abs(j)), rel=2e-15)


def test_host_basis_rejects_bad_specs():
    from paper_2509_01180_b200 import api
    with pytest.raises(ValueError):
        api.basis_roots(1, 3.0, 0)  # lambda_cut < pi drops the (0,1) root
    with pytest.raises(ValueError):
        api.basis_roots(4, 8.0, 5)
    r, _ = api.basis_roots(1, 4.0, 1)
    assert len(r) == 0  # (1, 4): degree 1 has no root below 4


def test_host_wigner_D_and_grid_count_match_oracle():
    """wigner_D (steer.cpp:158-178) on the host and the baseline grid count
    (optimize.cpp:541-544: ceil(2 pi/s)^2 (ceil(pi/s) + 1))."""
    from paper_2509_01180_b200 import api
    for s in range(3):
        q = bmo.haar_rotation(5, s)
        got = api.wigner_D(12, q)
        ref = bmo.wigner_D(12, q)
        assert np.abs(got - ref).max() <= 1e-12
    for deg in (5.0, 6.0, 22.5, 0.5):
        st = deg * math.pi / 180.0
        na, nb = math.ceil(2 * math.pi / st), math.ceil(math.pi / st) + 1
        assert api.baseline_evaluation_count(st) == na * na * nb == bmo.baseline_evaluation_count(st)


def test_expand_entry_points_reject_a_null_context():
    """bm_expand / bm_expand_windows without a context: an error code, no crash
    (the argument checks run before any device call)."""
    L = _lib.lib()
    assert L.bm_expand(None, None, 0, None, None, None) != 0
    assert L.bm_expand_windows(None, None, 0, None, None, 0, None, None) != 0
