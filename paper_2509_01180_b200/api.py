"""Python mirror of the reference's alignment API over the C ABI (libballmatch_b200).

Names and argument meaning follow the reference headers (proj/include/ballmatch):
``build_spec`` -> :class:`Context` (basis + operator for an n^3 grid on one
device), ``expand``, ``align`` / ``align_batch``, ``average``.  Errors map back
to the reference's exception types: ValueError for std::invalid_argument,
ArithmeticError for std::domain_error.

Device buffers are torch CUDA tensors; host numpy arrays are accepted where the
reference takes a Volume and are copied in.  There is no CPU implementation:
without a CUDA device every call raises.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise _lib.BallmatchError("libballmatch_b200 needs a CUDA device (no CPU fallback)")
    return torch


def default_lambda_cut(n: int, l_max: int) -> float:
    """default_lambda_cut (src/basis.cpp:117-138)."""
    return _lib.lib().bm_default_lambda_cut(n, l_max)


class Context:
    """Basis + pulled-back operator for an n^3 grid, resident on one device."""

    def __init__(self, n: int, l_max: int, lambda_cut: float = 0.0, device: int = 0):
        L = _lib.lib()
        h = C.c_void_p()
        _lib.check(L.bm_context_create(device, n, l_max, lambda_cut, C.byref(h)), "build_spec")
        self._h = h
        self.device = device
        info = (C.c_longlong * 10)()
        L.bm_context_info(self._h, info)
        (self.n, self.l_max, self.coeff_count, self.support, self.m_pad, self.k_pad, self.n_r,
         self.n_theta, self.n_phi, self.pair_count) = (int(v) for v in info)
        self.lambda_cut = L.bm_context_lambda_cut(self._h)

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().bm_context_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # BasisSpec accessors (include/ballmatch/basis.hpp:36-47)
    def radial_count(self, l: int) -> int:
        return _lib.lib().bm_context_roots(self._h, l, None, None)

    def roots(self, l: int):
        k = self.radial_count(l)
        r = (C.c_double * max(k, 1))()
        nm = (C.c_double * max(k, 1))()
        _lib.lib().bm_context_roots(self._h, l, r, nm)
        return np.array(r[:k]), np.array(nm[:k])

    def block_offset(self, l: int) -> int:
        return sum(self.radial_count(j) * (2 * j + 1) for j in range(l))

    def index_of(self, k: int, l: int, m: int) -> int:
        return self.block_offset(l) + (k - 1) * (2 * l + 1) + (m + l)

    # ------------------------------------------------------------------ expand
    def expand(self, vols, shifts=None):
        """expand(shift_volume(v, s)) for a batch: vols (count, n, n, n) float32 on the
        device (or numpy, copied in) -> complex128 (count, coeff_count) on the device."""
        torch = _torch()
        v = vols if isinstance(vols, torch.Tensor) else torch.as_tensor(np.asarray(vols))
        if v.dim() == 3:
            v = v.unsqueeze(0)
        v = v.to(device=f"cuda:{self.device}", dtype=torch.float32).contiguous()
        count = v.shape[0]
        out = torch.empty((count, self.coeff_count, 2), dtype=torch.float64, device=v.device)
        sh = None
        if shifts is not None:
            s = np.ascontiguousarray(np.asarray(shifts, dtype=np.int32).reshape(count, 3))
            sh = s.ctypes.data_as(C.c_void_p)
        stream = torch.cuda.current_stream(v.device).cuda_stream
        _lib.check(_lib.lib().bm_expand(self._h, C.c_void_p(v.data_ptr()), count, sh,
                                        C.c_void_p(out.data_ptr()), C.c_void_p(stream)), "expand")
        return torch.view_as_complex(out)
