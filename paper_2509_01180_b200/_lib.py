"""ctypes loader for libballmatch_b200.so (the C ABI in include/ballmatch_b200.h).

The product path has no CPU fallback: if the shared library is missing or a
CUDA device is absent, calls raise instead of degrading silently.
"""
from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libballmatch_b200.so"
HEADER = PKG.parent / "include" / "ballmatch_b200.h"

_lib = None


class BallmatchError(RuntimeError):
    pass


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise BallmatchError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2509_01180_b200.build`")
        _lib = C.CDLL(str(LIB_PATH))
        _declare(_lib)
    return _lib


def declared_symbols() -> list[str]:
    """Every bm_* function declared in include/ballmatch_b200.h."""
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(bm_[a-z0-9_]+)\s*\(", text)))


P = C.c_void_p
I = C.c_int
LL = C.c_longlong
D = C.c_double


def _declare(L: C.CDLL) -> None:
    L.bm_last_error.restype = C.c_char_p
    L.bm_abi_version.restype = I
    L.bm_split3_gemm.argtypes = [I, I, I, P, P, P, P, P, LL, LL, LL, LL, I, I, P, P, P]
    L.bm_split3_gemm.restype = I
    L.bm_context_create.argtypes = [I, I, I, D, C.POINTER(C.c_void_p)]
    L.bm_context_create.restype = I
    L.bm_context_destroy.argtypes = [P]
    L.bm_context_destroy.restype = I
    L.bm_context_info.argtypes = [P, P]
    L.bm_context_info.restype = I
    L.bm_context_lambda_cut.argtypes = [P]
    L.bm_context_lambda_cut.restype = D
    L.bm_context_roots.argtypes = [P, I, P, P]
    L.bm_context_roots.restype = I
    L.bm_default_lambda_cut.argtypes = [I, I]
    L.bm_default_lambda_cut.restype = D
    L.bm_expand.argtypes = [P, P, I, P, P, P]
    L.bm_expand.restype = I


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = lib().bm_last_error().decode()
        if rc == 1:
            raise ValueError(f"{what}: {msg}")
        if rc == 3:
            raise ArithmeticError(f"{what}: {msg}")
        raise BallmatchError(f"{what}: status {rc}: {msg}")
