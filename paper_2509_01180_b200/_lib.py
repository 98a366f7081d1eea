"""ctypes loader for libballmatch_b200.so (the C ABI in include/ballmatch_b200.h).

The product path has no CPU fallback: if the shared library is missing or a
CUDA device is absent, calls raise instead of degrading silently.
"""
from __future__ import annotations

import ctypes as C
import os
import re
from pathlib import Path

PKG = Path(__file__).resolve().parent
# BMB_LIB: alternative build of the same library (variant experiments, tools/build_variant.py)
LIB_PATH = Path(os.environ["BMB_LIB"]) if os.environ.get("BMB_LIB") else PKG / "libballmatch_b200.so"
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


class AlignConfig(C.Structure):
    """bm_align_config: OptimizerConfig (include/ballmatch/optimize.hpp:15-32)."""
    _fields_ = [("n_bands", C.c_int), ("bands", C.c_int * 16), ("seed_grid_step", C.c_double),
                ("max_candidates", C.c_int), ("newton_max_iter", C.c_int),
                ("grad_tol", C.c_double), ("step_damping", C.c_double),
                ("shift_radius", C.c_int), ("shift_step", C.c_int), ("accept_tol", C.c_double),
                ("auto_bands", C.c_int), ("prune_after_band", C.c_int), ("n_thresholds", C.c_int),
                ("thresholds", C.c_double * 8)]


class AlignResult(C.Structure):
    _fields_ = [("shift", C.c_int * 3), ("quat", C.c_double * 4), ("score", C.c_double),
                ("converged", C.c_int), ("candidates", C.c_longlong),
                ("evaluations", C.c_longlong), ("subtomo_norm", C.c_double),
                ("windows", C.c_int), ("n_bands", C.c_int), ("bands", C.c_int * 16),
                ("evaluations_per_band", C.c_longlong * 16), ("expand_template_s", C.c_double),
                ("coarse_search_s", C.c_double), ("fine_search_s", C.c_double)]


class WindowResult(C.Structure):
    _fields_ = [("volume", C.c_int), ("shift", C.c_int * 3), ("valid", C.c_int),
                ("n_candidates", C.c_int), ("converged", C.c_int), ("raw_score", C.c_double),
                ("norm_score", C.c_double), ("subtomo_norm", C.c_double),
                ("quat", C.c_double * 4), ("evaluations", C.c_longlong)]


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
    L.bm_expand_windows.argtypes = [P, P, I, P, P, I, P, P]
    L.bm_expand_windows.restype = I
    L.bm_set_template.argtypes = [P, P, D, P]
    L.bm_set_template.restype = I
    L.bm_template_norm.argtypes = [P]
    L.bm_template_norm.restype = D
    L.bm_align_batch.argtypes = [P, P, I, C.POINTER(AlignConfig), C.POINTER(AlignResult), P]
    L.bm_align_batch.restype = I
    L.bm_search_windows.argtypes = [P, P, I, P, P, I, C.POINTER(AlignConfig),
                                    C.POINTER(WindowResult), P]
    L.bm_search_windows.restype = I
    L.bm_eval_sweep.argtypes = [P, P, I, P, P, I, I, P, P]
    L.bm_eval_sweep.restype = I
    L.bm_apply_wedge_taper.argtypes = [P, P, P, I, P]
    L.bm_apply_wedge_taper.restype = I
    L.bm_average_accumulate.argtypes = [P, P, I, P, P, P]
    L.bm_average_accumulate.restype = I
    L.bm_context_set_timing.argtypes = [P, I]
    L.bm_context_set_timing.restype = I
    L.bm_context_timings.argtypes = [P, P, P, I]
    L.bm_context_timings.restype = I
    L.bm_synthesize.argtypes = [P, P, I, I, P, P]
    L.bm_synthesize.restype = I
    L.bm_context_set_lanes.argtypes = [P, I, I]
    L.bm_context_set_lanes.restype = I
    L.bm_context_eval_counts.argtypes = [P, I, P]
    L.bm_context_eval_counts.restype = I
    L.bm_context_band_timings.argtypes = [P, P]
    L.bm_context_band_timings.restype = I
    L.bm_context_set_expand_mode.argtypes = [P, I]
    L.bm_context_set_expand_mode.restype = I
    L.bm_eval_sweep_tc.argtypes = [P, P, I, P, P, I, P, P, P]
    L.bm_eval_sweep_tc.restype = I
    L.bm_xi_coefficients.argtypes = [P, P, I, P, P, P]
    L.bm_xi_coefficients.restype = I
    L.bm_xi_compose_right.argtypes = [P, P, P, I, P, P]
    L.bm_xi_compose_right.restype = I
    L.bm_rotate_expansion.argtypes = [P, P, P, P, P]
    L.bm_rotate_expansion.restype = I
    L.bm_wigner_D.argtypes = [I, P, P]
    L.bm_wigner_D.restype = I
    L.bm_exhaustive_baseline.argtypes = [P, P, I, D, P, P, P, P]
    L.bm_exhaustive_baseline.restype = I
    L.bm_baseline_evaluation_count.argtypes = [D]
    L.bm_baseline_evaluation_count.restype = C.c_longlong
    L.bm_basis_roots.argtypes = [I, D, I, P, P, P]
    L.bm_basis_roots.restype = I
    L.bm_objective_eval.argtypes = [P, P, P, P, P, I, I, I, P, P]
    L.bm_objective_eval.restype = I
    L.bm_seed_candidates.argtypes = [P, P, I, I, D, I, P, P, P, P]
    L.bm_seed_candidates.restype = I
    L.bm_template_coeffs.argtypes = [P, P, P]
    L.bm_template_coeffs.restype = I
    L.bm_wedge_power_kernel.argtypes = [P, P]
    L.bm_wedge_power_kernel.restype = I
    L.bm_context_set_expand_pairs.argtypes = [P, I]
    L.bm_context_set_expand_pairs.restype = I
    L.bm_context_set_stage_reuse.argtypes = [P, I]
    L.bm_context_set_stage_reuse.restype = I
    L.bm_context_eval_stats.argtypes = [P, P, P, I]
    L.bm_context_eval_stats.restype = I
    L.bm_make_template.argtypes = [I, I, I, C.c_ulonglong, P, P]
    L.bm_make_template.restype = I
    L.bm_make_particles.argtypes = [I, P, I, I, C.c_ulonglong, I, D, D, P, P, P, P]
    L.bm_make_particles.restype = I


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = lib().bm_last_error().decode()
        if rc == 1:
            raise ValueError(f"{what}: {msg}")
        if rc == 3:
            raise ArithmeticError(f"{what}: {msg}")
        raise BallmatchError(f"{what}: status {rc}: {msg}")
