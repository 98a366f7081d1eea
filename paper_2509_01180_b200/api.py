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
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise _lib.BallmatchError("libballmatch_b200 needs a CUDA device (no CPU fallback)")
    return torch


# FP32 evaluation: acceptance slack of the Newton line test and gradient
# tolerance floor (the reference's 1e-12 / 1e-7 assume FP64 scores)
FP32_ACCEPT_TOL = 1e-6
FP32_GRAD_TOL = 1e-5


def make_config(bands=(7, 12, 33), seed_grid_step=np.pi / 8, max_candidates=20,
                newton_max_iter=30, grad_tol=1e-7, step_damping=1e-3, shift_radius=4,
                shift_step=2, accept_tol=None, auto_bands=False, prune_after_band=False,
                band_thresholds=(0.5, 0.25, 0.05)) -> _lib.AlignConfig:
    """OptimizerConfig defaults (include/ballmatch/optimize.hpp:15-32); grad_tol is
    floored at the FP32 evaluation's resolution unless accept_tol is given explicitly."""
    c = _lib.AlignConfig()
    c.auto_bands = 1 if auto_bands else 0
    c.prune_after_band = 1 if prune_after_band else 0
    c.n_thresholds = len(band_thresholds)
    for i, t in enumerate(band_thresholds):
        c.thresholds[i] = float(t)
    c.n_bands = len(bands)
    for i, b in enumerate(bands):
        c.bands[i] = int(b)
    c.seed_grid_step = seed_grid_step
    c.max_candidates = max_candidates
    c.newton_max_iter = newton_max_iter
    c.grad_tol = max(grad_tol, FP32_GRAD_TOL) if accept_tol is None else grad_tol
    c.step_damping = step_damping
    c.shift_radius = shift_radius
    c.shift_step = shift_step
    c.accept_tol = FP32_ACCEPT_TOL if accept_tol is None else accept_tol
    return c


def default_lambda_cut(n: int, l_max: int) -> float:
    """default_lambda_cut (src/basis.cpp:117-138)."""
    return _lib.lib().bm_default_lambda_cut(n, l_max)


def make_template(n: int, blobs: int, seed: int, device: int = 0):
    """BASELINE template model on the device (float32 (n, n, n) tensor)."""
    torch = _torch()
    out = torch.empty((n, n, n), dtype=torch.float32, device=f"cuda:{device}")
    stream = torch.cuda.current_stream(out.device).cuda_stream
    _lib.check(_lib.lib().bm_make_template(device, n, blobs, seed, C.c_void_p(out.data_ptr()),
                                           C.c_void_p(stream)), "make_template")
    return out


def basis_roots(l_max: int, lambda_cut: float, l: int):
    """Host basis setup (build_spec): roots lambda_lk <= lambda_cut of degree l and
    their norms, as numpy arrays; no device needed."""
    cap = int(lambda_cut / math.pi) + 2
    r = np.zeros(cap)
    nm = np.zeros(cap)
    cnt = C.c_int(0)
    _lib.check(_lib.lib().bm_basis_roots(int(l_max), float(lambda_cut), int(l), r.ctypes.data_as(C.c_void_p),
                                         nm.ctypes.data_as(C.c_void_p), C.byref(cnt)), "basis_roots")
    return r[:cnt.value].copy(), nm[:cnt.value].copy()


def xi_count(L: int) -> int:
    return (L + 1) * (2 * L + 1) * (2 * L + 3) // 3


def wigner_D(L: int, quat):
    """wigner_D (src/steer.cpp:158-178) for degrees <= L: XiBlocks layout, numpy complex128."""
    q = np.ascontiguousarray(quat, dtype=np.float64)
    out = np.zeros(2 * xi_count(L))
    _lib.check(_lib.lib().bm_wigner_D(int(L), q.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p)),
               "wigner_D")
    return out.view(np.complex128)


def baseline_evaluation_count(step: float) -> int:
    """baseline_evaluation_count (src/optimize.cpp:541-544)."""
    return int(_lib.lib().bm_baseline_evaluation_count(float(step)))


def make_particles(tmpl, count: int, base_seed: int, shift_max: int, snr=None, wedge_deg=None):
    """Particles of a BASELINE config on the device: (count, n, n, n) float32 tensor plus
    the ground truth (quaternions (count, 4), shifts (count, 3))."""
    torch = _torch()
    n = tmpl.shape[-1]
    out = torch.empty((count, n, n, n), dtype=torch.float32, device=tmpl.device)
    q = np.zeros((count, 4))
    sh = np.zeros((count, 3), dtype=np.int32)
    stream = torch.cuda.current_stream(out.device).cuda_stream
    _lib.check(_lib.lib().bm_make_particles(
        tmpl.device.index or 0, C.c_void_p(tmpl.contiguous().data_ptr()), n, count, base_seed,
        shift_max, snr or 0.0, wedge_deg or 0.0, C.c_void_p(out.data_ptr()),
        q.ctypes.data_as(C.c_void_p), sh.ctypes.data_as(C.c_void_p), C.c_void_p(stream)),
        "make_particles")
    return out, q, sh


class Context:
    """Basis + pulled-back operator for an n^3 grid, resident on one device."""

    def __init__(self, n: int, l_max: int, lambda_cut: float = 0.0, device: int = 0):
        L = _lib.lib()
        h = C.c_void_p()
        _lib.check(L.bm_context_create(device, n, l_max, lambda_cut, C.byref(h)), "build_spec")
        self._h = h
        self.device = device
        self._refresh_info()
        self.lambda_cut = L.bm_context_lambda_cut(self._h)

    def _refresh_info(self):
        info = (C.c_longlong * 10)()
        _lib.lib().bm_context_info(self._h, info)
        (self.n, self.l_max, self.coeff_count, self.support, self.m_pad, self.k_pad, self.n_r,
         self.n_theta, self.n_phi, self.pair_count) = (int(v) for v in info)

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

    def expand_windows(self, vols, win_vol, shifts):
        """expand(shift_volume(vols[win_vol[w]], shifts[w])) for every window w (the
        shift search's expansions: many windows per volume) -> complex128
        (n_win, coeff_count) on the device."""
        torch = _torch()
        v = self._dev(vols)
        wv = np.ascontiguousarray(np.asarray(win_vol, dtype=np.int32))
        s = np.ascontiguousarray(np.asarray(shifts, dtype=np.int32).reshape(len(wv), 3))
        out = torch.empty((len(wv), self.coeff_count, 2), dtype=torch.float64, device=v.device)
        _lib.check(_lib.lib().bm_expand_windows(self._h, C.c_void_p(v.data_ptr()), v.shape[0],
                                                wv.ctypes.data_as(C.c_void_p), s.ctypes.data_as(C.c_void_p), len(wv),
                                                C.c_void_p(out.data_ptr()), self._stream(v)), "expand_windows")
        return torch.view_as_complex(out)

    # ------------------------------------------------------------------ align
    def _dev(self, vols):
        torch = _torch()
        v = vols if isinstance(vols, torch.Tensor) else torch.as_tensor(np.asarray(vols))
        if v.dim() == 3:
            v = v.unsqueeze(0)
        return v.to(device=f"cuda:{self.device}", dtype=torch.float32).contiguous()

    def _stream(self, t):
        dev = t.device if t.device.type == "cuda" else _torch().device(f"cuda:{self.device}")
        return C.c_void_p(_torch().cuda.current_stream(dev).cuda_stream)

    def _particles(self, vols):
        """float32 particle batch for bm_align_batch / bm_average_accumulate: CPU
        tensors (pinned for overlap) and arrays stay in host memory, the library
        stages them per lane; anything else goes to the context's device."""
        torch = _torch()
        v = vols if isinstance(vols, torch.Tensor) else torch.as_tensor(np.asarray(vols))
        if v.dim() == 3:
            v = v.unsqueeze(0)
        if v.device.type == "cpu":
            return v.to(dtype=torch.float32).contiguous()
        return v.to(device=f"cuda:{self.device}", dtype=torch.float32).contiguous()

    def set_template(self, tmpl, wedge_theta_deg: float = 0.0):
        """Template state of align() (src/optimize.cpp:438-454)."""
        t = self._dev(tmpl)
        _lib.check(_lib.lib().bm_set_template(self._h, C.c_void_p(t.data_ptr()), wedge_theta_deg,
                                              self._stream(t)), "set_template")
        self.template_norm = _lib.lib().bm_template_norm(self._h)
        self.wedge_theta_deg = wedge_theta_deg

    def align_batch(self, particles, cfg: _lib.AlignConfig):
        """align() for every particle of the batch (device or host tensor); list of
        dicts (AlignmentResult)."""
        v = self._particles(particles)
        count = v.shape[0]
        out = (_lib.AlignResult * max(count, 1))()
        _lib.check(_lib.lib().bm_align_batch(self._h, C.c_void_p(v.data_ptr()), count,
                                             C.byref(cfg), out, self._stream(v)), "align")
        return [dict(shift=tuple(r.shift), quat=np.array(r.quat[:]), score=r.score,
                     converged=bool(r.converged), candidates=r.candidates,
                     evaluations=r.evaluations, subtomo_norm=r.subtomo_norm, windows=r.windows,
                     bands=[int(b) for b in r.bands[:r.n_bands]],
                     evaluations_per_band={int(r.bands[j]): int(r.evaluations_per_band[j])
                                           for j in range(r.n_bands)},
                     expand_template_s=r.expand_template_s, coarse_search_s=r.coarse_search_s,
                     fine_search_s=r.fine_search_s)
                for r in out[:count]]

    def average_accumulate(self, particles, results, out=None):
        """Coefficient-space average numerator: out (complex128, coeff_count, device) +=
        sum_p rotate_expansion(f_hat_{p,s_p}, g_p^-1)."""
        torch = _torch()
        v = self._particles(particles)
        count = v.shape[0]
        if out is None:
            out = torch.zeros((self.coeff_count, 2), dtype=torch.float64, device=f"cuda:{self.device}")
        res = (_lib.AlignResult * max(count, 1))()
        for i, r in enumerate(results):
            for j in range(3):
                res[i].shift[j] = int(r["shift"][j])
            for j in range(4):
                res[i].quat[j] = float(r["quat"][j])
        _lib.check(_lib.lib().bm_average_accumulate(self._h, C.c_void_p(v.data_ptr()), count, res,
                                                    C.c_void_p(out.data_ptr()), self._stream(v)),
                   "average")
        return out

    def search_windows(self, vols, windows, cfg: _lib.AlignConfig):
        """search_one_shift for explicit (volume index, (sx, sy, sz)) windows."""
        v = self._dev(vols)
        n_win = len(windows)
        wv = np.ascontiguousarray([w[0] for w in windows], dtype=np.int32)
        ws = np.ascontiguousarray([w[1] for w in windows], dtype=np.int32).reshape(-1)
        out = (_lib.WindowResult * max(n_win, 1))()
        _lib.check(_lib.lib().bm_search_windows(
            self._h, C.c_void_p(v.data_ptr()), v.shape[0], wv.ctypes.data_as(C.c_void_p),
            ws.ctypes.data_as(C.c_void_p), n_win, C.byref(cfg), out, self._stream(v)),
            "search_windows")
        return [dict(volume=r.volume, shift=tuple(r.shift), valid=bool(r.valid),
                     candidates=r.n_candidates, converged=bool(r.converged),
                     raw_score=r.raw_score, norm_score=r.norm_score,
                     subtomo_norm=r.subtomo_norm, quat=np.array(r.quat[:]),
                     evaluations=r.evaluations) for r in out[:n_win]]

    def eval_sweep(self, f, t, euler, order: int = 1):
        """Rotate-score-gradient sweep (config 4): value and Euler gradient of
        C = Re sum xi D(g), xi = xi_coefficients(f_p, t), for every (p, g).
        f: complex (n_f, coeff_count), t: complex (coeff_count,), euler: (n_rot, 3);
        returns float64 (n_f, n_rot, 4) on the device."""
        torch = _torch()
        dev = torch.device(f"cuda:{self.device}")
        fa = torch.view_as_real(torch.as_tensor(f, dtype=torch.complex128)).to(dev).contiguous()
        ta = torch.view_as_real(torch.as_tensor(t, dtype=torch.complex128)).to(dev).contiguous()
        ea = torch.as_tensor(euler, dtype=torch.float64).to(dev).contiguous()
        n_f, n_rot = fa.shape[0], ea.shape[0]
        out = torch.empty((n_f, n_rot, 4), dtype=torch.float64, device=dev)
        _lib.check(_lib.lib().bm_eval_sweep(self._h, C.c_void_p(fa.data_ptr()), n_f,
                                            C.c_void_p(ta.data_ptr()), C.c_void_p(ea.data_ptr()),
                                            n_rot, order, C.c_void_p(out.data_ptr()),
                                            self._stream(out)), "eval_sweep")
        return out

    def objective_eval(self, f, euler, anchors=None, L=None, order: int = 2, t=None):
        """Objective::eval of the refinement (bm_objective_eval) on xi(f, t) (t None:
        the template) at chart angles euler (n, 3) with chart anchors (n, 4) or None;
        returns float64 numpy (n, 13): value, gradient, Hessian (row-major)."""
        torch = _torch()
        dev = torch.device(f"cuda:{self.device}")
        fa = torch.view_as_real(torch.as_tensor(f, dtype=torch.complex128)).to(dev).contiguous()
        ta = None if t is None else torch.view_as_real(torch.as_tensor(t, dtype=torch.complex128)).to(dev).contiguous()
        ea = torch.as_tensor(np.asarray(euler, dtype=np.float64).reshape(-1, 3)).to(dev).contiguous()
        aa = None if anchors is None else torch.as_tensor(np.asarray(anchors, dtype=np.float64).reshape(-1, 4)).to(dev).contiguous()
        n = ea.shape[0]
        out = torch.empty((n, 13), dtype=torch.float64, device=dev)
        _lib.check(_lib.lib().bm_objective_eval(
            self._h, C.c_void_p(fa.data_ptr()), None if ta is None else C.c_void_p(ta.data_ptr()),
            C.c_void_p(ea.data_ptr()), None if aa is None else C.c_void_p(aa.data_ptr()), n,
            self.l_max if L is None else int(L), int(order), C.c_void_p(out.data_ptr()), self._stream(out)),
            "objective_eval")
        torch.cuda.synchronize(dev)
        return out.cpu().numpy()

    def seed_candidates(self, f, L_low: int, step: float = math.pi / 8, max_candidates: int = 24):
        """seed_candidates of coefficient sets f (n_f, coeff_count) against the template:
        a list of (quaternions (count, 4), grid scores (count,)) in rank order."""
        torch = _torch()
        dev = torch.device(f"cuda:{self.device}")
        fa = torch.view_as_real(torch.as_tensor(f, dtype=torch.complex128)).to(dev).contiguous()
        if fa.dim() == 2:
            fa = fa.unsqueeze(0)
        n_f = fa.shape[0]
        q = np.zeros((n_f, max_candidates, 4))
        cnt = np.zeros(n_f, dtype=np.int32)
        sc = np.zeros((n_f, max_candidates))
        _lib.check(_lib.lib().bm_seed_candidates(
            self._h, C.c_void_p(fa.data_ptr()), n_f, int(L_low), float(step), int(max_candidates),
            q.ctypes.data_as(C.c_void_p), cnt.ctypes.data_as(C.c_void_p), sc.ctypes.data_as(C.c_void_p),
            self._stream(fa)), "seed_candidates")
        return [(q[i, :cnt[i]].copy(), sc[i, :cnt[i]].copy()) for i in range(n_f)]

    def _c128(self, x):
        torch = _torch()
        return torch.view_as_real(torch.as_tensor(np.asarray(x) if not isinstance(x, torch.Tensor) else x,
                                                  dtype=torch.complex128)).to(f"cuda:{self.device}").contiguous()

    def xi_coefficients(self, f, t):
        """xi_coefficients(f[p], t) (src/xcorr.cpp:21-50), FP64: complex (n, N_xi(l_max)) numpy."""
        torch = _torch()
        fa = self._c128(f)
        if fa.dim() == 2:
            fa = fa.unsqueeze(0)
        ta = self._c128(t)
        out = torch.empty((fa.shape[0], xi_count(self.l_max), 2), dtype=torch.float64, device=fa.device)
        _lib.check(_lib.lib().bm_xi_coefficients(self._h, C.c_void_p(fa.data_ptr()), fa.shape[0],
                                                 C.c_void_p(ta.data_ptr()), C.c_void_p(out.data_ptr()),
                                                 self._stream(out)), "xi_coefficients")
        return torch.view_as_complex(out).cpu().numpy()

    def xi_compose_right(self, xi, quat, l_limit: int = -1):
        """xi_compose_right (src/xcorr.cpp:149-155), FP64: complex N_xi(l_max) numpy."""
        torch = _torch()
        xa = self._c128(xi)
        q = np.ascontiguousarray(quat, dtype=np.float64)
        out = torch.empty_like(xa)
        _lib.check(_lib.lib().bm_xi_compose_right(self._h, C.c_void_p(xa.data_ptr()), q.ctypes.data_as(C.c_void_p),
                                                  int(l_limit), C.c_void_p(out.data_ptr()), self._stream(out)),
                   "xi_compose_right")
        return torch.view_as_complex(out).cpu().numpy()

    def rotate_expansion(self, f, quat):
        """rotate_expansion (src/steer.cpp:208-223), FP64: complex (coeff_count,) numpy."""
        torch = _torch()
        fa = self._c128(f)
        q = np.ascontiguousarray(quat, dtype=np.float64)
        out = torch.empty_like(fa)
        _lib.check(_lib.lib().bm_rotate_expansion(self._h, C.c_void_p(fa.data_ptr()), q.ctypes.data_as(C.c_void_p),
                                                  C.c_void_p(out.data_ptr()), self._stream(out)), "rotate_expansion")
        return torch.view_as_complex(out).cpu().numpy()

    def exhaustive_baseline(self, xi, l_cut: int, step: float):
        """exhaustive_baseline (src/optimize.cpp:523-539) of one kernel: (quat, score, evaluations)."""
        xa = self._c128(xi)
        q = np.zeros(4)
        sc = C.c_double()
        ev = C.c_longlong()
        _lib.check(_lib.lib().bm_exhaustive_baseline(self._h, C.c_void_p(xa.data_ptr()), int(l_cut), float(step),
                                                     q.ctypes.data_as(C.c_void_p), C.byref(sc), C.byref(ev),
                                                     self._stream(xa)), "exhaustive_baseline")
        return q, sc.value, ev.value

    def template_coeffs(self):
        """t_hat of the current template (complex128 (coeff_count,), device)."""
        torch = _torch()
        out = torch.empty((self.coeff_count, 2), dtype=torch.float64, device=f"cuda:{self.device}")
        _lib.check(_lib.lib().bm_template_coeffs(self._h, C.c_void_p(out.data_ptr()), self._stream(out)),
                   "template_coeffs")
        return torch.view_as_complex(out)

    def wedge_power_kernel(self):
        """The template's wedge-power kernel in the XiBlocks layout (numpy complex128)."""
        L = self.l_max
        nxi = (L + 1) * (2 * L + 1) * (2 * L + 3) // 3
        out = np.zeros(2 * nxi)
        _lib.check(_lib.lib().bm_wedge_power_kernel(self._h, out.ctypes.data_as(C.c_void_p)),
                   "wedge_power_kernel")
        return out.view(np.complex128)

    def eval_sweep_tc(self, f, t, euler, timing: bool = False):
        """The config-4 sweep as two tensor-core GEMMs (bm_eval_sweep_tc): same output
        as eval_sweep(order=1); with timing, also (tables ms, GEMM ms, gather ms, GEMM FLOPs)."""
        torch = _torch()
        dev = torch.device(f"cuda:{self.device}")
        fa = torch.view_as_real(torch.as_tensor(f, dtype=torch.complex128)).to(dev).contiguous()
        ta = torch.view_as_real(torch.as_tensor(t, dtype=torch.complex128)).to(dev).contiguous()
        ea = torch.as_tensor(euler, dtype=torch.float64).to(dev).contiguous()
        n_f, n_rot = fa.shape[0], ea.shape[0]
        out = torch.empty((n_f, n_rot, 4), dtype=torch.float64, device=dev)
        tm = np.zeros(4)
        _lib.check(_lib.lib().bm_eval_sweep_tc(self._h, C.c_void_p(fa.data_ptr()), n_f, C.c_void_p(ta.data_ptr()),
                                               C.c_void_p(ea.data_ptr()), n_rot, C.c_void_p(out.data_ptr()),
                                               tm.ctypes.data_as(C.c_void_p) if timing else None,
                                               self._stream(out)), "eval_sweep_tc")
        return (out, tuple(tm)) if timing else out

    def apply_wedge_taper(self, vols):
        torch = _torch()
        v = self._dev(vols)
        out = torch.empty_like(v)
        _lib.check(_lib.lib().bm_apply_wedge_taper(self._h, C.c_void_p(v.data_ptr()),
                                                   C.c_void_p(out.data_ptr()), v.shape[0],
                                                   self._stream(v)), "apply_wedge_taper")
        return out

    # ------------------------------------------------------------------ evidence
    def set_timing(self, on: bool = True):
        _lib.check(_lib.lib().bm_context_set_timing(self._h, 1 if on else 0), "set_timing")

    def synthesize(self, coeffs, n: int, real_volume: bool = True):
        """synthesize (src/basis.cpp:332-419): coefficients (complex128 (coeff_count,) or
        float64 (coeff_count, 2), device or host) -> float64 (n, n, n) voxel map on the device."""
        torch = _torch()
        dev = torch.device(f"cuda:{self.device}")
        c = torch.as_tensor(coeffs)
        if c.is_complex():
            c = torch.view_as_real(c.to(torch.complex128))
        c = c.to(device=dev, dtype=torch.float64).contiguous()
        if c.numel() != 2 * self.coeff_count:
            raise ValueError("synthesize: coefficient count does not match the basis")
        out = torch.empty((n, n, n), dtype=torch.float64, device=dev)
        _lib.check(_lib.lib().bm_synthesize(self._h, C.c_void_p(c.data_ptr()), 1 if real_volume else 0, n,
                                            C.c_void_p(out.data_ptr()), self._stream(out)), "synthesize")
        return out

    def eval_counts(self, L: int):
        """(order-2, order-0) evaluations at band L since the last eval_stats(reset=True)."""
        out = (C.c_longlong * 2)()
        _lib.check(_lib.lib().bm_context_eval_counts(self._h, L, out), "eval_counts")
        return out[0], out[1]

    def band_timings(self):
        """Per-band split of the refinement timers: {band index: {class: ms}} (timing on)."""
        ms = (C.c_double * 60)()
        _lib.check(_lib.lib().bm_context_band_timings(self._h, ms), "band_timings")
        names = ("gather", "expand", "seed", "refine", "wedge", "misc", "refine_band0",
                 "refine_band1", "refine_band2", "refine_band3+", "eval_order2", "eval_order0",
                 "compose", "newton", "xi_build")
        return {b: {n: ms[b * 15 + k] for k, n in enumerate(names) if ms[b * 15 + k] > 0} for b in range(4)}

    def set_lanes(self, lanes: int, min_per_lane: int = 64):
        """Concurrent lanes of align_batch (default 4 lanes of >= 64 particles)."""
        _lib.check(_lib.lib().bm_context_set_lanes(self._h, lanes, min_per_lane), "set_lanes")

    def set_expand_mode(self, mode: str):
        """'factored' (default) or 'gemm' (dense operator on the tensor cores)."""
        _lib.check(_lib.lib().bm_context_set_expand_mode(self._h, {"factored": 0, "gemm": 1}[mode]),
                   "set_expand_mode")
        self._refresh_info()

    def set_expand_pairs(self, mode: int):
        """Expansion gathers: 0 direct, 1 from a copy when a volume has >= 4 windows
        (default: zero-padded quad copy for |shift| <= 6, else x-paired copy), 2 always
        x-paired copy, 3 always quad copy.  Coefficients are bit-identical."""
        _lib.check(_lib.lib().bm_context_set_expand_pairs(self._h, int(mode)), "set_expand_pairs")

    def set_stage_reuse(self, on: bool):
        """Opt in: average_accumulate right after align_batch of the same (unmodified)
        host buffer reuses the device copy align_batch staged, once."""
        _lib.check(_lib.lib().bm_context_set_stage_reuse(self._h, 1 if on else 0), "set_stage_reuse")

    def eval_stats(self, reset: bool = False):
        """(order-2 evaluations, order-0 evaluations, algorithmic FLOPs) of the refinement."""
        ev = (C.c_longlong * 2)()
        fl = C.c_double()
        _lib.check(_lib.lib().bm_context_eval_stats(self._h, ev, C.byref(fl), 1 if reset else 0), "eval_stats")
        return ev[0], ev[1], fl.value

    def timings(self, reset: bool = False):
        ms = (C.c_double * 15)()
        cnt = (C.c_longlong * 4)()
        _lib.check(_lib.lib().bm_context_timings(self._h, ms, cnt, 1 if reset else 0), "timings")
        names = ("gather", "expand", "seed", "refine", "wedge", "misc", "refine_band0",
                 "refine_band1", "refine_band2", "refine_band3+", "eval_order2", "eval_order0",
                 "compose", "newton", "xi_build")
        return (dict(zip(names, ms[:])),
                dict(launches=cnt[0], windows_expanded=cnt[1], gemm_launches=cnt[2],
                     refine_launches=cnt[3]))


def run_bench(ctx: "Context", subtomo, cfg, true_rotation=None, baseline_step_deg: float = 5.0,
              baseline_band: int = 0, wedge: bool = False):
    """run_bench (src/optimize.cpp:546-584): align one subtomogram against the
    context's template, then the exhaustive grid baseline on the kernel of the
    winning shift, and the accuracy-matched evaluation ratio
    align_evaluations / |grid at max(align error, 0.01 deg)|.
    wedge: the template state has a wedge (the particle is taper-filtered first)."""
    import time
    torch = _torch()
    v = ctx._dev(subtomo)
    t0 = time.perf_counter()
    res = ctx.align_batch(v, cfg)[0]
    torch.cuda.synchronize()
    rep = {"alignment": res, "align_seconds": time.perf_counter() - t0,
           "align_evaluations": int(res["evaluations"]), "baseline_step_deg": baseline_step_deg,
           "baseline_band": baseline_band}
    fw = ctx.apply_wedge_taper(v) if wedge else v
    f_hat = ctx.expand(fw, [res["shift"]])
    xi = ctx.xi_coefficients(f_hat, ctx.template_coeffs())[0]
    t0 = time.perf_counter()
    bq, bs, bn = ctx.exhaustive_baseline(xi, baseline_band, baseline_step_deg * math.pi / 180.0)
    rep["baseline_seconds"] = time.perf_counter() - t0
    rep["baseline"] = {"quat": bq, "score": bs, "evaluations": bn}

    def geod(a, b):
        return math.degrees(2.0 * math.acos(min(1.0, abs(float(np.dot(a, b))))))
    if true_rotation is not None:
        rep["align_error_deg"] = geod(res["quat"], true_rotation)
        rep["baseline_error_deg"] = geod(bq, true_rotation)
        rep["matched_step_deg"] = max(rep["align_error_deg"], 0.01)
    else:
        rep["align_error_deg"] = rep["baseline_error_deg"] = -1.0
        rep["matched_step_deg"] = baseline_step_deg
    rep["matched_evaluations"] = baseline_evaluation_count(rep["matched_step_deg"] * math.pi / 180.0)
    rep["evaluation_ratio"] = rep["align_evaluations"] / rep["matched_evaluations"]
    return rep

