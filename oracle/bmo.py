"""numpy/ctypes wrapper of the CPU oracle (oracle/_build/libbm_oracle.so).

TEST INFRASTRUCTURE ONLY — the checker for the CUDA path and the CPU baseline
timed by bench.py.  Volumes are float64 arrays shaped (n, n, n) indexed
[z, y, x] (the reference's x-fastest storage, include/ballmatch/volume.hpp:24-31).
Quaternions are (w, x, y, z).  XiBlocks are packed: concatenated (2l+1)^2
row-major complex blocks, l = 0..L.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "libbm_oracle.so"
_lib = None

P = C.c_void_p
I = C.c_int
D = C.c_double
LL = C.c_longlong
U = C.c_uint
ULL = C.c_ulonglong


def build() -> Path:
    r = subprocess.run(["make", "-C", str(HERE)], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{r.stdout}\n{r.stderr}")
    return LIB


class Config(C.Structure):
    """Mirrors OptimizerConfig (include/ballmatch/optimize.hpp:15-32), fixed bands."""
    _fields_ = [("l_max", I), ("lambda_cut", D), ("n_bands", I), ("bands", I * 16),
                ("seed_grid_step", D), ("max_candidates", I), ("newton_max_iter", I),
                ("grad_tol", D), ("step_damping", D), ("shift_radius", I), ("shift_step", I),
                ("threads", I), ("auto_bands", I), ("prune_after_band", I), ("n_thresholds", I),
                ("thresholds", D * 8)]


class AlignOut(C.Structure):
    _fields_ = [("shift", I * 3), ("quat", D * 4), ("score", D), ("converged", I),
                ("candidates_evaluated", LL), ("evaluations", LL), ("template_norm", D),
                ("subtomo_norm", D), ("windows", I), ("n_bands", I), ("bands", I * 16)]


def make_config(l_max=42, lambda_cut=0.0, bands=(7, 12, 33), seed_grid_step=np.pi / 8,
                max_candidates=20, newton_max_iter=30, grad_tol=1e-7, step_damping=1e-3,
                shift_radius=4, shift_step=2, threads=0, auto_bands=False, prune_after_band=False,
                band_thresholds=(0.5, 0.25, 0.05)) -> Config:
    c = Config()
    c.l_max = l_max
    c.lambda_cut = lambda_cut
    c.n_bands = len(bands)
    for i, b in enumerate(bands):
        c.bands[i] = b
    c.seed_grid_step = seed_grid_step
    c.max_candidates = max_candidates
    c.newton_max_iter = newton_max_iter
    c.grad_tol = grad_tol
    c.step_damping = step_damping
    c.shift_radius = shift_radius
    c.shift_step = shift_step
    c.threads = threads
    c.auto_bands = 1 if auto_bands else 0
    c.prune_after_band = 1 if prune_after_band else 0
    c.n_thresholds = len(band_thresholds)
    for i, t in enumerate(band_thresholds):
        c.thresholds[i] = t
    return c


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = C.CDLL(str(LIB))
        sig = {
            "bmo_last_error": ([], C.c_char_p),
            "bmo_philox_round10": ([P, P, P], None),
            "bmo_philox_u32": ([ULL, U, LL, P], None),
            "bmo_philox_gaussian": ([ULL, U, LL, P], None),
            "bmo_sph_jl": ([I, D], D),
            "bmo_bessel_root": ([I, I], D),
            "bmo_default_lambda_cut": ([I, I], D),
            "bmo_spherical_harmonic": ([I, I, D, D, P], None),
            "bmo_gauss_legendre": ([I, P, P], None),
            "bmo_legendre_table": ([I, D, P], None),
            "bmo_spec_create": ([I, D], P),
            "bmo_spec_destroy": ([P], None),
            "bmo_spec_info": ([P, P], None),
            "bmo_spec_radial_count": ([P, I], I),
            "bmo_spec_root": ([P, I, I], D),
            "bmo_spec_norm": ([P, I, I], D),
            "bmo_spec_plan": ([P, P, P, P, P], None),
            "bmo_expand": ([P, I, P, P], I),
            "bmo_expand_many": ([P, I, I, P, P, I], I),
            "bmo_synthesize": ([P, P, I, P], I),
            "bmo_rotate_expansion": ([P, P, P, P], None),
            "bmo_little_d": ([I, D, I, P], None),
            "bmo_wigner_D": ([I, P, P], None),
            "bmo_xi": ([P, P, P, P], I),
            "bmo_corr_deriv": ([I, P, P, I, I, P], I),
            "bmo_corr_deriv_many": ([I, I, P, I, P, I, I, P, I], I),
            "bmo_xi_compose_right": ([I, P, P, I, P], None),
            "bmo_grid_scores": ([I, P, I, D, P], None),
            "bmo_exhaustive_baseline": ([I, P, I, D, P, P, P], I),
            "bmo_baseline_evaluation_count": ([D], LL),
            "bmo_seed_candidates": ([I, P, I, D, I, I, P, P, P, P], I),
            "bmo_refine": ([I, P, P, C.POINTER(Config), I, P, P, P, P, P, I, P, P], I),
            "bmo_energy_ratio": ([I, P, I, P], I),
            "bmo_select_bands": ([I, P, P, I, P], I),
            "bmo_align": ([I, P, P, C.POINTER(Config), D, C.POINTER(AlignOut)], I),
            "bmo_search_window": ([P, I, P, P, P, C.POINTER(Config), D, P, P, P, P, P], I),
            "bmo_apply_wedge": ([I, P, D, P], I),
            "bmo_apply_wedge_taper": ([I, P, D, D, P], I),
            "bmo_wedge_kept_fraction": ([I, D], D),
            "bmo_wedge_keep_profile": ([I, D, P, D], D),
            "bmo_wedge_power_kernel": ([I, P, D, I, P], I),
            "bmo_wedge_power_factors": ([I, P, D, I, P, P, P], I),
            "bmo_fft_r2c_3d": ([I, P, P], None),
            "bmo_sample_trilinear": ([I, P, D, D, D], D),
            "bmo_shift_volume": ([I, P, P, P], None),
            "bmo_rotate_volume_trilinear": ([I, P, P, P], None),
            "bmo_euler_zyz": ([P, P], None),
            "bmo_from_euler_zyz": ([P, P], None),
            "bmo_geodesic_degrees": ([P, P], D),
            "bmo_haar_rotation": ([ULL, U, P], None),
            "bmo_make_phantom": ([I, I, ULL, D, D, P, P, P, P, P, P], I),
            "bmo_gaussian_blob_template": ([I, I, ULL, P], None),
            "bmo_make_particle": ([I, P, ULL, I, D, D, P, P, P], I),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _chk(rc, what=""):
    if rc != 0:
        msg = lib().bmo_last_error().decode()
        if rc == 1:
            raise ValueError(f"{what}: {msg}")
        raise RuntimeError(f"{what}: status {rc}: {msg}")


def xi_count(L: int) -> int:
    return (L + 1) * (2 * L + 1) * (2 * L + 3) // 3


def xi_block(xi: np.ndarray, l: int) -> np.ndarray:
    off = xi_count(l - 1) if l > 0 else 0
    w = 2 * l + 1
    return xi[off:off + w * w].reshape(w, w)


# ------------------------------------------------------------------ numerics
def philox_round10(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().bmo_philox_round10(_p(c), _p(k), _p(out))
    return out


def philox_u32(seed, stream, n):
    out = np.zeros(n, dtype=np.uint32)
    lib().bmo_philox_u32(seed, stream, n, _p(out))
    return out


def philox_gaussian(seed, stream, n):
    out = np.zeros(n, dtype=np.float64)
    lib().bmo_philox_gaussian(seed, stream, n, _p(out))
    return out


def sph_jl(l, x):
    return lib().bmo_sph_jl(l, x)


def bessel_root(l, k):
    return lib().bmo_bessel_root(l, k)


def default_lambda_cut(n, l_max):
    return lib().bmo_default_lambda_cut(n, l_max)


def spherical_harmonic(l, m, theta, phi):
    out = np.zeros(2)
    lib().bmo_spherical_harmonic(l, m, theta, phi, _p(out))
    return complex(out[0], out[1])


def gauss_legendre(n):
    x = np.zeros(n)
    w = np.zeros(n)
    lib().bmo_gauss_legendre(n, _p(x), _p(w))
    return x, w


class Spec:
    """BasisSpec (include/ballmatch/basis.hpp:31-58) + its ExpandPlan."""

    def __init__(self, l_max: int, lambda_cut: float):
        h = lib().bmo_spec_create(l_max, lambda_cut)
        if not h:
            raise ValueError(lib().bmo_last_error().decode())
        self._h = C.c_void_p(h)
        info = np.zeros(6, dtype=np.int64)
        lib().bmo_spec_info(self._h, _p(info))
        self.l_max, self.coeff_count, self.pair_count, self.n_r, self.n_theta, self.n_phi = \
            (int(v) for v in info)
        self.lambda_cut = lambda_cut

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.bmo_spec_destroy(self._h)

    def radial_count(self, l):
        return lib().bmo_spec_radial_count(self._h, l)

    def root(self, l, k):
        return lib().bmo_spec_root(self._h, l, k)

    def norm(self, l, k):
        return lib().bmo_spec_norm(self._h, l, k)

    def block_offset(self, l):
        return sum(self.radial_count(j) * (2 * j + 1) for j in range(l))

    def index_of(self, k, l, m):
        return self.block_offset(l) + (k - 1) * (2 * l + 1) + (m + l)

    def plan(self):
        r = np.zeros(self.n_r)
        ct = np.zeros(self.n_theta)
        tri = (self.l_max + 1) * (self.l_max + 2) // 2
        ptab = np.zeros(tri * self.n_theta)
        radial = np.zeros(self.pair_count * self.n_r)
        lib().bmo_spec_plan(self._h, _p(r), _p(ct), _p(ptab), _p(radial))
        return r, ct, ptab.reshape(tri, self.n_theta), radial.reshape(self.pair_count, self.n_r)


def _vol(v):
    v = np.ascontiguousarray(v, dtype=np.float64)
    assert v.ndim == 3 and v.shape[0] == v.shape[1] == v.shape[2]
    return v


def expand(vol, spec: Spec) -> np.ndarray:
    v = _vol(vol)
    out = np.zeros(2 * spec.coeff_count)
    _chk(lib().bmo_expand(spec._h, v.shape[0], _p(v), _p(out)), "expand")
    return out.view(np.complex128)


def expand_many(vols, spec: Spec, threads=0) -> np.ndarray:
    v = np.ascontiguousarray(vols, dtype=np.float64)
    cnt, n = v.shape[0], v.shape[1]
    out = np.zeros((cnt, 2 * spec.coeff_count))
    import os
    _chk(lib().bmo_expand_many(spec._h, n, cnt, _p(v), _p(out), threads or os.cpu_count()))
    return out.view(np.complex128)


def synthesize(coeffs, spec: Spec, n: int) -> np.ndarray:
    c = np.ascontiguousarray(coeffs, dtype=np.complex128)
    out = np.zeros((n, n, n))
    _chk(lib().bmo_synthesize(spec._h, _p(c), n, _p(out)), "synthesize")
    return out


def rotate_expansion(coeffs, spec: Spec, quat) -> np.ndarray:
    c = np.ascontiguousarray(coeffs, dtype=np.complex128)
    q = np.asarray(quat, dtype=np.float64)
    out = np.zeros_like(c)
    lib().bmo_rotate_expansion(spec._h, _p(c), _p(q), _p(out))
    return out


def little_d(l_max, beta, order=0):
    n = xi_count(l_max)
    out = np.zeros(n * (order + 1))
    lib().bmo_little_d(l_max, beta, order, _p(out))
    return [out[i * n:(i + 1) * n] for i in range(order + 1)]


def wigner_D(l_max, quat):
    q = np.asarray(quat, dtype=np.float64)
    out = np.zeros(2 * xi_count(l_max))
    lib().bmo_wigner_D(l_max, _p(q), _p(out))
    return out.view(np.complex128)


def xi_coefficients(t, f, spec: Spec) -> np.ndarray:
    """xi_l[m,m'] = sum_k conj(t[k,l,m]) f[k,l,m'] (src/xcorr.cpp:34-50)."""
    t = np.ascontiguousarray(t, dtype=np.complex128)
    f = np.ascontiguousarray(f, dtype=np.complex128)
    out = np.zeros(2 * xi_count(spec.l_max))
    lib().bmo_xi(spec._h, _p(t), _p(f), _p(out))
    return out.view(np.complex128)


@dataclass
class Deriv:
    value: float
    imag: float
    grad: np.ndarray
    hess: np.ndarray


def correlation_derivatives(xi, L, euler, l_cut, order) -> Deriv:
    x = np.ascontiguousarray(xi, dtype=np.complex128)
    e = np.asarray(euler, dtype=np.float64)
    out = np.zeros(14)
    _chk(lib().bmo_corr_deriv(L, _p(x), _p(e), l_cut, order, _p(out)), "correlation")
    return Deriv(out[0], out[1], out[2:5].copy(), out[5:14].reshape(3, 3).copy())


def corr_deriv_many(xis, L, eulers, l_cut, order=1, threads=0):
    x = np.ascontiguousarray(xis, dtype=np.complex128)
    e = np.ascontiguousarray(eulers, dtype=np.float64)
    n_xi, n_rot = x.shape[0], e.shape[0]
    out = np.zeros((n_xi, n_rot, 4))
    import os
    _chk(lib().bmo_corr_deriv_many(L, n_xi, _p(x), n_rot, _p(e), l_cut, order, _p(out),
                                   threads or os.cpu_count()))
    return out


def xi_compose_right(xi, L, quat, l_limit=-1):
    x = np.ascontiguousarray(xi, dtype=np.complex128)
    q = np.asarray(quat, dtype=np.float64)
    out = np.zeros(2 * xi_count(L))
    lib().bmo_xi_compose_right(L, _p(x), _p(q), l_limit, _p(out))
    return out.view(np.complex128)


def euler_grid_shape(step):
    na = int(np.ceil(2 * np.pi / step))
    nb = int(np.ceil(np.pi / step)) + 1
    return na, nb, na


def grid_scores(xi, L, l_cut, step):
    x = np.ascontiguousarray(xi, dtype=np.complex128)
    na, nb, ng = euler_grid_shape(step)
    out = np.zeros(na * nb * ng)
    lib().bmo_grid_scores(L, _p(x), l_cut, step, _p(out))
    return out


def seed_candidates(xi, L, l_low, step, max_candidates, wp=None, L_wp=0):
    x = np.ascontiguousarray(xi, dtype=np.complex128)
    q = np.zeros((max_candidates, 4))
    s = np.zeros(max_candidates)
    idx = np.zeros(max_candidates, dtype=np.int64)
    w = None if wp is None else np.ascontiguousarray(wp, dtype=np.complex128)
    n = lib().bmo_seed_candidates(L, _p(x), l_low, step, max_candidates, L_wp,
                                  None if w is None else _p(w), _p(q), _p(s), _p(idx))
    if n < 0:
        raise ValueError(lib().bmo_last_error().decode())
    return q[:n], s[:n], idx[:n]


def energy_ratio(xi, L, l_cut):
    """energy_ratio (src/xcorr.cpp:129-137); ArithmeticError for a zero kernel."""
    x = np.ascontiguousarray(xi, dtype=np.complex128)
    out = np.zeros(1)
    rc = lib().bmo_energy_ratio(L, _p(x), l_cut, _p(out))
    if rc == 3:
        raise ArithmeticError(lib().bmo_last_error().decode())
    _chk(rc, "energy_ratio")
    return float(out[0])


def select_bands(xi, L, thresholds):
    """select_bands (src/optimize.cpp:179-195)."""
    x = np.ascontiguousarray(xi, dtype=np.complex128)
    t = np.ascontiguousarray(thresholds, dtype=np.float64)
    out = np.zeros(L + 1, dtype=np.int32)
    n = lib().bmo_select_bands(L, _p(x), _p(t), len(t), _p(out))
    if n < 0:
        raise ValueError(lib().bmo_last_error().decode())
    return [int(b) for b in out[:n]]


def refine(xi, L, start, cfg: Config, wp=None, L_wp=0, max_trace=4096):
    x = np.ascontiguousarray(xi, dtype=np.complex128)
    st = np.asarray(start, dtype=np.float64)
    w = None if wp is None else np.ascontiguousarray(wp, dtype=np.complex128)
    q = np.zeros(4)
    score = np.zeros(1)
    conv = np.zeros(1, dtype=np.int32)
    trace = np.zeros((max_trace, 7))
    nt = np.zeros(1, dtype=np.int32)
    ne = np.zeros(1, dtype=np.int64)
    _chk(lib().bmo_refine(L, _p(x), _p(st), C.byref(cfg), L_wp, None if w is None else _p(w),
                          _p(q), _p(score), _p(conv), _p(trace), max_trace, _p(nt), _p(ne)),
         "refine")
    return dict(quat=q, score=float(score[0]), converged=bool(conv[0]),
                trace=trace[:nt[0]].copy(), evaluations=int(ne[0]))


def align(tmpl, sub, cfg: Config, wedge_deg=0.0):
    t = _vol(tmpl)
    s = _vol(sub)
    out = AlignOut()
    _chk(lib().bmo_align(t.shape[0], _p(t), _p(s), C.byref(cfg), wedge_deg, C.byref(out)), "align")
    return dict(shift=tuple(out.shift), quat=np.array(out.quat[:]), score=out.score,
                converged=bool(out.converged), candidates=out.candidates_evaluated,
                evaluations=out.evaluations, template_norm=out.template_norm,
                subtomo_norm=out.subtomo_norm, windows=out.windows,
                bands=[int(b) for b in out.bands[:out.n_bands]])


def search_window(spec: Spec, tmpl, sub, shift, cfg: Config, wedge_deg=0.0):
    t = _vol(tmpl)
    s = _vol(sub)
    sh = np.asarray(shift, dtype=np.int32)
    q = np.zeros(4)
    ns, rs, sn = np.zeros(1), np.zeros(1), np.zeros(1)
    conv = np.zeros(1, dtype=np.int32)
    rc = lib().bmo_search_window(spec._h, t.shape[0], _p(t), _p(s), _p(sh), C.byref(cfg),
                                 wedge_deg, _p(q), _p(ns), _p(rs), _p(sn), _p(conv))
    if rc not in (0, 3):
        _chk(rc, "search_window")
    return dict(quat=q, norm_score=float(ns[0]), raw_score=float(rs[0]),
                subtomo_norm=float(sn[0]), converged=bool(conv[0]), valid=rc == 0)


def apply_wedge(v, theta):
    v = _vol(v)
    out = np.zeros_like(v)
    _chk(lib().bmo_apply_wedge(v.shape[0], _p(v), theta, _p(out)), "apply_wedge")
    return out


def apply_wedge_taper(v, theta, taper=6.0):
    v = _vol(v)
    out = np.zeros_like(v)
    _chk(lib().bmo_apply_wedge_taper(v.shape[0], _p(v), theta, taper, _p(out)), "taper")
    return out


def wedge_kept_fraction(n, theta):
    return lib().bmo_wedge_kept_fraction(n, theta)


def wedge_keep_profile(n, theta, nu, taper=6.0):
    v = np.asarray(nu, dtype=np.float64)
    return lib().bmo_wedge_keep_profile(n, theta, _p(v), taper)


def wedge_power_kernel(tmpl, theta, l_max):
    t = _vol(tmpl)
    out = np.zeros(2 * xi_count(l_max))
    _chk(lib().bmo_wedge_power_kernel(t.shape[0], _p(t), theta, l_max, _p(out)), "wpk")
    return out.view(np.complex128)


def wedge_power_factors(tmpl, theta, l_max):
    t = _vol(tmpl)
    tri = (l_max + 1) * (l_max + 2) // 2
    chi = np.zeros(2 * tri)
    q = np.zeros(2 * tri)
    tot = np.zeros(1)
    _chk(lib().bmo_wedge_power_factors(t.shape[0], _p(t), theta, l_max, _p(chi), _p(q), _p(tot)))
    return chi.view(np.complex128), q.view(np.complex128), float(tot[0])


def fft_r2c_3d(v):
    v = _vol(v)
    n = v.shape[0]
    out = np.zeros(2 * n * n * (n // 2 + 1))
    lib().bmo_fft_r2c_3d(n, _p(v), _p(out))
    return out.view(np.complex128).reshape(n, n, n // 2 + 1)


def sample_trilinear(v, x, y, z):
    v = _vol(v)
    return lib().bmo_sample_trilinear(v.shape[0], _p(v), x, y, z)


def shift_volume(v, s):
    v = _vol(v)
    sh = np.asarray(s, dtype=np.int32)
    out = np.zeros_like(v)
    lib().bmo_shift_volume(v.shape[0], _p(v), _p(sh), _p(out))
    return out


def rotate_volume_trilinear(v, quat):
    v = _vol(v)
    q = np.asarray(quat, dtype=np.float64)
    out = np.zeros_like(v)
    lib().bmo_rotate_volume_trilinear(v.shape[0], _p(v), _p(q), _p(out))
    return out


def euler_zyz(quat):
    q = np.asarray(quat, dtype=np.float64)
    out = np.zeros(3)
    lib().bmo_euler_zyz(_p(q), _p(out))
    return out


def from_euler_zyz(a, b, g):
    e = np.array([a, b, g], dtype=np.float64)
    out = np.zeros(4)
    lib().bmo_from_euler_zyz(_p(e), _p(out))
    return out


def geodesic_degrees(q1, q2):
    a = np.asarray(q1, dtype=np.float64)
    b = np.asarray(q2, dtype=np.float64)
    return lib().bmo_geodesic_degrees(_p(a), _p(b))


def haar_rotation(seed, stream):
    out = np.zeros(4)
    lib().bmo_haar_rotation(seed, stream, _p(out))
    return out


def make_phantom(n=64, blobs=6, seed=0, snr=None, wedge=None, quat=None, shift=None):
    t = np.zeros((n, n, n))
    s = np.zeros((n, n, n))
    q = np.zeros(4)
    sh = np.zeros(3, dtype=np.int32)
    qi = None if quat is None else np.asarray(quat, dtype=np.float64)
    si = None if shift is None else np.asarray(shift, dtype=np.int32)
    _chk(lib().bmo_make_phantom(n, blobs, seed, snr or 0.0, wedge or 0.0,
                                None if qi is None else _p(qi), None if si is None else _p(si),
                                _p(t), _p(s), _p(q), _p(sh)), "make_phantom")
    return t, s, q, tuple(int(x) for x in sh)


def gaussian_blob_template(n, blobs, seed):
    out = np.zeros((n, n, n))
    lib().bmo_gaussian_blob_template(n, blobs, seed, _p(out))
    return out


def make_particle(tmpl, seed, shift_max, snr=None, wedge=None):
    t = _vol(tmpl)
    s = np.zeros_like(t)
    q = np.zeros(4)
    sh = np.zeros(3, dtype=np.int32)
    _chk(lib().bmo_make_particle(t.shape[0], _p(t), seed, shift_max, snr or 0.0, wedge or 0.0,
                                 _p(s), _p(q), _p(sh)), "make_particle")
    return s, q, tuple(int(x) for x in sh)


def exhaustive_baseline(xi, L, l_cut, step):
    """exhaustive_baseline (src/optimize.cpp:523-539): (quat, score, evaluations)."""
    x = np.ascontiguousarray(xi, dtype=np.complex128)
    q = np.zeros(4)
    sc = np.zeros(1)
    ev = np.zeros(1, dtype=np.int64)
    _chk(lib().bmo_exhaustive_baseline(L, _p(x), l_cut, step, _p(q), _p(sc), _p(ev)), "baseline")
    return q, float(sc[0]), int(ev[0])


def baseline_evaluation_count(step):
    """baseline_evaluation_count (src/optimize.cpp:541-544)."""
    return int(lib().bmo_baseline_evaluation_count(step))
