"""Direct parity of the refinement's evaluation, seeding and wedge kernels.

- Objective::eval (src/optimize.cpp:102-131) at order 2 -- value, Euler gradient
  and Hessian of correlation_derivatives (src/xcorr.cpp:52-105) -- at L = 4, 8,
  16, 20, unanchored and on anchored charts: the oracle composes the chart kernel
  xi~ = xi D(a)^T (xi_compose_right, xcorr.cpp:149-155) as refine() does
  (optimize.cpp:268-299); the device evaluates the window / side kernels and maps
  the derivatives to the chart (refine.cu chart_transform).
- the wedge quotient C / sqrt(clamp(1 - rho, 0.02, 2)) with its chain rule;
- the wedge-power kernel xi_wp (xcorr.cpp:234-357);
- seed candidate lists (optimize.cpp:197-253): exact rotations and rank order.
Bars: value within 1e-4 relative (north_star's score tolerance); gradient and
Hessian within 1e-4 of the derivative scale (FP32 evaluation)."""
import math

import numpy as np
import pytest

from oracle import bmo
from paper_2509_01180_b200 import api

pytestmark = pytest.mark.gpu

KOFF = bmo.from_euler_zyz(0.0, math.pi / 2, 0.0)


def qmul(a, b):
    w1, x1, y1, z1 = a
    w2, x2, y2, z2 = b
    return np.array([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2, w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                     w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2, w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2])


def qinv(a):
    return np.array([a[0], -a[1], -a[2], -a[3]])


def random_coeffs(spec, rng, count):
    """config-4 recipe: N(0,1) + i N(0,1) scaled 1/(1+l), real-volume symmetric"""
    out = np.zeros((count, spec.coeff_count), dtype=np.complex128)
    for c in range(count):
        for l in range(spec.l_max + 1):
            for k in range(1, spec.radial_count(l) + 1):
                for m in range(0, l + 1):
                    z = (rng.standard_normal() + 1j * rng.standard_normal()) / (1 + l)
                    if m == 0:
                        z = z.real
                    out[c, spec.index_of(k, l, m)] = z
                    if m:
                        out[c, spec.index_of(k, l, -m)] = (-1) ** m * np.conj(z)
    return out


def chart_points(rng, n, anchored):
    """chart angles and anchors as refine() produces them: anchors a = K^-1 T with
    T within 0.05 rad of a gimbal pole, chart angles around K = ZYZ(0, pi/2, 0)"""
    eul, anc = [], []
    for i in range(n):
        if anchored:
            beta = rng.uniform(0, 0.05) if i % 2 == 0 else math.pi - rng.uniform(0, 0.05)
            T = bmo.from_euler_zyz(rng.uniform(-3, 3), beta, rng.uniform(-3, 3))
            anc.append(qmul(qinv(KOFF), T))
            e = np.array([0.0, math.pi / 2, 0.0]) + rng.normal(0, 0.4, 3)
        else:
            e = bmo.euler_zyz(bmo.haar_rotation(77, i))
            e[1] = min(max(e[1], 0.06), math.pi - 0.06)
        eul.append(e)
    return np.array(eul), (np.array(anc) if anchored else None)


def oracle_objective(xi, wp, L_xi, L_wp, e, L, order):
    """Objective::eval (optimize.cpp:106-130) on given kernels."""
    c = bmo.correlation_derivatives(xi, L_xi, e, L, order)
    if wp is None:
        return c.value, c.grad, c.hess
    r = bmo.correlation_derivatives(wp, L_wp, e, min(L, L_wp), order)
    v = min(max(1.0 - r.value, 0.02), 2.0)
    s = 1.0 / math.sqrt(v)
    val = c.value * s
    if order < 1:
        return val, None, None
    dv = -r.grad
    v32 = s / v
    grad = c.grad * s - 0.5 * c.value * v32 * dv
    v52 = v32 / v
    hess = (c.hess * s - 0.5 * v32 * (np.outer(c.grad, dv) + np.outer(dv, c.grad) + c.value * (-r.hess))
            + 0.75 * c.value * v52 * np.outer(dv, dv))
    return val, grad, hess


def check(got, want, tag):
    v, g, h = want
    scale = max(abs(v), np.abs(g).max(), np.abs(h).max(), 1e-12)
    assert abs(got[0] - v) <= 1e-4 * max(abs(v), 1e-12) + 1e-6 * scale, (tag, got[0], v)
    assert np.abs(got[1:4] - g).max() <= 1e-4 * scale, (tag, got[1:4], g)
    assert np.abs(got[4:].reshape(3, 3) - h).max() <= 1e-4 * scale, (tag, got[4:].reshape(3, 3), h)


@pytest.mark.parametrize("anchored", [False, True])
@pytest.mark.parametrize("L", [4, 8, 16, 20])
def test_objective_order2_matches_oracle(cuda_device, L, anchored):
    Lc = 20
    rng = np.random.default_rng(10 * L + anchored)
    spec = bmo.Spec(Lc, Lc * math.pi)
    ctx = api.Context(0, Lc, Lc * math.pi)  # basis-only context
    f = random_coeffs(spec, rng, 1)[0]
    t = random_coeffs(spec, rng, 1)[0]
    eul, anc = chart_points(rng, 24, anchored)
    got = ctx.objective_eval(f, eul, anc, L=L, order=2, t=t)
    got0 = ctx.objective_eval(f, eul, anc, L=L, order=0, t=t)
    xi = bmo.xi_coefficients(f, t, spec)
    for i in range(len(eul)):
        x = bmo.xi_compose_right(xi, Lc, anc[i], L) if anchored else xi
        want = oracle_objective(x, None, Lc, 0, eul[i], L, 2)
        check(got[i], want, (L, anchored, i))
        assert abs(got0[i, 0] - want[0]) <= 1e-4 * abs(want[0]) + 1e-6 * np.abs(want[1]).max()


@pytest.fixture(scope="module")
def wedge_ctx(cuda_device):
    n, L = 32, 8
    tmpl = bmo.gaussian_blob_template(n, 20, 3)
    ctx = api.Context(n, L, L * math.pi)
    ctx.set_template(tmpl.astype(np.float32), 60.0)
    parts = [bmo.make_particle(tmpl, 40 + i, 2, 0.5, 60.0)[0].astype(np.float32) for i in range(2)]
    f = ctx.expand(ctx.apply_wedge_taper(np.stack(parts))).cpu().numpy()
    return ctx, tmpl, f, bmo.Spec(L, L * math.pi)


@pytest.mark.parametrize("anchored", [False, True])
def test_objective_wedge_quotient_matches_oracle(wedge_ctx, anchored):
    ctx, _, f, spec = wedge_ctx
    L = spec.l_max
    t = ctx.template_coeffs().cpu().numpy()
    wp = ctx.wedge_power_kernel()
    rng = np.random.default_rng(5 + anchored)
    for p in range(len(f)):
        xi = bmo.xi_coefficients(f[p], t, spec)
        for band in (4, 8):
            eul, anc = chart_points(rng, 16, anchored)
            got = ctx.objective_eval(f[p], eul, anc, L=band, order=2)
            for i in range(len(eul)):
                x = bmo.xi_compose_right(xi, L, anc[i], band) if anchored else xi
                w = bmo.xi_compose_right(wp, L, anc[i], band) if anchored else wp
                check(got[i], oracle_objective(x, w, L, L, eul[i], band, 2), (p, band, anchored, i))


def test_wedge_power_kernel_matches_oracle(wedge_ctx):
    ctx, tmpl, _, spec = wedge_ctx
    got = ctx.wedge_power_kernel()
    ref = bmo.wedge_power_kernel(tmpl, 60.0, spec.l_max)
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err < 1e-6, err


def _off_pole(q, s):
    keep = [r for r in range(len(q)) if 1e-6 < bmo.euler_zyz(q[r])[1] < math.pi - 1e-6]
    return q[keep], s[keep]


@pytest.mark.parametrize("wedge", [0.0, 60.0])
def test_seed_candidates_match_oracle(cuda_device, wedge):
    """Identical FP32 expansions in: the device seed list (FP64 grid scores) equals
    the oracle's -- same grid rotations in the same rank order, scores within 1e-9.
    Grid points on the gimbal poles (beta = 0 or pi) form plateaus of one rotation
    whose scores differ only by rounding; which plateau member survives the strict
    local-maximum test (optimize.cpp:209-237) is decided by that rounding in the
    reference as well (either side may keep zero, one or two members of a
    plateau), so only the off-pole candidates are compared."""
    n, L = 64, 16
    tmpl = api.make_template(n, 40, 20250901)
    parts, _, _ = api.make_particles(tmpl, 6, 3000, 3, 0.1, wedge or None)
    ctx = api.Context(n, L, L * math.pi)
    ctx.set_template(tmpl, wedge)
    fw = ctx.apply_wedge_taper(parts) if wedge else parts
    shifts = [(0, 0, 0), (2, -2, 0), (-2, 2, 2), (0, 2, -2), (2, 2, 2), (-2, 0, 0)]
    f = ctx.expand(fw, shifts).cpu().numpy()
    t = ctx.template_coeffs().cpu().numpy()
    spec = bmo.Spec(L, L * math.pi)
    wp = ctx.wedge_power_kernel() if wedge else None
    got = ctx.seed_candidates(f, 4, math.pi / 8, 24)
    for p in range(len(f)):
        xi = bmo.xi_coefficients(f[p], t, spec)
        q, s, _ = bmo.seed_candidates(xi, L, 4, math.pi / 8, 24, wp, L if wedge else 0)
        gq, gs = got[p]
        oq, os_ = _off_pole(q, s)
        dq, ds = _off_pole(gq, gs)
        assert len(dq) == len(oq), (p, len(dq), len(oq))
        for r in range(len(oq)):
            assert np.allclose(dq[r], oq[r], atol=1e-12) or np.allclose(dq[r], -oq[r], atol=1e-12), (p, r)
            assert abs(ds[r] - os_[r]) <= 1e-9 * abs(os_[r]), (p, r, ds[r], os_[r])
