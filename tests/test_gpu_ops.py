"""Reference operators on the device (FP64, reference layouts) vs the oracle:
xi_coefficients (src/xcorr.cpp:21-50), xi_compose_right (xcorr.cpp:149-155),
rotate_expansion (src/steer.cpp:208-223), exhaustive_baseline
(src/optimize.cpp:523-539) and run_bench's evaluation ratio (optimize.cpp:546-584,
reference test proj/tests/test_optimize.cpp:324-344)."""
import math

import numpy as np
import pytest

from oracle import bmo
from paper_2509_01180_b200 import api

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sets(cuda_device):
    n, L = 32, 8
    spec = bmo.Spec(L, L * math.pi)
    ctx = api.Context(n, L, L * math.pi)
    t = bmo.gaussian_blob_template(n, 12, 4)
    f = bmo.gaussian_blob_template(n, 12, 5)
    return ctx, spec, bmo.expand(t, spec), bmo.expand(f, spec)


def test_xi_coefficients(sets):
    ctx, spec, t, f = sets
    got = ctx.xi_coefficients(np.stack([f, t]), t)
    for i, a in enumerate((f, t)):
        ref = bmo.xi_coefficients(a, t, spec)
        assert np.abs(got[i] - ref).max() <= 1e-12 * np.abs(ref).max()


def test_compose_and_rotate(sets):
    ctx, spec, t, f = sets
    xi = bmo.xi_coefficients(f, t, spec)
    for s in range(4):
        q = bmo.haar_rotation(31, s)
        for lim in (-1, 4):
            got = ctx.xi_compose_right(xi, q, lim)
            ref = bmo.xi_compose_right(xi, spec.l_max, q, lim)
            assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
        got = ctx.rotate_expansion(f, q)
        ref = bmo.rotate_expansion(f, spec, q)
        assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("l_cut,step_deg", [(4, 6.0), (8, 5.0), (8, 22.5)])
def test_exhaustive_baseline(sets, l_cut, step_deg):
    ctx, spec, t, f = sets
    xi = bmo.xi_coefficients(f, t, spec)
    step = step_deg * math.pi / 180.0
    q, s, n = ctx.exhaustive_baseline(xi, l_cut, step)
    rq, rs, rn = bmo.exhaustive_baseline(xi, spec.l_max, l_cut, step)
    assert n == rn == api.baseline_evaluation_count(step)
    assert abs(s - rs) <= 1e-12 * abs(rs)
    assert bmo.geodesic_degrees(q, rq) < 1e-9
    # self-correlation: the peak sits at the identity (test_optimize.cpp:292-301)
    qs, _, _ = ctx.exhaustive_baseline(bmo.xi_coefficients(t, t, spec), l_cut, step)
    assert bmo.geodesic_degrees(qs, [1.0, 0.0, 0.0, 0.0]) <= step_deg * math.sqrt(3.0)


def test_run_bench_reports_a_sane_efficiency_ratio(cuda_device):
    """The reference's run_bench acceptance (test_optimize.cpp:324-344): 48^3 phantom,
    4 blobs, seed 777, rotation ZYZ(0.9, 1.1, 0.2), shift (1, 1, -1), small_config with
    shift radius 2, baseline 6 deg at band 4: ratio <= 0.1 and align no less
    accurate than the baseline."""
    q_true = bmo.from_euler_zyz(0.9, 1.1, 0.2)
    tmpl, sub, q, sh = bmo.make_phantom(n=48, blobs=4, seed=777, quat=q_true, shift=(1, 1, -1))
    ctx = api.Context(48, 16, 0.0)  # lambda_cut 0: default_lambda_cut(48, 16)
    ctx.set_template(tmpl.astype(np.float32), 0.0)
    cfg = api.make_config(bands=(4, 8, 14), max_candidates=24, shift_radius=2, shift_step=2)
    rep = api.run_bench(ctx, sub.astype(np.float32), cfg, true_rotation=q, baseline_step_deg=6.0,
                        baseline_band=4)
    assert rep["align_evaluations"] > 0
    assert rep["matched_evaluations"] >= rep["align_evaluations"]
    assert 0.0 <= rep["align_error_deg"] <= rep["baseline_error_deg"] + 1e-12
    assert rep["evaluation_ratio"] <= 0.1
    assert tuple(rep["alignment"]["shift"]) == tuple(sh)
