"""Rotate-score-gradient kernel (K4+K5) vs the oracle's correlation_derivatives
(src/xcorr.cpp:52-105) on random real-symmetric coefficient sets (config-4
recipe: N(0,1) + i N(0,1) scaled 1/(1+l), f_{k,l,-m} = (-1)^m conj f_{k,l,m}).
Scores within 1e-4 relative (north_star); gradients within 1e-4 of the
gradient scale."""
import math

import numpy as np
import pytest

from oracle import bmo
from paper_2509_01180_b200 import api

pytestmark = pytest.mark.gpu


def random_coeffs(spec, rng, count):
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


@pytest.mark.parametrize("path", ["simt", "tensor"])
@pytest.mark.parametrize("L", [4, 8, 16, 24])
def test_eval_sweep_matches_oracle(cuda_device, L, path):
    rng = np.random.default_rng(L)
    spec = bmo.Spec(L, L * math.pi)
    ctx = api.Context(0, L, L * math.pi)  # basis-only context (no expansion operator)
    f = random_coeffs(spec, rng, 3)
    t = random_coeffs(spec, rng, 1)[0]
    eul = []
    for g in range(16):
        e = bmo.euler_zyz(bmo.haar_rotation(99, g))
        e[1] = min(max(e[1], 0.02), math.pi - 0.02)
        eul.append(e)
    eul = np.array(eul)
    got = (ctx.eval_sweep(f, t, eul, order=1) if path == "simt" else ctx.eval_sweep_tc(f, t, eul)).cpu().numpy()
    for p in range(len(f)):
        xi = bmo.xi_coefficients(f[p], t, spec)
        for g in range(len(eul)):
            d = bmo.correlation_derivatives(xi, L, eul[g], L, 1)
            scale = max(abs(d.value), np.abs(d.grad).max(), 1e-12)
            assert abs(got[p, g, 0] - d.value) <= 1e-4 * scale, (p, g, got[p, g, 0], d.value)
            assert np.abs(got[p, g, 1:] - d.grad).max() <= 1e-4 * scale, (p, g)
