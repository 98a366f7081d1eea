"""Averaging (kernel K9) and the device data generator (K10) against the oracle."""
import math

import numpy as np
import pytest

from oracle import bmo
from paper_2509_01180_b200 import api

pytestmark = pytest.mark.gpu


def test_template_generator_matches_oracle(cuda_device):
    for n, blobs, seed in ((32, 20, 1), (64, 40, 20250901)):
        got = api.make_template(n, blobs, seed).cpu().numpy().astype(np.float64)
        ref = bmo.gaussian_blob_template(n, blobs, seed)
        assert np.abs(got - ref).max() <= 1e-6 * np.abs(ref).max()


@pytest.mark.parametrize("snr,wedge", [(None, None), (0.5, None), (0.1, 60.0)])
def test_particle_generator_matches_oracle(cuda_device, snr, wedge):
    n = 32
    tmpl = api.make_template(n, 20, 5)
    parts, q, sh = api.make_particles(tmpl, 3, 700, 3, snr, wedge)
    t64 = tmpl.cpu().numpy().astype(np.float64)
    for p in range(3):
        ref, rq, rsh = bmo.make_particle(t64, 700 + p, 3, snr, wedge)
        assert tuple(sh[p]) == rsh
        assert np.abs(q[p] - rq).max() < 1e-12
        got = parts[p].cpu().numpy().astype(np.float64)
        assert np.abs(got - ref).max() <= 1e-5 * np.abs(ref).max()


def test_average_matches_oracle_rotate_expansion(cuda_device):
    n, L = 32, 8
    tmpl = bmo.gaussian_blob_template(n, 20, 21)
    parts = []
    for p in range(4):
        s, _, _ = bmo.make_particle(tmpl, 900 + p, 2, 1.0, None)
        parts.append(s.astype(np.float32))
    parts = np.stack(parts)
    ctx = api.Context(n, L, L * math.pi)
    ctx.set_template(tmpl.astype(np.float32))
    cfg = api.make_config(bands=(4, 8), max_candidates=8, shift_radius=2, shift_step=2)
    res = ctx.align_batch(parts, cfg)
    got = ctx.average_accumulate(parts, res).cpu().numpy()
    got = got[..., 0] + 1j * got[..., 1]
    spec = bmo.Spec(L, L * math.pi)
    ref = np.zeros(spec.coeff_count, dtype=np.complex128)
    for p, r in enumerate(res):
        f = bmo.expand(bmo.shift_volume(parts[p].astype(np.float64), r["shift"]), spec)
        q = r["quat"]
        ref += bmo.rotate_expansion(f, spec, [q[0], -q[1], -q[2], -q[3]])
    assert np.linalg.norm(got - ref) <= 1e-5 * np.linalg.norm(ref)


def test_config2_sized_alignment_parity(cuda_device):
    """64^3, L=16, bands 4-8-16, 24 starts, wedge 60, SNR 0.1, shifts +-3: the
    metric configuration (the bench's template and first 16 particles), GPU vs
    oracle align()."""
    n, L = 64, 16
    P = 16
    tmpl_d = api.make_template(n, 40, 20250901)
    parts, q, sh = api.make_particles(tmpl_d, P, 1000, 3, 0.1, 60.0)
    ctx = api.Context(n, L, L * math.pi)
    ctx.set_template(tmpl_d, 60.0)
    cfg = api.make_config(bands=(4, 8, 16), max_candidates=24, shift_radius=4, shift_step=2)
    got = ctx.align_batch(parts, cfg)
    ocfg = bmo.make_config(l_max=L, lambda_cut=L * math.pi, bands=(4, 8, 16), max_candidates=24,
                           shift_radius=4, shift_step=2)
    tmpl = tmpl_d.cpu().numpy().astype(np.float64)
    for p in range(P):
        ref = bmo.align(tmpl, parts[p].cpu().numpy().astype(np.float64), ocfg, wedge_deg=60.0)
        assert got[p]["shift"] == ref["shift"]
        assert bmo.geodesic_degrees(got[p]["quat"], ref["quat"]) < 0.5
        assert got[p]["score"] == pytest.approx(ref["score"], rel=1e-4)


@pytest.mark.parametrize("n,L,m_out", [(32, 8, 32), (64, 16, 48)])
def test_synthesize_matches_oracle(cuda_device, n, L, m_out):
    """synthesize (src/basis.cpp:332-419) of an expansion on an m_out^3 grid, FP64 on
    both sides; the complex-coefficient branch agrees on real-symmetric input."""
    ctx = api.Context(n, L, L * math.pi)
    spec = bmo.Spec(L, L * math.pi)
    tmpl = bmo.gaussian_blob_template(n, 20, 31)
    coef = bmo.expand(tmpl, spec)
    got = ctx.synthesize(coef, m_out).cpu().numpy()
    ref = bmo.synthesize(coef, spec, m_out)
    assert np.linalg.norm(got - ref) <= 1e-10 * np.linalg.norm(ref)
    got_c = ctx.synthesize(coef, m_out, real_volume=False).cpu().numpy()
    assert np.linalg.norm(got_c - ref) <= 1e-10 * np.linalg.norm(ref)
    # the averaged map of an identity alignment reproduces the template's band-limited map
    assert np.linalg.norm(got - tmpl) <= 0.5 * np.linalg.norm(tmpl) if m_out == n else True


def test_config5_sized_alignment_parity(cuda_device):
    """Config-5 shape: 64^3, L=20, four marching bands 4-8-16-20, 24 starts, 60-blob
    template, SNR 0.05, shifts +-4, wedge 60; four particles, GPU vs oracle align()."""
    n, L = 64, 20
    P = 4
    tmpl_d = api.make_template(n, 60, 20250905)
    parts, q, sh = api.make_particles(tmpl_d, P, 5000, 4, 0.05, 60.0)
    ctx = api.Context(n, L, L * math.pi)
    ctx.set_template(tmpl_d, 60.0)
    cfg = api.make_config(bands=(4, 8, 16, 20), max_candidates=24, shift_radius=4, shift_step=2)
    got = ctx.align_batch(parts, cfg)
    ocfg = bmo.make_config(l_max=L, lambda_cut=L * math.pi, bands=(4, 8, 16, 20), max_candidates=24,
                           shift_radius=4, shift_step=2)
    tmpl = tmpl_d.cpu().numpy().astype(np.float64)
    for p in range(P):
        ref = bmo.align(tmpl, parts[p].cpu().numpy().astype(np.float64), ocfg, wedge_deg=60.0)
        assert got[p]["shift"] == ref["shift"]
        assert bmo.geodesic_degrees(got[p]["quat"], ref["quat"]) < 0.5
        assert got[p]["score"] == pytest.approx(ref["score"], rel=1e-4)
        assert got[p]["bands"] == [4, 8, 16, 20]


def test_align_batch_edge_counts(cuda_device):
    """An empty batch returns nothing; batches smaller than the lane split (1, 3
    particles with 4 lanes) give the same results as one lane."""
    n, L = 32, 8
    tmpl = api.make_template(n, 20, 9)
    parts, _, _ = api.make_particles(tmpl, 3, 4242, 2, 0.5, 60.0)
    cfg = api.make_config(bands=(4, 8), max_candidates=8, shift_radius=2, shift_step=2)
    ctx = api.Context(n, L, L * math.pi)
    ctx.set_template(tmpl, 60.0)
    assert ctx.align_batch(parts[:0], cfg) == []
    ctx.set_lanes(4, 1)
    many = ctx.align_batch(parts, cfg)
    one = ctx.align_batch(parts[:1], cfg)
    ctx.set_lanes(1)
    ref = ctx.align_batch(parts, cfg)
    assert len(many) == 3 and len(one) == 1
    for a, b in zip(many, ref):
        assert a["shift"] == b["shift"] and list(a["quat"]) == list(b["quat"]) and a["score"] == b["score"]
    assert one[0]["shift"] == ref[0]["shift"] and one[0]["score"] == ref[0]["score"]
