"""Alignment parity (kernels K4-K7 + host driver) against the CPU oracle on
identical float32 inputs.  Bars (BASELINE.json north_star): rotations within
0.5 deg geodesic, shifts exact, scores within 1e-4 relative."""
import math

import numpy as np
import pytest

from oracle import bmo
from paper_2509_01180_b200 import api

pytestmark = pytest.mark.gpu


def _particles(n, blobs, seed, count, shift_max, snr, wedge):
    tmpl = bmo.gaussian_blob_template(n, blobs, seed)
    parts, truth = [], []
    for p in range(count):
        s, q, sh = bmo.make_particle(tmpl, seed * 1000 + p + 1, shift_max, snr, wedge)
        parts.append(s)
        truth.append((q, sh))
    return tmpl, np.stack(parts), truth


def test_single_window_cfg1_like(cuda_device):
    """Config-1 slice: 32^3, L=8, single window s=0, 8 starts, one band."""
    n, L = 32, 8
    tmpl, parts, truth = _particles(n, 20, 11, 6, 0, 0.5, None)
    ctx = api.Context(n, L, L * math.pi)
    ctx.set_template(tmpl.astype(np.float32))
    cfg = api.make_config(bands=(8,), max_candidates=8)
    got = ctx.search_windows(parts.astype(np.float32), [(i, (0, 0, 0)) for i in range(len(parts))], cfg)
    spec = bmo.Spec(L, L * math.pi)
    ocfg = bmo.make_config(l_max=L, lambda_cut=L * math.pi, bands=(8,), max_candidates=8)
    for i, g in enumerate(got):
        ref = bmo.search_window(spec, tmpl, parts[i].astype(np.float32).astype(np.float64),
                                (0, 0, 0), ocfg)
        ang = bmo.geodesic_degrees(g["quat"], ref["quat"])
        assert ang < 0.5, f"particle {i}: {ang:.3f} deg"
        assert g["norm_score"] == pytest.approx(ref["norm_score"], rel=1e-4)
        assert g["subtomo_norm"] == pytest.approx(ref["subtomo_norm"], rel=1e-5)


def test_windows_with_shifts_and_wedge(cuda_device):
    n, L = 32, 8
    tmpl, parts, truth = _particles(n, 20, 12, 3, 2, 0.5, 60.0)
    ctx = api.Context(n, L, L * math.pi)
    ctx.set_template(tmpl.astype(np.float32), 60.0)
    cfg = api.make_config(bands=(4, 8), max_candidates=8)
    f32 = parts.astype(np.float32)
    filt = ctx.apply_wedge_taper(f32).cpu().numpy()
    wins = [(i, s) for i in range(len(parts)) for s in [(0, 0, 0), (1, -1, 2), (-2, 0, 1)]]
    got = ctx.search_windows(filt, wins, cfg)
    spec = bmo.Spec(L, L * math.pi)
    ocfg = bmo.make_config(l_max=L, lambda_cut=L * math.pi, bands=(4, 8), max_candidates=8)
    for (i, s), g in zip(wins, got):
        ref = bmo.search_window(spec, tmpl, f32[i].astype(np.float64), s, ocfg, wedge_deg=60.0)
        ang = bmo.geodesic_degrees(g["quat"], ref["quat"])
        assert ang < 0.5, f"window {(i, s)}: {ang:.3f} deg"
        assert g["norm_score"] == pytest.approx(ref["norm_score"], rel=1e-4)


def test_align_batch_matches_oracle(cuda_device):
    n, L = 32, 8
    tmpl, parts, truth = _particles(n, 20, 13, 3, 2, 1.0, None)
    ctx = api.Context(n, L, L * math.pi)
    ctx.set_template(tmpl.astype(np.float32))
    cfg = api.make_config(bands=(4, 8), max_candidates=8, shift_radius=2, shift_step=2)
    got = ctx.align_batch(parts.astype(np.float32), cfg)
    ocfg = bmo.make_config(l_max=L, lambda_cut=L * math.pi, bands=(4, 8), max_candidates=8,
                           shift_radius=2, shift_step=2)
    for i, g in enumerate(got):
        ref = bmo.align(tmpl, parts[i].astype(np.float32).astype(np.float64), ocfg)
        assert g["shift"] == ref["shift"]
        assert bmo.geodesic_degrees(g["quat"], ref["quat"]) < 0.5
        assert g["score"] == pytest.approx(ref["score"], rel=1e-4)
        assert g["windows"] == ref["windows"]
        # ground truth: shift recovered exactly, rotation close
        assert g["shift"] == truth[i][1]


def test_config1_all_particles_match_oracle(cuda_device):
    """BASELINE config 1 in full: 32^3, L=8, 20-blob template, 128 particles (Haar
    rotations, SNR 0.5, no wedge, no shift), one window s = 0, band {8}, 8 starts —
    every particle's rotation within 0.5 deg and score within 1e-4 of the oracle's
    search_one_shift (src/optimize.cpp:361-419) on the same float32 bytes."""
    import math

    import numpy as np

    from oracle import bmo
    from paper_2509_01180_b200 import api

    n, L, P = 32, 8, 128
    cut = L * math.pi
    tmpl_d = api.make_template(n, 20, 1)
    parts, q_true, _ = api.make_particles(tmpl_d, P, 100, 0, 0.5, None)
    ctx = api.Context(n, L, cut)
    ctx.set_template(tmpl_d)
    cfg = api.make_config(bands=(8,), max_candidates=8)
    got = ctx.search_windows(parts, [(p, (0, 0, 0)) for p in range(P)], cfg)
    spec = bmo.Spec(L, cut)
    ocfg = bmo.make_config(l_max=L, lambda_cut=cut, bands=(8,), max_candidates=8)
    tmpl = tmpl_d.cpu().numpy().astype(np.float64)
    host = parts.cpu().numpy().astype(np.float64)
    worst_ang, worst_score = 0.0, 0.0
    for p in range(P):
        ref = bmo.search_window(spec, tmpl, host[p], (0, 0, 0), ocfg)
        ang = bmo.geodesic_degrees(got[p]["quat"], ref["quat"])
        rel = abs(got[p]["norm_score"] - ref["norm_score"]) / abs(ref["norm_score"])
        worst_ang, worst_score = max(worst_ang, ang), max(worst_score, rel)
    assert worst_ang < 0.5, worst_ang
    assert worst_score < 1e-4, worst_score


@pytest.mark.parametrize("mode", ["prune", "auto"])
def test_prune_after_band_and_auto_bands_match_oracle(cuda_device, mode):
    """OptimizerConfig.prune_after_band (optimize.cpp:391-403) and auto_bands
    (optimize.cpp:455-460, select_bands 179-195) through align_batch vs the oracle's
    align on the same float32 bytes: same band schedule, same shift, rotation within
    0.5 deg, score within 1e-4."""
    import math

    import numpy as np

    from oracle import bmo
    from paper_2509_01180_b200 import api

    n, L = 32, 8
    tmpl_d = api.make_template(n, 20, 3)
    parts, _, _ = api.make_particles(tmpl_d, 3, 500, 2, 1.0, 60.0)
    ctx = api.Context(n, L, L * math.pi)
    ctx.set_template(tmpl_d, 60.0)
    kw = dict(max_candidates=8, shift_radius=2, shift_step=2)
    if mode == "prune":
        cfg = api.make_config(bands=(4, 8), prune_after_band=True, **kw)
        ocfg = bmo.make_config(l_max=L, lambda_cut=L * math.pi, bands=(4, 8), prune_after_band=True, **kw)
    else:
        th = (0.05, 0.01, 0.002)
        cfg = api.make_config(bands=(), auto_bands=True, band_thresholds=th, **kw)
        ocfg = bmo.make_config(l_max=L, lambda_cut=L * math.pi, bands=(), auto_bands=True, band_thresholds=th, **kw)
    got = ctx.align_batch(parts, cfg)
    tmpl = tmpl_d.cpu().numpy().astype(np.float64)
    for p in range(3):
        ref = bmo.align(tmpl, parts[p].cpu().numpy().astype(np.float64), ocfg, wedge_deg=60.0)
        if mode == "auto":
            assert got[p]["bands"] == ref["bands"]
        assert got[p]["shift"] == ref["shift"]
        assert bmo.geodesic_degrees(got[p]["quat"], ref["quat"]) < 0.5
        assert got[p]["score"] == pytest.approx(ref["score"], rel=1e-4)
        # (candidate counters are not compared: a near-tied seed-grid maximum can add or
        # drop a candidate in a few windows, FP64 seed scores from FP32 vs FP64 expansions)


def test_lanes_give_identical_results(cuda_device):
    """bm_context_set_lanes: the batch split across concurrent lanes (own streams,
    buffers and host threads) gives bit-identical results to one lane."""
    import math

    from paper_2509_01180_b200 import api

    n, L = 32, 8
    tmpl = api.make_template(n, 20, 5)
    parts, _, _ = api.make_particles(tmpl, 12, 800, 2, 0.5, 60.0)
    cfg = api.make_config(bands=(4, 8), max_candidates=8, shift_radius=2, shift_step=2)
    out = {}
    for lanes in (1, 3):
        ctx = api.Context(n, L, L * math.pi)
        ctx.set_template(tmpl, 60.0)
        ctx.set_lanes(lanes, 2)
        out[lanes] = ctx.align_batch(parts, cfg)
    for a, b in zip(out[1], out[3]):
        assert a["shift"] == b["shift"]
        assert list(a["quat"]) == list(b["quat"])
        assert a["score"] == b["score"]
        assert a["evaluations"] == b["evaluations"]


def test_lanes_raised_after_set_template(cuda_device):
    """set_lanes to more lanes after set_template: the new lanes adopt the
    template (regression: they used to raise 'set_template first')."""
    import math

    n, L = 32, 8
    tmpl = api.make_template(n, 20, 5)
    parts, _, _ = api.make_particles(tmpl, 8, 700, 2, 0.5, 60.0)
    cfg = api.make_config(bands=(4, 8), max_candidates=8, shift_radius=2, shift_step=2)
    ctx = api.Context(n, L, L * math.pi)
    ctx.set_template(tmpl, 60.0)
    ctx.set_lanes(2, 2)
    a = ctx.align_batch(parts, cfg)
    ctx.set_lanes(4, 2)
    b = ctx.align_batch(parts, cfg)
    for x, y in zip(a, b):
        assert x["shift"] == y["shift"] and list(x["quat"]) == list(y["quat"]) and x["score"] == y["score"]


def test_host_particles_match_device(cuda_device):
    """bm_align_batch / bm_average_accumulate with host (pinned) particles give the
    same results as with device particles (per-lane staging)."""
    import math

    import torch

    n, L = 32, 8
    tmpl = api.make_template(n, 20, 5)
    parts, _, _ = api.make_particles(tmpl, 12, 800, 2, 0.5, 60.0)
    cfg = api.make_config(bands=(4, 8), max_candidates=8, shift_radius=2, shift_step=2)
    ctx = api.Context(n, L, L * math.pi)
    ctx.set_template(tmpl, 60.0)
    ctx.set_lanes(3, 2)
    dev = ctx.align_batch(parts, cfg)
    avg_d = ctx.average_accumulate(parts, dev)
    host = parts.cpu().pin_memory()
    hst = ctx.align_batch(host, cfg)
    avg_h = ctx.average_accumulate(host, hst)
    for a, b in zip(dev, hst):
        assert a["shift"] == b["shift"] and list(a["quat"]) == list(b["quat"]) and a["score"] == b["score"]
    # (the FP64 numerator is summed with atomics: order-dependent in the last bits)
    assert torch.allclose(avg_d, avg_h, rtol=1e-12, atol=1e-12)


def test_refilled_host_buffer_is_restaged(cuda_device):
    """A host buffer refilled between align_batch and average_accumulate is staged
    again (reuse is opt-in and use-once), so the average is built from the new bytes."""
    import math

    import torch

    n, L = 32, 8
    tmpl = api.make_template(n, 20, 5)
    parts, _, _ = api.make_particles(tmpl, 6, 900, 2, 0.5, None)
    other, _, _ = api.make_particles(tmpl, 6, 950, 2, 0.5, None)
    cfg = api.make_config(bands=(8,), max_candidates=4, shift_radius=2, shift_step=2)
    ctx = api.Context(n, L, L * math.pi)
    ctx.set_template(tmpl, 0.0)
    ctx.set_lanes(1, 1)
    host = parts.cpu().pin_memory()
    res = ctx.align_batch(host, cfg)
    want = ctx.average_accumulate(other, res)          # device reference on the new bytes
    host.copy_(other.cpu())                            # refill the same pinned buffer
    got = ctx.average_accumulate(host, res)
    assert torch.allclose(got, want, rtol=1e-12, atol=1e-12)
    # opt-in reuse serves exactly one average of an unmodified buffer
    ctx.set_stage_reuse(True)
    host.copy_(parts.cpu())
    res = ctx.align_batch(host, cfg)
    a1 = ctx.average_accumulate(host, res)
    a2 = ctx.average_accumulate(host, res)
    assert torch.allclose(a1, a2, rtol=1e-12, atol=1e-12)


def test_evaluations_per_band_and_phase_timings(cuda_device):
    """AlignmentResult's evaluations_per_band (optimize.hpp:83; optimize.cpp:507-511):
    per band of the schedule, summing to the total; the seed grid is counted at the
    first band; phase timings are filled."""
    import math

    n, L = 32, 8
    tmpl = api.make_template(n, 20, 5)
    parts, _, _ = api.make_particles(tmpl, 4, 1200, 2, 0.5, 60.0)
    cfg = api.make_config(bands=(4, 8), max_candidates=8, shift_radius=2, shift_step=2)
    ctx = api.Context(n, L, L * math.pi)
    ctx.set_template(tmpl, 60.0)
    for r in ctx.align_batch(parts, cfg):
        epb = r["evaluations_per_band"]
        assert set(epb) == {4, 8}
        assert sum(epb.values()) == r["evaluations"]
        assert epb[4] >= r["windows"] * 16 * 9 * 16  # the 16 x 9 x 16 seed grid of every window
        assert epb[8] > 0
        assert r["coarse_search_s"] > 0 and r["fine_search_s"] > 0 and r["expand_template_s"] > 0
