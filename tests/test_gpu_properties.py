"""Size-independent properties at BASELINE.json's full sizes, where the CPU oracle
is too slow to run the whole case (it checks small samples of the same
configurations elsewhere): linearity and shift covariance of the expansion on
the alignment's whole shift grids, and the generate -> align -> recover round
trip on the full 1024-particle batch of the metric configuration."""
import math

import numpy as np
import pytest
import torch

from paper_2509_01180_b200 import api

pytestmark = pytest.mark.gpu


def _shifted(v, s):
    """shift_volume (src/volume.cpp:50-67) on the device: out[z, y, x] = v[z+sz, y+sy, x+sx],
    zero where the source leaves the grid."""
    n = v.shape[-1]
    out = torch.zeros_like(v)
    sx, sy, sz = s

    def rng(d):
        return (max(0, -d), min(n, n - d))

    (x0, x1), (y0, y1), (z0, z1) = rng(sx), rng(sy), rng(sz)
    out[z0:z1, y0:y1, x0:x1] = v[z0 + sz:z1 + sz, y0 + sy:y1 + sy, x0 + sx:x1 + sx]
    return out


def test_expansion_is_linear_on_a_config3_batch(cuda_device):
    """expand(a u + b v) = a expand(u) + b expand(v) on 2048 volumes of config 3's
    64^3 / L = 16 case (i.i.d. N(0,1) voxels): FP32 rounding only."""
    n, L, count = 64, 16, 2048
    ctx = api.Context(n, L, L * math.pi)
    g = torch.Generator(device=cuda_device).manual_seed(31)
    u = torch.randn((count, n, n, n), generator=g, device=cuda_device)
    v = torch.randn((count, n, n, n), generator=g, device=cuda_device)
    a, b = 0.75, -1.5
    eu, ev = ctx.expand(u), ctx.expand(v)
    ew = ctx.expand(a * u + b * v)
    ref = a * eu + b * ev
    err = torch.linalg.norm(ew - ref, dim=1) / torch.linalg.norm(ref, dim=1)
    assert float(err.max()) < 5e-6, float(err.max())
    assert float(torch.linalg.norm(eu, dim=1).min()) > 0  # non-trivial expansions


@pytest.mark.parametrize("L", [16, 20])
def test_window_expansions_equal_expansions_of_shifted_volumes(cuda_device, L):
    """The shift search expands windows of a volume in place (padded quad copy,
    x-neighbour windows sharing their loads).  Every window of the coarse grid
    (radius 4, step 2) and of a fine cube must give exactly the bits of the plain
    expansion of the explicitly shifted volume (same taps, same FP32 order), for
    configs 2 (L = 16) and 5 (L = 20)."""
    n = 64
    ctx = api.Context(n, L, L * math.pi)
    tmpl = api.make_template(n, 40, 7)
    parts, _, _ = api.make_particles(tmpl, 2, 4100, 3, 0.1, 60.0)
    coarse = [(x, y, z) for z in range(-4, 5, 2) for y in range(-4, 5, 2) for x in range(-4, 5, 2)]
    fine = [(2 + x, -2 + y, 0 + z) for z in range(-2, 3) for y in range(-2, 3) for x in range(-2, 3)
            if (x % 2, y % 2, z % 2) != (0, 0, 0)]
    shifts = coarse + fine
    win_vol = [0] * len(shifts) + [1] * len(shifts)
    got = ctx.expand_windows(parts, win_vol, shifts + shifts)
    ctx.set_expand_pairs(0)
    for p in range(2):
        vols = torch.stack([_shifted(parts[p], s) for s in shifts])
        ref = ctx.expand(vols)
        assert torch.equal(got[p * len(shifts):(p + 1) * len(shifts)], ref)


def test_config2_round_trip_on_the_full_batch(cuda_device):
    """Generate the metric configuration's 1024 particles from the template with known
    rotations and shifts (SNR 0.1, +-60 degree wedge, shifts +-3), align them, and
    recover the truth: the reference's acceptance criteria are statistical at this
    noise level (tests/acceptance.cpp), so the bars are >= 90% exact shifts and a
    median rotation error below 1 degree; every result must be finite and every
    particle must have searched its 125 coarse and 98 to 117 fine windows."""
    n, L, count = 64, 16, 1024
    ctx = api.Context(n, L, L * math.pi)
    tmpl = api.make_template(n, 40, 7)
    ctx.set_template(tmpl, 60.0)
    parts, q, sh = api.make_particles(tmpl, count, 1000, 3, 0.1, 60.0)
    cfg = api.make_config(bands=(4, 8, 16), max_candidates=24, shift_radius=4, shift_step=2)
    res = ctx.align_batch(parts, cfg)
    assert len(res) == count
    exact = sum(tuple(r["shift"]) == tuple(int(x) for x in sh[i]) for i, r in enumerate(res))
    errs = []
    for i, r in enumerate(res):
        assert all(math.isfinite(x) for x in r["quat"]) and math.isfinite(r["score"])
        assert abs(sum(x * x for x in r["quat"]) - 1.0) < 1e-9
        assert 125 + 98 <= r["windows"] <= 125 + 117  # the fine cube minus the 8 to 27 coarse points inside it
        d = min(1.0, abs(float(np.dot(r["quat"], q[i]))))
        errs.append(math.degrees(2 * math.acos(d)))
    assert exact >= 0.9 * count, exact
    assert float(np.median(errs)) < 1.0, float(np.median(errs))
    # the batch is deterministic: a second pass gives the same bits
    again = ctx.align_batch(parts, cfg)
    assert all(a["shift"] == b["shift"] and list(a["quat"]) == list(b["quat"]) and a["score"] == b["score"]
               for a, b in zip(res, again))


def _config4_inputs(L, n_p, n_g):
    """BASELINE config 4: complex coefficient sets N(0,1) + i N(0,1) scaled by 1/(1+l) with the
    real-volume symmetry, Euler triples of Haar-random rotations."""
    ctx = api.Context(0, L, L * math.pi)
    rng = np.random.default_rng(4)

    def coeffs(count):
        out = np.zeros((count, ctx.coeff_count), dtype=np.complex128)
        for l in range(L + 1):
            for k in range(1, ctx.radial_count(l) + 1):
                base = ctx.index_of(k, l, 0)
                z = (rng.standard_normal((count, l + 1)) + 1j * rng.standard_normal((count, l + 1))) / (1 + l)
                z[:, 0] = z[:, 0].real
                for m in range(l + 1):
                    out[:, base + m] = z[:, m]
                    if m:
                        out[:, base - m] = (-1) ** m * np.conj(z[:, m])
        return out

    u = np.random.default_rng(5).random((n_g, 3))
    w, x = np.sqrt(1 - u[:, 0]) * np.sin(2 * np.pi * u[:, 1]), np.sqrt(1 - u[:, 0]) * np.cos(2 * np.pi * u[:, 1])
    y, z = np.sqrt(u[:, 0]) * np.sin(2 * np.pi * u[:, 2]), np.sqrt(u[:, 0]) * np.cos(2 * np.pi * u[:, 2])
    m02, m12, m22 = 2 * (x * z + w * y), 2 * (y * z - w * x), 1 - 2 * (x * x + y * y)
    m20, m21 = 2 * (x * z - w * y), 2 * (y * z + w * x)
    eul = np.stack([np.arctan2(m12, m02), np.arctan2(np.hypot(m02, m12), m22), np.arctan2(m21, -m20)], 1)
    return ctx, coeffs(n_p), coeffs(1)[0], eul


def test_config4_sweep_gradient_and_tensor_path_at_full_size(cuda_device):
    """Config 4 at its full size (L = 24, 512 particles x 4096 rotations): the closed-form
    Euler gradient agrees with central differences of the score (the same kernel at
    e +- h along each angle), and the tensor-core sweep (two tcgen05 GEMMs) agrees with
    the SIMT sweep on all 2.1 M (particle, rotation) pairs within the north_star's 1e-4."""
    L, n_p, n_g = 24, 512, 4096
    ctx, f, t, eul = _config4_inputs(L, n_p, n_g)
    eul[:, 1] = np.clip(eul[:, 1], 0.05, math.pi - 0.05)  # central differences need room at the poles
    base = ctx.eval_sweep(f, t, eul, order=1)
    scale = float(base[..., 0].abs().max())
    tc = ctx.eval_sweep_tc(f, t, eul)
    assert float((tc - base).abs().max()) <= 1e-4 * max(scale, float(base[..., 1:].abs().max()))
    h = 1e-3
    for axis in range(3):
        ep, em = eul.copy(), eul.copy()
        ep[:, axis] += h
        em[:, axis] -= h
        fd = (ctx.eval_sweep(f, t, ep, order=1)[..., 0] - ctx.eval_sweep(f, t, em, order=1)[..., 0]) / (2 * h)
        g = base[..., 1 + axis]
        gscale = float(g.abs().max())
        # truncation h^2 |C'''| / 6 ~ 1e-6 L^2 relative, FP32 score noise / h ~ 1e-3 relative
        assert float((fd - g).abs().max()) <= 5e-3 * gscale, (axis, float((fd - g).abs().max()), gscale)


def test_config5_average_is_additive_over_shards(cuda_device):
    """Config 5's averaging step shards the particles over the GPUs and combines the
    partial averages with one allreduce (a sum).  On one device: the FP64 average of a
    batch equals the sum of the averages of its shards (the alignment of a particle
    does not depend on the batch it is in), and it correlates with the template's own
    expansion (the aligned particles add up coherently)."""
    n, L, count = 64, 20, 96
    ctx = api.Context(n, L, L * math.pi)
    tmpl = api.make_template(n, 60, 20250905)
    ctx.set_template(tmpl, 60.0)
    parts, _, _ = api.make_particles(tmpl, count, 5000, 4, 0.05, 60.0)
    cfg = api.make_config(bands=(4, 8, 16, 20), max_candidates=24, shift_radius=4, shift_step=2)
    res = ctx.align_batch(parts, cfg)
    whole = ctx.average_accumulate(parts, res)
    shards = [(0, 40), (40, 41), (41, 96)]
    total = torch.zeros_like(whole)
    for a, b in shards:
        r = ctx.align_batch(parts[a:b], cfg)
        assert all(x["shift"] == y["shift"] and list(x["quat"]) == list(y["quat"]) for x, y in zip(r, res[a:b]))
        total += ctx.average_accumulate(parts[a:b], r)
    assert float(torch.linalg.norm(total - whole)) <= 1e-12 * float(torch.linalg.norm(whole))
    t_hat = ctx.expand(tmpl[None])[0]
    avg = torch.view_as_complex(whole.contiguous()) if whole.shape[-1] == 2 and not whole.is_complex() else whole
    corr = abs(complex(torch.vdot(t_hat, avg.to(t_hat.dtype)))) / (
        float(torch.linalg.norm(t_hat)) * float(torch.linalg.norm(avg)))
    assert corr > 0.5, corr
