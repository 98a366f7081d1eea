"""Throughput on the other BASELINE.json configurations (1 GPU), one JSON line each:
  cfg3  expansion sweep: 8192 volumes of N(0,1) voxels masked to the ball, 48^3/64^3, L = 8/16/24
  cfg4  rotate-score-gradient sweep: 512 coefficient sets x 4096 Haar rotations at L = 24
  cfg5  production alignment: 64^3, L = 20, bands 4-8-16-20, 24 starts, shifts +-4, SNR 0.05,
        +-60 deg wedge, 60-blob template (a seeded subset of the 131072 particles)
Device-resident inputs, CUDA-event timing after a warm-up."""
import json
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2509_01180_b200 import api


def timed(fn, reps=1):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


def cfg3(batch=8192, ns=(48, 64), Ls=(8, 16, 24)):
    for n in ns:
        g = torch.Generator(device="cuda").manual_seed(3)
        vols = torch.randn((batch, n, n, n), device="cuda", generator=g)
        c = (torch.arange(n, device="cuda") - n // 2) * (2.0 / n)
        r2 = c[None, None, :] ** 2 + c[None, :, None] ** 2 + c[:, None, None] ** 2
        vols *= (r2 < 1.0).float()
        for L in Ls:
            ctx = api.Context(n, L, L * math.pi)
            ms, _ = timed(lambda: ctx.expand(vols))
            S = ctx.n_r * ctx.n_theta * ctx.n_phi
            ntri = (L + 1) * (L + 2) // 2
            per = 16.0 * S + 4.0 * ctx.n_phi * ctx.n_r * ctx.n_theta * (L + 1) + 4.0 * ctx.n_r * ntri * ctx.n_theta \
                + 2.0 * ctx.n_r * ctx.coeff_count
            print(json.dumps({"config": 3, "n": n, "L": L, "volumes": batch, "ms": ms,
                              "expansions_per_s": batch / ms * 1e3,
                              "algorithmic_tflops": per * batch / ms / 1e9, "mflop_per_expansion": per / 1e6,
                              "coeff_count": ctx.coeff_count}), flush=True)
            del ctx
        del vols


def random_coeffs(ctx, rng, count):
    L = ctx.l_max
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


def haar_euler(count, seed):
    rng = np.random.default_rng(seed)
    u = rng.random((count, 3))
    q = np.stack([np.sqrt(1 - u[:, 0]) * np.sin(2 * np.pi * u[:, 1]), np.sqrt(1 - u[:, 0]) * np.cos(2 * np.pi * u[:, 1]),
                  np.sqrt(u[:, 0]) * np.sin(2 * np.pi * u[:, 2]), np.sqrt(u[:, 0]) * np.cos(2 * np.pi * u[:, 2])], 1)
    w, x, y, z = q.T
    m02, m12, m22 = 2 * (x * z + w * y), 2 * (y * z - w * x), 1 - 2 * (x * x + y * y)
    m20, m21 = 2 * (x * z - w * y), 2 * (y * z + w * x)
    return np.stack([np.arctan2(m12, m02), np.arctan2(np.hypot(m02, m12), m22), np.arctan2(m21, -m20)], 1)


def cfg4(n_p=512, n_g=4096, L=24):
    ctx = api.Context(0, L, L * math.pi)
    rng = np.random.default_rng(4)
    f = torch.view_as_real(torch.as_tensor(random_coeffs(ctx, rng, n_p))).cuda().contiguous()
    t = torch.view_as_real(torch.as_tensor(random_coeffs(ctx, rng, 1)[0])).cuda().contiguous()
    e = torch.as_tensor(haar_euler(n_g, 5)).cuda().contiguous()
    fc, tc = torch.view_as_complex(f), torch.view_as_complex(t)
    ms, _ = timed(lambda: ctx.eval_sweep(fc, tc, e), reps=3)
    nxi = (L + 1) * (2 * L + 1) * (2 * L + 3) // 3
    # 8 N_xi + 24 (2L+1)^2 per (particle, rotation) unit, plus the
    # d, d' recursion 12 N_xi once per rotation (amortised over the particles)
    flop = n_p * n_g * (8.0 * nxi + 24 * (2 * L + 1) ** 2) + n_g * 12.0 * nxi
    peak = json.loads((Path(__file__).resolve().parent.parent / "profiles" / "fp32_peak.json").read_text())
    tf = flop / ms / 1e9
    ms_tc, _ = timed(lambda: ctx.eval_sweep_tc(fc, tc, e), reps=3)
    _, tm = ctx.eval_sweep_tc(fc, tc, e, timing=True)
    peaks = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text()) \
        if (Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").exists() else {"bf16_tflops": 1590.0}
    tensor_tf = tm[3] / (tm[1] / 1e3) / 1e12
    print(json.dumps({"config": 4, "path": "tensor (bm_eval_sweep_tc)", "L": L, "particles": n_p, "rotations": n_g,
                      "ms": ms_tc, "evaluations_per_s": n_p * n_g / ms_tc * 1e3,
                      "algorithmic_tflops": flop / ms_tc / 1e9, "phases_ms": {"tables": tm[0], "gemm": tm[1],
                                                                             "gather": tm[2]},
                      "gemm_tensor_tflops": tensor_tf, "tensor_frac_of_bf16_peak": tensor_tf / peaks["bf16_tflops"],
                      "flop_accounting": "algorithmic as the SIMT line; GEMM: 2 K N (3P + P) x 3 FP16 passes"}),
          flush=True)
    print(json.dumps({"config": 4, "path": "simt (bm_eval_sweep)", "L": L, "particles": n_p, "rotations": n_g, "ms": ms,
                      "evaluations_per_s": n_p * n_g / ms * 1e3, "algorithmic_tflops": tf,
                      "frac_fp32_peak": tf / float(peak["fp32_fma_tflops"]),
                      "flop_accounting": "SURVEY.md §8(d): n_p n_g (8 N_xi + 24 (2L+1)^2) + n_g 12 N_xi"}),
          flush=True)


def cfg5(P=2048):
    n, L = 64, 20
    ctx = api.Context(n, L, L * math.pi)
    tmpl = api.make_template(n, 60, 20250905)
    ctx.set_template(tmpl, 60.0)
    parts, q, sh = api.make_particles(tmpl, P, 5000, 4, 0.05, 60.0)
    cfg = api.make_config(bands=(4, 8, 16, 20), max_candidates=24, shift_radius=4, shift_step=2)
    ctx.align_batch(parts[:64], cfg)
    ms, res = timed(lambda: ctx.align_batch(parts, cfg))
    errs = [math.degrees(2 * math.acos(min(1.0, abs(float(np.dot(r["quat"], q[i])))))) for i, r in enumerate(res)]
    ok = sum(tuple(r["shift"]) == tuple(int(x) for x in sh[i]) for i, r in enumerate(res))
    print(json.dumps({"config": 5, "particles_timed": P, "ms": ms, "subtomograms_per_s": P / ms * 1e3,
                      "projected_131072_s_per_gpu": 131072 / (P / ms * 1e3),
                      "shift_exact": f"{ok}/{P}", "rot_err_deg_median": float(np.median(errs))}), flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["3", "4", "5"]
    if "3" in which:
        cfg3()
    if "3x" in which:  # one case: 64^3, L = 16 (profiling)
        cfg3(ns=(64,), Ls=(16,))
    if "4" in which:
        cfg4()
    if "5" in which:
        cfg5()
