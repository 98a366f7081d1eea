"""Config-4 probe: rotate-score-gradient sweep at L=24 (512 x 4096 in full; scaled by argv)."""
import math
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2509_01180_b200 import api
from oracle import bmo


def random_coeffs(spec, rng, count):
    """Config-4 recipe: N(0,1) + i N(0,1) scaled 1/(1+l), real-volume symmetric."""
    out = np.zeros((count, spec.coeff_count), dtype=np.complex128)
    for l in range(spec.l_max + 1):
        for k in range(1, spec.radial_count(l) + 1):
            base = spec.index_of(k, l, 0)
            z = (rng.standard_normal((count, l + 1)) + 1j * rng.standard_normal((count, l + 1))) / (1 + l)
            z[:, 0] = z[:, 0].real
            for m in range(l + 1):
                out[:, base + m] = z[:, m]
                if m:
                    out[:, base - m] = (-1) ** m * np.conj(z[:, m])
    return out


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    n_p = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    n_g = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
    spec = bmo.Spec(L, L * math.pi)
    rng = np.random.default_rng(0)
    f = random_coeffs(spec, rng, n_p)
    t = random_coeffs(spec, rng, 1)[0]
    eul = np.array([bmo.euler_zyz(bmo.haar_rotation(5, g)) for g in range(n_g)])
    ctx = api.Context(0, L, L * math.pi)
    out = ctx.eval_sweep(f[:4], t, eul[:16])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = ctx.eval_sweep(f, t, eul)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    nxi = (L + 1) * (2 * L + 1) * (2 * L + 3) // 3
    flop = n_p * n_g * (8.0 * nxi + 24 * (2 * L + 1) ** 2) + n_g * 12.0 * nxi
    print(f"L={L} {n_p}x{n_g}: {ms:.2f} ms  {n_p*n_g/ms/1e3:.1f} M evals/s  "
          f"{flop/ms/1e9:.1f} TFLOP/s algorithmic", flush=True)


if __name__ == "__main__":
    main()
