import sys, math
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from oracle import bmo
from paper_2509_01180_b200 import api

for n, L in ((32, 8), (48, 8), (64, 8), (32, 12), (64, 12), (64, 16)):
    ctx = api.Context(n, L, L * math.pi)
    spec = bmo.Spec(L, L * math.pi)
    v = bmo.gaussian_blob_template(n, 20, 2)
    got = ctx.expand(v[None].astype(np.float32)).cpu().numpy()[0]
    ref = bmo.expand(v, spec)
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    # per-degree error
    per = []
    for l in range(L + 1):
        a, b = ctx.block_offset(l), ctx.block_offset(l + 1)
        per.append(np.linalg.norm(got[a:b] - ref[a:b]) / max(np.linalg.norm(ref[a:b]), 1e-30))
    print(n, L, "support", ctx.support, "k_pad", ctx.k_pad, "m_pad", ctx.m_pad, f"err {err:.2e}",
          "worst-l", int(np.argmax(per)), f"{max(per):.2e}", "first rows", got[:3], ref[:3], flush=True)
    ctx.close()
