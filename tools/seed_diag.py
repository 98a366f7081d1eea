import math, sys
sys.path.insert(0, '/root/repo')
import numpy as np
from oracle import bmo
from paper_2509_01180_b200 import api
n, L = 64, 16
tmpl = api.make_template(n, 40, 20250901)
parts, _, _ = api.make_particles(tmpl, 6, 3000, 3, 0.1, None)
ctx = api.Context(n, L, L * math.pi)
ctx.set_template(tmpl, 0.0)
shifts = [(0, 0, 0), (2, -2, 0), (-2, 2, 2), (0, 2, -2), (2, 2, 2), (-2, 0, 0)]
f = ctx.expand(parts, shifts).cpu().numpy()
t = ctx.template_coeffs().cpu().numpy()
spec = bmo.Spec(L, L * math.pi)
got = ctx.seed_candidates(f, 4, math.pi / 8, 24)
p = 4
xi = bmo.xi_coefficients(f[p], t, spec)
q, s, idx = bmo.seed_candidates(xi, L, 4, math.pi / 8, 24, None, 0)
gq, gs = got[p]
for r in range(max(len(q), len(gq))):
    print(r, idx[r] if r < len(q) else None, np.round(q[r], 4) if r < len(q) else None, s[r] if r < len(q) else None, '|', np.round(gq[r], 4) if r < len(gq) else None, gs[r] if r < len(gs) else None)
gsc = bmo.grid_scores(xi, L, 4, math.pi / 8)
print(sorted(gsc)[-30:])
