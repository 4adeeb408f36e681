"""One-off check of the extensions against the restated oracle at moderate
sizes: smoothed aggregation + CG, Chebyshev + BiCGStab, SPAI0 + BiCGStab.
usage: python tools/ext_check.py kind g"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_02054_b200 as amg  # noqa: E402
from oracle import oracle as O  # noqa: E402
from oracle import problems as P  # noqa: E402


def bits(x):
    return np.asarray(x, np.float64).view(np.int64)


kind, g = sys.argv[1], int(sys.argv[2])
A = P.grid3d_values(kind, g, 7) if kind != "convdiff" else O.grid3d("convdiff", g, 7)
n = g ** 3
fr = P.rhs(n)
f = np.random.default_rng(3).uniform(-1, 1, n)
for name, kw, solver in (("SA + CG", dict(coarsening="smoothed"), "cg"),
                         ("SPAI0 + BiCGStab", dict(smoother="spai0"), "bicgstab"),
                         ("Chebyshev + BiCGStab", dict(smoother="chebyshev", cheb_degree=3, power_iters=10), "bicgstab")):
    try:
        h = amg.setup(A, amg.AmgParams(**kw))
    except amg.AmgrError as e:
        h = e
    try:
        o = O.setup(A, O.params(**kw))
    except Exception as e:
        o = e
    if isinstance(h, Exception) or isinstance(o, Exception):
        print(f"{kind} {g}^3 {name}: device: {h if isinstance(h, Exception) else 'ok'}; "
              f"oracle: {o if isinstance(o, Exception) else 'ok'}", flush=True)
        continue
    vals = all(np.array_equal(bits(h.level_A(l)[2]), bits(L.A[2])) for l, L in enumerate(o.levels))
    u, uo = amg.vcycle(h, f), O.vcycle(o, f)
    vdiff = np.linalg.norm(u - uo) / np.linalg.norm(uo)
    _, st = getattr(amg, solver)(h, fr)
    so = getattr(O, solver)(o, fr)
    print(f"{kind} {g}^3 {name}: levels {h.num_levels()}/{len(o.levels)}, A_i values bit-exact {vals}, "
          f"V-cycle rel diff {vdiff:.1e}, {solver} {st.iterations} vs oracle {so.iterations} "
          f"(converged {st.converged}/{so.converged})", flush=True)
