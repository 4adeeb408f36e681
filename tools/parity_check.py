"""One-off parity check at larger sizes than the unit tests: device hierarchy
(patterns, values, aggregates, smoother, coarse LU), V-cycle and BiCGStab vs
the unmodified reference (oracle/_ref).  usage: python tools/parity_check.py kind g [k]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_02054_b200 as amg  # noqa: E402
from oracle import problems as P  # noqa: E402
from oracle import ref  # noqa: E402


def bits(x):
    return np.asarray(x, np.float64).view(np.int64)


def main():
    kind, g = sys.argv[1], int(sys.argv[2])
    k = int(sys.argv[3]) if len(sys.argv) > 3 else 7
    A = P.grid3d_values(kind, g, k)
    n = g ** 3
    t0 = time.time()
    r = ref.setup(A, ref.params())
    t_ref = time.time() - t0
    h = amg.setup(A)
    ok = h.num_levels() == len(r.levels)
    for l, L in enumerate(r.levels):
        rp, ci, v = h.level_A(l)
        ok &= np.array_equal(rp, L.A[0]) and np.array_equal(ci, L.A[1]) and np.array_equal(bits(v), bits(L.A[2]))
        if L.agg is not None:
            ok &= np.array_equal(h.level_agg(l), L.agg)
            ok &= np.array_equal(bits(h.level_smoother(l)), bits(L.inv_diag))
    lu, piv = h.coarse_lu()
    ok &= np.array_equal(piv, r.piv) and np.array_equal(bits(lu), bits(r.lu))
    f = np.random.default_rng(1).uniform(-1, 1, n)
    vok = np.array_equal(bits(amg.vcycle(h, f)), bits(ref.vcycle(r, f, fixed=True)))
    fr = P.rhs(n)
    _, st = amg.bicgstab(h, fr)
    rs = ref.bicgstab(r, fr, fixed=True)
    # partial update to a later step: frozen transfers, new Galerkin values
    A2 = P.grid3d_values(kind, g, k + 9)
    r2 = ref.partial_update(r, A2, ref.params())
    h2 = amg.partial_update(h, A2)
    pok = all(np.array_equal(bits(h2.level_A(l)[2]), bits(L.A[2])) for l, L in enumerate(r2.levels))
    pvok = np.array_equal(bits(amg.vcycle(h2, f)), bits(ref.vcycle(r2, f, fixed=True)))
    print(f"  partial update to k={k + 9}: level values bit-exact {pok}, V-cycle bit-exact {pvok}", flush=True)
    print(f"{kind} {g}^3 k={k}: levels {h.num_levels()}, hierarchy bit-exact {ok}, V-cycle bit-exact {vok}, "
          f"BiCGStab {st.iterations} vs reference {rs.iterations} (converged {st.converged}/{rs.converged}); "
          f"reference setup {t_ref:.1f} s", flush=True)


if __name__ == "__main__":
    main()
