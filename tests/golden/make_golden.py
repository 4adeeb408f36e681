"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference
(oracle/_ref/libamgref.so, compiled from /root/reference/proj/src by
oracle/Makefile).  Run here (where /root/reference exists):

    make -C oracle ref && python tests/golden/make_golden.py

The fixtures let the CPU test suite pin the C restatement (oracle/amg_oracle.c)
against the reference without the reference being present (GPU box).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import problems as P  # noqa: E402
from oracle import ref  # noqa: E402

CASES = {
    "poisson1d_64_ce10": (lambda: P.poisson1d(64), dict(coarse_enough=10)),
    "poisson2d_24": (lambda: P.poisson2d(24), {}),
    "dambreak_12_k30": (lambda: P.grid3d_values("dambreak", 12, 30), {}),
    "poisson3d_10_k2": (lambda: P.grid3d_values("poisson", 10, 2), {}),
    "random_200": (lambda: P.random_csr(200, 200, 0.03, 5, diag=3.0), {}),
    "random_150_eps0.3": (lambda: P.random_csr(150, 150, 0.05, 9, diag=2.0), dict(eps=0.3)),
}


def dump_case(name, make, kw):
    A = make()
    prm = ref.params(**kw)
    h = ref.setup(A, prm)
    out = {"A_rp": A[0], "A_ci": A[1], "A_v": A[2], "nlev": len(h.levels), "params": np.array(
        [prm.eps, prm.omega, prm.pre_sweeps, prm.post_sweeps, prm.coarse_enough, prm.max_direct_size], np.float64)}
    for l, L in enumerate(h.levels):
        out[f"L{l}_rp"], out[f"L{l}_ci"], out[f"L{l}_v"] = L.A
        if L.agg is not None:
            out[f"L{l}_agg"] = L.agg
        if L.inv_diag is not None:
            out[f"L{l}_invd"] = L.inv_diag
    out["lu"], out["piv"] = h.lu, h.piv
    n = len(A[0]) - 1
    f = np.random.default_rng(7).uniform(-1, 1, n)
    out["vc_f"] = f
    out["vc_u_fixed"] = ref.vcycle(h, f, fixed=True, prm=prm)
    out["vc_u_shipped"] = ref.vcycle(h, f, fixed=False, prm=prm)
    s = ref.bicgstab(h, P.rhs(n), fixed=True, prm=prm)
    out["solve_fixed"] = np.array([s.iterations, s.converged, s.breakdown, s.relative_residual])
    out["solve_fixed_u"] = s.u
    s2 = ref.bicgstab(h, P.rhs(n), fixed=False, prm=prm)
    out["solve_shipped"] = np.array([s2.iterations, s2.converged, s2.breakdown, s2.relative_residual])
    # partial update with perturbed values
    B = (A[0], A[1], A[2] * (1.0 + 0.05 * np.random.default_rng(11).random(len(A[2]))))
    hu = ref.partial_update(h, B, prm)
    out["pu_v"] = B[2]
    for l, L in enumerate(hu.levels):
        out[f"PU{l}_v"] = L.A[2]
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    return len(h.levels)


def dump_aggregation():
    rng = np.random.default_rng(4242)
    graphs = {}
    for t in range(200):
        n = int(rng.integers(5, 60))
        m = int(rng.integers(0, 3 * n))
        e = set()
        for _ in range(m):
            a, b = int(rng.integers(0, n)), int(rng.integers(0, n))
            if a != b:
                e.add((a, b))
                e.add((b, a))
        rows = [[] for _ in range(n)]
        for a, b in sorted(e):
            rows[a].append(b)
        ptr = np.zeros(n + 1, np.int64)
        ptr[1:] = np.cumsum([len(r) for r in rows])
        adj = np.array([b for r in rows for b in r], np.int64)
        agg, nc = ref.aggregate(ptr, adj)
        graphs[f"g{t}_ptr"], graphs[f"g{t}_adj"], graphs[f"g{t}_agg"] = ptr, adj, agg
        graphs[f"g{t}_nc"] = np.array([nc])
    np.savez_compressed(os.path.join(HERE, "aggregation_200.npz"), **graphs)


if __name__ == "__main__":
    for name, (make, kw) in CASES.items():
        print(name, dump_case(name, make, kw), "levels")
    dump_aggregation()
    print("aggregation_200")
