"""TEST INFRASTRUCTURE ONLY — host generators of parity inputs (numpy).

* poisson1d / poisson2d / identity: the reference test oracles
  (proj/tests/unit/oracles.hpp:137-167), same entry order and values.
* grid3d: the g^3 7-point sequences of SURVEY.md §8(d), the 3D
  lift of the reference's 2D generator (proj/src/diffusion.cpp:54-118).  Every
  operation is an elementwise IEEE op in the same order as the device
  generator (paper_2108_02054_b200/csrc/kernels_gen.cu) and the C restatement
  (oracle/amg_oracle.c), so Poisson and dam-break values are bit-identical.
* random_csr: seeded random sparse matrices (not the reference's mt19937_64
  stream; the reference's own random matrices come via oracle/ref.py).
"""
from __future__ import annotations

import math

import numpy as np

POISSON, BLOB, DAMBREAK, CONVDIFF = 0, 1, 2, 3
KINDS = {"poisson": POISSON, "blob": BLOB, "dambreak": DAMBREAK, "convdiff": CONVDIFF}


def csr_from_dense_rows(rows, n, ncols=None):
    rp = [0]
    ci, v = [], []
    for r in rows:
        for c, x in sorted(r):
            ci.append(c)
            v.append(x)
        rp.append(len(ci))
    return (np.array(rp, np.int64), np.array(ci, np.int64), np.array(v, np.float64))


def poisson1d(n):
    """tridiag(-1, 2, -1) (oracles.hpp:137-145)."""
    rows = []
    for i in range(n):
        r = []
        if i > 0:
            r.append((i - 1, -1.0))
        r.append((i, 2.0))
        if i < n - 1:
            r.append((i + 1, -1.0))
        rows.append(r)
    return csr_from_dense_rows(rows, n)


def poisson2d(g):
    """5-point Laplacian, h = 1 (oracles.hpp:148-161)."""
    rows = []
    for iy in range(g):
        for ix in range(g):
            i = iy * g + ix
            r = [(i, 4.0)]
            if iy > 0:
                r.append((i - g, -1.0))
            if ix > 0:
                r.append((i - 1, -1.0))
            if ix < g - 1:
                r.append((i + 1, -1.0))
            if iy < g - 1:
                r.append((i + g, -1.0))
            rows.append(r)
    return csr_from_dense_rows(rows, g * g)


def identity(n):
    return (np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64), np.ones(n))


def diagonal(d):
    d = np.asarray(d, np.float64)
    n = len(d)
    return (np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64), d.copy())


def random_csr(n, ncols, fill, seed, diag=None):
    """Seeded random sparse matrix; optional dominant diagonal value base."""
    rng = np.random.default_rng(seed)
    rows = []
    for i in range(n):
        mask = rng.random(ncols) < fill
        cols = np.nonzero(mask)[0]
        vals = rng.uniform(-1.0, 1.0, len(cols))
        r = dict(zip(cols.tolist(), vals.tolist()))
        if diag is not None and i < ncols:
            r[i] = r.get(i, 0.0) + diag + rng.random()
        rows.append(list(r.items()))
    return csr_from_dense_rows(rows, n, ncols)


def grid3d_pattern(g):
    n = g ** 3
    idx = np.arange(n, dtype=np.int64)
    x, y, z = idx % g, (idx // g) % g, idx // (g * g)
    offs = [(-(g * g), z > 0), (-g, y > 0), (-1, x > 0), (0, np.ones(n, bool)), (1, x < g - 1),
            (g, y < g - 1), (g * g, z < g - 1)]
    counts = sum(m.astype(np.int64) for _, m in offs)
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=rp[1:])
    ci = np.zeros(rp[-1], np.int64)
    pos = rp[:-1].copy()
    for o, m in offs:
        ci[pos[m]] = idx[m] + o
        pos[m] += 1
    return rp, ci


def gen_params(kind, g, k, nsteps):
    """Same derivation as problem_values() in kernels_gen.cu."""
    h = 1.0 / float(g + 1)
    inv_h2 = 1.0 / (h * h)
    den = float(nsteps - 1 if nsteps > 1 else 1)
    gd = float(g)
    p = {"inv_h2": inv_h2}
    if kind == POISSON:
        p["shift"] = 0.01 * float(k + 1) * (6.0 * inv_h2)
    elif kind in (BLOB, CONVDIFF):
        p["contrast"] = 10.0
        sigma = 0.2 * gd
        p["inv_sigma2"] = 1.0 / (sigma * sigma)
        limit = gd - 1.0
        travel = float(k) * 0.25 / math.sqrt(3.0)
        pos = math.fmod(travel, 2.0 * limit)
        if pos > limit:
            pos = 2.0 * limit - pos
        p["c"] = pos
        if kind == CONVDIFF:
            th = 2.0 * math.pi * float(k) / den
            speed = 10.0 / h
            p["b"] = (speed * math.cos(th) / h, speed * math.sin(th) / h, 0.5 * speed / h)
    elif kind == DAMBREAK:
        p["a"] = gd * (0.25 + 0.5 * float(k) / den)
        p["bk"] = gd * (0.5 - 0.25 * float(k) / den)
    return p


def _node_coef(kind, p, x, y, z):
    if kind in (BLOB, CONVDIFF):
        dx = x.astype(np.float64) - p["c"]
        dy = y.astype(np.float64) - p["c"]
        dz = z.astype(np.float64) - p["c"]
        r2 = (dx * dx + dy * dy) + dz * dz
        return 1.0 + (p["contrast"] - 1.0) * np.exp(-(r2 * p["inv_sigma2"]))
    if kind == DAMBREAK:
        water = (x.astype(np.float64) < p["a"]) & (z.astype(np.float64) < p["bk"])
        return np.where(water, 1.0 / 1000.0, 1.0)
    return np.ones(x.shape)


def _harm(a, b):
    return ((2.0 * a) * b) / (a + b)


def grid3d_values(kind, g, k, nsteps=50):
    """Values of step k in grid3d_pattern(g) order."""
    kind = KINDS.get(kind, kind)
    p = gen_params(kind, g, k, nsteps)
    inv_h2 = p["inv_h2"]
    n = g ** 3
    idx = np.arange(n, dtype=np.int64)
    x, y, z = idx % g, (idx // g) % g, idx // (g * g)
    k0 = _node_coef(kind, p, x, y, z)

    def face(m, dx, dy, dz):
        out = k0.copy()
        out[m] = _harm(k0[m], _node_coef(kind, p, x[m] + dx, y[m] + dy, z[m] + dz))
        return out

    mz0, my0, mx0 = z > 0, y > 0, x > 0
    mx1, my1, mz1 = x < g - 1, y < g - 1, z < g - 1
    zlo, ylo, xlo = face(mz0, 0, 0, -1), face(my0, 0, -1, 0), face(mx0, -1, 0, 0)
    xhi, yhi, zhi = face(mx1, 1, 0, 0), face(my1, 0, 1, 0), face(mz1, 0, 0, 1)
    dg = (((((zlo + ylo) + xlo) + xhi) + yhi) + zhi) * inv_h2
    conv = {d: np.zeros(n) for d in ("zlo", "ylo", "xlo", "xhi", "yhi", "zhi")}
    if kind == CONVDIFF:
        bx, by, bz = p["b"]
        ax, ay, az = abs(bx), abs(by), abs(bz)
        dg = dg + ((ax + ay) + az)
        conv["xlo" if bx > 0 else "xhi"][:] = ax
        conv["ylo" if by > 0 else "yhi"][:] = ay
        conv["zlo" if bz > 0 else "zhi"][:] = az
    if kind == POISSON:
        dg = dg + p["shift"]
    rp, ci = grid3d_pattern(g)
    v = np.zeros(rp[-1])
    pos = rp[:-1].copy()
    entries = [(mz0, -(zlo * inv_h2 + conv["zlo"])), (my0, -(ylo * inv_h2 + conv["ylo"])),
               (mx0, -(xlo * inv_h2 + conv["xlo"])), (np.ones(n, bool), dg),
               (mx1, -(xhi * inv_h2 + conv["xhi"])), (my1, -(yhi * inv_h2 + conv["yhi"])),
               (mz1, -(zhi * inv_h2 + conv["zhi"]))]
    for m, val in entries:
        v[pos[m]] = val[m]
        pos[m] += 1
    return rp, ci, v


def rhs(n, seed=42):
    """f_i ~ U(0.1, 1.0).  The exact std::mt19937_64 stream of diffusion.cpp:38-41
    comes from the library (amgr_problem_rhs); this is a numpy stand-in for tests."""
    return np.random.default_rng(seed).uniform(0.1, 1.0, n)
