"""TEST INFRASTRUCTURE ONLY — ctypes wrapper over oracle/liboracle.so, the
plain-C restatement of the reference path (oracle/amg_oracle.c).  Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline leg may import this.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")

_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


class OCsr(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("rp", C.c_void_p), ("ci", C.c_void_p),
                ("v", C.c_void_p)]


class OParams(C.Structure):
    _fields_ = [("eps", C.c_double), ("omega", C.c_double), ("pre_sweeps", C.c_int32),
                ("post_sweeps", C.c_int32), ("coarse_enough", C.c_int64), ("max_direct_size", C.c_int64),
                ("smoother", C.c_int32), ("coarsening", C.c_int32), ("sa_omega", C.c_double),
                ("cheb_degree", C.c_int32), ("power_iters", C.c_int32), ("cheb_lower", C.c_double),
                ("cheb_safety", C.c_double)]


SMOOTHER = {"jacobi": 0, "spai0": 1, "chebyshev": 2}


def params(eps=0.08, omega=0.72, pre_sweeps=1, post_sweeps=1, coarse_enough=100, max_direct_size=2000,
           smoother="jacobi", coarsening="plain", sa_omega=2.0 / 3.0, cheb_degree=3, power_iters=10,
           cheb_lower=0.3, cheb_safety=1.1) -> OParams:
    return OParams(eps, omega, pre_sweeps, post_sweeps, coarse_enough, max_direct_size, SMOOTHER[smoother],
                   {"plain": 0, "smoothed": 1}[coarsening], sa_omega, cheb_degree, power_iters, cheb_lower,
                   cheb_safety)


class OracleError(Exception):
    def __init__(self, kind, msg):
        super().__init__(msg)
        self.kind = {1: "invalid_argument", 2: "runtime_error"}.get(kind, "error")


_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle oracle`")
        L = C.CDLL(LIB_PATH)
        vp, i64, f64, cp = C.c_void_p, C.c_int64, C.c_double, C.c_char_p
        L.o_spmv.argtypes = [C.POINTER(OCsr), _f64p, _f64p]
        L.o_transpose.argtypes = [C.POINTER(OCsr), C.POINTER(OCsr)]
        L.o_spmm.argtypes = [C.POINTER(OCsr), C.POINTER(OCsr), C.POINTER(OCsr), cp, C.c_int]
        L.o_galerkin.argtypes = [C.POINTER(OCsr)] * 4 + [cp, C.c_int]
        L.o_free_csr.argtypes = [C.POINTER(OCsr)]
        L.o_strength.argtypes = [C.POINTER(OCsr), f64, C.POINTER(vp), C.POINTER(vp), cp, C.c_int]
        L.o_aggregate.argtypes = [i64, _i64p, _i64p, _i64p]
        L.o_aggregate.restype = i64
        L.o_factorize.argtypes = [C.POINTER(OCsr), _f64p, _i64p, cp, C.c_int]
        L.o_coarse_solve.argtypes = [i64, _f64p, _i64p, _f64p, _f64p]
        L.o_setup.argtypes = [C.POINTER(OCsr), C.POINTER(OParams), C.POINTER(vp), cp, C.c_int]
        L.o_partial_update.argtypes = [vp, C.POINTER(OCsr), C.POINTER(OParams), C.POINTER(vp), cp, C.c_int]
        L.o_vcycle.argtypes = [vp, _f64p, _f64p]
        L.o_free_hier.argtypes = [vp]
        L.o_num_levels.argtypes = [vp]
        L.o_level_dims.argtypes = [vp, C.c_int, _i64p]
        L.o_level_A.argtypes = [vp, C.c_int, _i64p, _i64p, _f64p]
        L.o_level_P.argtypes = [vp, C.c_int, _i64p, _i64p, _f64p]
        L.o_level_R.argtypes = [vp, C.c_int, _i64p, _i64p, _f64p]
        L.o_level_smoother.argtypes = [vp, C.c_int, _f64p, C.POINTER(f64)]
        L.o_coarse_n.argtypes = [vp]
        L.o_coarse_n.restype = i64
        L.o_coarse.argtypes = [vp, _f64p, _i64p]
        L.o_bicgstab.argtypes = [vp, _f64p, _f64p, _f64p, f64, i64, _i64p, C.POINTER(f64)]
        L.o_cg.argtypes = [vp, _f64p, _f64p, _f64p, f64, i64, _i64p, C.POINTER(f64)]
        L.o_grid3d.argtypes = [C.c_int, i64, i64, i64, _i64p, _i64p, _f64p]
        _lib = L
    return _lib


_keep = []


def _ocsr(A, ncols=None):
    rp = np.ascontiguousarray(A[0], np.int64)
    ci = np.ascontiguousarray(A[1], np.int64)
    v = np.ascontiguousarray(A[2], np.float64)
    n = len(rp) - 1
    o = OCsr(n, n if ncols is None else ncols, rp.ctypes.data, ci.ctypes.data, v.ctypes.data)
    o._keep = (rp, ci, v)
    return o


def _from_ocsr(o: OCsr, free=True):
    n = o.nrows
    rp = np.ctypeslib.as_array(C.cast(o.rp, C.POINTER(C.c_int64)), shape=(n + 1,)).copy()
    nnz = int(rp[-1])
    ci = np.ctypeslib.as_array(C.cast(o.ci, C.POINTER(C.c_int64)), shape=(max(nnz, 1),))[:nnz].copy()
    v = np.ctypeslib.as_array(C.cast(o.v, C.POINTER(C.c_double)), shape=(max(nnz, 1),))[:nnz].copy()
    if free:
        lib().o_free_csr(C.byref(o))
    return rp, ci, v


def _err():
    return C.create_string_buffer(1024)


def spmv(A, x):
    o = _ocsr(A, len(x))
    y = np.zeros(o.nrows)
    lib().o_spmv(C.byref(o), np.ascontiguousarray(x, np.float64), y)
    return y


def transpose(A, ncols):
    o = _ocsr(A, ncols)
    T = OCsr()
    lib().o_transpose(C.byref(o), C.byref(T))
    return _from_ocsr(T)


def spmm(A, B, a_ncols, b_ncols):
    a, b = _ocsr(A, a_ncols), _ocsr(B, b_ncols)
    Cc = OCsr()
    e = _err()
    rc = lib().o_spmm(C.byref(a), C.byref(b), C.byref(Cc), e, 1024)
    if rc:
        raise OracleError(rc, e.value.decode())
    return _from_ocsr(Cc)


def galerkin(A, agg, nc):
    n = len(A[0]) - 1
    P = (np.arange(n + 1, dtype=np.int64), np.asarray(agg, np.int64), np.ones(n))
    R = transpose(P, nc)
    r, a, p = _ocsr(R, n), _ocsr(A), _ocsr(P, nc)
    Cc = OCsr()
    e = _err()
    rc = lib().o_galerkin(C.byref(r), C.byref(a), C.byref(p), C.byref(Cc), e, 1024)
    if rc:
        raise OracleError(rc, e.value.decode())
    return _from_ocsr(Cc)


def strength(A, eps):
    o = _ocsr(A)
    ap, adj = C.c_void_p(), C.c_void_p()
    e = _err()
    rc = lib().o_strength(C.byref(o), eps, C.byref(ap), C.byref(adj), e, 1024)
    if rc:
        raise OracleError(rc, e.value.decode())
    n = o.nrows
    ptr = np.ctypeslib.as_array(C.cast(ap, C.POINTER(C.c_int64)), shape=(n + 1,)).copy()
    m = int(ptr[-1])
    a = np.ctypeslib.as_array(C.cast(adj, C.POINTER(C.c_int64)), shape=(max(m, 1),))[:m].copy()
    libc = C.CDLL(None)
    libc.free.argtypes = [C.c_void_p]
    libc.free(ap)
    libc.free(adj)
    return ptr, a


def aggregate(adj_ptr, adj):
    adj_ptr = np.ascontiguousarray(adj_ptr, np.int64)
    adj = np.ascontiguousarray(adj if len(adj) else np.zeros(1, np.int64), np.int64)
    n = len(adj_ptr) - 1
    out = np.zeros(max(n, 1), np.int64)
    nc = lib().o_aggregate(n, adj_ptr, adj, out)
    return out[:n], int(nc)


def factorize(A):
    o = _ocsr(A)
    n = o.nrows
    lu = np.zeros(max(n * n, 1))
    piv = np.zeros(max(n, 1), np.int64)
    e = _err()
    rc = lib().o_factorize(C.byref(o), lu, piv, e, 1024)
    if rc:
        raise OracleError(rc, e.value.decode())
    return lu[:n * n], piv[:n]


def coarse_solve(lu, piv, b):
    n = len(piv)
    x = np.zeros(n)
    lib().o_coarse_solve(n, np.ascontiguousarray(lu), np.ascontiguousarray(piv, np.int64),
                         np.ascontiguousarray(b, np.float64), x)
    return x


@dataclass
class OLevel:
    A: tuple
    P: tuple | None
    R: tuple | None
    w: np.ndarray | None
    lam_max: float | None

    @property
    def agg(self):
        return None if self.P is None else self.P[1]


@dataclass
class OHierarchy:
    levels: list = field(default_factory=list)
    lu: np.ndarray | None = None
    piv: np.ndarray | None = None
    handle: int | None = None

    def __del__(self):
        if self.handle:
            try:
                lib().o_free_hier(self.handle)
            except Exception:
                pass
            self.handle = None


def _extract(h) -> OHierarchy:
    L = lib()
    out = OHierarchy(handle=h)
    for l in range(L.o_num_levels(h)):
        d = np.zeros(6, np.int64)
        L.o_level_dims(h, l, d)
        n, nnz, has_p, nc, has_s, nnzp = (int(x) for x in d)
        rp, ci, v = np.zeros(n + 1, np.int64), np.zeros(max(nnz, 1), np.int64), np.zeros(max(nnz, 1))
        L.o_level_A(h, l, rp, ci, v)
        P = R = w = lam = None
        if has_p:
            prp, pci, pv = np.zeros(n + 1, np.int64), np.zeros(max(nnzp, 1), np.int64), np.zeros(max(nnzp, 1))
            L.o_level_P(h, l, prp, pci, pv)
            P = (prp, pci[:nnzp], pv[:nnzp])
            rrp, rci, rv = np.zeros(nc + 1, np.int64), np.zeros(max(nnzp, 1), np.int64), np.zeros(max(nnzp, 1))
            L.o_level_R(h, l, rrp, rci, rv)
            R = (rrp, rci[:nnzp], rv[:nnzp])
        if has_s:
            w = np.zeros(n)
            x = C.c_double()
            L.o_level_smoother(h, l, w, C.byref(x))
            lam = x.value
        out.levels.append(OLevel((rp, ci[:nnz], v[:nnz]), P, R, w, lam))
    nL = L.o_coarse_n(h)
    out.lu = np.zeros(max(nL * nL, 1))
    out.piv = np.zeros(max(nL, 1), np.int64)
    L.o_coarse(h, out.lu, out.piv)
    out.lu, out.piv = out.lu[:nL * nL], out.piv[:nL]
    return out


def setup(A, prm: OParams | None = None) -> OHierarchy:
    """hierarchy.cpp:45-105 restated."""
    o = _ocsr(A)
    h = C.c_void_p()
    e = _err()
    rc = lib().o_setup(C.byref(o), C.byref(prm or params()), C.byref(h), e, 1024)
    if rc:
        raise OracleError(rc, e.value.decode())
    return _extract(h.value)


def partial_update(h: OHierarchy, A, prm: OParams | None = None) -> OHierarchy:
    o = _ocsr(A)
    out = C.c_void_p()
    e = _err()
    rc = lib().o_partial_update(h.handle, C.byref(o), C.byref(prm or params()), C.byref(out), e, 1024)
    if rc:
        raise OracleError(rc, e.value.decode())
    return _extract(out.value)


def vcycle(h: OHierarchy, f):
    f = np.ascontiguousarray(f, np.float64)
    u = np.zeros_like(f)
    lib().o_vcycle(h.handle, f, u)
    return u


@dataclass
class OSolve:
    u: np.ndarray
    iterations: int
    converged: bool
    breakdown: bool
    relative_residual: float


def _solve(fn, h, f, u0, tol, max_iter):
    f = np.ascontiguousarray(f, np.float64)
    u0 = np.zeros_like(f) if u0 is None else np.ascontiguousarray(u0, np.float64)
    u = np.zeros_like(f)
    st = np.zeros(3, np.int64)
    rr = C.c_double()
    fn(h.handle, f, u0, u, tol, max_iter, st, C.byref(rr))
    return OSolve(u, int(st[0]), bool(st[1]), bool(st[2]), rr.value)


def bicgstab(h, f, u0=None, tol=1e-8, max_iter=100):
    return _solve(lib().o_bicgstab, h, f, u0, tol, max_iter)


def cg(h, f, u0=None, tol=1e-8, max_iter=100):
    return _solve(lib().o_cg, h, f, u0, tol, max_iter)


def grid3d(kind, g, k, nsteps=50):
    kinds = {"poisson": 0, "blob": 1, "dambreak": 2, "convdiff": 3}
    kind = kinds.get(kind, kind)
    n = g ** 3
    nnz = 7 * g ** 3 - 6 * g ** 2
    rp, ci, v = np.zeros(n + 1, np.int64), np.zeros(nnz, np.int64), np.zeros(nnz)
    lib().o_grid3d(kind, g, k, nsteps, rp, ci, v)
    return rp, ci, v
