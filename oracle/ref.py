"""TEST INFRASTRUCTURE ONLY — ctypes wrapper over oracle/_ref/libamgref.so.

libamgref.so is the UNMODIFIED reference library (/root/reference/proj/src,
compiled by oracle/Makefile with -O2 -ffp-contract=off) plus oracle/ref_shim.cpp.
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference arm
may import this module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libamgref.so")

_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


class RefParams(C.Structure):
    _fields_ = [("eps", C.c_double), ("omega", C.c_double), ("pre_sweeps", C.c_int32),
                ("post_sweeps", C.c_int32), ("coarse_enough", C.c_int64),
                ("max_direct_size", C.c_int64)]


def params(eps=0.08, omega=0.72, pre_sweeps=1, post_sweeps=1, coarse_enough=100,
           max_direct_size=2000) -> RefParams:
    """AmgParams defaults: proj/include/amgreuse/hierarchy.hpp:14-21."""
    return RefParams(eps, omega, pre_sweeps, post_sweeps, coarse_enough, max_direct_size)


class RefError(Exception):
    def __init__(self, kind: int, msg: str):
        super().__init__(msg)
        self.kind = {1: "invalid_argument", 2: "runtime_error"}.get(kind, "error")


_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle ref`")
        L = C.CDLL(LIB_PATH)
        vp, cp, i64, f64 = C.c_void_p, C.c_char_p, C.c_int64, C.c_double
        L.ref_setup.argtypes = [i64, _i64p, _i64p, _f64p, C.POINTER(RefParams),
                                C.POINTER(vp), C.POINTER(f64), cp, C.c_int]
        L.ref_setup_rect.argtypes = [i64, i64, _i64p, _i64p, _f64p, C.POINTER(RefParams),
                                     C.POINTER(vp), cp, C.c_int]
        L.ref_partial_update.argtypes = [vp, i64, i64, _i64p, _i64p, _f64p,
                                         C.POINTER(RefParams), C.POINTER(vp), C.POINTER(f64),
                                         cp, C.c_int]
        L.ref_mm_read.argtypes = [cp, _i64p, vp, vp, vp, cp, C.c_int]
        L.ref_mm_read.restype = C.c_int
        L.ref_mm_read_vector.argtypes = [cp, C.POINTER(i64), vp, cp, C.c_int]
        L.ref_mm_read_vector.restype = C.c_int
        L.ref_render.restype = C.c_int
        L.ref_free.argtypes = [vp]
        L.ref_num_levels.argtypes = [vp]
        L.ref_num_levels.restype = i64
        L.ref_level_dims.argtypes = [vp, i64, _i64p]
        L.ref_level_A.argtypes = [vp, i64, _i64p, _i64p, _f64p]
        L.ref_level_P.argtypes = [vp, i64, _i64p, _i64p, _f64p]
        L.ref_level_R.argtypes = [vp, i64, _i64p, _i64p, _f64p]
        L.ref_level_invdiag.argtypes = [vp, i64, _f64p, C.POINTER(f64)]
        L.ref_coarse_n.argtypes = [vp]
        L.ref_coarse_n.restype = i64
        L.ref_coarse.argtypes = [vp, _f64p, _i64p]
        L.ref_timings.argtypes = [vp, _f64p]
        L.ref_operator_complexity.argtypes = [vp]
        L.ref_operator_complexity.restype = f64
        L.ref_vcycle.argtypes = [vp, _f64p, _f64p, C.c_int, C.POINTER(RefParams),
                                 C.POINTER(f64), cp, C.c_int]
        L.ref_bicgstab.argtypes = [vp, _f64p, _f64p, _f64p, f64, i64, C.c_int,
                                   C.POINTER(RefParams), _i64p, C.POINTER(f64), C.POINTER(f64),
                                   cp, C.c_int]
        L.ref_strength.argtypes = [i64, _i64p, _i64p, _f64p, f64, C.c_void_p, C.c_void_p, i64,
                                   cp, C.c_int]
        L.ref_strength.restype = i64
        L.ref_aggregate.argtypes = [i64, _i64p, _i64p, _i64p]
        L.ref_aggregate.restype = i64
        L.ref_spmv.argtypes = [i64, i64, _i64p, _i64p, _f64p, _f64p, _f64p]
        L.ref_galerkin.argtypes = [i64, i64, _i64p, _i64p, _f64p, _i64p, C.c_void_p,
                                   C.c_void_p, C.c_void_p]
        L.ref_galerkin.restype = i64
        L.ref_coarse_factorize.argtypes = [i64, _i64p, _i64p, _f64p, _f64p, _i64p, cp, C.c_int]
        _lib = L
    return _lib


def _csr(A):
    rp = np.ascontiguousarray(A[0], dtype=np.int64)
    ci = np.ascontiguousarray(A[1], dtype=np.int64)
    v = np.ascontiguousarray(A[2], dtype=np.float64)
    return rp, ci, v


@dataclass
class RefLevel:
    A: tuple                    # (row_ptr, col_idx, values) int64/int64/float64
    agg: np.ndarray | None      # P col_idx (aggregate id per fine row)
    R: tuple | None             # (row_ptr, col_idx, values)
    inv_diag: np.ndarray | None
    omega: float | None


@dataclass
class RefHierarchy:
    levels: list = field(default_factory=list)
    lu: np.ndarray | None = None
    piv: np.ndarray | None = None
    timings: np.ndarray | None = None
    seconds: float = 0.0
    handle: int | None = None

    def free(self):
        if self.handle:
            lib().ref_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _extract(h: int) -> RefHierarchy:
    L = lib()
    out = RefHierarchy(handle=h)
    nl = L.ref_num_levels(h)
    for i in range(nl):
        d = np.zeros(5, np.int64)
        L.ref_level_dims(h, i, d)
        n, nnz, has_p, nc, has_s = (int(x) for x in d)
        rp = np.zeros(n + 1, np.int64)
        ci = np.zeros(nnz, np.int64)
        v = np.zeros(nnz, np.float64)
        L.ref_level_A(h, i, rp, ci, v)
        agg = R = invd = om = None
        if has_p:
            prp, pci, pv = np.zeros(n + 1, np.int64), np.zeros(n, np.int64), np.zeros(n)
            L.ref_level_P(h, i, prp, pci, pv)
            agg = pci
            rrp, rci, rv = np.zeros(nc + 1, np.int64), np.zeros(n, np.int64), np.zeros(n)
            L.ref_level_R(h, i, rrp, rci, rv)
            R = (rrp, rci, rv)
        if has_s:
            invd = np.zeros(n)
            o = C.c_double()
            L.ref_level_invdiag(h, i, invd, C.byref(o))
            om = o.value
        out.levels.append(RefLevel((rp, ci, v), agg, R, invd, om))
    nc = L.ref_coarse_n(h)
    out.lu = np.zeros(nc * nc)
    out.piv = np.zeros(nc, np.int64)
    L.ref_coarse(h, out.lu, out.piv)
    out.timings = np.zeros(4)
    L.ref_timings(h, out.timings)
    return out


def _err():
    return C.create_string_buffer(1024)


def setup(A, prm: RefParams | None = None) -> RefHierarchy:
    """proj/src/hierarchy.cpp:45-105 (as shipped)."""
    rp, ci, v = _csr(A)
    n = len(rp) - 1
    h = C.c_void_p()
    secs = C.c_double()
    e = _err()
    rc = lib().ref_setup(n, rp, ci, v, C.byref(prm or params()), C.byref(h), C.byref(secs), e, 1024)
    if rc:
        raise RefError(rc, e.value.decode())
    out = _extract(h.value)
    out.seconds = secs.value
    return out


def partial_update(h: RefHierarchy, A, prm: RefParams | None = None, ncols=None) -> RefHierarchy:
    """proj/src/hierarchy.cpp:107-150 (as shipped)."""
    rp, ci, v = _csr(A)
    n = len(rp) - 1
    out = C.c_void_p()
    secs = C.c_double()
    e = _err()
    rc = lib().ref_partial_update(h.handle, n, n if ncols is None else ncols, rp, ci, v,
                                  C.byref(prm or params()), C.byref(out), C.byref(secs), e, 1024)
    if rc:
        raise RefError(rc, e.value.decode())
    res = _extract(out.value)
    res.seconds = secs.value
    return res


def vcycle(h: RefHierarchy, f, fixed=True, prm: RefParams | None = None):
    f = np.ascontiguousarray(f, dtype=np.float64)
    u = np.zeros_like(f)
    secs = C.c_double()
    e = _err()
    rc = lib().ref_vcycle(h.handle, f, u, int(fixed), C.byref(prm or params()), C.byref(secs), e, 1024)
    if rc:
        raise RefError(rc, e.value.decode())
    return u


@dataclass
class RefSolve:
    u: np.ndarray
    iterations: int
    converged: bool
    breakdown: bool
    relative_residual: float
    seconds: float


def bicgstab(h: RefHierarchy, f, u0=None, tol=1e-8, max_iter=100, fixed=True,
             prm: RefParams | None = None) -> RefSolve:
    """proj/src/bicgstab.cpp:21-135 with A = finest matrix, M = V-cycle."""
    f = np.ascontiguousarray(f, dtype=np.float64)
    u0 = np.zeros_like(f) if u0 is None else np.ascontiguousarray(u0, dtype=np.float64)
    u = np.zeros_like(f)
    st = np.zeros(3, np.int64)
    rr = C.c_double()
    secs = C.c_double()
    e = _err()
    rc = lib().ref_bicgstab(h.handle, f, u0, u, tol, max_iter, int(fixed), C.byref(prm or params()),
                            st, C.byref(rr), C.byref(secs), e, 1024)
    if rc:
        raise RefError(rc, e.value.decode())
    return RefSolve(u, int(st[0]), bool(st[1]), bool(st[2]), rr.value, secs.value)


def strength(A, eps):
    rp, ci, v = _csr(A)
    n = len(rp) - 1
    e = _err()
    adj_ptr = np.zeros(n + 1, np.int64)
    m = lib().ref_strength(n, rp, ci, v, eps, adj_ptr.ctypes.data, None, 0, e, 1024)
    if m < 0:
        raise RefError(1, e.value.decode())
    adj = np.zeros(max(m, 1), np.int64)
    lib().ref_strength(n, rp, ci, v, eps, adj_ptr.ctypes.data, adj.ctypes.data, m, e, 1024)
    return adj_ptr, adj[:m]


def aggregate(adj_ptr, adj):
    adj_ptr = np.ascontiguousarray(adj_ptr, np.int64)
    adj = np.ascontiguousarray(adj if len(adj) else np.zeros(1, np.int64), np.int64)
    n = len(adj_ptr) - 1
    out = np.zeros(max(n, 1), np.int64)
    nc = lib().ref_aggregate(n, adj_ptr, adj, out)
    return out[:n], int(nc)


def spmv(A, x, ncols=None):
    rp, ci, v = _csr(A)
    n = len(rp) - 1
    x = np.ascontiguousarray(x, np.float64)
    y = np.zeros(n)
    lib().ref_spmv(n, len(x) if ncols is None else ncols, rp, ci, v, x, y)
    return y


def galerkin(A, agg, nc):
    rp, ci, v = _csr(A)
    n = len(rp) - 1
    agg = np.ascontiguousarray(agg, np.int64)
    nnz = lib().ref_galerkin(n, nc, rp, ci, v, agg, None, None, None)
    crp, cci, cv = np.zeros(nc + 1, np.int64), np.zeros(nnz, np.int64), np.zeros(nnz)
    lib().ref_galerkin(n, nc, rp, ci, v, agg, crp.ctypes.data, cci.ctypes.data, cv.ctypes.data)
    return crp, cci, cv


def mm_read(path):
    """amgreuse::mm_read through the unmodified reference -> (rp, ci, v, ncols)."""
    dims = np.zeros(3, np.int64)
    err = C.create_string_buffer(1024)
    rc = lib().ref_mm_read(str(path).encode(), dims, None, None, None, err, 1024)
    if rc:
        raise RefError(rc, err.value.decode())
    rp = np.zeros(dims[0] + 1, np.int64)
    ci = np.zeros(max(dims[2], 1), np.int64)
    v = np.zeros(max(dims[2], 1))
    rc = lib().ref_mm_read(str(path).encode(), dims, rp.ctypes.data, ci.ctypes.data, v.ctypes.data, err, 1024)
    if rc:
        raise RefError(rc, err.value.decode())
    return rp, ci[:dims[2]], v[:dims[2]], int(dims[1])


def mm_read_vector(path):
    n = C.c_int64()
    err = C.create_string_buffer(1024)
    rc = lib().ref_mm_read_vector(str(path).encode(), C.byref(n), None, err, 1024)
    if rc:
        raise RefError(rc, err.value.decode())
    v = np.zeros(max(n.value, 1))
    rc = lib().ref_mm_read_vector(str(path).encode(), C.byref(n), v.ctypes.data, err, 1024)
    if rc:
        raise RefError(rc, err.value.decode())
    return v[:n.value]


def render(which, fmt, seqdir, amg, solve, reuse_iter_limit, rebuild_every, kinds, steps):
    """tools/bench_app.cpp render_report (which 0) / write_per_step_csv (which 1)
    of the unmodified reference over given run data.  steps[s][k] =
    (action, setup, solve, iterations, converged, (4 phase times))."""
    ns = len(steps[0])
    act = np.array([[x[0] for x in row] for row in steps], np.int32).ravel()
    se = np.array([[x[1] for x in row] for row in steps], np.float64).ravel()
    so = np.array([[x[2] for x in row] for row in steps], np.float64).ravel()
    it = np.array([[x[3] for x in row] for row in steps], np.int64).ravel()
    cv = np.array([[x[4] for x in row] for row in steps], np.int32).ravel()
    ph = np.array([[x[5] for x in row] for row in steps], np.float64).ravel()
    kk = np.array(kinds, np.int32)
    buf = C.create_string_buffer(1 << 20)
    f64, i64 = C.c_double, C.c_int64
    rc = lib().ref_render(C.c_int(which), C.c_int(fmt), str(seqdir).encode(), f64(amg[0]), f64(amg[1]),
                          C.c_int(amg[2]), C.c_int(amg[3]), i64(amg[4]), f64(solve[0]), i64(solve[1]),
                          i64(reuse_iter_limit), i64(rebuild_every or 0), C.c_int(len(kinds)),
                          kk.ctypes.data_as(C.c_void_p), i64(ns), act.ctypes.data_as(C.c_void_p),
                          se.ctypes.data_as(C.c_void_p), so.ctypes.data_as(C.c_void_p),
                          it.ctypes.data_as(C.c_void_p), cv.ctypes.data_as(C.c_void_p),
                          ph.ctypes.data_as(C.c_void_p), buf, C.c_int(1 << 20))
    if rc:
        raise RefError(1, buf.value.decode())
    return buf.value.decode()
