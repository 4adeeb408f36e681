"""B200-native partial-reuse AMG (arXiv 2108.02054) — Python mirror of the
reference's C++ solver API over the C-ABI of ``libamgr_b200.so``.

The reference (``/root/reference/proj``, library ``amgreuse``) exposes
``setup`` / ``partial_update`` / ``vcycle`` / ``bicgstab`` (+ ``run_sequence``
with reuse modes none|full|partial).  This module keeps those names, argument
meanings and error behaviour (``InvalidArgument`` <-> ``std::invalid_argument``,
``RuntimeFailure`` <-> ``std::runtime_error``, same message text) while every
computation runs in hand-written sm_100a kernels behind ``include/amgr.h``.

There is no CPU fallback: importing works without a GPU (for introspection
and the symbol checks), but every compute call requires the CUDA library and a
B200; if ``libamgr_b200.so`` is missing, import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import weakref
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "AmgParams", "SolveParams", "SolveStats", "PhaseTimings", "CsrMatrix", "Context", "Hierarchy",
    "setup", "partial_update", "vcycle", "bicgstab", "cg", "InvalidArgument", "RuntimeFailure",
    "DimensionChange", "CudaFailure", "LIB_PATH", "lib", "run_sequence",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libamgr_b200.so")
# development A/B of kernel variants: AMGR_LIB=<path to another build>
LIB_PATH = os.environ.get("AMGR_LIB", LIB_PATH)

HOST, DEVICE, DEVICE_ADOPT, STAGED = 0, 1, 2, 3


class _StagedRhs:
    def __repr__(self):
        return "STAGED_RHS"


STAGED_RHS = _StagedRhs()  # bicgstab(h, STAGED_RHS, (u0_ptr, u_ptr)): f = the staged RHS
SMOOTHER = {"jacobi": 0, "spai0": 1, "chebyshev": 2}
COARSENING = {"plain": 0, "smoothed": 1}
COARSE_SOLVE = {"exact": 0, "inverse": 1}
PROBLEM = {"poisson": 0, "blob": 1, "dambreak": 2, "convdiff": 3}


class AmgrError(Exception):
    pass


class InvalidArgument(AmgrError, ValueError):
    """std::invalid_argument in the reference."""


class DimensionChange(InvalidArgument):
    """partial update impossible, full rebuild required (reuse.cpp:69-70)."""


class RuntimeFailure(AmgrError, RuntimeError):
    """std::runtime_error in the reference (coarsening stalled, singular)."""


class CudaFailure(AmgrError, RuntimeError):
    pass


_ERR = {1: InvalidArgument, 2: RuntimeFailure, 3: CudaFailure, 4: CudaFailure, 5: DimensionChange}


class _Csr(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("nnz", C.c_int64), ("row_ptr", C.c_void_p),
                ("col_idx", C.c_void_p), ("values", C.c_void_p), ("index_bits", C.c_int32),
                ("location", C.c_int32)]


class _AmgParams(C.Structure):
    _fields_ = [("eps", C.c_double), ("omega", C.c_double), ("pre_sweeps", C.c_int32),
                ("post_sweeps", C.c_int32), ("coarse_enough", C.c_int64), ("max_direct_size", C.c_int64),
                ("smoother", C.c_int32), ("coarsening", C.c_int32), ("sa_omega", C.c_double),
                ("cheb_degree", C.c_int32), ("power_iters", C.c_int32), ("cheb_lower", C.c_double),
                ("cheb_safety", C.c_double), ("coarse_solve", C.c_int32), ("reserved", C.c_int32)]


class _SolveParams(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iter", C.c_int64)]


class _SolveStats(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("relative_residual", C.c_double), ("converged", C.c_int32),
                ("breakdown", C.c_int32)]


class _Timings(C.Structure):
    _fields_ = [("transfer_ops", C.c_double), ("galerkin", C.c_double), ("smoother", C.c_double),
                ("coarse_solver", C.c_double)]


# exported symbols and their prototypes (kept in sync with include/amgr.h;
# tests/test_abi.py checks both directions)
_V, _P, _I, _L, _D = C.c_void_p, C.POINTER, C.c_int, C.c_int64, C.c_double
PROTOTYPES = {
    "amgr_ctx_create": (_I, [_I, _V, _P(_V)]),
    "amgr_ctx_destroy": (None, [_V]),
    "amgr_last_error": (C.c_char_p, [_V]),
    "amgr_ctx_stream": (_V, [_V]),
    "amgr_ctx_synchronize": (_I, [_V]),
    "amgr_ctx_set_dot_order": (_I, [_V, _I]),
    "amgr_ctx_dot_order": (_I, [_V]),
    "amgr_version": (C.c_char_p, []),
    "amgr_amg_params_default": (None, [_P(_AmgParams)]),
    "amgr_solve_params_default": (None, [_P(_SolveParams)]),
    "amgr_setup": (_I, [_V, _P(_Csr), _P(_AmgParams), _P(_V)]),
    "amgr_partial_update": (_I, [_V, _P(_Csr), _P(_AmgParams), _P(_V)]),
    "amgr_rebuild": (_I, [_V, _P(_Csr)]),
    "amgr_rebuild_values": (_I, [_V, _V, _I]),
    "amgr_vcycle": (_I, [_V, _V, _V, _I]),
    "amgr_hier_destroy": (None, [_V]),
    "amgr_bicgstab": (_I, [_V, _V, _V, _V, _P(_SolveParams), _P(_SolveStats), _I]),
    "amgr_cg": (_I, [_V, _V, _V, _V, _P(_SolveParams), _P(_SolveStats), _I]),
    "amgr_spmv": (_I, [_V, _I, _V, _V, _I]),
    "amgr_csr_spmv": (_I, [_V, _P(_Csr), _V, _V, _I]),
    "amgr_build_smoother": (_I, [_V, _P(_Csr), _V, _I]),
    "amgr_smooth": (_I, [_V, _P(_Csr), _V, _D, _V, _V, _I, _I]),
    "amgr_coarse_factorize": (_I, [_V, _P(_Csr), _V, _V]),
    "amgr_coarse_solve": (_I, [_V, _L, _V, _V, _V, _V]),
    "amgr_hier_num_levels": (_I, [_V]),
    "amgr_hier_level_dims": (_I, [_V, _I, _V]),
    "amgr_hier_level_layout": (_I, [_V, _I, _V, _V]),
    "amgr_hier_level_stencil": (_I, [_V, _I, _V, _V]),
    "amgr_hier_level_A": (_I, [_V, _I, _V, _V, _V]),
    "amgr_hier_level_P": (_I, [_V, _I, _V]),
    "amgr_hier_level_R": (_I, [_V, _I, _V, _V]),
    "amgr_hier_level_smoother": (_I, [_V, _I, _V]),
    "amgr_hier_level_lambda": (_I, [_V, _I, _P(_D)]),
    "amgr_hier_coarse_n": (_L, [_V]),
    "amgr_hier_coarse_lu": (_I, [_V, _V, _V]),
    "amgr_hier_operator_complexity": (_D, [_V]),
    "amgr_hier_timings": (_I, [_V, _P(_Timings)]),
    "amgr_hier_shares_transfer": (_I, [_V, _V, _I]),
    "amgr_problem_nnz": (_L, [_L]),
    "amgr_problem_pattern": (_I, [_V, _L, _V, _V]),
    "amgr_problem_values": (_I, [_V, _I, _L, _L, _L, _V]),
    "amgr_problem_rhs": (_I, [_V, _L, C.c_uint64, _V, _I]),
    "amgr_probe_enable": (_I, [_V, C.c_char_p]),
    "amgr_probe_read": (_I, [_V, _P(_L), _P(_D), _P(_D)]),
    "amgr_launch_count": (_L, [_V]),
    "amgr_copy_to_host": (_I, [_V, _V, _V, C.c_size_t]),
    "amgr_run_sequence": (_I, [_V, _L, _V, _V, _V, _V, _V, _V, _V, _V]),
    "amgr_speedup_percent": (_D, [_D, _D]),
    "amgr_hier_level_transfer": (_I, [_V, _I, _I, _P(_L), _V, _V, _V]),
    "amgr_stage_values": (_I, [_V, _V, _I]),
    "amgr_stage_rhs": (_I, [_V, _V, _I]),
    "amgr_download_async": (_I, [_V, _V, _V, _L]),
    "amgr_mm_read": (_I, [_V, C.c_char_p, _P(_V)]),
    "amgr_matrix_csr": (_I, [_V, _P(_Csr)]),
    "amgr_csr_from_triplets": (_I, [_V, _L, _L, _L, _V, _V, _V, _P(_V)]),
    "amgr_matrix_free": (None, [_V]),
    "amgr_mm_read_vector": (_I, [_V, C.c_char_p, _P(_L), _V]),
    "amgr_nccl_unique_id": (_I, [_V]),
    "amgr_dist_create": (_I, [_V, _V, _I, _I, _I, _V, _L, _V, _P(_V)]),
    "amgr_dist_loopback_create": (_I, [_I, _P(_V)]),
    "amgr_dist_loopback_destroy": (None, [_V]),
    "amgr_dist_create_loopback": (_I, [_V, _V, _I, _I, _I, _V, _L, _V, _P(_V)]),
    "amgr_dist_rebuild_values": (_I, [_V, _V, _I]),
    "amgr_dist_create_auto": (_I, [_V, _V, _I, _I, _L, _P(_V)]),
    "amgr_dist_create_auto_loopback": (_I, [_V, _V, _I, _I, _L, _P(_V)]),
    "amgr_dist_level_dims": (_I, [_V, _I, _V]),
    "amgr_dist_level_maps": (_I, [_V, _I, _V, _V]),
    "amgr_dist_level_code": (_I, [_V, _I, _V]),
    "amgr_dist_rebuild_local": (_I, [_V, _V, _I]),
    "amgr_dist_vcycle": (_I, [_V, _V, _V]),
    "amgr_dist_bicgstab": (_I, [_V, _V, _V, _P(_SolveParams), _P(_SolveStats)]),
    "amgr_dist_destroy": (None, [_V]),
}

DOTS_BLOCKED, DOTS_SEQUENTIAL = 0, 1

_lib = None


def lib():
    """Load libamgr_b200.so (in-tree).  Fails loudly when it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing — build it with `make -C paper_2108_02054_b200/csrc` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in PROTOTYPES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


@dataclass
class AmgParams:
    """AmgParams (proj/include/amgreuse/hierarchy.hpp:14-21) + extensions."""
    eps: float = 0.08
    omega: float = 0.72
    pre_sweeps: int = 1
    post_sweeps: int = 1
    coarse_enough: int = 100
    max_direct_size: int = 2000
    smoother: str = "jacobi"
    coarsening: str = "plain"
    sa_omega: float = 2.0 / 3.0
    cheb_degree: int = 3
    power_iters: int = 10
    cheb_lower: float = 0.3
    cheb_safety: float = 1.1
    coarse_solve: str = "exact"

    def _c(self) -> _AmgParams:
        return _AmgParams(self.eps, self.omega, self.pre_sweeps, self.post_sweeps, self.coarse_enough,
                          self.max_direct_size, SMOOTHER[self.smoother], COARSENING[self.coarsening],
                          self.sa_omega, self.cheb_degree, self.power_iters, self.cheb_lower, self.cheb_safety,
                          COARSE_SOLVE[self.coarse_solve], 0)


@dataclass
class SolveParams:
    """SolveParams (bicgstab.hpp:17-20)."""
    tol: float = 1e-8
    max_iter: int = 100


@dataclass
class SolveStats:
    """SolveStats (bicgstab.hpp:22-27)."""
    iterations: int = 0
    relative_residual: float = 0.0
    converged: bool = False
    breakdown: bool = False


@dataclass
class PhaseTimings:
    """SetupPhaseTimings (hierarchy.hpp:24-38), seconds."""
    transfer_ops: float = 0.0
    galerkin: float = 0.0
    smoother: float = 0.0
    coarse_solver: float = 0.0

    def total(self) -> float:
        return self.transfer_ops + self.galerkin + self.smoother + self.coarse_solver


@dataclass
class CsrMatrix:
    """Host CSR (csr.hpp:25-45): int64 indices, fp64 values."""
    nrows: int
    ncols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(len(self.col_idx))

    @staticmethod
    def of(A) -> "CsrMatrix":
        if isinstance(A, CsrMatrix):
            return A
        rp, ci, v = A[:3]
        n = len(rp) - 1
        ncols = A[3] if len(A) > 3 else n
        return CsrMatrix(n, ncols, np.ascontiguousarray(rp, np.int64), np.ascontiguousarray(ci, np.int64),
                         np.ascontiguousarray(v, np.float64))

    def _c(self) -> _Csr:
        return _Csr(self.nrows, self.ncols, self.nnz, self.row_ptr.ctypes.data, self.col_idx.ctypes.data,
                    self.values.ctypes.data, 64, HOST)


@dataclass
class DeviceCsr:
    """CSR already resident on the device (raw pointers, e.g. torch data_ptr())."""
    nrows: int
    ncols: int
    nnz: int
    row_ptr: int
    col_idx: int
    values: int
    index_bits: int = 32

    def _c(self) -> _Csr:
        return _Csr(self.nrows, self.ncols, self.nnz, self.row_ptr, self.col_idx, self.values, self.index_bits,
                    DEVICE)


def _check(st: int, ctx_ptr):
    if st != 0:
        msg = lib().amgr_last_error(ctx_ptr) if ctx_ptr is not None else b""
        msg = msg.decode() if msg else ""
        raise _ERR.get(st, AmgrError)(msg)


class Context:
    """One device + one stream (amgr_ctx)."""

    def __init__(self, device: int = 0, stream: int | None = None):
        self._p = C.c_void_p()
        st = lib().amgr_ctx_create(device, stream, C.byref(self._p))
        if st != 0:
            msg = lib().amgr_last_error(None)
            raise _ERR.get(st, AmgrError)(msg.decode() if msg else "amgr_ctx_create failed")
        self.device = device

    @property
    def ptr(self):
        return self._p

    @property
    def stream(self) -> int:
        return lib().amgr_ctx_stream(self._p) or 0

    def synchronize(self):
        """amgr_ctx_synchronize: the context stream and the copy / download streams."""
        _check(lib().amgr_ctx_synchronize(self._p), self._p)

    def download_async(self, device_ptr: int, host_ptr: int, n: int):
        """amgr_download_async: snapshot n doubles at device_ptr (stream-ordered)
        and copy them to host_ptr on the download stream; complete after
        synchronize()."""
        _check(lib().amgr_download_async(self._p, device_ptr, host_ptr, n), self._p)

    def launches(self) -> int:
        return int(lib().amgr_launch_count(self._p))

    @property
    def sequential_dots(self) -> bool:
        """amgr_ctx_dot_order: True when every Krylov dot/norm is summed strictly
        left to right as the reference's dot (bicgstab.cpp:11-17)."""
        return int(lib().amgr_ctx_dot_order(self._p)) == DOTS_SEQUENTIAL

    @sequential_dots.setter
    def sequential_dots(self, on: bool):
        _check(lib().amgr_ctx_set_dot_order(self._p, DOTS_SEQUENTIAL if on else DOTS_BLOCKED), self._p)

    def probe(self, family: str | None):
        _check(lib().amgr_probe_enable(self._p, (family or "").encode()), self._p)

    def probe_read(self):
        n, ms, b = C.c_int64(), C.c_double(), C.c_double()
        _check(lib().amgr_probe_read(self._p, C.byref(n), C.byref(ms), C.byref(b)), self._p)
        return int(n.value), float(ms.value), float(b.value)

    def _adopt(self, obj):
        """Register an object owning device state of this context: closed
        before the context is (garbage collection of reference cycles may
        finalize a context before the objects using it)."""
        if not hasattr(self, "_children"):
            self._children = weakref.WeakSet()
        self._children.add(obj)
        return obj

    def close(self):
        if self._p:
            for ch in list(getattr(self, "_children", ())):
                try:
                    ch.close()
                except Exception:
                    pass
            lib().amgr_ctx_destroy(self._p)
            self._p = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def _f64(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float64)


class Hierarchy:
    """Device-resident AMG hierarchy (Hierarchy, hierarchy.hpp:49-59)."""

    def __init__(self, ptr, ctx: Context, prm: AmgParams):
        self._p = ptr
        self.ctx = ctx
        self.prm = prm
        ctx._adopt(self)

    # --- introspection (parity dumps) ---
    def num_levels(self) -> int:
        return int(lib().amgr_hier_num_levels(self._p))

    def level_dims(self, lvl: int):
        d = np.zeros(4, np.int64)
        _check(lib().amgr_hier_level_dims(self._p, lvl, d.ctypes.data), self.ctx.ptr)
        return {"nrows": int(d[0]), "nnz": int(d[1]), "n_coarse": int(d[2]), "has_smoother": bool(d[3])}

    def level_layout(self, lvl: int):
        """Row-pass layout of A_lvl: bytes per stored column (4 raw, 1/2
        coded) and the offset-dictionary size (amgr_hier_level_layout)."""
        cb, nd = C.c_int32(), C.c_int32()
        _check(lib().amgr_hier_level_layout(self._p, lvl, C.byref(cb), C.byref(nd)), self.ctx.ptr)
        return {"col_bytes": int(cb.value), "ndict": int(nd.value)}

    def level_stencil(self, lvl: int):
        """(K, offsets) when the row passes read A_lvl in its symmetric-stencil
        form (diagonal + K upper diagonals), (0, ()) when they read the CSR
        arrays (amgr_hier_level_stencil)."""
        k = C.c_int32()
        off = np.zeros(3, np.int32)
        _check(lib().amgr_hier_level_stencil(self._p, lvl, C.byref(k), off.ctypes.data), self.ctx.ptr)
        return int(k.value), tuple(int(x) for x in off[:k.value])

    def finest_size(self) -> int:
        return self.level_dims(0)["nrows"]

    def level_A(self, lvl: int):
        d = self.level_dims(lvl)
        rp = np.zeros(d["nrows"] + 1, np.int64)
        ci = np.zeros(max(d["nnz"], 1), np.int64)
        v = np.zeros(max(d["nnz"], 1))
        _check(lib().amgr_hier_level_A(self._p, lvl, rp.ctypes.data, ci.ctypes.data, v.ctypes.data), self.ctx.ptr)
        return rp, ci[:d["nnz"]], v[:d["nnz"]]

    def level_agg(self, lvl: int) -> np.ndarray:
        d = self.level_dims(lvl)
        a = np.zeros(d["nrows"], np.int64)
        _check(lib().amgr_hier_level_P(self._p, lvl, a.ctypes.data), self.ctx.ptr)
        return a

    def level_R(self, lvl: int):
        d = self.level_dims(lvl)
        rp = np.zeros(d["n_coarse"] + 1, np.int64)
        ci = np.zeros(d["nrows"], np.int64)
        _check(lib().amgr_hier_level_R(self._p, lvl, rp.ctypes.data, ci.ctypes.data), self.ctx.ptr)
        return rp, ci

    def level_transfer(self, lvl: int, which: str = "P"):
        """General CSR (row_ptr, col, values) of P or R = P^T (tentative or, under
        smoothed aggregation, the smoothed prolongator)."""
        w = {"P": 0, "R": 1}[which]
        d = self.level_dims(lvl)
        nnz = C.c_int64()
        _check(lib().amgr_hier_level_transfer(self._p, lvl, w, C.byref(nnz), None, None, None), self.ctx.ptr)
        rows = d["nrows"] if w == 0 else d["n_coarse"]
        rp = np.zeros(rows + 1, np.int64)
        ci = np.zeros(max(nnz.value, 1), np.int64)
        v = np.zeros(max(nnz.value, 1))
        _check(lib().amgr_hier_level_transfer(self._p, lvl, w, C.byref(nnz), rp.ctypes.data, ci.ctypes.data,
                                              v.ctypes.data), self.ctx.ptr)
        return rp, ci[:nnz.value], v[:nnz.value]

    def level_smoother(self, lvl: int) -> np.ndarray:
        d = self.level_dims(lvl)
        w = np.zeros(d["nrows"])
        _check(lib().amgr_hier_level_smoother(self._p, lvl, w.ctypes.data), self.ctx.ptr)
        return w

    def level_lambda(self, lvl: int) -> float:
        """Chebyshev extension: power-iteration lambda_max(D^-1 A) of a level."""
        x = C.c_double()
        _check(lib().amgr_hier_level_lambda(self._p, lvl, C.byref(x)), self.ctx.ptr)
        return float(x.value)

    def coarse_n(self) -> int:
        return int(lib().amgr_hier_coarse_n(self._p))

    def coarse_lu(self):
        n = int(lib().amgr_hier_coarse_n(self._p))
        lu = np.zeros(max(n * n, 1))
        piv = np.zeros(max(n, 1), np.int64)
        _check(lib().amgr_hier_coarse_lu(self._p, lu.ctypes.data, piv.ctypes.data), self.ctx.ptr)
        return lu[:n * n], piv[:n]

    def operator_complexity(self) -> float:
        return float(lib().amgr_hier_operator_complexity(self._p))

    def setup_timings(self) -> PhaseTimings:
        t = _Timings()
        _check(lib().amgr_hier_timings(self._p, C.byref(t)), self.ctx.ptr)
        return PhaseTimings(t.transfer_ops, t.galerkin, t.smoother, t.coarse_solver)

    def shares_transfer(self, other: "Hierarchy", lvl: int) -> bool:
        return bool(lib().amgr_hier_shares_transfer(self._p, other._p, lvl))

    # --- in-place perf path ---
    def rebuild(self, A):
        """In-place partial update (amgr_rebuild)."""
        A = A if isinstance(A, DeviceCsr) else CsrMatrix.of(A)
        c = A._c()
        _check(lib().amgr_rebuild(self._p, C.byref(c)), self.ctx.ptr)

    def rebuild_values(self, values, adopt: bool = False):
        """Values-only rebuild (amgr_rebuild_values).  A device pointer may be
        adopted zero-copy (AMGR_DEVICE_ADOPT): it must stay valid until the next
        rebuild and carry >= 32 bytes of slack."""
        if isinstance(values, int):
            _check(lib().amgr_rebuild_values(self._p, values, DEVICE_ADOPT if adopt else DEVICE), self.ctx.ptr)
        else:
            v = _f64(values)
            _check(lib().amgr_rebuild_values(self._p, v.ctypes.data, HOST), self.ctx.ptr)

    def stage_values(self, values, host: bool | None = None):
        """Pipelining (amgr_stage_values): copy the next step's values on the
        context's copy stream while the current work runs.  `values` is a
        device pointer (int; host=True for a pinned host pointer) or a numpy
        array (kept alive until the copy completed: call rebuild_staged)."""
        if isinstance(values, int):
            _check(lib().amgr_stage_values(self._p, values, HOST if host else DEVICE), self.ctx.ptr)
        else:
            self._staged_keep = _f64(values)
            _check(lib().amgr_stage_values(self._p, self._staged_keep.ctypes.data, HOST), self.ctx.ptr)

    def stage_rhs(self, f, host: bool | None = None):
        """Pipelining (amgr_stage_rhs): the next step's right-hand side, like
        stage_values; committed by the next rebuild_staged, then read by
        bicgstab(h, STAGED_RHS, ...)."""
        if isinstance(f, int):
            _check(lib().amgr_stage_rhs(self._p, f, HOST if host else DEVICE), self.ctx.ptr)
        else:
            self._rhs_keep = _f64(f)
            _check(lib().amgr_stage_rhs(self._p, self._rhs_keep.ctypes.data, HOST), self.ctx.ptr)

    def rebuild_staged(self):
        """amgr_rebuild_values(h, NULL, AMGR_STAGED): swap the staged values in."""
        _check(lib().amgr_rebuild_values(self._p, None, STAGED), self.ctx.ptr)
        self._staged_keep = None

    def spmv(self, lvl: int, x):
        d = self.level_dims(lvl)
        x = _f64(x)
        y = np.zeros(d["nrows"])
        _check(lib().amgr_spmv(self._p, lvl, x.ctypes.data, y.ctypes.data, HOST), self.ctx.ptr)
        return y

    def close(self):
        if self._p and self.ctx._p:
            lib().amgr_hier_destroy(self._p)
        self._p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def setup(A, prm: AmgParams | None = None, ctx: Context | None = None) -> Hierarchy:
    """Hierarchy setup(const CsrMatrix&, const AmgParams&) — hierarchy.hpp:65."""
    ctx = ctx or default_context()
    prm = prm or AmgParams()
    A = A if isinstance(A, DeviceCsr) else CsrMatrix.of(A)
    c = A._c()
    p = prm._c()
    out = C.c_void_p()
    _check(lib().amgr_setup(ctx.ptr, C.byref(c), C.byref(p), C.byref(out)), ctx.ptr)
    return Hierarchy(out, ctx, prm)


def partial_update(h: Hierarchy, A, prm: AmgParams | None = None) -> Hierarchy:
    """Hierarchy partial_update(const Hierarchy&, CsrMatrix, const AmgParams&) — hierarchy.hpp:71."""
    prm = prm or h.prm
    A = A if isinstance(A, DeviceCsr) else CsrMatrix.of(A)
    c = A._c()
    p = prm._c()
    out = C.c_void_p()
    _check(lib().amgr_partial_update(h._p, C.byref(c), C.byref(p), C.byref(out)), h.ctx.ptr)
    return Hierarchy(out, h.ctx, prm)


def vcycle(h: Hierarchy, f, prm: AmgParams | None = None) -> np.ndarray:
    """std::vector<double> vcycle(const Hierarchy&, span f, const AmgParams&) — hierarchy.hpp:75-76.

    The smoothing parameters are the hierarchy's (fixed at setup/partial_update)."""
    if isinstance(f, int):  # device pointers: f and out=u (device address via prm-free call)
        raise InvalidArgument("use vcycle_device(h, f_ptr, u_ptr) for device buffers")
    f = _f64(f)
    if len(f) != h.finest_size():
        raise InvalidArgument("vcycle: dimension mismatch")
    u = np.zeros_like(f)
    _check(lib().amgr_vcycle(h._p, f.ctypes.data, u.ctypes.data, HOST), h.ctx.ptr)
    return u


def vcycle_device(h: Hierarchy, f_ptr: int, u_ptr: int) -> None:
    """V-cycle on device-resident buffers (stream-ordered on h.ctx.stream)."""
    _check(lib().amgr_vcycle(h._p, f_ptr, u_ptr, DEVICE), h.ctx.ptr)


def _solve(fn, h, f, u0, prm):
    prm = prm or SolveParams()
    if f is STAGED_RHS:  # staged RHS (amgr_stage_rhs); u0 = (u0_ptr, u_ptr) device addresses
        u0_ptr, u_ptr = u0
        sp = _SolveParams(prm.tol, prm.max_iter)
        st = _SolveStats()
        _check(fn(h._p, None, u0_ptr, u_ptr, C.byref(sp), C.byref(st), STAGED), h.ctx.ptr)
        return None, SolveStats(int(st.iterations), float(st.relative_residual), bool(st.converged),
                                bool(st.breakdown))
    if isinstance(f, int):  # device pointers: (f, u0, u) all device addresses
        u0_ptr, u_ptr = u0
        sp = _SolveParams(prm.tol, prm.max_iter)
        st = _SolveStats()
        _check(fn(h._p, f, u0_ptr, u_ptr, C.byref(sp), C.byref(st), DEVICE), h.ctx.ptr)
        return None, SolveStats(int(st.iterations), float(st.relative_residual), bool(st.converged),
                                bool(st.breakdown))
    f = _f64(f)
    if u0 is None:
        u0 = np.zeros_like(f)
    u0 = _f64(u0)
    if len(u0) != len(f):
        raise InvalidArgument("bicgstab: dimension mismatch")
    u = np.zeros_like(f)
    sp = _SolveParams(prm.tol, prm.max_iter)
    st = _SolveStats()
    _check(fn(h._p, f.ctypes.data, u0.ctypes.data, u.ctypes.data, C.byref(sp), C.byref(st), HOST), h.ctx.ptr)
    return u, SolveStats(int(st.iterations), float(st.relative_residual), bool(st.converged), bool(st.breakdown))


def bicgstab(h: Hierarchy, f, u0=None, prm: SolveParams | None = None):
    """bicgstab(make_operator(A), make_preconditioner(h), f, u0, prm) — bicgstab.hpp:34-44."""
    return _solve(lib().amgr_bicgstab, h, f, u0, prm)


def cg(h: Hierarchy, f, u0=None, prm: SolveParams | None = None):
    """Preconditioned CG (extension; not in the reference)."""
    return _solve(lib().amgr_cg, h, f, u0, prm)


# ---- single-operator entry points (the reference's free functions) ----------------
def spmv(A, x, ctx: Context | None = None) -> np.ndarray:
    """y = A x (csr.cpp:76-91), on the device (amgr_csr_spmv)."""
    ctx = ctx or default_context()
    A = CsrMatrix.of(A)
    x = _f64(x)
    if len(x) != A.ncols:
        raise InvalidArgument("spmv: dimension mismatch")
    y = np.zeros(A.nrows)
    c = A._c()
    _check(lib().amgr_csr_spmv(ctx.ptr, C.byref(c), x.ctypes.data, y.ctypes.data, HOST), ctx.ptr)
    return y


def build_smoother(A, omega: float = 0.72, ctx: Context | None = None) -> np.ndarray:
    """JacobiSmoother::inv_diag of build_smoother(A, omega) (smoother.cpp:8-32)."""
    ctx = ctx or default_context()
    A = CsrMatrix.of(A)
    w = np.zeros(A.nrows)
    c = A._c()
    _check(lib().amgr_build_smoother(ctx.ptr, C.byref(c), w.ctypes.data, HOST), ctx.ptr)
    return w


def smooth(inv_diag, A, f, u, sweeps: int, omega: float = 0.72, ctx: Context | None = None) -> np.ndarray:
    """smooth(s, A, f, u, sweeps) (smoother.cpp:34-48); returns the smoothed u."""
    ctx = ctx or default_context()
    A = CsrMatrix.of(A)
    w, f, u = _f64(inv_diag), _f64(f), _f64(u).copy()
    if not (len(w) == len(f) == len(u) == A.nrows):
        raise InvalidArgument("smooth: dimension mismatch")
    c = A._c()
    _check(lib().amgr_smooth(ctx.ptr, C.byref(c), w.ctypes.data, float(omega), f.ctypes.data, u.ctypes.data,
                             int(sweeps), HOST), ctx.ptr)
    return u


def coarse_factorize(A, ctx: Context | None = None):
    """DenseFactorization (lu row-major n*n, piv) of coarse_factorize(A) (dense_lu.cpp:10-50)."""
    ctx = ctx or default_context()
    A = CsrMatrix.of(A)
    n = A.nrows
    lu = np.zeros(n * n)
    piv = np.zeros(n, np.int64)
    c = A._c()
    _check(lib().amgr_coarse_factorize(ctx.ptr, C.byref(c), lu.ctypes.data, piv.ctypes.data), ctx.ptr)
    return lu, piv


def coarse_solve(lu, piv, rhs, ctx: Context | None = None) -> np.ndarray:
    """coarse_solve(f, rhs) (dense_lu.cpp:52-73)."""
    ctx = ctx or default_context()
    lu, rhs = _f64(lu), _f64(rhs)
    piv = np.ascontiguousarray(piv, np.int64)
    n = len(piv)
    if len(rhs) != n:
        raise InvalidArgument("coarse_solve: dimension mismatch")
    x = np.zeros(n)
    _check(lib().amgr_coarse_solve(ctx.ptr, n, lu.ctypes.data, piv.ctypes.data, rhs.ctypes.data, x.ctypes.data),
           ctx.ptr)
    return x


def run_sequence(*args, **kwargs):
    """RunResult run_sequence(systems, StrategyConfig, AmgParams, SolveParams) — reuse.hpp:70-71."""
    from .reuse import run_sequence as _rs
    return _rs(*args, **kwargs)


# ---- Matrix Market ingestion (matrix_market.hpp) -------------------------------------
class Matrix:
    """A device CSR owned by the library (amgr_matrix), e.g. from mm_read."""

    def __init__(self, ptr, ctx: Context):
        self._p = ptr
        self.ctx = ctx
        ctx._adopt(self)
        c = _Csr()
        _check(lib().amgr_matrix_csr(self._p, C.byref(c)), ctx.ptr)
        self.nrows, self.ncols, self.nnz = int(c.nrows), int(c.ncols), int(c.nnz)
        self._view = DeviceCsr(self.nrows, self.ncols, self.nnz, c.row_ptr, c.col_idx, c.values, 32)

    def device_csr(self) -> DeviceCsr:
        """Device view (setup / partial_update / rebuild accept it directly)."""
        return self._view

    def to_host(self):
        """(row_ptr int64, col int64, values) host copies."""
        v = self._view
        rp = np.zeros(self.nrows + 1, np.int32)
        ci = np.zeros(max(self.nnz, 1), np.int32)
        val = np.zeros(max(self.nnz, 1))
        L = lib()
        _check(L.amgr_copy_to_host(self.ctx.ptr, rp.ctypes.data, v.row_ptr, 4 * (self.nrows + 1)), self.ctx.ptr)
        if self.nnz:
            _check(L.amgr_copy_to_host(self.ctx.ptr, ci.ctypes.data, v.col_idx, 4 * self.nnz), self.ctx.ptr)
            _check(L.amgr_copy_to_host(self.ctx.ptr, val.ctypes.data, v.values, 8 * self.nnz), self.ctx.ptr)
        return rp.astype(np.int64), ci[:self.nnz].astype(np.int64), val[:self.nnz]

    def close(self):
        if self._p and self.ctx._p:
            lib().amgr_matrix_free(self._p)
        self._p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def mm_read(path, ctx: Context | None = None) -> Matrix:
    """CsrMatrix mm_read(path) (matrix_market.hpp:17): parsed on the host,
    assembled on the device; raises RuntimeFailure with the reference's text."""
    ctx = ctx or default_context()
    p = C.c_void_p()
    _check(lib().amgr_mm_read(ctx.ptr, os.fspath(path).encode(), C.byref(p)), ctx.ptr)
    return Matrix(p, ctx)


def mm_read_vector(path, ctx: Context | None = None) -> np.ndarray:
    """std::vector<double> mm_read_vector(path) (matrix_market.hpp:25)."""
    ctx = ctx or default_context()
    n = C.c_int64(0)
    _check(lib().amgr_mm_read_vector(ctx.ptr, os.fspath(path).encode(), C.byref(n), None), ctx.ptr)
    v = np.zeros(max(n.value, 1))
    n2 = C.c_int64(n.value)
    _check(lib().amgr_mm_read_vector(ctx.ptr, os.fspath(path).encode(), C.byref(n2), v.ctypes.data), ctx.ptr)
    return v[:n.value]
