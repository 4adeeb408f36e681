"""Row-partitioned multi-GPU solve over the C-ABI (amgr_dist_*), one process
per GPU.  torch.distributed is only the plumbing that broadcasts the NCCL
unique id; the data path (halo exchange, transition allgather, dot
reductions) is NCCL inside libamgr_b200.so on the context stream.

    h = amg.setup(A_global)                      # same hierarchy on every rank
    ds = DistSolver(h, rank, world, nccl_id)     # partition (partition.py) + NCCL comm
    ds.rebuild_local(local_values)               # partial reuse step from this rank's rows
    stats = ds.bicgstab(f_local_ptr, u_local_ptr)
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch  # noqa: F401  -- loads torch's libnccl.so.2 before the library binds NCCL

from . import Hierarchy, SolveParams, SolveStats, _check, _SolveParams, _SolveStats, lib
from . import partition as PT


class _DistLevel(C.Structure):
    _fields_ = [("n_own", C.c_int64), ("n_halo", C.c_int64), ("nnz", C.c_int64), ("n_coarse_owned", C.c_int64),
                ("row_ptr", C.c_void_p), ("col", C.c_void_p), ("nnz_map", C.c_void_p), ("owned", C.c_void_p),
                ("agg", C.c_void_p), ("mptr", C.c_void_p), ("midx", C.c_void_p), ("n_send_peers", C.c_int32),
                ("n_recv_peers", C.c_int32), ("send_peer", C.c_void_p), ("send_cnt", C.c_void_p),
                ("send_idx", C.c_void_p), ("recv_peer", C.c_void_p), ("recv_off", C.c_void_p),
                ("recv_cnt", C.c_void_p)]


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().amgr_nccl_unique_id(buf), None)
    return buf.raw


class Loopback:
    """In-process test transport (amgr_dist_loopback_create): all ranks of the
    job live in one process, one host thread and one Context each, on the
    same GPU; exchanges are stream-ordered device copies + host barriers."""

    def __init__(self, world: int):
        self._p = C.c_void_p()
        _check(lib().amgr_dist_loopback_create(world, C.byref(self._p)), None)
        self.world = world

    def close(self):
        if self._p:
            lib().amgr_dist_loopback_destroy(self._p)
            self._p = None


def hierarchy_structure(h: Hierarchy):
    """Download the structure build_plan needs (patterns and aggregates)."""
    out = []
    for l in range(h.num_levels()):
        rp, ci, _ = h.level_A(l)
        d = h.level_dims(l)
        out.append({"n": d["nrows"], "rp": rp, "col": ci, "agg": h.level_agg(l) if d["n_coarse"] else None})
    return out


class _DeviceLevel:
    """What the caller needs of a device-built plan level (sizes; level 0 maps)."""

    def __init__(self, dims, owned=None, nnz_map=None):
        self.n_own, n_halo, nnz, self.n_coarse_owned, _ = (int(x) for x in dims)
        self.halo = np.zeros(n_halo, np.int64)  # only its length is meaningful
        self.nnz = nnz
        self.owned, self.nnz_map = owned, nnz_map


class _DevicePlan:
    def __init__(self, top, levels):
        self.top, self.levels = top, levels


class DistSolver:
    def __init__(self, h: Hierarchy, rank: int, world: int, nccl_id: bytes | None = None,
                 replicate_below: int = 20000, plan: PT.Plan | None = None, loopback: Loopback | None = None,
                 device_plan: bool = False):
        self.h, self.rank, self.world = h, rank, world
        self._keep = []
        if device_plan:
            # partition built on the device (amgr_dist_create_auto): no host plan, no pattern download
            self._p = C.c_void_p()
            if loopback is not None:
                _check(lib().amgr_dist_create_auto_loopback(h._p, loopback._p, rank, world, int(replicate_below),
                                                            C.byref(self._p)), h.ctx.ptr)
            else:
                idb = C.create_string_buffer(nccl_id, 128)
                _check(lib().amgr_dist_create_auto(h._p, idb, rank, world, int(replicate_below), C.byref(self._p)),
                       h.ctx.ptr)
            d = np.zeros(5, np.int64)
            _check(lib().amgr_dist_level_dims(self._p, 0, d.ctypes.data), h.ctx.ptr)
            top = int(d[4])
            levels = []
            for lvl in range(top + 1):
                d = np.zeros(5, np.int64)
                _check(lib().amgr_dist_level_dims(self._p, lvl, d.ctypes.data), h.ctx.ptr)
                if lvl == 0:
                    own = np.zeros(int(d[0]), np.int64)
                    nm = np.zeros(int(d[2]), np.int64)
                    _check(lib().amgr_dist_level_maps(self._p, 0, own.ctypes.data, nm.ctypes.data), h.ctx.ptr)
                    levels.append(_DeviceLevel(d, own, nm))
                else:
                    levels.append(_DeviceLevel(d))
            self.plan = _DevicePlan(top, levels)
            self.owned0 = levels[0].owned
            h.ctx._adopt(self)
            return
        struct = hierarchy_structure(h)
        self.plan = plan or PT.build_plan(struct, rank, world, replicate_below)
        T = self.plan.top
        if T < 0:
            raise ValueError("hierarchy too small to partition (raise replicate_below or the problem size)")

        def arr(a, dt=np.int64):
            a = np.ascontiguousarray(a, dt)
            self._keep.append(a)
            return a.ctypes.data

        levels = (_DistLevel * (T + 1))()
        for i, L in enumerate(self.plan.levels):
            sp = sorted(L.send)
            rpeers = sorted(L.recv)
            levels[i] = _DistLevel(
                L.n_own, len(L.halo), len(L.col), len(L.mptr) - 1, arr(L.rp), arr(L.col), arr(L.nnz_map),
                arr(L.owned), arr(L.agg), arr(L.mptr), arr(L.midx if len(L.midx) else np.zeros(1)),
                len(sp), len(rpeers), arr(sp, np.int32), arr([len(L.send[p]) for p in sp]),
                arr(np.concatenate([L.send[p] for p in sp]) if sp else np.zeros(1)), arr(rpeers, np.int32),
                arr([L.recv[p][0] for p in rpeers]), arr([L.recv[p][1] for p in rpeers]))
        own_t = self.plan.owner[T + 1]
        t_counts = np.bincount(own_t, minlength=world).astype(np.int64)
        self._keep.append(t_counts)
        self._p = C.c_void_p()
        if loopback is not None:
            _check(lib().amgr_dist_create_loopback(h._p, loopback._p, rank, world, T, levels, int(t_counts.sum()),
                                                   t_counts.ctypes.data, C.byref(self._p)), h.ctx.ptr)
        else:
            idb = C.create_string_buffer(nccl_id, 128)
            _check(lib().amgr_dist_create(h._p, idb, rank, world, T, levels, int(t_counts.sum()),
                                          t_counts.ctypes.data, C.byref(self._p)), h.ctx.ptr)
        self.owned0 = self.plan.levels[0].owned
        h.ctx._adopt(self)

    @property
    def n_local(self) -> int:
        return int(len(self.owned0))

    def rebuild_values(self, global_values_ptr: int, device: bool = True):
        _check(lib().amgr_dist_rebuild_values(self._p, global_values_ptr, 1 if device else 0), self.h.ctx.ptr)

    def local_values(self, global_values) -> np.ndarray:
        """This rank's A_0 entries in local CSR order (global_values[nnz_map])."""
        return np.ascontiguousarray(np.asarray(global_values, np.float64)[self.plan.levels[0].nnz_map])

    def rebuild_local(self, local_values, device: bool | None = None):
        """Partial rebuild from rank-local values (amgr_dist_rebuild_local):
        a device pointer (int) or a host array of len(nnz_map) entries."""
        if isinstance(local_values, int):
            _check(lib().amgr_dist_rebuild_local(self._p, local_values, 1 if device in (None, True) else 0),
                   self.h.ctx.ptr)
            return
        v = np.ascontiguousarray(local_values, np.float64)
        if len(v) != len(self.plan.levels[0].nnz_map):
            raise ValueError("rebuild_local: expected the rank's local entries")
        _check(lib().amgr_dist_rebuild_local(self._p, v.ctypes.data, 0), self.h.ctx.ptr)

    def vcycle(self, f_ptr: int, u_ptr: int):
        _check(lib().amgr_dist_vcycle(self._p, f_ptr, u_ptr), self.h.ctx.ptr)

    def bicgstab(self, f_ptr: int, u_ptr: int, prm: SolveParams | None = None) -> SolveStats:
        prm = prm or SolveParams()
        sp = _SolveParams(prm.tol, prm.max_iter)
        st = _SolveStats()
        _check(lib().amgr_dist_bicgstab(self._p, f_ptr, u_ptr, C.byref(sp), C.byref(st)), self.h.ctx.ptr)
        return SolveStats(int(st.iterations), float(st.relative_residual), bool(st.converged), bool(st.breakdown))

    def level_col_bytes(self, level: int) -> int:
        """Bytes per entry of the partitioned level's column stream (1/2: coded, 4: int32)."""
        v = C.c_int(0)
        _check(lib().amgr_dist_level_code(self._p, int(level), C.byref(v)), self.h.ctx.ptr)
        return int(v.value)

    def close(self):
        if self._p and self.h.ctx._p:
            lib().amgr_dist_destroy(self._p)
        self._p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
