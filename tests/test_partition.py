"""Multi-GPU host logic on CPU: the aggregate-consistent row
partition (paper_2108_02054_b200/partition.py) executed by a world-size-2
gloo run.  A numpy executor plays each rank's device: it runs the V-cycle on
the local rows with halo exchanges (send/recv) and the transition allgather,
and the assembled result must equal the single-domain V-cycle of the C oracle
bit for bit (every row sum and restriction keeps the reference's order).
A distributed BiCGStab with rank-ordered dot reductions converges within +-1
iteration of the oracle; with the sequential-dot mode's global-order dots it
is the oracle's BiCGStab bit for bit.  The numpy executor is test infrastructure standing
in for the kernels (which are the single-GPU ones, tested in -m gpu)."""
import os
import socket

import numpy as np
import pytest

from oracle import oracle as O
from oracle import problems as P
from paper_2108_02054_b200 import partition as PT

OMEGA = 0.72


def spmv_seq(rp, col, val, x):
    """y_i = sum_k a_ik x_col in stored order, from 0.0 (csr.cpp:79-84)."""
    n = len(rp) - 1
    y = np.zeros(n)
    lens = np.diff(rp)
    for k in range(int(lens.max()) if n else 0):
        m = lens > k
        idx = rp[:-1][m] + k
        y[m] = y[m] + val[idx] * x[col[idx]]
    return y


def restrict_seq(mptr, midx, r):
    nc = len(mptr) - 1
    f = np.zeros(nc)
    lens = np.diff(mptr)
    for k in range(int(lens.max()) if nc else 0):
        m = lens > k
        f[m] = f[m] + r[midx[mptr[:-1][m] + k]]
    return f


class Comm:
    def __init__(self, dist):
        self.dist = dist

    def halo(self, L, x_own):
        import torch

        x = np.concatenate([x_own, np.zeros(len(L.halo))])
        reqs = []
        for p, idx in L.send.items():
            reqs.append(self.dist.isend(torch.from_numpy(np.ascontiguousarray(x_own[idx])), p))
        bufs = {}
        for p, (s, c) in L.recv.items():
            bufs[p] = torch.zeros(c, dtype=torch.float64)
            reqs.append(self.dist.irecv(bufs[p], p))
        for q in reqs:
            q.wait()
        for p, (s, c) in L.recv.items():
            x[L.n_own + s:L.n_own + s + c] = bufs[p].numpy()
        return x

    def allgather_concat(self, v):
        import torch

        t = torch.from_numpy(np.ascontiguousarray(v))
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(self.dist.get_world_size())]
        self.dist.all_gather(sizes, torch.tensor([len(v)]))
        # padded blocks (gloo wants equal sizes; the device path pads the same way)
        pad = max(int(s.item()) for s in sizes)
        tp = torch.zeros(pad, dtype=torch.float64)
        tp[:len(v)] = t
        out = [torch.zeros(pad, dtype=torch.float64) for _ in sizes]
        self.dist.all_gather(out, tp)
        return np.concatenate([o.numpy()[:int(s.item())] for o, s in zip(out, sizes)])

    def dot_global_order(self, a, b, owned, n):
        """the sequential-dot mode's algorithm (dist.cu seq_dot_dist): rounded
        local products, one allgather, the reference's left-to-right sum over
        the global index (bicgstab.cpp:11-17) through the gathered owned ids"""
        prods = self.allgather_concat(np.asarray(a) * np.asarray(b))
        ids = self.allgather_concat(np.asarray(owned, np.float64)).astype(np.int64)
        g = np.empty(n)
        g[ids] = prods
        s = 0.0
        for v in g.tolist():
            s += v
        return s

    def sum_ordered(self, x):
        """deterministic: gather per-rank partials, add in rank order"""
        parts = self.allgather_concat(np.array([x]))
        s = 0.0
        for p in parts:
            s += p
        return s


def local_vcycle(plan, H, f_own, comm):
    """One V-cycle (hierarchy.cpp:152-186 with smoothing) on the partition."""
    T = plan.top
    Ls = plan.levels
    u0s, rs, fs = [], [], [f_own]
    for i in range(T + 1):
        L = Ls[i]
        val = H.levels[i].A[2][L.nnz_map]
        w = H.levels[i].w[L.owned]
        u0 = 0.0 + (OMEGA * w) * fs[i]
        r = fs[i] - spmv_seq(L.rp, L.col, val, comm.halo(L, u0))
        fc = restrict_seq(L.mptr, L.midx, r)
        u0s.append(u0)
        fs.append(fc if i < T else comm.allgather_concat(fc))
    # replicated levels T+1..: single-domain V-cycle on every rank
    uc = replicated_vcycle(H, T + 1, fs[T + 1])
    for i in range(T, -1, -1):
        L = Ls[i]
        val = H.levels[i].A[2][L.nnz_map]
        w = H.levels[i].w[L.owned]
        x = u0s[i] + (0.0 + uc[L.agg])
        s = spmv_seq(L.rp, L.col, val, comm.halo(L, x))
        uc = x + (OMEGA * w) * (fs[i] - s)
    return uc


def replicated_vcycle(H, start, f):
    Lv = H.levels
    nL = len(Lv)
    us, fs = {}, {start: f}
    for i in range(start, nL - 1):
        A = Lv[i].A
        u0 = 0.0 + (OMEGA * Lv[i].w) * fs[i]
        r = fs[i] - spmv_seq(A[0], A[1], A[2], u0)
        R = Lv[i].R
        fs[i + 1] = spmv_seq(R[0], R[1], R[2], r)
        us[i] = u0
    u = O.coarse_solve(H.lu, H.piv, fs[nL - 1])
    for i in range(nL - 2, start - 1, -1):
        A = Lv[i].A
        P_ = Lv[i].P
        x = us[i] + spmv_seq(P_[0], P_[1], P_[2], u)
        u = x + (OMEGA * Lv[i].w) * (fs[i] - spmv_seq(A[0], A[1], A[2], x))
    return u


def local_bicgstab(plan, H, f_own, comm, tol=1e-8, max_iter=100, seq=False):
    """bicgstab.cpp:21-135 with distributed SpMV and rank-ordered dots (seq:
    the reference's global-order dots)."""
    L0 = plan.levels[0]
    val0 = H.levels[0].A[2][L0.nnz_map]
    A = lambda x: spmv_seq(L0.rp, L0.col, val0, comm.halo(L0, x))  # noqa: E731
    M = lambda x: local_vcycle(plan, H, x, comm)  # noqa: E731
    if seq:
        n = len(H.levels[0].A[0]) - 1
        dot = lambda a, b: comm.dot_global_order(a, b, L0.owned, n)  # noqa: E731
    else:
        dot = lambda a, b: comm.sum_ordered(float(np.dot(a, b)))  # noqa: E731
    nf = np.sqrt(dot(f_own, f_own))
    u = np.zeros_like(f_own)
    r = f_own - A(u)
    rt = r.copy()
    floor = 1e-30 * nf * nf
    rho_old = alpha = omega = 1.0
    p = v = np.zeros_like(r)
    for it in range(1, max_iter + 1):
        rho = dot(rt, r)
        if abs(rho) < floor:
            return u, it, False
        p = r.copy() if it == 1 else r + ((rho / rho_old) * (alpha / omega)) * (p - omega * v)
        ph = M(p)
        v = A(ph)
        alpha = rho / dot(rt, v)
        s = r - alpha * v
        if np.sqrt(dot(s, s)) / nf <= tol:
            u = u + alpha * ph
            if np.sqrt(dot(f_own - A(u), f_own - A(u))) / nf <= tol:
                return u, it, True
            r, rho_old = s, rho
            continue
        sh = M(s)
        t = A(sh)
        omega = dot(t, s) / dot(t, t)
        u = u + (alpha * ph + omega * sh)
        r = s - omega * t
        rho_old = rho
        if np.sqrt(dot(r, r)) / nf <= tol:
            res = f_own - A(u)
            if np.sqrt(dot(res, res)) / nf <= tol:
                return u, it, True
    return u, max_iter, False


def _worker(rank, world, port, out_path):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    A = P.grid3d_values("dambreak", 14, 21)
    H = O.setup(A)
    plan = PT.build_plan(PT.hierarchy_from_oracle(H), rank, world, replicate_below=100)
    comm = Comm(dist)
    n = len(A[0]) - 1
    f = np.random.default_rng(3).uniform(-1, 1, n)
    u_own = local_vcycle(plan, H, f[plan.levels[0].owned], comm)
    fr = P.rhs(n)
    us, it, conv = local_bicgstab(plan, H, fr[plan.levels[0].owned], comm)
    uq, itq, convq = local_bicgstab(plan, H, fr[plan.levels[0].owned], comm, seq=True)
    np.savez(out_path + f".{rank}.npz", owned=plan.levels[0].owned, u=u_own, us=us, it=it, conv=conv,
             uq=uq, itq=itq, convq=convq,
             top=plan.top, halos=[len(L.halo) for L in plan.levels])
    dist.destroy_process_group()


def _rebuild_worker(rank, world, port, out_path):
    """Partitioned rebuild from rank-local values (amgr_dist_rebuild_local's
    algorithm, host statement partition.local_galerkin): local Jacobi weights
    and the Galerkin rows of the rank's coarse rows from ONLY its own A_k
    entries, the level-(top+1) rows allgathered."""
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    A = P.grid3d_values("dambreak", 14, 21)
    A2 = P.grid3d_values("dambreak", 14, 35)
    H = O.setup(A)
    struct = PT.hierarchy_from_oracle(H)
    plan = PT.build_plan(struct, rank, world, replicate_below=100)
    comm = Comm(dist)
    T = plan.top
    vals = np.asarray(A2[2], np.float64)[plan.levels[0].nnz_map]  # the only A_k data this rank sees
    res = {}
    for i in range(T + 1):
        L = plan.levels[i]
        diag = np.array([vals[L.rp[r] + np.nonzero(L.col[L.rp[r]:L.rp[r + 1]] == r)[0][0]] for r in range(L.n_own)])
        res[f"w{i}"] = 1.0 / diag
        res[f"own{i}"] = L.owned
        crp, ccol = struct[i + 1]["rp"], struct[i + 1]["col"]
        if i < T:
            rows = plan.levels[i + 1].owned
        else:
            rows = np.nonzero(plan.owner[T + 1] == rank)[0]
        cv = PT.local_galerkin(L, vals, struct[i]["agg"], rows, crp, ccol)
        if i < T:
            vals = cv  # owned rows of level i+1 in local CSR order (= global order per row)
        else:
            res["AT1"] = comm.allgather_concat(cv)
    np.savez(out_path + f".{rank}.npz", top=T, **res)
    dist.destroy_process_group()


def test_partitioned_rebuild_from_local_values_gloo(tmp_path):
    import torch.multiprocessing as mp

    out = str(tmp_path / "rb")
    world = 2
    mp.spawn(_rebuild_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    A = P.grid3d_values("dambreak", 14, 21)
    A2 = P.grid3d_values("dambreak", 14, 35)
    Hu = O.partial_update(O.setup(A), A2)
    for r in range(world):
        d = np.load(out + f".{r}.npz")
        T = int(d["top"])
        assert T >= 1
        for i in range(T + 1):
            w_ref = Hu.levels[i].w[d[f"own{i}"]]
            np.testing.assert_array_equal(d[f"w{i}"].view(np.int64), w_ref.view(np.int64))
        np.testing.assert_array_equal(d["AT1"].view(np.int64), np.asarray(Hu.levels[T + 1].A[2]).view(np.int64))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_partition_plan_invariants():
    A = P.grid3d_values("dambreak", 12, 5)
    H = O.setup(A)
    hier = PT.hierarchy_from_oracle(H)
    W = 3
    plans = [PT.build_plan(hier, r, W, replicate_below=50) for r in range(W)]
    T = plans[0].top
    assert T >= 1
    for i in range(T + 1):
        owned = np.concatenate([p.levels[i].owned for p in plans])
        assert np.array_equal(np.sort(owned), np.arange(hier[i]["n"]))  # a partition
        for p in plans:
            L = p.levels[i]
            # halo completeness and send/recv symmetry
            for q, (s, c) in L.recv.items():
                peer = plans[q].levels[i]
                np.testing.assert_array_equal(peer.owned[peer.send[p.rank]], L.halo[s:s + c])
        # aggregate consistency: every fine row's aggregate is owned by the same rank
        if i < T:
            for p in plans:
                L = p.levels[i]
                assert (p.owner[i + 1][hier[i]["agg"][L.owned]] == p.rank).all()


def test_distributed_vcycle_and_bicgstab_gloo(tmp_path):
    import torch.multiprocessing as mp

    out = str(tmp_path / "dist")
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    A = P.grid3d_values("dambreak", 14, 21)
    H = O.setup(A)
    n = len(A[0]) - 1
    f = np.random.default_rng(3).uniform(-1, 1, n)
    u_ref = O.vcycle(H, f)
    u = np.zeros(n)
    us = np.zeros(n)
    its = []
    for r in range(world):
        d = np.load(out + f".{r}.npz")
        u[d["owned"]] = d["u"]
        us[d["owned"]] = d["us"]
        its.append(int(d["it"]))
        assert bool(d["conv"])
        assert int(d["top"]) >= 1 and sum(d["halos"]) > 0  # really partitioned, real halos
    np.testing.assert_array_equal(u.view(np.int64), u_ref.view(np.int64))
    so = O.bicgstab(H, P.rhs(n))
    assert its[0] == its[1] and abs(its[0] - so.iterations) <= 1
    res = np.linalg.norm(P.rhs(n) - O.spmv(A, us)) / np.linalg.norm(P.rhs(n))
    assert res <= 1e-8
    # global-order dots: the oracle's BiCGStab iteration for iteration
    uq = np.zeros(n)
    for r in range(world):
        d = np.load(out + f".{r}.npz")
        uq[d["owned"]] = d["uq"]
        assert bool(d["convq"]) and int(d["itq"]) == so.iterations, (int(d["itq"]), so.iterations)
    np.testing.assert_array_equal(uq.view(np.int64), np.asarray(so.u).view(np.int64))
