"""Partitioned multi-GPU solve on the device (amgr_dist_*), exercised with
world size 1 on the single GPU this run has: the full code path (local CSR
views, halo pack, transition allgather through NCCL, replicated coarse levels
via vcycle_from, rank-ordered dot reductions) must reproduce the single-GPU
V-cycle bit for bit and the same BiCGStab iterates.  The world > 1 exchange
plan is validated on CPU (tests/test_partition.py)."""
import numpy as np
import pytest

from oracle import problems as P

pytestmark = pytest.mark.gpu
amg = pytest.importorskip("paper_2108_02054_b200")


def test_dist_world1_matches_single_gpu(ctx):
    import torch

    from paper_2108_02054_b200 import distributed as D

    A = P.grid3d_values("dambreak", 20, 9)
    h = amg.setup(A, ctx=ctx)
    ds = D.DistSolver(h, 0, 1, D.nccl_unique_id(), replicate_below=300)
    assert ds.plan.top >= 1
    n = 20 ** 3
    f = np.random.default_rng(2).uniform(-1, 1, n)
    fd = torch.from_numpy(f[ds.owned0]).cuda()
    ud = torch.zeros(ds.n_local, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    ds.vcycle(fd.data_ptr(), ud.data_ptr())
    ctx.synchronize()
    u = np.zeros(n)
    u[ds.owned0] = ud.cpu().numpy()
    np.testing.assert_array_equal(u.view(np.int64), amg.vcycle(h, f).view(np.int64))
    fr = P.rhs(n)
    frd = torch.from_numpy(fr[ds.owned0]).cuda()
    ur = torch.zeros(ds.n_local, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    st = ds.bicgstab(frd.data_ptr(), ur.data_ptr())
    _, st1 = amg.bicgstab(h, fr)
    assert st.converged and st.iterations == st1.iterations
    # rebuild through the distributed handle (global rebuild + local gathers)
    A2 = P.grid3d_values("dambreak", 20, 30)
    vals = torch.from_numpy(np.concatenate([A2[2], np.zeros(8)])).cuda()
    torch.cuda.synchronize()
    ds.rebuild_values(vals.data_ptr())
    ur.zero_()
    torch.cuda.synchronize()
    st2 = ds.bicgstab(frd.data_ptr(), ur.data_ptr())
    h2 = amg.setup(A2, ctx=ctx)
    _, st3 = amg.bicgstab(h2, fr)
    assert st2.converged and st2.iterations == st3.iterations
    ds.close()


@pytest.mark.parametrize("overlap", ["1", "0"])
@pytest.mark.parametrize("world", [2, 3, 4])
def test_dist_multirank_loopback_matches_single_gpu(world, overlap, monkeypatch):
    """The multi-rank device path (local CSR views with real halos, per-peer
    halo exchange, transition allgather of padded blocks, replicated coarse
    levels, rank-ordered dot sums, distributed rebuild) with `world` ranks in
    one process on the one GPU, exchanging through the loopback test
    transport: the assembled V-cycle is bit-identical to the single-GPU one
    and every rank takes the single-GPU BiCGStab iteration count.  With
    overlap (the default for world > 1) each V-cycle pass runs on stale halo
    values while the exchange is in flight on a second stream, then the
    boundary rows are recomputed (k_rowlist): still the same bits."""
    import threading

    monkeypatch.setenv("AMGR_DIST_OVERLAP", overlap)

    import torch

    from paper_2108_02054_b200 import distributed as D

    A = P.grid3d_values("dambreak", 20, 9)
    n = 20 ** 3
    f = np.random.default_rng(2).uniform(-1, 1, n)
    fr = P.rhs(n)
    A2 = P.grid3d_values("dambreak", 20, 30)
    ref_ctx = amg.Context(0)
    h_ref = amg.setup(A, ctx=ref_ctx)
    u_ref = amg.vcycle(h_ref, f)
    _, st_ref = amg.bicgstab(h_ref, fr)
    h2_ref = amg.setup(A2, ctx=ref_ctx)
    _, st2_ref = amg.bicgstab(h2_ref, fr)

    lb = D.Loopback(world)
    ranks = []
    for r in range(world):
        ctx = amg.Context(0)
        h = amg.setup(A, ctx=ctx)
        ds = D.DistSolver(h, r, world, replicate_below=300, loopback=lb)
        assert ds.plan.top >= 1 and (world == 1 or sum(len(L.halo) for L in ds.plan.levels) > 0)
        # level 0 keeps a coded column stream despite its halo columns (2 bytes at most)
        assert ds.level_col_bytes(0) in (1, 2), ds.level_col_bytes(0)
        own = torch.from_numpy(ds.owned0).cuda()
        ranks.append({"ctx": ctx, "h": h, "ds": ds, "own": own})
    torch.cuda.synchronize()
    vals2 = torch.from_numpy(np.concatenate([A2[2], np.zeros(8)])).cuda()
    out = [None] * world
    errs = []

    def run(r):
        try:
            R = ranks[r]
            ds = R["ds"]
            fd = torch.from_numpy(f).cuda()[R["own"]].contiguous()
            ud = torch.zeros(ds.n_local, dtype=torch.float64, device="cuda")
            frd = torch.from_numpy(fr).cuda()[R["own"]].contiguous()
            ur = torch.zeros(ds.n_local, dtype=torch.float64, device="cuda")
            torch.cuda.synchronize()
            R["ctx"].probe("vcycle_rows")
            ds.vcycle(fd.data_ptr(), ud.data_ptr())
            R["ctx"].synchronize()
            R["rows_launches"] = R["ctx"].probe_read()[0]
            R["ctx"].probe(None)
            st = ds.bicgstab(frd.data_ptr(), ur.data_ptr())
            ds.rebuild_values(vals2.data_ptr())
            ur.zero_()
            torch.cuda.synchronize()
            st2 = ds.bicgstab(frd.data_ptr(), ur.data_ptr())
            R["ctx"].synchronize()
            out[r] = (ud.cpu().numpy(), st, st2)
        except Exception as e:  # surfaced below
            errs.append(e)

    threads = [threading.Thread(target=run, args=(r,), daemon=True) for r in range(world)]
    for t_ in threads:
        t_.start()
    for t_ in threads:
        t_.join(timeout=120)
    assert not errs, errs
    assert all(o is not None for o in out), "a rank did not finish"
    u = np.zeros(n)
    for r in range(world):
        u[ranks[r]["ds"].owned0] = out[r][0]
    np.testing.assert_array_equal(u.view(np.int64), u_ref.view(np.int64))
    if overlap == "1":  # the boundary-row passes ran (2 per partitioned level with a halo)
        assert all(R["rows_launches"] > 0 for R in ranks), [R["rows_launches"] for R in ranks]
    else:
        assert all(R["rows_launches"] == 0 for R in ranks)
    for r in range(world):
        assert out[r][1].converged and out[r][1].iterations == st_ref.iterations
        assert out[r][2].converged and out[r][2].iterations == st2_ref.iterations
    for R in ranks:
        R["ds"].close()
    lb.close()


def _run_ranks(world, fn):
    import threading

    out, errs = [None] * world, []

    def run(r):
        try:
            out[r] = fn(r)
        except Exception as e:  # surfaced below
            errs.append((r, e))

    threads = [threading.Thread(target=run, args=(r,), daemon=True) for r in range(world)]
    for t_ in threads:
        t_.start()
    for t_ in threads:
        t_.join(timeout=180)
    return out, errs


@pytest.mark.parametrize("world", [1, 2, 3])
def test_dist_rebuild_from_rank_local_values_bit_exact(world):
    """amgr_dist_rebuild_local: every rank passes ONLY its own rows of A_k
    (global_values[nnz_map]); local Jacobi + local Galerkin products (device
    plans restricted to the rank's coarse rows), one allgather of A_{top+1},
    replicated tail rebuild.  The assembled V-cycle equals the single-GPU
    V-cycle of partial_update(h, A_k) bit for bit and the BiCGStab iteration
    counts agree; a zero diagonal raises the reference's message on every
    rank.  world 1 runs through NCCL, 2 and 3 through the loopback transport."""
    import torch

    from paper_2108_02054_b200 import distributed as D

    A = P.grid3d_values("dambreak", 20, 9)
    A2 = P.grid3d_values("dambreak", 20, 30)
    n = 20 ** 3
    f = np.random.default_rng(7).uniform(-1, 1, n)
    fr = P.rhs(n)
    ref_ctx = amg.Context(0)
    h_ref = amg.setup(A, ctx=ref_ctx)
    h_ref.rebuild_values(A2[2])
    u_ref = amg.vcycle(h_ref, f)
    _, st_ref = amg.bicgstab(h_ref, fr)
    bad = np.asarray(A2[2]).copy()
    rp, ci = np.asarray(A2[0]), np.asarray(A2[1])
    brow = 4321
    bad[rp[brow] + np.nonzero(ci[rp[brow]:rp[brow + 1]] == brow)[0][0]] = 0.0
    with pytest.raises(amg.InvalidArgument) as e_ref:
        h_ref.rebuild_values(bad)

    lb = D.Loopback(world) if world > 1 else None
    ranks = []
    for r in range(world):
        ctx = amg.Context(0)
        h = amg.setup(A, ctx=ctx)
        ds = D.DistSolver(h, r, world, D.nccl_unique_id() if lb is None else None, replicate_below=300, loopback=lb)
        assert ds.plan.top >= 1
        ranks.append({"ctx": ctx, "ds": ds, "own": ds.owned0})

    def fn(r):
        R = ranks[r]
        ds = R["ds"]
        ds.rebuild_local(ds.local_values(A2[2]))
        fd = torch.from_numpy(f[R["own"]]).cuda()
        ud = torch.zeros(ds.n_local, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        ds.vcycle(fd.data_ptr(), ud.data_ptr())
        R["ctx"].synchronize()
        frd = torch.from_numpy(fr[R["own"]]).cuda()
        ur = torch.zeros(ds.n_local, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        st = ds.bicgstab(frd.data_ptr(), ur.data_ptr())
        msg = None
        try:
            ds.rebuild_local(ds.local_values(bad))
        except amg.InvalidArgument as e:
            msg = str(e)
        return ud.cpu().numpy(), st, msg

    out, errs = _run_ranks(world, fn)
    assert not errs, errs
    u = np.zeros(n)
    for r in range(world):
        u[ranks[r]["own"]] = out[r][0]
    np.testing.assert_array_equal(u.view(np.int64), u_ref.view(np.int64))
    for r in range(world):
        assert out[r][1].converged and out[r][1].iterations == st_ref.iterations
        assert out[r][2] == str(e_ref.value), (out[r][2], str(e_ref.value))
    for R in ranks:
        R["ds"].close()
    if lb:
        lb.close()


def test_dist_create_validates_the_plan_before_connecting(ctx):
    """A corrupt plan is rejected with a message before any NCCL
    communicator exists (indices and transition counts checked)."""
    from paper_2108_02054_b200 import distributed as D
    from paper_2108_02054_b200 import partition as PT

    A = P.grid3d_values("dambreak", 12, 3)
    h = amg.setup(A, ctx=ctx)
    for corrupt, msg in ((lambda p: p.levels[0].col.__setitem__(0, 10 ** 8), "column id"),
                         (lambda p: p.levels[0].send.__setitem__(0, np.array([1])), "send peer"),
                         (lambda p: setattr(p.levels[p.top], "mptr", p.levels[p.top].mptr[:-1]),
                          "owned coarse rows")):
        plan = PT.build_plan(D.hierarchy_structure(h), 0, 1, replicate_below=100)
        corrupt(plan)
        with pytest.raises(amg.InvalidArgument, match=msg):
            D.DistSolver(h, 0, 1, D.nccl_unique_id(), plan=plan)


@pytest.mark.parametrize("world", [2, 3])
def test_device_built_plan_matches_host_plan_and_solves(world):
    """amgr_dist_create_auto builds the partition on the device (dist_plan.cu):
    owned rows, local CSR maps and halo sizes equal partition.py's on every
    rank, and a loopback run on the device plans (rank-local rebuild, V-cycle,
    BiCGStab) is bit-identical to the single-GPU path."""
    import torch

    from paper_2108_02054_b200 import distributed as D
    from paper_2108_02054_b200 import partition as PT

    A = P.grid3d_values("dambreak", 20, 9)
    A2 = P.grid3d_values("dambreak", 20, 30)
    n = 20 ** 3
    f = np.random.default_rng(11).uniform(-1, 1, n)
    fr = P.rhs(n)
    ref_ctx = amg.Context(0)
    h_ref = amg.setup(A, ctx=ref_ctx)
    h_ref.rebuild_values(A2[2])
    u_ref = amg.vcycle(h_ref, f)
    _, st_ref = amg.bicgstab(h_ref, fr)
    struct = D.hierarchy_structure(h_ref)

    lb = D.Loopback(world)
    ranks = []
    for r in range(world):
        ctx = amg.Context(0)
        h = amg.setup(A, ctx=ctx)
        ds = D.DistSolver(h, r, world, replicate_below=300, loopback=lb, device_plan=True)
        hp = PT.build_plan(struct, r, world, replicate_below=300)
        assert ds.plan.top == hp.top
        for lvl in range(hp.top + 1):
            assert ds.plan.levels[lvl].n_own == hp.levels[lvl].n_own
            assert len(ds.plan.levels[lvl].halo) == len(hp.levels[lvl].halo)
            assert ds.plan.levels[lvl].n_coarse_owned == len(hp.levels[lvl].mptr) - 1
        np.testing.assert_array_equal(ds.owned0, hp.levels[0].owned)
        np.testing.assert_array_equal(ds.plan.levels[0].nnz_map, hp.levels[0].nnz_map)
        ranks.append({"ctx": ctx, "ds": ds, "own": ds.owned0})

    def fn(r):
        R = ranks[r]
        ds = R["ds"]
        ds.rebuild_local(ds.local_values(A2[2]))
        fd = torch.from_numpy(f[R["own"]]).cuda()
        ud = torch.zeros(ds.n_local, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        ds.vcycle(fd.data_ptr(), ud.data_ptr())
        R["ctx"].synchronize()
        frd = torch.from_numpy(fr[R["own"]]).cuda()
        ur = torch.zeros(ds.n_local, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        st = ds.bicgstab(frd.data_ptr(), ur.data_ptr())
        return ud.cpu().numpy(), st

    out, errs = _run_ranks(world, fn)
    assert not errs, errs
    u = np.zeros(n)
    for r in range(world):
        u[ranks[r]["own"]] = out[r][0]
    np.testing.assert_array_equal(u.view(np.int64), u_ref.view(np.int64))
    for r in range(world):
        assert out[r][1].converged and out[r][1].iterations == st_ref.iterations
    for R in ranks:
        R["ds"].close()
    lb.close()


@pytest.mark.parametrize("world,g", [(4, 48), (8, 48), (8, 64), (2, 128), (8, 128)])
def test_device_built_plan_c4_rank_counts_bit_exact(world, g):
    """C4's rank counts (4 and 8) on larger dam-break grids, all on the
    device-built plan through the loopback transport with halo overlap: the
    rank-local rebuild and the assembled V-cycle equal the single-GPU partial
    update's bit for bit.  BiCGStab: every rank takes the same iteration count
    and the assembled solution's true residual is <= tol; the count equals the
    single-GPU one up to 64^3, while at 128^3 the rank-ordered dot sums (a
    different summation order from the single-GPU blocked dots) move it by a
    few iterations, as any dot order does at that size (test_gpu_parity_large)."""
    import torch

    from paper_2108_02054_b200 import distributed as D

    A = P.grid3d_values("dambreak", g, 9)
    A2 = P.grid3d_values("dambreak", g, 30)
    n = g ** 3
    f = np.random.default_rng(13).uniform(-1, 1, n)
    fr = P.rhs(n)
    ref_ctx = amg.Context(0)
    h_ref = amg.setup(A, ctx=ref_ctx)
    h_ref.rebuild_values(A2[2])
    u_ref = amg.vcycle(h_ref, f)
    _, st_ref = amg.bicgstab(h_ref, fr)

    lb = D.Loopback(world)
    ranks = []
    for r in range(world):
        ctx = amg.Context(0)
        h = amg.setup(A, ctx=ctx)
        ds = D.DistSolver(h, r, world, replicate_below=2000, loopback=lb, device_plan=True)
        assert ds.plan.top >= 2, ds.plan.top
        ranks.append({"ctx": ctx, "ds": ds, "own": ds.owned0})
    assert sorted(np.concatenate([R["own"] for R in ranks]).tolist()) == list(range(n))

    def fn(r):
        R = ranks[r]
        ds = R["ds"]
        ds.rebuild_local(ds.local_values(A2[2]))
        fd = torch.from_numpy(f[R["own"]]).cuda()
        ud = torch.zeros(ds.n_local, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        ds.vcycle(fd.data_ptr(), ud.data_ptr())
        R["ctx"].synchronize()
        frd = torch.from_numpy(fr[R["own"]]).cuda()
        ur = torch.zeros(ds.n_local, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        st = ds.bicgstab(frd.data_ptr(), ur.data_ptr())
        return ud.cpu().numpy(), st, ur.cpu().numpy()

    out, errs = _run_ranks(world, fn)
    assert not errs, errs
    assert all(o is not None for o in out), "a rank did not finish"
    u = np.zeros(n)
    for r in range(world):
        u[ranks[r]["own"]] = out[r][0]
    np.testing.assert_array_equal(u.view(np.int64), u_ref.view(np.int64))
    its = {out[r][1].iterations for r in range(world)}
    assert len(its) == 1 and all(out[r][1].converged for r in range(world)), [out[r][1] for r in range(world)]
    x = np.zeros(n)
    for r in range(world):
        x[ranks[r]["own"]] = out[r][2]
    from oracle import ref

    assert np.linalg.norm(fr - ref.spmv(A2, x)) <= 1e-8 * np.linalg.norm(fr)
    if g <= 64:
        assert its == {st_ref.iterations}
    else:
        assert abs(its.pop() - st_ref.iterations) <= 0.25 * st_ref.iterations
    for R in ranks:
        R["ds"].close()
    lb.close()


@pytest.mark.parametrize("world,g", [(1, 20), (2, 20), (3, 32), (4, 48), (8, 128)])
def test_dist_sequential_dots_bit_identical(world, g):
    """Sequential-dot parity mode on the partition (every rank's context set
    to AMGR_DOTS_SEQUENTIAL): each dot is the reference's left-to-right sum
    over the GLOBAL index (products allgathered, summed through the global
    order), so the row-partitioned BiCGStab after a rank-local rebuild is the
    reference's bicgstab on partial_update(A_k) bit for bit — same iteration
    count, same assembled iterate, same residual — at any rank count, checked
    against oracle/_ref itself (128^3 at W = 8: 2.1M rows, about a minute of
    reference CPU time).  World 1 runs over NCCL (graph-captured), the others
    through loopback."""
    import torch

    from oracle import ref
    from paper_2108_02054_b200 import distributed as D

    A = P.grid3d_values("dambreak", g, 9)
    A2 = P.grid3d_values("dambreak", g, 30)
    n = g ** 3
    fr = P.rhs(n)
    r0 = ref.setup(A)
    r2 = ref.partial_update(r0, A2)
    r0.free()
    rs = ref.bicgstab(r2, fr, fixed=True)
    want_u, want_it, want_res = rs.u, rs.iterations, rs.relative_residual
    r2.free()

    lb = D.Loopback(world) if world > 1 else None
    ranks = []
    for r in range(world):
        ctx = amg.Context(0)
        ctx.sequential_dots = True
        h = amg.setup(A, amg.AmgParams(coarse_solve="exact"), ctx=ctx)
        ds = D.DistSolver(h, r, world, D.nccl_unique_id() if lb is None else None, replicate_below=2000,
                          loopback=lb, device_plan=True)
        ranks.append({"ctx": ctx, "ds": ds, "own": ds.owned0})

    def fn(r):
        R = ranks[r]
        ds = R["ds"]
        ds.rebuild_local(ds.local_values(A2[2]))
        frd = torch.from_numpy(fr[R["own"]]).cuda()
        ur = torch.zeros(ds.n_local, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        st = ds.bicgstab(frd.data_ptr(), ur.data_ptr())
        return st, ur.cpu().numpy()

    out, errs = _run_ranks(world, fn)
    assert not errs, errs
    assert all(o is not None for o in out), "a rank did not finish"
    x = np.zeros(n)
    for r in range(world):
        st = out[r][0]
        assert st.converged and st.iterations == want_it, (r, st, want_it)
        assert np.float64(st.relative_residual).view(np.int64) == np.float64(want_res).view(np.int64), \
            (st.relative_residual, want_res)
        x[ranks[r]["own"]] = out[r][1]
    np.testing.assert_array_equal(x.view(np.int64), np.asarray(want_u).view(np.int64))
    for R in ranks:
        R["ds"].close()
    if lb:
        lb.close()


def test_dist_mixed_dot_orders_fail_on_every_rank():
    """Ranks whose contexts disagree on the dot order would run different
    collective sequences: every rank raises instead of hanging."""
    import torch

    from paper_2108_02054_b200 import distributed as D

    g, world = 16, 2
    A = P.grid3d_values("dambreak", g, 9)
    fr = P.rhs(g ** 3)
    lb = D.Loopback(world)
    ranks = []
    for r in range(world):
        ctx = amg.Context(0)
        ctx.sequential_dots = r == 0
        h = amg.setup(A, ctx=ctx)
        ds = D.DistSolver(h, r, world, replicate_below=300, loopback=lb, device_plan=True)
        ranks.append({"ctx": ctx, "ds": ds, "own": ds.owned0})

    def fn(r):
        R = ranks[r]
        frd = torch.from_numpy(fr[R["own"]]).cuda()
        ur = torch.zeros(R["ds"].n_local, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        try:
            R["ds"].bicgstab(frd.data_ptr(), ur.data_ptr())
        except amg.InvalidArgument as e:
            return str(e)
        return None

    out, errs = _run_ranks(world, fn)
    assert not errs, errs
    assert all(o is not None and "different dot orders" in o for o in out), out
    for R in ranks:
        R["ds"].close()
    lb.close()


def test_device_built_plan_world1_nccl(ctx):
    """World 1 over NCCL on a device-built plan (no halos, no send lists):
    rank-local rebuild + BiCGStab equal the single-GPU path."""
    import torch

    from paper_2108_02054_b200 import distributed as D

    A = P.grid3d_values("dambreak", 20, 9)
    A2 = P.grid3d_values("dambreak", 20, 30)
    n = 20 ** 3
    fr = P.rhs(n)
    h = amg.setup(A, ctx=ctx)
    ds = D.DistSolver(h, 0, 1, D.nccl_unique_id(), replicate_below=300, device_plan=True)
    assert ds.plan.top >= 1 and len(ds.plan.levels[0].halo) == 0
    ds.rebuild_local(ds.local_values(A2[2]))
    frd = torch.from_numpy(fr[ds.owned0]).cuda()
    ur = torch.zeros(ds.n_local, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    st = ds.bicgstab(frd.data_ptr(), ur.data_ptr())
    h2 = amg.setup(A, ctx=ctx)
    h2.rebuild_values(A2[2])
    u2, st2 = amg.bicgstab(h2, fr)
    assert st.converged and st.iterations == st2.iterations
    u = np.zeros(n)
    u[ds.owned0] = ur.cpu().numpy()
    np.testing.assert_array_equal(u.view(np.int64), u2.view(np.int64))
    ds.close()
