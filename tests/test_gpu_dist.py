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
