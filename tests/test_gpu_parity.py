"""GPU parity: the CUDA path (through the C-ABI) against the reference itself
(oracle/_ref, the unmodified reference compiled from /root/reference sources).

Bar (BASELINE.json north_star): hierarchy structure bit-exact (aggregates,
patterns of P, R and every A_i); level values within 1e-12 relative — we
assert bit-exactness, which holds because the device replays the reference's
summation order; solve: iteration count within +-1 and final
residual <= tol against the fixed-V-cycle oracle.
"""
import numpy as np
import pytest

from oracle import problems as P
from oracle import ref

pytestmark = pytest.mark.gpu

amg = pytest.importorskip("paper_2108_02054_b200")


def _bits(a):
    return np.asarray(a, np.float64).view(np.int64)


def assert_same_hierarchy(g, r, values=True, lu=True):
    assert g.num_levels() == len(r.levels), (g.num_levels(), len(r.levels))
    for l, RL in enumerate(r.levels):
        rp, ci, v = g.level_A(l)
        np.testing.assert_array_equal(rp, RL.A[0], err_msg=f"level {l} row_ptr")
        np.testing.assert_array_equal(ci, RL.A[1], err_msg=f"level {l} col_idx")
        if values:
            np.testing.assert_array_equal(_bits(v), _bits(RL.A[2]), err_msg=f"level {l} values")
        if RL.agg is not None:
            np.testing.assert_array_equal(g.level_agg(l), RL.agg, err_msg=f"level {l} aggregates")
            rrp, rci = g.level_R(l)
            np.testing.assert_array_equal(rrp, RL.R[0], err_msg=f"level {l} R row_ptr")
            np.testing.assert_array_equal(rci, RL.R[1], err_msg=f"level {l} R col_idx")
        if RL.inv_diag is not None and values:
            np.testing.assert_array_equal(_bits(g.level_smoother(l)), _bits(RL.inv_diag),
                                          err_msg=f"level {l} inv_diag")
    if values and lu:
        lu, piv = g.coarse_lu()
        np.testing.assert_array_equal(piv, r.piv)
        np.testing.assert_array_equal(_bits(lu), _bits(r.lu))


CASES = {
    "poisson1d_64_ce10": (lambda: P.poisson1d(64), dict(coarse_enough=10)),
    "poisson2d_16": (lambda: P.poisson2d(16), {}),
    "poisson2d_40": (lambda: P.poisson2d(40), {}),
    "poisson2d_64": (lambda: P.poisson2d(64), {}),
    "poisson3d_12": (lambda: P.grid3d_values("poisson", 12, 3), {}),
    "dambreak_16": (lambda: P.grid3d_values("dambreak", 16, 0), {}),
    "dambreak_24_k20": (lambda: P.grid3d_values("dambreak", 24, 20), {}),
    "blob_20": (lambda: P.grid3d_values("blob", 20, 5), {}),
    "random_300": (lambda: P.random_csr(300, 300, 0.02, 7, diag=3.0), {}),
    "random_500_eps0": (lambda: P.random_csr(500, 500, 0.01, 11, diag=2.0), dict(eps=0.0)),
}


@pytest.mark.parametrize("name", list(CASES))
def test_setup_bit_exact(ctx, name):
    make, kw = CASES[name]
    A = make()
    h = amg.setup(A, amg.AmgParams(**kw), ctx=ctx)
    r = ref.setup(A, ref.params(**kw))
    assert_same_hierarchy(h, r)


@pytest.mark.parametrize("name", ["poisson2d_40", "dambreak_24_k20", "random_300"])
def test_partial_update_bit_exact(ctx, name):
    make, kw = CASES[name]
    A = make()
    h = amg.setup(A, amg.AmgParams(**kw), ctx=ctx)
    r = ref.setup(A, ref.params(**kw))
    rp, ci, v = A
    rng = np.random.default_rng(5)
    B = (rp, ci, v * (1.0 + 0.1 * rng.random(len(v))))
    hu = amg.partial_update(h, B)
    ru = ref.partial_update(r, B, ref.params(**kw))
    assert_same_hierarchy(hu, ru)
    for l in range(h.num_levels() - 1):
        assert hu.shares_transfer(h, l)
    # in-place rebuild gives the same hierarchy
    h.rebuild(B)
    assert_same_hierarchy(h, ru)


def test_partial_update_fixed_point(ctx):
    A = P.grid3d_values("dambreak", 16, 7)
    h = amg.setup(A, ctx=ctx)
    r = ref.setup(A)
    assert_same_hierarchy(amg.partial_update(h, A), r)


def test_dambreak_sequence_partial_reuse(ctx):
    # values drift, pattern fixed: device rebuild == reference partial_update
    A0 = P.grid3d_values("dambreak", 20, 0)
    h = amg.setup(A0, ctx=ctx)
    r = ref.setup(A0)
    for k in (5, 17, 49):
        Ak = P.grid3d_values("dambreak", 20, k)
        h.rebuild_values(Ak[2])
        r = ref.partial_update(r, Ak)
        assert_same_hierarchy(h, r)


def test_pattern_change_same_dims(ctx):
    A = P.random_csr(200, 200, 0.03, 1, diag=2.0)
    B = P.random_csr(200, 200, 0.03, 2, diag=2.0)
    h = amg.setup(A, ctx=ctx)
    r = ref.setup(A)
    assert_same_hierarchy(amg.partial_update(h, B), ref.partial_update(r, B))


@pytest.mark.parametrize("name", ["poisson2d_64", "dambreak_24_k20", "blob_20", "random_300"])
def test_vcycle_bit_exact(ctx, name):
    make, kw = CASES[name]
    A = make()
    h = amg.setup(A, amg.AmgParams(**kw), ctx=ctx)
    r = ref.setup(A, ref.params(**kw))
    f = np.random.default_rng(3).uniform(-1, 1, len(A[0]) - 1)
    u = amg.vcycle(h, f)
    ur = ref.vcycle(r, f, fixed=True, prm=ref.params(**kw))
    np.testing.assert_array_equal(_bits(u), _bits(ur))


@pytest.mark.parametrize("pre,post", [(0, 0), (2, 1), (1, 3)])
def test_vcycle_sweeps(ctx, pre, post):
    A = P.poisson2d(32)
    h = amg.setup(A, amg.AmgParams(pre_sweeps=pre, post_sweeps=post), ctx=ctx)
    r = ref.setup(A, ref.params(pre_sweeps=pre, post_sweeps=post))
    f = np.random.default_rng(4).uniform(-1, 1, 32 * 32)
    u = amg.vcycle(h, f)
    ur = ref.vcycle(r, f, fixed=True, prm=ref.params(pre_sweeps=pre, post_sweeps=post))
    np.testing.assert_array_equal(_bits(u), _bits(ur))


@pytest.mark.parametrize("name", ["poisson2d_64", "dambreak_24_k20", "blob_20", "poisson3d_12"])
def test_bicgstab_parity(ctx, name):
    make, kw = CASES[name]
    A = make()
    h = amg.setup(A, amg.AmgParams(**kw), ctx=ctx)
    r = ref.setup(A, ref.params(**kw))
    f = P.rhs(len(A[0]) - 1)
    u, st = amg.bicgstab(h, f)
    rs = ref.bicgstab(r, f, fixed=True, prm=ref.params(**kw))
    assert st.converged and rs.converged
    assert abs(st.iterations - rs.iterations) <= 1, (st.iterations, rs.iterations)
    assert st.relative_residual <= 1e-8
    # true residual from the reference's own spmv
    res = np.linalg.norm(f - ref.spmv(A, u)) / np.linalg.norm(f)
    assert res <= 1e-8


def test_bicgstab_zero_rhs(ctx):
    A = P.poisson2d(8)
    h = amg.setup(A, ctx=ctx)
    u, st = amg.bicgstab(h, np.zeros(64))
    assert st.converged and st.iterations == 0 and np.all(u == 0)


def test_errors_match_reference(ctx):
    # dimension change (hierarchy.cpp:110-116)
    h = amg.setup(P.poisson2d(12), ctx=ctx)
    with pytest.raises(amg.DimensionChange, match="partial update impossible, full rebuild required"):
        amg.partial_update(h, P.poisson2d(13))
    # zero diagonal with level prefix (hierarchy.cpp:31-35)
    A = (np.array([0, 2, 3]), np.array([0, 1, 0]), np.array([1.0, 1.0, 1.0]))
    with pytest.raises(amg.InvalidArgument, match="level 0"):
        amg.setup(A, amg.AmgParams(coarse_enough=1), ctx=ctx)
    # stall beyond the direct budget (hierarchy.cpp:70-77)
    D = P.diagonal(np.full(20, 2.0))
    with pytest.raises(amg.RuntimeFailure, match="coarsening stalled"):
        amg.setup(D, amg.AmgParams(coarse_enough=5, max_direct_size=10), ctx=ctx)
    hd = amg.setup(D, amg.AmgParams(coarse_enough=5, max_direct_size=50), ctx=ctx)
    assert hd.num_levels() == 1
    # singular coarse matrix (dense_lu.cpp:38-42)
    S = (np.array([0, 2, 4]), np.array([0, 1, 0, 1]), np.array([1.0, 1.0, 1.0, 1.0]))
    with pytest.raises(amg.RuntimeFailure, match="singular"):
        amg.setup(S, ctx=ctx)


@pytest.mark.parametrize("name", ["poisson2d_64", "dambreak_24_k20", "random_300"])
def test_inverse_coarse_mode_solve_parity(ctx, name):
    """AMGR_COARSE_INVERSE (extension): same hierarchy bits, V-cycle within
    1e-12 of the exact mode, solve within +-1 iteration of the reference."""
    make, kw = CASES[name]
    A = make()
    he = amg.setup(A, amg.AmgParams(**kw), ctx=ctx)
    hi = amg.setup(A, amg.AmgParams(coarse_solve="inverse", **kw), ctx=ctx)
    r = ref.setup(A, ref.params(**kw))
    assert_same_hierarchy(hi, r, lu=hi.coarse_n() > 160)  # small coarse systems: direct inverse, no LU
    if hi.coarse_n() <= 160:
        with pytest.raises(amg.InvalidArgument, match="inverse"):
            hi.coarse_lu()
    f = np.random.default_rng(3).uniform(-1, 1, len(A[0]) - 1)
    ue, ui = amg.vcycle(he, f), amg.vcycle(hi, f)
    assert np.linalg.norm(ue - ui) <= 1e-12 * np.linalg.norm(ue)
    fr = P.rhs(len(A[0]) - 1)
    _, st = amg.bicgstab(hi, fr)
    rs = ref.bicgstab(r, fr, fixed=True, prm=ref.params(**kw))
    assert st.converged and abs(st.iterations - rs.iterations) <= 1


def test_device_generator_matches_host(ctx):
    """The device dam-break / Poisson generators (used by bench.py) produce the
    same bits as the host restatement the parity tests feed the reference."""
    import torch

    L = amg.lib()
    g = 20
    n, nnz = g ** 3, int(L.amgr_problem_nnz(g))
    rp = torch.empty(n + 1, dtype=torch.int32, device="cuda")
    ci = torch.empty(nnz, dtype=torch.int32, device="cuda")
    v = torch.empty(nnz, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    amg._check(L.amgr_problem_pattern(ctx.ptr, g, rp.data_ptr(), ci.data_ptr()), ctx.ptr)
    for kind, k in (("dambreak", 0), ("dambreak", 31), ("poisson", 4), ("convdiff", 7)):
        amg._check(L.amgr_problem_values(ctx.ptr, amg.PROBLEM[kind], g, k, 50, v.data_ptr()), ctx.ptr)
        ctx.synchronize()
        hrp, hci, hv = P.grid3d_values(kind, g, k, 50)
        np.testing.assert_array_equal(rp.cpu().numpy(), hrp)
        np.testing.assert_array_equal(ci.cpu().numpy(), hci)
        if kind == "convdiff":  # exp() may differ in the last bit between libm and CUDA
            np.testing.assert_allclose(v.cpu().numpy(), hv, rtol=1e-14)
        else:
            np.testing.assert_array_equal(v.cpu().numpy().view(np.int64), hv.view(np.int64))


def test_rebuild_adopted_device_values(ctx):
    import torch

    A0 = P.grid3d_values("dambreak", 16, 2)
    A1 = P.grid3d_values("dambreak", 16, 40)
    h = amg.setup(A0, ctx=ctx)
    buf = torch.zeros(len(A1[2]) + 8, dtype=torch.float64, device="cuda")
    buf[: len(A1[2])] = torch.from_numpy(A1[2]).cuda()
    torch.cuda.synchronize()
    h.rebuild_values(buf.data_ptr(), adopt=True)
    r = ref.partial_update(ref.setup(A0), A1)
    assert_same_hierarchy(h, r)


def test_cg_extension_converges(ctx):
    from oracle import oracle as O

    A = P.grid3d_values("poisson", 16, 0)
    h = amg.setup(A, ctx=ctx)
    f = P.rhs(16 ** 3)
    u, st = amg.cg(h, f)
    so = O.cg(O.setup(A), f)
    assert st.converged and so.converged
    assert abs(st.iterations - so.iterations) <= 1
    res = np.linalg.norm(f - ref.spmv(A, u)) / np.linalg.norm(f)
    assert res <= 1e-8


def test_many_levels_and_launch_count(ctx):
    A = P.grid3d_values("dambreak", 32, 10)
    h = amg.setup(A, ctx=ctx)
    l0 = ctx.launches()
    amg.vcycle(h, P.rhs(32 ** 3))
    assert ctx.launches() > l0 + 3 * (h.num_levels() - 1)


@pytest.mark.parametrize("name", ["poisson2d_64", "dambreak_24_k20", "random_300"])
@pytest.mark.parametrize("cluster", ["0", "8", "16"])
def test_vcycle_tail_kernels_bit_exact(ctx, name, monkeypatch, cluster):
    """The persistent V-cycle tail (AMGR_TAIL_NNZ) runs every level in two
    kernels with prolongation fused into smoothing, as a cooperative grid
    (grid barriers) or as one thread-block cluster (AMGR_TAIL_CLUSTER = 8 /
    16 CTAs, cluster barriers): same bits as the reference's (fixed) V-cycle
    and the same solve."""
    monkeypatch.setenv("AMGR_TAIL_CLUSTER", cluster)
    make, kw = CASES[name]
    A = make()
    r = ref.setup(A, ref.params(**kw))
    f = np.random.default_rng(7).uniform(-1, 1, len(A[0]) - 1)
    uref = ref.vcycle(r, f, fixed=True, prm=ref.params(**kw))
    monkeypatch.setenv("AMGR_TAIL_NNZ", "100000000")
    h = amg.setup(A, amg.AmgParams(**kw), ctx=ctx)
    l0 = ctx.launches()
    u = amg.vcycle(h, f)
    assert ctx.launches() - l0 <= 6  # premul, tail down, coarse, tail up (+ copies)
    np.testing.assert_array_equal(_bits(u), _bits(uref))
    fr = P.rhs(len(A[0]) - 1)
    _, st = amg.bicgstab(h, fr)
    rs = ref.bicgstab(r, fr, fixed=True, prm=ref.params(**kw))
    assert st.converged and abs(st.iterations - rs.iterations) <= 1


# ---------------------------------------------------------------- extensions vs the restated oracle
@pytest.mark.parametrize("name,sa_omega", [("poisson2d_40", 2.0 / 3.0), ("poisson3d_12", 2.0 / 3.0),
                                           ("dambreak_16", 0.5), ("random_300", 2.0 / 3.0)])
def test_smoothed_aggregation_vs_oracle(ctx, name, sa_omega):
    """Smoothed aggregation (extension, parity pinned to the restated oracle):
    the device-built smoothed prolongator P, R = P^T, every A_i (two device
    SpGEMMs), the V-cycle with general R/P, a partial update and the solves."""
    from oracle import oracle as O

    make, kw = CASES[name]
    A = make()
    kw = dict(kw, coarsening="smoothed", sa_omega=sa_omega)
    h = amg.setup(A, amg.AmgParams(**kw), ctx=ctx)
    o = O.setup(A, O.params(**kw))
    assert h.num_levels() == len(o.levels)
    for l, L in enumerate(o.levels):
        rp, ci, v = h.level_A(l)
        np.testing.assert_array_equal(rp, L.A[0], err_msg=f"level {l} row_ptr")
        np.testing.assert_array_equal(ci, L.A[1], err_msg=f"level {l} col")
        np.testing.assert_array_equal(_bits(v), _bits(L.A[2]), err_msg=f"level {l} values")
        if L.P is not None:
            for which, ref_m in (("P", L.P), ("R", L.R)):
                mrp, mci, mv = h.level_transfer(l, which)
                np.testing.assert_array_equal(mrp, ref_m[0], err_msg=f"level {l} {which} row_ptr")
                np.testing.assert_array_equal(mci, ref_m[1], err_msg=f"level {l} {which} col")
                np.testing.assert_array_equal(_bits(mv), _bits(ref_m[2]), err_msg=f"level {l} {which} values")
            np.testing.assert_array_equal(_bits(h.level_smoother(l)), _bits(L.w))
    lu, piv = h.coarse_lu()
    np.testing.assert_array_equal(piv, o.piv)
    np.testing.assert_array_equal(_bits(lu), _bits(o.lu))
    n = len(A[0]) - 1
    f = np.random.default_rng(4).uniform(-1, 1, n)
    np.testing.assert_array_equal(_bits(amg.vcycle(h, f)), _bits(O.vcycle(o, f)))
    fr = P.rhs(n)
    _, st = amg.bicgstab(h, fr)
    so = O.bicgstab(o, fr)
    assert st.converged and abs(st.iterations - so.iterations) <= 1
    _, sc = amg.cg(h, fr)
    oc = O.cg(o, fr)
    assert sc.converged == oc.converged and abs(sc.iterations - oc.iterations) <= 1
    # partial update: frozen P/R values, new Galerkin products
    A2 = (A[0], A[1], A[2] * np.linspace(1.0, 1.5, len(A[2])))
    h2 = amg.partial_update(h, A2, amg.AmgParams(**kw))
    o2 = O.partial_update(o, A2, O.params(**kw))
    for l, L in enumerate(o2.levels):
        np.testing.assert_array_equal(_bits(h2.level_A(l)[2]), _bits(L.A[2]), err_msg=f"update level {l}")
    np.testing.assert_array_equal(_bits(amg.vcycle(h2, f)), _bits(O.vcycle(o2, f)))



@pytest.mark.parametrize("problem", ["poisson", "convdiff"])
def test_chebyshev_smoother_vs_oracle(ctx, problem):
    """Chebyshev + power iteration (extension, parity unpinned by the
    reference): same hierarchy bits as the oracle, lambda_max within 1e-12,
    V-cycle within 1e-10 (lambda comes from parallel dots), solve +-1 iter."""
    from oracle import oracle as O

    g = 16
    A = P.grid3d_values(problem, g, 3) if problem == "poisson" else O.grid3d(problem, g, 3)
    kw = dict(smoother="chebyshev", cheb_degree=3, power_iters=12)
    h = amg.setup(A, amg.AmgParams(**kw), ctx=ctx)
    o = O.setup(A, O.params(**kw))
    assert h.num_levels() == len(o.levels)
    for l, L in enumerate(o.levels[:-1]):
        np.testing.assert_array_equal(_bits(h.level_A(l)[2]), _bits(L.A[2]))
        assert h.level_lambda(l) * 1.1 == pytest.approx(L.lam_max, rel=1e-12)
    f = np.random.default_rng(5).uniform(-1, 1, g ** 3)
    u, uo = amg.vcycle(h, f), O.vcycle(o, f)
    assert np.linalg.norm(u - uo) <= 1e-10 * np.linalg.norm(uo)
    fr = P.rhs(g ** 3)
    _, st = amg.bicgstab(h, fr)
    so = O.bicgstab(o, fr)
    assert st.converged == so.converged and abs(st.iterations - so.iterations) <= 1


def test_spai0_smoother_vs_oracle(ctx):
    from oracle import oracle as O

    A = P.grid3d_values("dambreak", 16, 12)
    h = amg.setup(A, amg.AmgParams(smoother="spai0"), ctx=ctx)
    o = O.setup(A, O.params(smoother="spai0"))
    for l, L in enumerate(o.levels[:-1]):
        np.testing.assert_array_equal(_bits(h.level_A(l)[2]), _bits(L.A[2]))
        np.testing.assert_array_equal(_bits(h.level_smoother(l)), _bits(L.w))
    f = np.random.default_rng(6).uniform(-1, 1, 16 ** 3)
    np.testing.assert_array_equal(_bits(amg.vcycle(h, f)), _bits(O.vcycle(o, f)))
    fr = P.rhs(16 ** 3)
    _, st = amg.bicgstab(h, fr)
    so = O.bicgstab(o, fr)
    assert st.converged and abs(st.iterations - so.iterations) <= 1


@pytest.mark.parametrize("n", [72, 75, 78, 150, 160, 161, 400])
def test_direct_solve_sizes_around_the_smem_opt_in(ctx, n):
    """Stalled coarsening (no strong couplings) -> the whole matrix is the
    coarsest system; n = 72..78 is where dynamic + static shared memory of the
    register LU kernel first exceeds 48 KB (regression: missing opt-in);
    160 | 161 is the register kernel's limit (k_dense_reg -> k_lu_factor)."""
    A = P.random_csr(n, n, 0.05, 3, diag=4.0)
    kw = dict(eps=0.99)
    h = amg.setup(A, amg.AmgParams(**kw), ctx=ctx)
    r = ref.setup(A, ref.params(**kw))
    assert h.num_levels() == 1 and h.coarse_n() == n
    lu, piv = h.coarse_lu()
    np.testing.assert_array_equal(piv, r.piv)
    np.testing.assert_array_equal(_bits(lu), _bits(r.lu))
    f = np.random.default_rng(2).uniform(-1, 1, n)
    np.testing.assert_array_equal(_bits(amg.vcycle(h, f)), _bits(ref.vcycle(r, f, fixed=True, prm=ref.params(**kw))))


def test_staged_values_rebuild_matches_plain_rebuild(ctx):
    """amgr_stage_values + AMGR_STAGED (copy-stream pipelining) gives the same
    hierarchy as a plain values rebuild, over two consecutive steps (the
    staging buffer is recycled)."""
    A0 = P.grid3d_values("dambreak", 16, 0)
    h = amg.setup(A0, ctx=ctx)
    g = amg.setup(A0, ctx=ctx)
    for k in (11, 23):
        Ak = P.grid3d_values("dambreak", 16, k)
        h.stage_values(Ak[2])
        h.rebuild_staged()
        g.rebuild_values(Ak[2])
        for l in range(h.num_levels()):
            np.testing.assert_array_equal(_bits(h.level_A(l)[2]), _bits(g.level_A(l)[2]))
        f = np.random.default_rng(k).uniform(-1, 1, 16 ** 3)
        np.testing.assert_array_equal(_bits(amg.vcycle(h, f)), _bits(amg.vcycle(g, f)))
    with pytest.raises(amg.InvalidArgument, match="no staged values"):
        h.rebuild_staged()


def test_pipelined_steps_match_plain_steps(ctx):
    """The fully pipelined step sequence (amgr_stage_values + amgr_stage_rhs
    one step ahead, STAGED rebuild, STAGED solve on device-resident u,
    amgr_download_async of each solution) gives the plain host-path results
    bit for bit: per-step solutions, iteration counts, and the staged RHS is
    the step's own (a different RHS per step)."""
    import torch

    g = 16
    n = g ** 3
    mats = [P.grid3d_values("dambreak", g, k) for k in (0, 7, 15, 22)]
    rhs = [np.random.default_rng(k).uniform(0.1, 1, n) for k in range(4)]
    # plain path: host buffers, u0 = previous solution
    h = amg.setup(mats[0], ctx=ctx)
    u = np.zeros(n)
    plain = []
    for k in range(1, 4):
        h.rebuild_values(mats[k][2])
        u, st = amg.bicgstab(h, rhs[k], u)
        plain.append((u.copy(), st.iterations))
    # pipelined path
    hp = amg.setup(mats[0], ctx=ctx)
    dev = torch.device("cuda", ctx.device)
    ub = [torch.zeros(n, dtype=torch.float64, device=dev) for _ in range(2)]
    hv = [torch.from_numpy(mats[k][2]).pin_memory() for k in range(4)]
    hf = [torch.from_numpy(rhs[k]).pin_memory() for k in range(4)]
    out = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(3)]
    torch.cuda.synchronize()
    hp.stage_values(hv[1].data_ptr(), host=True)
    hp.stage_rhs(hf[1].data_ptr(), host=True)
    its = []
    for j, k in enumerate(range(1, 4)):
        hp.rebuild_staged()
        if k + 1 < 4:
            hp.stage_values(hv[k + 1].data_ptr(), host=True)
            hp.stage_rhs(hf[k + 1].data_ptr(), host=True)
        _, st = amg.bicgstab(hp, amg.STAGED_RHS, (ub[(j + 1) % 2].data_ptr(), ub[j % 2].data_ptr()))
        its.append(st.iterations)
        ctx.download_async(ub[j % 2].data_ptr(), out[j].data_ptr(), n)
    ctx.synchronize()
    for j in range(3):
        assert its[j] == plain[j][1]
        np.testing.assert_array_equal(_bits(out[j].numpy()), _bits(plain[j][0]))
    # a staged solve with no staged RHS ever is an error
    h2 = amg.setup(mats[0], ctx=ctx)
    with pytest.raises(amg.InvalidArgument, match="no staged right-hand side"):
        amg.bicgstab(h2, amg.STAGED_RHS, (ub[0].data_ptr(), ub[1].data_ptr()))


@pytest.mark.parametrize("kind,g", [("dambreak", 20), ("blob", 24)])
def test_coded_columns_match_raw_columns(ctx, kind, g, monkeypatch):
    """Coded column stream (encode_columns: col = row + dict[code], uint8 on the
    7-point level, uint16 on the wider levels) against the raw int32 layout
    (AMGR_COLCODE=0): identical hierarchy, V-cycle and solve, bit for bit; and
    against the oracle."""
    from oracle import oracle as O

    A = P.grid3d_values(kind, g, 9)
    n = g ** 3
    monkeypatch.delenv("AMGR_COLCODE", raising=False)
    h = amg.setup(A, ctx=ctx)  # default: uint8 on the 7-point level, uint16 on 8..12 entries/row
    lay = [h.level_layout(l) for l in range(h.num_levels())]
    assert lay[0] == {"col_bytes": 1, "ndict": 7}
    for l in range(1, h.num_levels() - 1):
        d = h.level_dims(l)
        mid = 8 * d["nrows"] < d["nnz"] <= 12 * d["nrows"]
        assert lay[l]["col_bytes"] == (2 if mid else 4), (l, d, lay[l])
    monkeypatch.setenv("AMGR_COLCODE", "16")
    hw = amg.setup(A, ctx=ctx)
    assert all(hw.level_layout(l)["col_bytes"] == 2 for l in range(1, hw.num_levels() - 1))
    monkeypatch.setenv("AMGR_COLCODE", "0")
    hr = amg.setup(A, ctx=ctx)
    assert all(hr.level_layout(l)["col_bytes"] == 4 for l in range(hr.num_levels()))
    f = np.random.default_rng(11).uniform(-1, 1, n)
    ref_v = _bits(O.vcycle(O.setup(A), f))
    for x in (h, hw, hr):
        np.testing.assert_array_equal(_bits(amg.vcycle(x, f)), ref_v)
    fr = P.rhs(n)
    u2, s2 = amg.bicgstab(hr, fr)
    for x in (h, hw):
        u1, s1 = amg.bicgstab(x, fr)
        assert s1.iterations == s2.iterations
        np.testing.assert_array_equal(_bits(u1), _bits(u2))
    # partial reuse keeps the coded pattern
    A2 = P.grid3d_values(kind, g, 10)
    h2 = amg.partial_update(h, A2)
    assert h2.level_layout(0)["col_bytes"] == 1
    np.testing.assert_array_equal(_bits(amg.vcycle(h2, f)), _bits(O.vcycle(O.partial_update(O.setup(A), A2), f)))


def test_coded_columns_fallback_many_offsets(ctx):
    """A pattern whose offsets exceed the code dictionary keeps int32 columns."""
    rng = np.random.default_rng(3)
    n = 3000
    rows = []
    for i in range(n):
        cols = set(rng.choice(n, 5, replace=False).tolist()) | {i}
        rows.append([(c, (4.0 if c == i else -0.5)) for c in cols])
    A = P.csr_from_dense_rows(rows, n)
    h = amg.setup(A, amg.AmgParams(coarse_enough=50), ctx=ctx)
    assert h.level_layout(0)["col_bytes"] == 4
    from oracle import oracle as O

    f = rng.uniform(-1, 1, n)
    np.testing.assert_array_equal(_bits(amg.vcycle(h, f)), _bits(O.vcycle(O.setup(A, O.params(coarse_enough=50)), f)))


def test_chebyshev_solve_without_prior_vcycle(ctx):
    """The first Chebyshev sweep used to allocate its direction vectors lazily;
    when that happened inside the solver's CUDA-graph capture the allocation
    became graph-owned and relaunching the graph failed (cudaGraphLaunch:
    invalid argument).  A solve as the very first call must work."""
    from oracle import oracle as O

    g = 20
    A = O.grid3d("convdiff", g, 4)
    kw = dict(smoother="chebyshev")
    h = amg.setup(A, amg.AmgParams(**kw), ctx=ctx)
    fr = P.rhs(g ** 3)
    _, st = amg.bicgstab(h, fr)
    so = O.bicgstab(O.setup(A, O.params(**kw)), fr)
    assert st.converged and so.converged and abs(st.iterations - so.iterations) <= 1


def test_pipelining_entry_points_validate_arguments(ctx):
    """amgr_stage_rhs / amgr_download_async / STAGED solve argument checks
    (the reference-style error texts come back through amgr_last_error)."""
    import ctypes

    import torch

    L = amg.lib()
    A = P.grid3d_values("poisson", 8, 0)
    h = amg.setup(A, ctx=ctx)
    n = 8 ** 3
    u = torch.zeros(n, dtype=torch.float64, device=torch.device("cuda", ctx.device))
    host = torch.empty(n, dtype=torch.float64).pin_memory()
    assert L.amgr_download_async(ctx.ptr, u.data_ptr(), host.data_ptr(), -1) != 0
    assert L.amgr_download_async(ctx.ptr, None, host.data_ptr(), n) != 0
    assert L.amgr_download_async(ctx.ptr, u.data_ptr(), host.data_ptr(), 0) == 0
    assert L.amgr_stage_rhs(h._p, None, amg.HOST) != 0
    with pytest.raises(amg.InvalidArgument, match="location must be HOST or DEVICE"):
        amg._check(L.amgr_stage_rhs(h._p, u.data_ptr(), amg.STAGED), ctx.ptr)
    # f = NULL is only accepted with AMGR_STAGED
    sp, st = amg._SolveParams(1e-8, 10), amg._SolveStats()
    assert L.amgr_bicgstab(h._p, None, u.data_ptr(), u.data_ptr(), ctypes.byref(sp), ctypes.byref(st),
                           amg.DEVICE) != 0
    # a staged RHS is consumed by the next STAGED rebuild, then solved with
    h.stage_values(A[2])
    h.stage_rhs(np.ones(n))
    h.rebuild_staged()
    _, s1 = amg.bicgstab(h, amg.STAGED_RHS, (u.data_ptr(), u.data_ptr()))
    u2, s2 = amg.bicgstab(h, np.ones(n))
    assert s1.iterations == s2.iterations and s1.converged
    np.testing.assert_array_equal(_bits(u.cpu().numpy()), _bits(u2))


def test_pattern_change_keeps_coded_columns(ctx):
    """A pattern-changing partial update re-encodes the column streams
    (hierarchy.cu rebuild_into), so the row passes keep their 1-byte coded
    level 0 instead of silently falling back to int32 columns."""
    A = P.grid3d_values("dambreak", 16, 3)
    h = amg.setup(A, ctx=ctx)
    before = [h.level_layout(l)["col_bytes"] for l in range(h.num_levels() - 1)]
    assert before[0] == 1
    # drop the couplings of every 5th row to its +x neighbour (and the
    # symmetric entry): same dimensions, new sparsity pattern
    rp, ci, v = (np.asarray(x) for x in A)
    n = len(rp) - 1
    keep = np.ones(len(ci), bool)
    for i in range(0, n - 1, 5):
        for a, b in ((i, i + 1), (i + 1, i)):
            s, e = rp[a], rp[a + 1]
            hit = np.nonzero(ci[s:e] == b)[0]
            keep[s + hit] = False
    rows = np.repeat(np.arange(n), np.diff(rp))[keep]
    rp2 = np.zeros(n + 1, np.int64)
    np.add.at(rp2, rows + 1, 1)
    B = (np.cumsum(rp2), ci[keep], v[keep])
    hu = amg.partial_update(h, B)
    ru = ref.partial_update(ref.setup(A), B)
    assert_same_hierarchy(hu, ru)
    after = [hu.level_layout(l)["col_bytes"] for l in range(hu.num_levels() - 1)]
    assert after[0] == 1, after
    f = P.rhs(n)
    assert np.array_equal(_bits(amg.vcycle(hu, f)), _bits(ref.vcycle(ru, f, fixed=True)))


@pytest.mark.parametrize("groups,rows,fuse", [("1", "0", "0"), ("0", "1", "1"), ("0", "0", "0"), ("0", "0", "1")])
def test_rebuild_zero_diagonal_error_fused_and_separate(ctx, monkeypatch, groups, rows, fuse):
    """A partial update whose new A_0 has a zero diagonal fails with the
    reference's message (hierarchy.cpp:124-132 + :31-35), both when the
    Jacobi rebuild is fused into a Galerkin kernel (warp-group, the default;
    member-row) and when it runs separately; a coarse-level zero diagonal
    names its level."""
    monkeypatch.setenv("AMGR_RAP_GROUPS", groups)
    monkeypatch.setenv("AMGR_RAP_ROWS", rows)
    monkeypatch.setenv("AMGR_FUSE_JACOBI", fuse)
    A = P.grid3d_values("dambreak", 12, 3)
    h = amg.setup(A, ctx=ctx)
    r = ref.setup(A)
    rp, ci, v = (np.asarray(x).copy() for x in A)
    row = 37
    v[rp[row] + np.nonzero(ci[rp[row]:rp[row + 1]] == row)[0][0]] = 0.0
    with pytest.raises(ref.RefError) as er:
        ref.partial_update(r, (rp, ci, v))
    with pytest.raises(amg.InvalidArgument) as eg:
        h.rebuild((rp, ci, v))
    assert str(eg.value) == str(er.value), (str(eg.value), str(er.value))
    # the hierarchy stays usable: rebuild with valid values again
    h.rebuild(A)
    assert_same_hierarchy(h, r)


@pytest.mark.parametrize("name", ["poisson2d_64", "dambreak_24_k20", "blob_20", "random_300", "poisson1d_64_ce10"])
def test_member_row_rap_matches_contrib_rap(ctx, monkeypatch, name):
    """k_rap_grp (warp-group plan, fused fine Jacobi; the default),
    k_rap_rows (member-row plan, fused Jacobi), k_rap_tma with the coarse
    Jacobi fused, and k_rap_tma + separate k_jacobi give the same bits, and
    all match the reference."""
    make, kw = CASES[name]
    A = make()
    h = amg.setup(A, amg.AmgParams(**kw), ctx=ctx)
    r = ref.setup(A, ref.params(**kw))
    rp, ci, v = A
    B = (rp, ci, np.asarray(v) * (1.0 + 0.05 * np.random.default_rng(9).random(len(v))))
    ru = ref.partial_update(r, B, ref.params(**kw))
    for groups, rows, fuse in (("1", "0", "0"), ("0", "1", "1"), ("0", "0", "0"), ("0", "0", "1"), ("0", "1", "0"),
                               ("1", "0", "1")):
        monkeypatch.setenv("AMGR_RAP_GROUPS", groups)
        monkeypatch.setenv("AMGR_RAP_ROWS", rows)
        monkeypatch.setenv("AMGR_FUSE_JACOBI", fuse)
        h.rebuild_values(B[2])
        assert_same_hierarchy(h, ru)


def _wide_row_poisson(g=24, eps=1e-3):
    """2-D Poisson plus one node coupled (weakly, symmetrically) to every
    other node: row 0 has g*g entries (> 255), beyond the warp-group Galerkin
    plan's 8-bit row offsets, so that level falls back to k_rap_tma + k_jacobi."""
    rp, ci, v = (np.asarray(x) for x in P.poisson2d(g))
    n = len(rp) - 1
    rows = []
    for i in range(n):
        cols = dict(zip(ci[rp[i]:rp[i + 1]].tolist(), v[rp[i]:rp[i + 1]].tolist()))
        if i == 0:
            for j in range(1, n):
                cols[j] = cols.get(j, 0.0) - eps
            cols[0] += eps * (n - 1)
        else:
            cols[0] = cols.get(0, 0.0) - eps
            cols[i] += eps
        rows.append(sorted(cols.items()))
    rp2 = np.zeros(n + 1, np.int64)
    rp2[1:] = np.cumsum([len(r) for r in rows])
    ci2 = np.array([c for r in rows for c, _ in r], np.int64)
    v2 = np.array([x for r in rows for _, x in r])
    return rp2, ci2, v2


@pytest.mark.parametrize("groups", ["1", "0"])
def test_galerkin_group_plan_falls_back_on_long_rows(ctx, monkeypatch, groups):
    """A level whose rows exceed the warp-group plan's bounds (a 576-entry
    row) runs k_rap_tma + k_jacobi while the other levels run k_rap_grp: the
    partial update is still bit-exact against the reference."""
    monkeypatch.setenv("AMGR_RAP_GROUPS", groups)
    A = _wide_row_poisson()
    assert np.max(np.diff(A[0])) > 255
    h = amg.setup(A, ctx=ctx)
    r = ref.setup(A)
    assert_same_hierarchy(h, r)
    B = (A[0], A[1], A[2] * (1.0 + 0.05 * np.random.default_rng(4).random(len(A[2]))))
    hu = amg.partial_update(h, B)
    ru = ref.partial_update(r, B)
    assert_same_hierarchy(hu, ru)
    h.rebuild_values(B[2])
    assert_same_hierarchy(h, ru)


def test_rebuild_coarse_level_zero_diagonal_names_its_level(ctx, monkeypatch):
    """A zero diagonal that first appears on a coarse level during a partial
    update (the fused coarse-Jacobi epilogue) is reported with that level,
    as build_smoother inside partial_update does (hierarchy.cpp:124-132)."""
    A = P.poisson1d(8)  # aggregates {0,1},{2,3},... -> levels of 8, 4, 2, 1 rows
    prm = dict(coarse_enough=1)
    rp, ci, v = (np.asarray(x).copy() for x in A)
    # rows 0 and 1: [[1, -1], [-1, 1]] block -> coarse (0, 0) = 1 - 1 - 1 + 1 = 0
    for i, j, x in ((0, 0, 1.0), (0, 1, -1.0), (1, 0, -1.0), (1, 1, 1.0)):
        v[rp[i] + np.nonzero(ci[rp[i]:rp[i + 1]] == j)[0][0]] = x
    r = ref.setup(A, ref.params(**prm))
    with pytest.raises(ref.RefError) as er:
        ref.partial_update(r, (rp, ci, v), ref.params(**prm))
    assert "level 1" in str(er.value)
    for groups, fuse in (("1", "0"), ("0", "1"), ("0", "0")):
        monkeypatch.setenv("AMGR_RAP_GROUPS", groups)
        monkeypatch.setenv("AMGR_FUSE_JACOBI", fuse)
        h = amg.setup(A, amg.AmgParams(**prm), ctx=ctx)
        with pytest.raises(amg.InvalidArgument) as eg:
            h.rebuild((rp, ci, v))
        assert str(eg.value) == str(er.value)


@pytest.mark.parametrize("g,k", [(48, 7), (96, 20)])
def test_lag_fused_smoothing_spmv_is_bit_identical(ctx, monkeypatch, g, k):
    """k_rowpass_lag (last level-0 smoothing sweep + the Krylov SpMV/dots in
    one pass over A_0) gives exactly the separate kernels' BiCGStab: same
    iterations, same iterate bits, same residual."""
    A = P.grid3d_values("dambreak", g, k)
    f = P.rhs(g ** 3)
    out = {}
    for lag in ("0", "1"):
        monkeypatch.setenv("AMGR_LAG_FUSE", lag)  # opt-in fused kernel vs the default separate passes
        h = amg.setup(A, ctx=ctx)
        u, st = amg.bicgstab(h, f)
        out[lag] = (u, st)
    (u0, s0), (u1, s1) = out["0"], out["1"]
    assert s0.iterations == s1.iterations and s0.converged == s1.converged
    assert np.array_equal(_bits(u0), _bits(u1))
    assert _bits([s0.relative_residual])[0] == _bits([s1.relative_residual])[0]


@pytest.mark.parametrize("name", ["dambreak_24_k20", "blob_20", "random_300", "poisson2d_64"])
def test_level_spmv_bit_exact(ctx, name):
    """amgr_spmv (k_rowpass<OpSpmv> on every level: coded 1-/2-byte and raw
    column streams) and the single-operator amgr_csr_spmv equal the
    reference's spmv (csr.cpp:76-85) bit for bit."""
    make, kw = CASES[name]
    A = make()
    h = amg.setup(A, amg.AmgParams(**kw), ctx=ctx)
    r = ref.setup(A, ref.params(**kw))
    rng = np.random.default_rng(4)
    for l, RL in enumerate(r.levels):
        x = rng.uniform(-1, 1, len(RL.A[0]) - 1)
        assert np.array_equal(_bits(h.spmv(l, x)), _bits(ref.spmv(RL.A, x))), f"level {l}"
    x = rng.uniform(-1, 1, len(A[0]) - 1)
    assert np.array_equal(_bits(amg.spmv(A, x, ctx=ctx)), _bits(ref.spmv(A, x)))


def test_single_operator_entry_points(ctx):
    """build_smoother / smooth / coarse_factorize / coarse_solve on one matrix
    (the reference's free functions) against the hierarchy's own results and
    the reference's arithmetic, incl. error texts."""
    A = P.grid3d_values("dambreak", 10, 4)
    r = ref.setup(A)
    w = amg.build_smoother(A, 0.72, ctx=ctx)
    assert np.array_equal(_bits(w), _bits(r.levels[0].inv_diag))
    f = P.rhs(1000)
    # one sweep from u0: u + (om*w)(f - A u), elementwise IEEE ops as smoother.cpp:46
    u0 = np.random.default_rng(2).uniform(-1, 1, 1000)
    expect = u0.copy()
    for _ in range(3):
        expect = expect + (0.72 * w) * (f - ref.spmv(A, expect))
    assert np.array_equal(_bits(amg.smooth(w, A, f, u0, 3, 0.72, ctx=ctx)), _bits(expect))
    # coarsest matrix of the hierarchy: factor and solve as the hierarchy does
    Lc = r.levels[-1].A
    lu, piv = amg.coarse_factorize(Lc, ctx=ctx)
    assert np.array_equal(piv, r.piv) and np.array_equal(_bits(lu), _bits(r.lu))
    b = np.random.default_rng(3).uniform(-1, 1, len(piv))
    x = amg.coarse_solve(lu, piv, b, ctx=ctx)
    assert np.allclose(ref.spmv(Lc, x), b, rtol=1e-9, atol=1e-12)
    bad = (np.array([0, 1, 2]), np.array([0, 0]), np.array([1.0, 1.0]))
    with pytest.raises(amg.InvalidArgument, match="build_smoother: zero diagonal at row 1"):
        amg.build_smoother(bad, ctx=ctx)
    sing = P.csr_from_dense_rows([[(0, 1.0), (1, 1.0)], [(0, 1.0), (1, 1.0)]], 2)
    with pytest.raises(amg.RuntimeFailure, match="singular"):
        amg.coarse_factorize(sing, ctx=ctx)


def test_tiny_and_empty_systems_match_reference(ctx):
    """Edge sizes (hierarchy.cpp:45-105, dense_lu.cpp, bicgstab.cpp): the
    empty matrix is rejected with the reference's text; 1x1 and 2x2 systems
    are a single direct level whose factor, V-cycle and BiCGStab (iterations,
    iterate, residual) are bit-identical to the reference's."""
    empty = (np.array([0]), np.array([], dtype=np.int64), np.array([]))
    with pytest.raises(ref.RefError, match="setup: empty matrix"):
        ref.setup(empty)
    with pytest.raises(amg.InvalidArgument, match="setup: empty matrix"):
        amg.setup(empty, ctx=ctx)
    systems = [((np.array([0, 1]), np.array([0]), np.array([4.0])), np.array([2.0])),
               (P.csr_from_dense_rows([[(0, 4.0), (1, -1.0)], [(0, -1.0), (1, 4.0)]], 2), np.array([1.0, 2.0])),
               # pivoting: |a_10| > |a_00|
               (P.csr_from_dense_rows([[(0, 1.0), (1, 2.0)], [(0, 3.0), (1, 1.0)]], 2), np.array([1.0, -1.0]))]
    for A, f in systems:
        h = amg.setup(A, ctx=ctx)
        r = ref.setup(A)
        assert h.num_levels() == len(r.levels) == 1
        assert_same_hierarchy(h, r)
        assert np.array_equal(_bits(amg.vcycle(h, f)), _bits(ref.vcycle(r, f, fixed=True)))
        u, st = amg.bicgstab(h, f)
        rs = ref.bicgstab(r, f, fixed=True)
        assert st.iterations == rs.iterations and bool(st.converged) == rs.converged
        assert np.array_equal(_bits(u), _bits(rs.u))
        r.free()


def test_isolated_rows_and_ragged_lengths_match_reference(ctx):
    """Rows with only a diagonal entry (no strong neighbours: singleton
    aggregates, coarsening.cpp:77-120) mixed with long rows: hierarchy, partial
    update and V-cycle bit-exact."""
    n = 600
    rng = np.random.default_rng(5)
    rows = []
    for i in range(n):
        if i % 7 == 3:
            rows.append([(i, 2.5)])  # isolated
            continue
        cols = {i}
        k = 2 if i % 11 else 40  # a few long rows
        for j in rng.integers(0, n, k):
            if int(j) % 7 != 3:
                cols.add(int(j))
        ent = [(j, -rng.uniform(0.1, 1.0)) for j in sorted(cols) if j != i]
        ent.append((i, 1.0 + sum(-v for _, v in ent)))
        rows.append(sorted(ent))
    A = P.csr_from_dense_rows(rows, n)
    prm = dict(coarse_enough=20)
    h = amg.setup(A, amg.AmgParams(**prm), ctx=ctx)
    r = ref.setup(A, ref.params(**prm))
    assert h.num_levels() >= 2
    assert_same_hierarchy(h, r)
    A2 = (A[0], A[1], A[2] * rng.uniform(0.9, 1.1, len(A[2])))
    h.rebuild_values(A2[2])
    r2 = ref.partial_update(r, A2, ref.params(**prm))
    assert_same_hierarchy(h, r2)
    f = np.random.default_rng(6).uniform(-1, 1, n)
    assert np.array_equal(_bits(amg.vcycle(h, f)), _bits(ref.vcycle(r2, f, fixed=True, prm=ref.params(**prm))))
    r2.free()
    r.free()


def test_symmetric_stencil_form_bit_exact(ctx, monkeypatch):
    """Level 0 of a grid stencil with bitwise-symmetric values runs its row
    passes on the symmetric-stencil form (diagonal + K upper diagonals, k_dia):
    V-cycle, level SpMV and partial update stay bit-exact against the
    reference; values that are not bitwise symmetric (one a_ij != a_ji)
    switch the passes back to the CSR arrays at that rebuild, and back again
    when symmetry returns; AMGR_SYM_DIA=0 gives the same bits."""
    A = P.grid3d_values("dambreak", 24, 7)
    n = 24 ** 3
    f = np.random.default_rng(8).uniform(-1, 1, n)
    h = amg.setup(A, ctx=ctx)
    r = ref.setup(A)
    assert h.level_stencil(0) == (3, (1, 24, 576))
    assert h.level_stencil(1) == (0, ())
    assert np.array_equal(_bits(amg.vcycle(h, f)), _bits(ref.vcycle(r, f, fixed=True)))
    assert np.array_equal(_bits(h.spmv(0, f)), _bits(ref.spmv(A, f)))
    # one asymmetric entry: a(i, i+1) != a(i+1, i)
    rp, ci, v = (np.asarray(x) for x in A)
    i = 5000
    e = rp[i] + int(np.nonzero(ci[rp[i]:rp[i + 1]] == i + 1)[0][0])
    v2 = v.copy()
    v2[e] = np.nextafter(v2[e], 0.0)
    A2 = (rp, ci, v2)
    h.rebuild_values(v2)
    assert h.level_stencil(0) == (0, ())
    r2 = ref.partial_update(r, A2)
    assert np.array_equal(_bits(amg.vcycle(h, f)), _bits(ref.vcycle(r2, f, fixed=True)))
    assert np.array_equal(_bits(h.spmv(0, f)), _bits(ref.spmv(A2, f)))
    r2.free()
    h.rebuild_values(v)
    assert h.level_stencil(0) == (3, (1, 24, 576))
    u_on = amg.vcycle(h, f)
    assert np.array_equal(_bits(u_on), _bits(ref.vcycle(r, f, fixed=True)))
    _, st_on = amg.bicgstab(h, P.rhs(n))
    monkeypatch.setenv("AMGR_SYM_DIA", "0")
    h.rebuild_values(v)
    assert h.level_stencil(0) == (0, ())
    assert np.array_equal(_bits(amg.vcycle(h, f)), _bits(u_on))
    _, st_off = amg.bicgstab(h, P.rhs(n))
    assert abs(st_on.iterations - st_off.iterations) <= 1
    monkeypatch.delenv("AMGR_SYM_DIA")
    # 2D 5-point stencil: K = 2
    h2 = amg.setup(P.poisson2d(64), ctx=ctx)
    assert h2.level_stencil(0) == (2, (1, 64))
    r.free()
