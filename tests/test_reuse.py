"""Reuse driver (run_sequence, reuse.cpp:46-154).  CPU: speedup arithmetic
(SPEC.md Table-2 examples).  GPU: the device driver against the restated
run_sequence over the C oracle on the same host sequences."""
import math

import numpy as np
import pytest

from oracle import problems as P


def test_speedup_arithmetic_table2():
    import paper_2108_02054_b200 as amg

    L = amg.lib()
    # SPEC.md:411-423 / PAPER.md Table 2 level-set OpenMP row
    assert L.amgr_speedup_percent(1.235, 0.021) == pytest.approx(5781.0, abs=1.0)
    assert L.amgr_speedup_percent(1.235 + 2.893, 0.021 + 3.132) == pytest.approx(31.0, abs=1.0)
    assert L.amgr_speedup_percent(1.235 + 2.893, 0.423 + 2.794) == pytest.approx(28.0, abs=1.0)
    assert L.amgr_speedup_percent(2.0, 2.0) == 0.0
    assert math.isinf(L.amgr_speedup_percent(1.0, 0.0))


class HostSeq:
    def __init__(self, mats, rhs):
        self.mats, self.rhs = mats, rhs

    def size(self):
        return len(self.mats)

    def step(self, k):
        return self.mats[k], self.rhs[k] if isinstance(self.rhs, list) else self.rhs


def dambreak_seq(g, ks):
    return HostSeq([P.grid3d_values("dambreak", g, k) for k in ks], P.rhs(g ** 3))


@pytest.mark.gpu
@pytest.mark.parametrize("kind,extra", [("none", {}), ("partial", {}), ("partial", {"rebuild_every": 2}),
                                        ("full", {}), ("full", {"reuse_iter_limit": 10})])
def test_run_sequence_matches_oracle(ctx, kind, extra):
    import paper_2108_02054_b200 as amg
    from paper_2108_02054_b200 import reuse as R
    from oracle import reuse_oracle as RO

    seq = dambreak_seq(14, [0, 10, 20, 30, 40, 49])
    st = R.StrategyConfig(R.StrategyKind[kind], extra.get("reuse_iter_limit", 0), extra.get("rebuild_every"))
    res = R.run_sequence(seq, st, ctx=ctx)
    ref = RO.run_sequence(seq, kind, extra.get("reuse_iter_limit", 0), extra.get("rebuild_every"))
    assert [int(s.action) for s in res.report.steps] == [r[0] for r in ref]
    for s, r in zip(res.report.steps, ref):
        assert abs(s.iterations - r[1]) <= 1 and s.converged == r[2]
    # the reference solves with the hierarchy's finest matrix (reuse.cpp:104): under
    # full reuse that is the matrix of the last full build, not A_k
    A_solved = None
    for u, s, k in zip(res.solutions, res.report.steps, range(6)):
        if s.action != R.StepAction.reused_unchanged:
            A_solved = seq.mats[k]
        res_true = np.linalg.norm(seq.rhs - P_spmv(A_solved, u)) / np.linalg.norm(seq.rhs)
        assert res_true <= 1e-8
    rep = res.report
    assert rep.full_rebuilds == sum(1 for s in rep.steps if s.action == R.StepAction.full_build)
    assert rep.avg_iterations == pytest.approx(np.mean([s.iterations for s in rep.steps]))
    if kind == "none":
        assert rep.full_rebuilds == 6
    if kind == "partial" and not extra:
        assert rep.full_rebuilds == 1
        assert all(s.phase_timings.transfer_ops == 0.0 for s in rep.steps[1:])


def P_spmv(A, x):
    from oracle import ref

    return ref.spmv(A, x)


@pytest.mark.gpu
def test_constant_sequence_partial_identical_iterations(ctx):
    from paper_2108_02054_b200 import reuse as R

    A = P.grid3d_values("dambreak", 12, 5)
    f = P.rhs(12 ** 3)
    seq = HostSeq([A] * 4, [f, f * 1.5, f * 0.5, f])  # fresh solves: vary the RHS
    res = R.run_sequence(seq, R.StrategyConfig(R.StrategyKind.partial), ctx=ctx)
    assert [s.action for s in res.report.steps] == [R.StepAction.full_build] + [R.StepAction.partial_update] * 3
    res_full = R.run_sequence(seq, R.StrategyConfig(R.StrategyKind.full, reuse_iter_limit=100), ctx=ctx)
    assert res_full.report.full_rebuilds == 1


@pytest.mark.gpu
def test_dimension_change_falls_back_to_full_build(ctx):
    from paper_2108_02054_b200 import reuse as R

    seq = HostSeq([P.grid3d_values("poisson", 10, 0), P.grid3d_values("poisson", 11, 1),
                   P.grid3d_values("poisson", 11, 2)], None)
    seq.rhs = None

    class S(HostSeq):
        def step(self, k):
            A = self.mats[k]
            return A, P.rhs(len(A[0]) - 1)

    s = S(seq.mats, None)
    res = R.run_sequence(s, R.StrategyConfig(R.StrategyKind.partial), ctx=ctx)
    assert [s_.action for s_ in res.report.steps] == [R.StepAction.full_build, R.StepAction.full_build,
                                                      R.StepAction.partial_update]


@pytest.mark.gpu
def test_device_generated_sequence(ctx):
    from paper_2108_02054_b200 import reuse as R

    seq = R.DeviceGridSequence("dambreak", 24, 4, ctx=ctx)
    res = R.run_sequence(seq, R.StrategyConfig(R.StrategyKind.partial), ctx=ctx, keep_solutions=False)
    assert res.report.full_rebuilds == 1 and all(s.converged for s in res.report.steps)
    base = R.run_sequence(seq, R.StrategyConfig(R.StrategyKind.none), ctx=ctx, keep_solutions=False)
    assert base.report.full_rebuilds == 4
    assert R.speedup_percent(base.report, res.report, R.SpeedupBasis.setup) > 0.0


def test_file_sequence_directory_rules(tmp_path):
    """read_sequence (matrix_market.cpp:225-256): directory scan, gaps, missing
    files — host logic, no device needed."""
    from paper_2108_02054_b200 import RuntimeFailure
    from paper_2108_02054_b200 import reuse as R

    with pytest.raises(RuntimeFailure, match="not a directory"):
        R.FileSequence(tmp_path / "nope")
    with pytest.raises(RuntimeFailure, match="no step_NNNN.mtx files"):
        R.FileSequence(tmp_path)
    for k in (3, 4, 6):
        (tmp_path / f"step_{k:04d}.mtx").write_text("x")
    with pytest.raises(RuntimeFailure, match="gap in step numbering, expected step 5 but found step 6"):
        R.FileSequence(tmp_path)
    (tmp_path / "step_0006.mtx").unlink()
    (tmp_path / "step_0004.rhs.mtx").write_text("x")
    (tmp_path / "notes.txt").write_text("x")
    s = R.FileSequence(tmp_path)
    assert s.size() == 2 and s.rhs[0] is None and s.rhs[1].endswith("step_0004.rhs.mtx")


def _synthetic_outcomes():
    """Three strategies x 4 steps of made-up timings (inf speedup for the
    setup-free full reuse, sub-microsecond and large values)."""
    from paper_2108_02054_b200 import PhaseTimings
    from paper_2108_02054_b200 import reuse as R

    rng = np.random.default_rng(5)
    spec = {R.StrategyKind.none: [0, 0, 0, 0], R.StrategyKind.full: [0, 2, 2, 2],
            R.StrategyKind.partial: [0, 1, 1, 0]}
    outcomes, raw = [], []
    for kind, acts in spec.items():
        steps, rrow = [], []
        for k, a in enumerate(acts):
            setup = 0.0 if a == 2 else float(rng.uniform(1e-4, 3.0))
            solve = float(rng.uniform(1e-7, 40.0))
            it = int(rng.integers(1, 101))
            conv = bool(rng.integers(0, 2))
            ph = [float(x) for x in rng.uniform(0, 1.0, 4)] if a == 0 else [0.0, float(rng.uniform(0, 1)),
                                                                              float(rng.uniform(0, 1)), 1e-6]
            steps.append(R.StepMetrics(k, setup, solve, it, conv, R.StepAction(a), PhaseTimings(*ph)))
            rrow.append((a, setup, solve, it, int(conv), ph))
        rep = R.RunReport(strategy=R.StrategyConfig(kind), steps=steps)
        rep.total_setup = sum(s.setup_time for s in steps)
        rep.total_solve = sum(s.solve_time for s in steps)
        rep.full_rebuilds = sum(1 for s in steps if s.action == R.StepAction.full_build)
        rep.avg_iterations = sum(s.iterations for s in steps) / len(steps)
        outcomes.append(R.StrategyOutcome(kind, [rep], rep))
        raw.append(rrow)
    return outcomes, raw


@pytest.mark.parametrize("fmt", ["markdown", "csv"])
def test_report_renderer_matches_reference_bench_app(fmt):
    """Table-1/Table-2-style report and per-step CSV (tools/bench_app.cpp:129-281)
    are byte-identical to the unmodified reference's renderers on the same run data."""
    from oracle import ref
    from paper_2108_02054_b200 import AmgParams, SolveParams
    from paper_2108_02054_b200 import reuse as R

    if not ref.available():
        pytest.skip("oracle/_ref not built")
    outcomes, raw = _synthetic_outcomes()
    amg = AmgParams(eps=0.08, omega=0.72, coarse_enough=100)
    sp = SolveParams(tol=1e-8, max_iter=100)
    for rie, rbe in ((0, None), (25, 3)):
        mine = R.render_report(outcomes, fmt, source="sequence directory /data/seq", amg=amg, solve=sp,
                               reuse_iter_limit=rie, rebuild_every=rbe)
        theirs = ref.render(0, 0 if fmt == "markdown" else 1, "/data/seq",
                            (0.08, 0.72, 1, 1, 100), (1e-8, 100), rie, rbe, [int(o.kind) for o in outcomes], raw)
        assert mine == theirs
    assert R.per_step_csv(outcomes) == ref.render(1, 0, "/data/seq", (0.08, 0.72, 1, 1, 100), (1e-8, 100), 0, None,
                                                  [int(o.kind) for o in outcomes], raw)
    assert R.effective_strategies([R.StrategyKind.partial, R.StrategyKind.partial]) == [R.StrategyKind.none,
                                                                                       R.StrategyKind.partial]


@pytest.mark.gpu
def test_bench_app_cli_on_device(tmp_path, capsys):
    """The reuse benchmark CLI end to end on the device (3 strategies over a
    generated sequence): report + per-step CSV with one row per step."""
    from paper_2108_02054_b200 import bench_app

    per = tmp_path / "steps.csv"
    assert bench_app.main(["--generate", "dambreak", "--grid", "16", "--steps", "3", "--per-step", str(per)]) == 0
    out = capsys.readouterr().out
    assert out.startswith("# AMG setup reuse benchmark") and "| Partial reuse |" in out
    assert len(per.read_text().strip().splitlines()) == 1 + 3 * 3


@pytest.mark.gpu
def test_partial_reuse_escalation_matches_restated_rule(ctx):
    """Extension: partial reuse with convergence-triggered
    escalation — a solve that needed >= reuse_iter_limit iterations makes the
    next step a full build (the reference's full-reuse rule, reuse.cpp:116-117,
    applied to partial reuse); actions match the restated driver."""
    from oracle import reuse_oracle as RO
    from paper_2108_02054_b200 import reuse as R

    seq = dambreak_seq(14, [0, 1, 49, 0, 1, 49])
    st = R.StrategyConfig(R.StrategyKind.partial, reuse_iter_limit=1, escalate=True)
    res = R.run_sequence(seq, st, ctx=ctx)
    ref = RO.run_sequence(seq, "partial", 1, escalate=True)
    assert [int(s.action) for s in res.report.steps] == [r[0] for r in ref]
    assert 1 < res.report.full_rebuilds < len(ref)  # escalated, but not every step
    plain = R.run_sequence(seq, R.StrategyConfig(R.StrategyKind.partial), ctx=ctx)
    assert plain.report.full_rebuilds == 1
