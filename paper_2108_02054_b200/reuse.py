"""Reuse driver — mirror of the reference's run_sequence / RunReport API
(proj/include/amgreuse/reuse.hpp:13-81, proj/src/reuse.cpp) over
`amgr_run_sequence`.  The per-step loop (action choice, setup / in-place
partial update, BiCGStab from the previous solution, the full-reuse rebuild
flag) runs in the library's C++; Python only adapts the problem sequence.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field

import numpy as np

from . import (AmgParams, Context, CsrMatrix, DeviceCsr, InvalidArgument, PhaseTimings, SolveParams, _check,
               _Csr, _SolveParams, _Timings, default_context, lib)


class StrategyKind(enum.IntEnum):
    """reuse.hpp:13"""
    none = 0
    full = 1
    partial = 2


def strategy_kind_from_string(name: str) -> StrategyKind:
    """reuse.cpp:31-36"""
    try:
        return StrategyKind[name]
    except KeyError:
        raise InvalidArgument(f"unknown strategy '{name}' (expected none, full or partial)") from None


class StepAction(enum.IntEnum):
    """reuse.hpp:31"""
    full_build = 0
    partial_update = 1
    reused_unchanged = 2


@dataclass
class StrategyConfig:
    """reuse.hpp:20-28.  escalate (extension): partial reuse
    falls back to a full build after a solve that did not converge or used
    >= reuse_iter_limit iterations (the reference's full-reuse rule)."""
    kind: StrategyKind = StrategyKind.none
    reuse_iter_limit: int = 0
    rebuild_every: int | None = None
    escalate: bool = False


@dataclass
class StepMetrics:
    """reuse.hpp:33-41"""
    step: int
    setup_time: float
    solve_time: float
    iterations: int
    converged: bool
    action: StepAction
    phase_timings: PhaseTimings


@dataclass
class RunReport:
    """reuse.hpp:43-50"""
    strategy: StrategyConfig
    steps: list = field(default_factory=list)
    total_setup: float = 0.0
    total_solve: float = 0.0
    full_rebuilds: int = 0
    avg_iterations: float = 0.0


@dataclass
class RunResult:
    solutions: list
    report: RunReport


class _Strategy(C.Structure):
    _fields_ = [("kind", C.c_int32), ("flags", C.c_int32), ("reuse_iter_limit", C.c_int64),
                ("rebuild_every", C.c_int64)]


class _StepMetrics(C.Structure):
    _fields_ = [("step", C.c_int64), ("setup_time", C.c_double), ("solve_time", C.c_double),
                ("iterations", C.c_int64), ("converged", C.c_int32), ("action", C.c_int32),
                ("phase_timings", _Timings)]


STEP_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.POINTER(_Csr), C.POINTER(C.c_void_p), C.POINTER(C.c_int32))
SINK_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64)


def run_sequence(systems, strategy: StrategyConfig, amg: AmgParams | None = None, solve: SolveParams | None = None,
                 ctx: Context | None = None, keep_solutions: bool = True) -> RunResult:
    """RunResult run_sequence(const ProblemSequence&, const StrategyConfig&,
    const AmgParams&, const SolveParams&) — reuse.hpp:70-71.

    `systems` needs size() and step(k) -> (A, rhs); A is a host CSR tuple /
    CsrMatrix or a DeviceCsr, rhs a numpy array or a device pointer (int)."""
    ctx = ctx or default_context()
    amg = amg or AmgParams()
    solve = solve or SolveParams()
    if strategy.rebuild_every is not None and strategy.rebuild_every < 1:
        raise InvalidArgument("run_sequence: rebuild_every must be >= 1")
    n_steps = systems.size()
    keep = {}
    solutions = []
    errors = []

    def step_cb(_user, k, a_out, rhs_out, loc_out):
        try:
            A, rhs = systems.step(int(k))
            A = A if isinstance(A, DeviceCsr) else CsrMatrix.of(A)
            if isinstance(rhs, int):
                rhs_ptr, loc = rhs, 1
            else:
                rhs = np.ascontiguousarray(rhs, np.float64)
                if len(rhs) != A.nrows:
                    raise InvalidArgument("run_sequence: RHS length does not match matrix size")
                rhs_ptr, loc = rhs.ctypes.data, 0
            keep["A"], keep["rhs"] = A, rhs
            a_out[0] = A._c()
            rhs_out[0] = rhs_ptr
            loc_out[0] = loc
            return 0
        except Exception as e:  # surfaced after the call
            errors.append(e)
            return 1

    def sink_cb(_user, k, u_dev, n):
        host = np.empty(int(n))
        _check(lib().amgr_copy_to_host(ctx.ptr, host.ctypes.data, u_dev, 8 * int(n)), ctx.ptr)
        solutions.append(host)

    step_fn = STEP_FN(step_cb)
    sink_fn = SINK_FN(sink_cb) if keep_solutions else SINK_FN()
    st = _Strategy(int(strategy.kind), 1 if strategy.escalate else 0, strategy.reuse_iter_limit,
                   strategy.rebuild_every if strategy.rebuild_every is not None else 0)
    metrics = (_StepMetrics * n_steps)()
    p = amg._c()
    sp = _SolveParams(solve.tol, solve.max_iter)
    rc = lib().amgr_run_sequence(ctx.ptr, n_steps, step_fn, None, C.byref(st), C.byref(p), C.byref(sp), metrics,
                                 sink_fn, None)
    if errors:
        raise errors[0]
    _check(rc, ctx.ptr)
    rep = RunReport(strategy=strategy)
    for m in metrics:
        pt = m.phase_timings
        rep.steps.append(StepMetrics(int(m.step), m.setup_time, m.solve_time, int(m.iterations), bool(m.converged),
                                     StepAction(m.action),
                                     PhaseTimings(pt.transfer_ops, pt.galerkin, pt.smoother, pt.coarse_solver)))
    # totals (reuse.cpp:126-134)
    rep.total_setup = sum(s.setup_time for s in rep.steps)
    rep.total_solve = sum(s.solve_time for s in rep.steps)
    rep.full_rebuilds = sum(1 for s in rep.steps if s.action == StepAction.full_build)
    rep.avg_iterations = sum(s.iterations for s in rep.steps) / len(rep.steps)
    return RunResult(solutions, rep)


class SpeedupBasis(enum.IntEnum):
    total = 0
    setup = 1


def speedup_percent(base: RunReport, other: RunReport, which: SpeedupBasis = SpeedupBasis.total) -> float:
    """reuse.cpp:138-147: (t_base / t_other - 1) * 100, +inf when t_other == 0."""
    if len(base.steps) != len(other.steps):
        raise InvalidArgument("speedup_percent: reports cover different step counts")
    tb = base.total_setup + (base.total_solve if which == SpeedupBasis.total else 0.0)
    to = other.total_setup + (other.total_solve if which == SpeedupBasis.total else 0.0)
    return float(lib().amgr_speedup_percent(tb, to))


def speedup_from_times(t_base: float, t_other: float) -> float:
    return math.inf if t_other == 0.0 else (t_base / t_other - 1.0) * 100.0


def full_build_phase_totals(report: RunReport) -> PhaseTimings:
    """reuse.cpp:149-154"""
    t = PhaseTimings()
    for s in report.steps:
        if s.action == StepAction.full_build:
            t.transfer_ops += s.phase_timings.transfer_ops
            t.galerkin += s.phase_timings.galerkin
            t.smoother += s.phase_timings.smoother
            t.coarse_solver += s.phase_timings.coarse_solver
    return t


class DeviceGridSequence:
    """ProblemSequence (sequence.hpp:17-23) generated on the device: the 3D
    synthetic sequences of SURVEY.md 8(d) (poisson / blob / dambreak /
    convdiff), fixed RHS U(0.1, 1) from std::mt19937_64(seed).

    `steps` systems are served; with `total` and `first` they are the window
    first .. first+steps-1 of a `total`-step sequence (e.g. steps 0..5 of the
    50-step C3 dam-break sequence)."""

    def __init__(self, kind: str, g: int, steps: int, seed: int = 42, ctx: Context | None = None,
                 total: int | None = None, first: int = 0):
        import torch

        from . import DEVICE, PROBLEM

        self.ctx = ctx or default_context()
        self.kind, self.g, self.steps = PROBLEM[kind], g, steps
        self.total, self.first = (total or steps), first
        if first < 0 or first + steps > self.total:
            raise ValueError("DeviceGridSequence: window outside the sequence")
        L = lib()
        n, nnz = g ** 3, int(L.amgr_problem_nnz(g))
        self.n, self.nnz = n, nnz
        dev = torch.device("cuda", self.ctx.device)
        self.rp = torch.empty(n + 1, dtype=torch.int32, device=dev)
        self.ci = torch.empty(nnz + 8, dtype=torch.int32, device=dev)
        self.v = torch.empty(nnz + 8, dtype=torch.float64, device=dev)
        self.f = torch.empty(n, dtype=torch.float64, device=dev)
        torch.cuda.synchronize()
        _check(L.amgr_problem_pattern(self.ctx.ptr, g, self.rp.data_ptr(), self.ci.data_ptr()), self.ctx.ptr)
        _check(L.amgr_problem_rhs(self.ctx.ptr, n, seed, self.f.data_ptr(), DEVICE), self.ctx.ptr)
        self.ctx.synchronize()

    def size(self) -> int:
        return self.steps

    def step(self, k: int):
        L = lib()
        _check(L.amgr_problem_values(self.ctx.ptr, self.kind, self.g, self.first + k, self.total, self.v.data_ptr()),
               self.ctx.ptr)
        self.ctx.synchronize()
        return DeviceCsr(self.n, self.n, self.nnz, self.rp.data_ptr(), self.ci.data_ptr(), self.v.data_ptr()), \
            self.f.data_ptr()


class FileSequence:
    """FileSequence / read_sequence (matrix_market.hpp:29-47,
    matrix_market.cpp:205-256): `step_NNNN.mtx` (+ optional `step_NNNN.rhs.mtx`,
    else an RHS of ones) in one directory, read lazily in index order; the
    matrices are assembled on the device (mm_read)."""

    def __init__(self, directory, ctx: Context | None = None):
        import os
        import re

        from . import RuntimeFailure

        self.ctx = ctx  # resolved lazily: the directory scan needs no device
        d = os.fspath(directory)
        if not os.path.isdir(d):
            raise RuntimeFailure("read_sequence: not a directory: " + d)
        mats, rhs = {}, {}
        for name in os.listdir(d):
            path = os.path.join(d, name)
            if not os.path.isfile(path):
                continue
            m = re.match(r"^step_(\d{1,4})(.{1,15})$", name)  # sscanf("step_%4ld%15s")
            if not m:
                continue
            idx, tail = int(m.group(1)), m.group(2)
            if tail == ".mtx":
                mats[idx] = path
            elif tail == ".rhs.mtx":
                rhs[idx] = path
        if not mats:
            raise RuntimeFailure("read_sequence: no step_NNNN.mtx files in " + d)
        self.mats, self.rhs = [], []
        expected = min(mats)
        for idx in sorted(mats):
            if idx != expected:
                raise RuntimeFailure(f"read_sequence: gap in step numbering, expected step {expected} but found "
                                     f"step {idx}")
            expected += 1
            self.mats.append(mats[idx])
            self.rhs.append(rhs.get(idx))
        self._keep = None

    def size(self) -> int:
        return len(self.mats)

    def step(self, k: int):
        from . import RuntimeFailure, mm_read, mm_read_vector

        if k >= self.size():
            raise IndexError("FileSequence::step: index out of range")
        ctx = self.ctx or default_context()
        M = mm_read(self.mats[k], ctx)
        if self.rhs[k] is None:
            f = np.ones(M.nrows)
        else:
            f = mm_read_vector(self.rhs[k], ctx)
            if len(f) != M.nrows:
                raise RuntimeFailure(f"step {k}: RHS length {len(f)} does not match matrix size {M.nrows} "
                                     f"({self.rhs[k]})")
        self._keep = M  # the device CSR must outlive the driver's use of this step
        return M.device_csr(), f


# ---- benchmark driver and report (tools/bench_app.cpp) -----------------------------
@dataclass
class StrategyOutcome:
    """bench_app.hpp:36-41: all runs of one strategy and the per-cell median."""
    kind: StrategyKind
    runs: list
    median: RunReport


def _median(v):
    v = sorted(v)
    n = len(v)
    return v[n // 2] if n % 2 == 1 else 0.5 * (v[n // 2 - 1] + v[n // 2])


def median_report(runs) -> RunReport:
    """bench_app.cpp:24-40"""
    import copy

    out = copy.deepcopy(runs[0])
    if len(runs) == 1:
        return out
    for s in range(len(out.steps)):
        out.steps[s].setup_time = _median([r.steps[s].setup_time for r in runs])
        out.steps[s].solve_time = _median([r.steps[s].solve_time for r in runs])
    out.total_setup = _median([r.total_setup for r in runs])
    out.total_solve = _median([r.total_solve for r in runs])
    return out


def effective_strategies(kinds) -> list:
    """bench_app.cpp:83-93: `none` is the implicit speedup baseline."""
    out = []
    if any(k != StrategyKind.none for k in kinds):
        out.append(StrategyKind.none)
    for k in kinds:
        if k not in out:
            out.append(k)
    return out


def run_benchmark(systems, kinds=(StrategyKind.none, StrategyKind.full, StrategyKind.partial),
                  amg: AmgParams | None = None, solve: SolveParams | None = None, reuse_iter_limit: int = 0,
                  rebuild_every: int | None = None, repeat: int = 1, ctx: Context | None = None) -> list:
    """run_benchmark (bench_app.cpp:223-246): every strategy `repeat` times over
    the same sequence on the device; rebuild_every applies to `partial`."""
    if not kinds:
        raise InvalidArgument("at least one strategy is required")
    if repeat < 1:
        raise InvalidArgument("--repeat must be >= 1")
    outcomes = []
    for k in effective_strategies(list(kinds)):
        cfg = StrategyConfig(k, reuse_iter_limit, rebuild_every if k == StrategyKind.partial else None)
        runs = [run_sequence(systems, cfg, amg, solve, ctx=ctx, keep_solutions=False).report for _ in range(repeat)]
        outcomes.append(StrategyOutcome(k, runs, median_report(runs)))
    return outcomes


_DISPLAY = {StrategyKind.none: "No reuse", StrategyKind.full: "Full reuse", StrategyKind.partial: "Partial reuse"}
_ACTION = {StepAction.full_build: "full_build", StepAction.partial_update: "partial_update",
           StepAction.reused_unchanged: "reused_unchanged"}


def _fmt_speedup(p: float) -> str:
    if math.isinf(p):
        return "inf" if p > 0 else "-inf"
    return f"{p:.0f}"


def _header(p: str, amg: AmgParams, solve: SolveParams, source: str, reuse_iter_limit: int,
            rebuild_every: int | None, repeat: int, parallel: bool) -> str:
    """render_header (bench_app.cpp:98-126)"""
    s = f"{p}source: {source}\n"
    s += (f"{p}amg: eps {amg.eps:g}, omega {amg.omega:g}, sweeps {amg.pre_sweeps}+{amg.post_sweeps}, "
          f"coarse_enough {amg.coarse_enough}\n")
    s += f"{p}solver: bicgstab, tol {solve.tol:g}, max_iter {solve.max_iter}"
    if reuse_iter_limit > 0:
        s += f", reuse_iter_limit {reuse_iter_limit}"
    if rebuild_every:
        s += f", rebuild_every {rebuild_every}"
    s += "\n"
    if repeat > 1:
        s += f"{p}repeat: {repeat} (per-cell medians)\n"
    if parallel:
        s += f"{p}timings: contended (strategies ran in parallel)\n"
    return s


def render_report(outcomes, fmt: str = "markdown", source: str = "", amg: AmgParams | None = None,
                  solve: SolveParams | None = None, reuse_iter_limit: int = 0, rebuild_every: int | None = None,
                  repeat: int = 1, parallel: bool = False) -> str:
    """render_report (bench_app.cpp:248-266): Table-1-style strategy comparison
    (setup, solve, rebuilds, iterations, speedups vs `none`) and the Table-2-style
    setup-phase breakdown of the full builds; markdown or csv.  `source` is the
    header's source description, e.g. "sequence directory <dir>"."""
    amg = amg or AmgParams()
    solve = solve or SolveParams()
    base = next((o.median for o in outcomes if o.kind == StrategyKind.none), None)
    speedups = base is not None and len(outcomes) > 1
    # breakdown (bench_app.cpp:176-206): the last `none` outcome, else the first
    pick = outcomes[0]
    for o in outcomes:
        if o.kind == StrategyKind.none:
            pick = o
    t = full_build_phase_totals(pick.median)
    rows = [("Transfer operators", t.transfer_ops), ("Galerkin operator", t.galerkin), ("Smoother", t.smoother),
            ("Direct solver for the coarsest system", t.coarse_solver)]
    total = sum(x for _, x in rows) or 1.0
    s = ""
    if fmt == "markdown":
        s += "# AMG setup reuse benchmark\n\n"
        s += _header("- ", amg, solve, source, reuse_iter_limit, rebuild_every, repeat, parallel)
        s += "\n## Strategy comparison\n\n"
        s += "| Strategy | Setup (s) | Solve (s) | Rebuilds | Average iterations |"
        if speedups:
            s += " Total speedup (%) | Setup speedup (%) |"
        s += "\n|---|---|---|---|---|" + ("---|---|" if speedups else "") + "\n"
        for o in outcomes:
            r = o.median
            s += (f"| {_DISPLAY[o.kind]} | {r.total_setup:.3f} | {r.total_solve:.3f} | {r.full_rebuilds} | "
                  f"{r.avg_iterations:.1f} |")
            if speedups:
                if o.kind == StrategyKind.none:
                    s += "  |  |"
                else:
                    s += (f" {_fmt_speedup(speedup_percent(base, r, SpeedupBasis.total))} | "
                          f"{_fmt_speedup(speedup_percent(base, r, SpeedupBasis.setup))} |")
            s += "\n"
        s += "\n## Setup phase breakdown (full builds)\n\n"
        s += "| Setup phase | Share (%) |\n|---|---|\n"
        for label, x in rows:
            s += f"| {label} | {100.0 * x / total:.1f} |\n"
    else:
        s += _header("# ", amg, solve, source, reuse_iter_limit, rebuild_every, repeat, parallel)
        s += "strategy,setup_s,solve_s,rebuilds,avg_iterations"
        if speedups:
            s += ",total_speedup_pct,setup_speedup_pct"
        s += "\n"
        for o in outcomes:
            r = o.median
            s += f"{o.kind.name},{r.total_setup:.3f},{r.total_solve:.3f},{r.full_rebuilds},{r.avg_iterations:.1f}"
            if speedups:
                if o.kind == StrategyKind.none:
                    s += ",,"
                else:
                    s += (f",{_fmt_speedup(speedup_percent(base, r, SpeedupBasis.total))},"
                          f"{_fmt_speedup(speedup_percent(base, r, SpeedupBasis.setup))}")
            s += "\n"
        s += "\nsetup_phase,share_pct\n"
        for label, x in rows:
            s += f'"{label}",{100.0 * x / total:.1f}\n'
    return s


def per_step_csv(outcomes) -> str:
    """write_per_step_csv (bench_app.cpp:268-281)"""
    s = ("strategy,step,action,setup_s,solve_s,iterations,converged,"
         "transfer_ops_s,galerkin_s,smoother_s,coarse_solver_s\n")
    for o in outcomes:
        for m in o.median.steps:
            p = m.phase_timings
            s += (f"{o.kind.name},{m.step},{_ACTION[m.action]},{m.setup_time:.9g},{m.solve_time:.9g},"
                  f"{m.iterations},{1 if m.converged else 0},{p.transfer_ops:.9g},{p.galerkin:.9g},"
                  f"{p.smoother:.9g},{p.coarse_solver:.9g}\n")
    return s
