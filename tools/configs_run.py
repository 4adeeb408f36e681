"""BASELINE.json configs other than the bench's C3, run on one B200 through
the library (they are parity / coverage cases, not bench lines):

  C1  Poisson 32^3 with a time-varying shift, smoothed aggregation + Jacobi,
      CG, 10 steps of partial reuse; iterations against the restated oracle
  C2  moving-blob diffusion 128^3, SPAI0, none / full / partial over 20 steps
      (run_sequence)
  C5  convection-diffusion 200^3 (nonsymmetric), Chebyshev smoother,
      BiCGStab, partial reuse over 20 steps (run_sequence)

usage: python tools/configs_run.py [C1 C2 C5] > gpurun_out/configs.json"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_02054_b200 as amg  # noqa: E402
from paper_2108_02054_b200 import reuse as R  # noqa: E402


def strategy_summary(res):
    st = res.report.steps
    return {"setup_s": res.report.total_setup, "solve_s": res.report.total_solve,
            "full_rebuilds": res.report.full_rebuilds, "avg_iterations": res.report.avg_iterations,
            "iterations": [s.iterations for s in st], "converged": all(s.converged for s in st)}


def c1(ctx):
    from oracle import oracle as O
    from oracle import problems as P

    g, steps = 32, 10
    prm = amg.AmgParams(coarsening="smoothed")
    f = P.rhs(g ** 3)
    mats = [P.grid3d_values("poisson", g, k, steps) for k in range(steps)]
    h = amg.setup(mats[0], prm, ctx=ctx)
    o = O.setup(mats[0], O.params(coarsening="smoothed"))
    u = np.zeros(g ** 3)
    uo = np.zeros(g ** 3)
    its, its_o, t = [], [], []
    for k in range(steps):
        t0 = time.perf_counter()
        if k:
            h = amg.partial_update(h, mats[k], prm)
        u, st = amg.cg(h, f, u)
        t.append(time.perf_counter() - t0)
        if k:
            o = O.partial_update(o, mats[k], O.params(coarsening="smoothed"))
        so = O.cg(o, f, uo)
        uo = so.u
        its.append(st.iterations)
        its_o.append(so.iterations)
    return {"config": "C1 Poisson 32^3, SA + Jacobi, CG, 10 partial-reuse steps", "iterations": its,
            "oracle_iterations": its_o, "host_wall_s_per_step": float(np.mean(t[1:])),
            "max_abs_diff_last_solution": float(np.max(np.abs(u - uo)))}


def c2(ctx):
    out = {"config": "C2 moving-blob 128^3, SPAI0, 20 steps"}
    prm = amg.AmgParams(smoother="spai0")
    for kind in ("none", "full", "partial"):
        seq = R.DeviceGridSequence("blob", 128, 20, ctx=ctx)
        res = R.run_sequence(seq, R.StrategyConfig(R.StrategyKind[kind]), prm, amg.SolveParams(), ctx=ctx,
                             keep_solutions=False)
        out[kind] = strategy_summary(res)
        del seq
    return out


def c5(ctx):
    prm = amg.AmgParams(smoother="chebyshev")
    seq = R.DeviceGridSequence("convdiff", 200, 20, ctx=ctx)
    res = R.run_sequence(seq, R.StrategyConfig(R.StrategyKind.partial), prm, amg.SolveParams(), ctx=ctx,
                         keep_solutions=False)
    out = {"config": "C5 convection-diffusion 200^3, Chebyshev(3, [0.3, 1.1] x lambda_max), BiCGStab, "
                     "partial reuse, 20 steps", "partial": strategy_summary(res)}
    prmj = amg.AmgParams()
    res = R.run_sequence(seq, R.StrategyConfig(R.StrategyKind.partial), prmj, amg.SolveParams(), ctx=ctx,
                         keep_solutions=False)
    out["partial_jacobi_for_comparison"] = strategy_summary(res)
    return out


if __name__ == "__main__":
    which = sys.argv[1:] or ["C1", "C2", "C5"]
    ctx = amg.Context(0)
    res = {}
    for w in which:
        res[w] = {"C1": c1, "C2": c2, "C5": c5}[w](ctx)
        print(json.dumps({w: res[w]}), flush=True)
