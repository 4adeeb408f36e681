"""Command-line reuse benchmark (the reference's tools/amg_bench.cpp +
bench_app.cpp) on the device: runs the strategies over a sequence with the
library's run_sequence and prints the Table-1/Table-2 report (markdown or
csv), optionally the per-step CSV.

  python -m paper_2108_02054_b200.bench_app --sequence DIR
  python -m paper_2108_02054_b200.bench_app --generate dambreak --grid 64 --steps 10

--sequence reads step_NNNN.mtx files (FileSequence); --generate uses the
device 3D generators (poisson / blob / dambreak / convdiff; the reference's
2D diffusion generator is not ported)."""
from __future__ import annotations

import argparse
import sys

from . import AmgParams, SolveParams
from . import reuse as R


def main(argv=None) -> int:
    a = argparse.ArgumentParser(prog="amg_bench")
    src = a.add_mutually_exclusive_group(required=True)
    src.add_argument("--sequence")
    src.add_argument("--generate", choices=["poisson", "blob", "dambreak", "convdiff"])
    a.add_argument("--grid", type=int, default=64)
    a.add_argument("--steps", type=int, default=10)
    a.add_argument("--seed", type=int, default=42)
    a.add_argument("--strategies", default="none,full,partial")
    a.add_argument("--eps", type=float, default=0.08)
    a.add_argument("--omega", type=float, default=0.72)
    a.add_argument("--pre-sweeps", type=int, default=1)
    a.add_argument("--post-sweeps", type=int, default=1)
    a.add_argument("--coarse-enough", type=int, default=100)
    a.add_argument("--max-direct-size", type=int, default=2000)
    a.add_argument("--tol", type=float, default=1e-8)
    a.add_argument("--max-iter", type=int, default=100)
    a.add_argument("--reuse-iter-limit", type=int, default=0)
    a.add_argument("--rebuild-every", type=int)
    a.add_argument("--format", choices=["markdown", "csv"], default="markdown")
    a.add_argument("--output")
    a.add_argument("--per-step")
    a.add_argument("--repeat", type=int, default=1)
    x = a.parse_args(argv)
    kinds = [R.strategy_kind_from_string(s) for s in x.strategies.split(",")]
    amg = AmgParams(eps=x.eps, omega=x.omega, pre_sweeps=x.pre_sweeps, post_sweeps=x.post_sweeps,
                    coarse_enough=x.coarse_enough, max_direct_size=x.max_direct_size)
    sp = SolveParams(tol=x.tol, max_iter=x.max_iter)
    if x.sequence:
        seq = R.FileSequence(x.sequence)
        source = f"sequence directory {x.sequence}"
    else:
        seq = R.DeviceGridSequence(x.generate, x.grid, x.steps, seed=x.seed)
        source = f"generated 3D {x.generate} sequence (device), grid {x.grid}^3, steps {x.steps}, seed {x.seed}"
    outcomes = R.run_benchmark(seq, kinds, amg, sp, x.reuse_iter_limit, x.rebuild_every, x.repeat)
    text = R.render_report(outcomes, x.format, source, amg, sp, x.reuse_iter_limit, x.rebuild_every, x.repeat)
    if x.output:
        open(x.output, "w").write(text)
    else:
        sys.stdout.write(text)
    if x.per_step:
        open(x.per_step, "w").write(R.per_step_csv(outcomes))
    return 0


if __name__ == "__main__":
    sys.exit(main())
