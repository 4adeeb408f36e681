"""run_sequence at g^3 dam-break for one strategy, printing per-step setup and
solve times (setup/alloc traces via AMGR_TRACE_SETUP / AMGR_TRACE_ALLOC).
usage: python tools/strategy_probe.py [g] [strategy] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_02054_b200 as amg  # noqa: E402
from paper_2108_02054_b200 import reuse as R  # noqa: E402

g = int(sys.argv[1]) if len(sys.argv) > 1 else 256
kind = sys.argv[2] if len(sys.argv) > 2 else "none"
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
ctx = amg.Context(0)
seq = R.DeviceGridSequence("dambreak", g, steps, ctx=ctx)
res = R.run_sequence(seq, R.StrategyConfig(R.StrategyKind[kind]), amg.AmgParams(coarse_solve="inverse"),
                     amg.SolveParams(), ctx=ctx, keep_solutions=False)
for s in res.report.steps:
    print(f"step {s.step}: setup {1e3 * s.setup_time:.1f} ms solve {1e3 * s.solve_time:.1f} ms its {s.iterations} "
          f"{s.action} {s.phase_timings}", flush=True)
