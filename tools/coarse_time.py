"""Development probe: per-call device time of the coarse solve (probe family
"coarse_solve") and the coarse factorization ("coarse") at g^3 dam-break in
the exact mode, for the kernels selected by an environment knob read per
call.  usage: python tools/coarse_time.py g [VAR v1 v2 ...]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_02054_b200 as amg  # noqa: E402
from oracle import problems as P  # noqa: E402

g = int(sys.argv[1])
var = sys.argv[2] if len(sys.argv) > 2 else None
values = sys.argv[3:] if var else [None]
ctx = amg.Context(0)
A = P.grid3d_values("dambreak", g, 1)
h = amg.setup(A, amg.AmgParams(coarse_solve="exact"), ctx=ctx)
f = P.rhs(g ** 3)
print(f"levels {h.num_levels()}, coarse n {h.coarse_n()}", flush=True)
ref_u = None
for rep in range(2):
    for val in values:
        if var:
            os.environ[var] = val
        for fam in ("coarse_solve", "coarse"):
            ctx.probe(fam)
            if fam == "coarse":
                for _ in range(5):
                    h.rebuild_values(A[2])
            else:
                for _ in range(10):
                    u = amg.vcycle(h, f)
            cnt, ms, _ = ctx.probe_read()
            ctx.probe(None)
            print(f"{var}={val} {fam}: {cnt} launches, {1e3 * ms / max(cnt, 1):.1f} us/launch", flush=True)
        u = amg.vcycle(h, f)
        if ref_u is None:
            ref_u = u
        print(f"  V-cycle bit-identical across variants: {np.array_equal(u.view(np.int64), ref_u.view(np.int64))}")
