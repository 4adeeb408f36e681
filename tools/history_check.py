"""Diagnostic: relative-residual history of the device BiCGStab vs the
reference (fixed V-cycle) by re-running with max_iter = 1..K (each run is
deterministic from u0 = 0).  usage: python tools/history_check.py kind g k K"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_02054_b200 as amg  # noqa: E402
from oracle import problems as P  # noqa: E402
from oracle import ref  # noqa: E402

kind, g, k, K = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
A = P.grid3d_values(kind, g, k)
n = g ** 3
fr = P.rhs(n)
h = amg.setup(A)
r = ref.setup(A, ref.params())
step = int(sys.argv[5]) if len(sys.argv) > 5 else 1
for it in range(1, K + 1, step):
    _, st = amg.bicgstab(h, fr, prm=amg.SolveParams(tol=1e-8, max_iter=it))
    rs = ref.bicgstab(r, fr, max_iter=it, fixed=True, prm=ref.params())
    print(f"it {it:3d}: device relres {st.relative_residual:.3e} ({st.iterations})   reference "
          f"{rs.relative_residual:.3e} ({rs.iterations})", flush=True)
