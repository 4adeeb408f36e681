"""Per-level column-offset statistics (j - i) of the bench hierarchy: how many
distinct offsets, and the largest |offset| (layout study for a coded column
stream).  usage: python tools/offset_stats.py [g]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_02054_b200 as amg  # noqa: E402
from paper_2108_02054_b200 import reuse as R  # noqa: E402

g = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ctx = amg.Context()
seq = R.DeviceGridSequence("dambreak", g, 2, ctx=ctx)
A, _ = seq.step(0)
h = amg.setup(A, amg.AmgParams(), ctx=ctx)
for l in range(h.num_levels()):
    rp, ci, _ = h.level_A(l)
    n = len(rp) - 1
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
    d = ci.astype(np.int64) - rows
    u = np.unique(d)
    print(f"level {l}: n={n} nnz={len(ci)} nnz/row={len(ci)/n:.2f} distinct offsets={len(u)} "
          f"max|off|={np.abs(d).max()} frac|off|<=32767={np.mean(np.abs(d) <= 32767):.4f} "
          f"frac|off|<=127={np.mean(np.abs(d) <= 127):.4f}", flush=True)
