"""Per-level row-pass timing of the bench hierarchy (probe families
vcycle_down@l / vcycle_smooth@l over one V-cycle batch).  Used for layout
A/B runs (AMGR_COLCODE).  usage: python tools/level_time.py [g]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_02054_b200 as amg  # noqa: E402
from paper_2108_02054_b200 import reuse as R  # noqa: E402

g = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ctx = amg.Context()
seq = R.DeviceGridSequence("dambreak", g, 2, ctx=ctx)
A, fptr = seq.step(0)
h = amg.setup(A, amg.AmgParams(), ctx=ctx)
n = g ** 3
u = torch.zeros(n, dtype=torch.float64, device="cuda")
for _ in range(3):
    amg.vcycle_device(h, fptr, u.data_ptr())
ctx.synchronize()
out = []
for l in range(min(h.num_levels() - 1, int(os.environ.get("LEVELS", "6")))):
    row = [l, h.level_layout(l)["col_bytes"]]
    for fam in (f"vcycle_down@{l}", f"vcycle_smooth@{l}"):
        ctx.probe(fam)
        for _ in range(10):
            amg.vcycle_device(h, fptr, u.data_ptr())
        ctx.synchronize()
        c, ms, b = ctx.probe_read()
        row.append(1e3 * ms / c if c else 0.0)
    ctx.probe(None)
    out.append(row)
    print(f"level {row[0]} col_bytes {row[1]}: down {row[2]:.1f} us, smooth {row[3]:.1f} us", flush=True)
