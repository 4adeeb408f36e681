"""Development probe: device time of one in-place partial rebuild
(amgr_rebuild_values from device values) at g^3 dam-break while varying an
environment knob read per call.  usage: python tools/rebuild_time.py g VAR v1 v2 ..."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_02054_b200 as amg  # noqa: E402

g = int(sys.argv[1])
var = sys.argv[2]
values = sys.argv[3:]
ctx = amg.Context(0)
L = amg.lib()
n, nnz = g ** 3, int(L.amgr_problem_nnz(g))
rp = torch.empty(n + 1, dtype=torch.int32, device="cuda")
ci = torch.empty(nnz + 8, dtype=torch.int32, device="cuda")
vals = [torch.empty(nnz + 8, dtype=torch.float64, device="cuda") for _ in range(2)]
torch.cuda.synchronize()
amg._check(L.amgr_problem_pattern(ctx.ptr, g, rp.data_ptr(), ci.data_ptr()), ctx.ptr)
for k, v in enumerate(vals):
    amg._check(L.amgr_problem_values(ctx.ptr, 2, g, 1 + k, 50, v.data_ptr()), ctx.ptr)
ctx.synchronize()
h = amg.setup(amg.DeviceCsr(n, n, nnz, rp.data_ptr(), ci.data_ptr(), vals[0].data_ptr()),
              amg.AmgParams(coarse_solve=os.environ.get("COARSE", "exact")), ctx=ctx)
s = torch.cuda.ExternalStream(ctx.stream)
for rep in range(2):
    for val in values:
        os.environ[var] = val
        for k in range(3):
            h.rebuild_values(vals[k & 1].data_ptr(), adopt=True)
        ts = []
        for k in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                e0.record()
            h.rebuild_values(vals[k & 1].data_ptr(), adopt=True)
            with torch.cuda.stream(s):
                e1.record()
            ctx.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(f"{var}={val}: rebuild {sum(ts) / len(ts):.3f} ms (min {min(ts):.3f}), stencil {h.level_stencil(0)}",
              flush=True)
