"""Development probe: device time of one V-cycle (stream-launched) and of
one BiCGStab iteration (CUDA-graph path, 30 iterations from a zero guess) at
g^3 dam-break while varying an environment knob read per call
(AMGR_TAIL_NNZ, AMGR_FOLD_PREMUL, ...).  usage: python tools/vcycle_time.py g VAR v1 v2 ..."""
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
v = torch.empty(nnz + 8, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
amg._check(L.amgr_problem_pattern(ctx.ptr, g, rp.data_ptr(), ci.data_ptr()), ctx.ptr)
amg._check(L.amgr_problem_values(ctx.ptr, 2, g, 1, 50, v.data_ptr()), ctx.ptr)
f = torch.empty(n, dtype=torch.float64, device="cuda")
amg._check(L.amgr_problem_rhs(ctx.ptr, n, 42, f.data_ptr(), amg.DEVICE), ctx.ptr)
u = torch.zeros(n, dtype=torch.float64, device="cuda")
ctx.synchronize()
h = amg.setup(amg.DeviceCsr(n, n, nnz, rp.data_ptr(), ci.data_ptr(), v.data_ptr()),
              amg.AmgParams(coarse_solve=os.environ.get("COARSE", "inverse")), ctx=ctx)
s = torch.cuda.ExternalStream(ctx.stream)
for rep in range(2):
    for val in values:
        os.environ[var] = val
        for _ in range(3):
            amg.vcycle_device(h, f.data_ptr(), u.data_ptr())
        ctx.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record()
            for _ in range(20):
                amg.vcycle_device(h, f.data_ptr(), u.data_ptr())
            e1.record()
        ctx.synchronize()
        vc = e0.elapsed_time(e1) / 20
        it = []
        for _ in range(3):
            u.zero_()
            torch.cuda.synchronize()
            with torch.cuda.stream(s):
                e0.record()
            _, st = amg.bicgstab(h, f.data_ptr(), (u.data_ptr(), u.data_ptr()), amg.SolveParams(max_iter=30))
            with torch.cuda.stream(s):
                e1.record()
            ctx.synchronize()
            it.append(e0.elapsed_time(e1) / max(st.iterations, 1))
        print(f"{var}={val}: vcycle {vc:.3f} ms, bicgstab {min(it):.3f} ms/iteration ({st.iterations} its)", flush=True)
