"""Development driver: one full setup at g^3 dam-break inside a profiler
region (use with ncu --profile-from-start off)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_02054_b200 as amg  # noqa: E402

g = int(sys.argv[1]) if len(sys.argv) > 1 else 128
ctx = amg.Context(0)
L = amg.lib()
n, nnz = g ** 3, int(L.amgr_problem_nnz(g))
rp = torch.empty(n + 1, dtype=torch.int32, device="cuda")
ci = torch.empty(nnz + 8, dtype=torch.int32, device="cuda")
v = torch.empty(nnz + 8, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
amg._check(L.amgr_problem_pattern(ctx.ptr, g, rp.data_ptr(), ci.data_ptr()), ctx.ptr)
amg._check(L.amgr_problem_values(ctx.ptr, 2, g, 0, 50, v.data_ptr()), ctx.ptr)
ctx.synchronize()
A = amg.DeviceCsr(n, n, nnz, rp.data_ptr(), ci.data_ptr(), v.data_ptr())
h = amg.setup(A, amg.AmgParams(coarse_solve="inverse"), ctx=ctx)  # warm-up
ctx.synchronize()
import time  # noqa: E402

reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
torch.cuda.profiler.start()
for _ in range(reps):
    del h
    t0 = time.perf_counter()
    h = amg.setup(A, amg.AmgParams(coarse_solve="inverse"), ctx=ctx)
    ctx.synchronize()
    t = time.perf_counter() - t0
    print(f"setup {t*1e3:.1f} ms, levels {h.num_levels()}, timings {h.setup_timings()}", flush=True)
torch.cuda.profiler.stop()
