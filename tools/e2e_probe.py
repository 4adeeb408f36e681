"""Where does the e2e time go?  Host-timed step loops at 256^3 through the
C-ABI: (a) device-resident values (adopt), (b) staged from device memory,
(c) staged from pinned host memory (the bench's e2e), (d) = (c) with per-step
host timestamps.  usage: python tools/e2e_probe.py [g] [K]"""
import ctypes
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_02054_b200 as amg  # noqa: E402

g = int(sys.argv[1]) if len(sys.argv) > 1 else 256
K = int(sys.argv[2]) if len(sys.argv) > 2 else 5
ctx = amg.Context(0)
L = amg.lib()
n = g ** 3
nnz = int(L.amgr_problem_nnz(g))
rp = torch.empty(n + 1, dtype=torch.int32, device="cuda")
ci = torch.empty(nnz + 8, dtype=torch.int32, device="cuda")
vals = [torch.empty(nnz + 8, dtype=torch.float64, device="cuda") for _ in range(K + 2)]
torch.cuda.synchronize()
amg._check(L.amgr_problem_pattern(ctx.ptr, g, rp.data_ptr(), ci.data_ptr()), ctx.ptr)
for k in range(K + 2):
    amg._check(L.amgr_problem_values(ctx.ptr, 2, g, k, 50, vals[k].data_ptr()), ctx.ptr)
f = torch.empty(n, dtype=torch.float64, device="cuda")
amg._check(L.amgr_problem_rhs(ctx.ptr, n, 42, f.data_ptr(), amg.DEVICE), ctx.ptr)
ctx.synchronize()
h = amg.setup(amg.DeviceCsr(n, n, nnz, rp.data_ptr(), ci.data_ptr(), vals[0].data_ptr()),
              amg.AmgParams(coarse_solve="inverse"), ctx=ctx)
sp = amg._SolveParams(1e-8, 100)
st = amg._SolveStats()
ub = [torch.zeros(n, dtype=torch.float64, device="cuda"), torch.zeros(n, dtype=torch.float64, device="cuda")]
amg._check(L.amgr_bicgstab(h._p, f.data_ptr(), ub[0].data_ptr(), ub[0].data_ptr(), ctypes.byref(sp),
                           ctypes.byref(st), amg.DEVICE), ctx.ptr)
hv = [torch.empty(nnz, dtype=torch.float64, pin_memory=True) for _ in range(K)]
hf = [torch.empty(n, dtype=torch.float64, pin_memory=True) for _ in range(K)]
for k in range(K):
    hv[k].copy_(vals[k + 1][:nnz])
    hf[k].copy_(f)
uo = [torch.empty(n, dtype=torch.float64, pin_memory=True) for _ in range(K)]
torch.cuda.synchronize()


def run(mode):
    ub[0].copy_(ub[1]) if False else None
    ctx.synchronize()
    t0 = time.perf_counter()
    stamps = []
    if mode in ("staged_dev", "staged_host"):
        src = (lambda k: hv[k].data_ptr()) if mode == "staged_host" else (lambda k: vals[k + 1].data_ptr())
        loc = amg.HOST if mode == "staged_host" else amg.DEVICE
        fsrc = (lambda k: hf[k].data_ptr()) if mode == "staged_host" else (lambda k: f.data_ptr())
        amg._check(L.amgr_stage_values(h._p, src(0), loc), ctx.ptr)
        amg._check(L.amgr_stage_rhs(h._p, fsrc(0), loc), ctx.ptr)
    for j in range(K):
        if mode == "adopt":
            amg._check(L.amgr_rebuild_values(h._p, vals[j + 1].data_ptr(), amg.DEVICE_ADOPT), ctx.ptr)
            amg._check(L.amgr_bicgstab(h._p, f.data_ptr(), ub[j % 2].data_ptr(), ub[(j + 1) % 2].data_ptr(),
                                       ctypes.byref(sp), ctypes.byref(st), amg.DEVICE), ctx.ptr)
        else:
            amg._check(L.amgr_rebuild_values(h._p, None, amg.STAGED), ctx.ptr)
            if j + 1 < K:
                amg._check(L.amgr_stage_values(h._p, src(j + 1), loc), ctx.ptr)
                amg._check(L.amgr_stage_rhs(h._p, fsrc(j + 1), loc), ctx.ptr)
            amg._check(L.amgr_bicgstab(h._p, None, ub[j % 2].data_ptr(), ub[(j + 1) % 2].data_ptr(),
                                       ctypes.byref(sp), ctypes.byref(st), amg.STAGED), ctx.ptr)
            if mode == "staged_host":
                amg._check(L.amgr_download_async(ctx.ptr, ub[(j + 1) % 2].data_ptr(), uo[j].data_ptr(), n), ctx.ptr)
        stamps.append((time.perf_counter() - t0) * 1e3)
    ctx.synchronize()
    total = (time.perf_counter() - t0) * 1e3
    print(f"{mode:12s} {total / K:8.1f} ms/step  step ends {[round(x, 1) for x in stamps]}  total {total:.1f}",
          flush=True)


for mode in ("adopt", "staged_dev", "staged_host", "adopt", "staged_host"):
    run(mode)
