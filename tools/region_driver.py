"""Small driver for ncu launch lists: set up a g^3 dam-break hierarchy, then run
the profiled region (cudaProfilerStart/Stop) = 1 rebuild + 2 V-cycles + 1 solve
iteration budget.  Use with `ncu --profile-from-start off`.

usage: python tools/region_driver.py [g] [what: vcycle|rebuild|solve|all]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_02054_b200 as amg  # noqa: E402


def main():
    g = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    what = sys.argv[2] if len(sys.argv) > 2 else "all"
    ctx = amg.Context(0)
    L = amg.lib()
    n = g ** 3
    nnz = int(L.amgr_problem_nnz(g))
    rp = torch.empty(n + 1, dtype=torch.int32, device="cuda")
    ci = torch.empty(nnz, dtype=torch.int32, device="cuda")
    v0 = torch.empty(nnz, dtype=torch.float64, device="cuda")
    v1 = torch.empty(nnz, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    amg._check(L.amgr_problem_pattern(ctx.ptr, g, rp.data_ptr(), ci.data_ptr()), ctx.ptr)
    amg._check(L.amgr_problem_values(ctx.ptr, 2, g, 0, 50, v0.data_ptr()), ctx.ptr)
    amg._check(L.amgr_problem_values(ctx.ptr, 2, g, 1, 50, v1.data_ptr()), ctx.ptr)
    f = torch.empty(n, dtype=torch.float64, device="cuda")
    amg._check(L.amgr_problem_rhs(ctx.ptr, n, 42, f.data_ptr(), amg.DEVICE), ctx.ptr)
    u = torch.zeros(n, dtype=torch.float64, device="cuda")
    ctx.synchronize()
    prm = amg.AmgParams(coarse_solve=os.environ.get("AMGR_COARSE", "exact"))  # bench default
    h = amg.setup(amg.DeviceCsr(n, n, nnz, rp.data_ptr(), ci.data_ptr(), v0.data_ptr()), prm, ctx=ctx)
    # warm-up
    h.rebuild_values(v1.data_ptr())
    amg.vcycle_device(h, f.data_ptr(), u.data_ptr())
    ctx.synchronize()
    torch.cuda.profiler.start()
    if what in ("rebuild", "all"):
        h.rebuild_values(v1.data_ptr())
    if what in ("vcycle", "all"):
        amg.vcycle_device(h, f.data_ptr(), u.data_ptr())
        amg.vcycle_device(h, f.data_ptr(), u.data_ptr())
    if what in ("solve", "all"):
        u.zero_()
        torch.cuda.synchronize()
        _, st = amg.bicgstab(h, f.data_ptr(), (u.data_ptr(), u.data_ptr()), amg.SolveParams(max_iter=2))
    ctx.synchronize()
    torch.cuda.profiler.stop()
    print("levels", h.num_levels(), [h.level_dims(l)["nrows"] for l in range(h.num_levels())])


if __name__ == "__main__":
    main()
