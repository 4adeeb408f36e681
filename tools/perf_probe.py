"""Development probe: setup / rebuild / V-cycle / solve timings and per-kernel
family device time on one GPU.  Not the bench (bench.py is); used to see where
time goes while iterating on kernels.

usage: python tools/perf_probe.py [g] [kind] [steps]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_02054_b200 as amg  # noqa: E402


def main():
    g = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    kind = sys.argv[2] if len(sys.argv) > 2 else "dambreak"
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    ctx = amg.Context(0)
    L = amg.lib()
    n = g ** 3
    nnz = int(L.amgr_problem_nnz(g))
    rp = torch.empty(n + 1, dtype=torch.int32, device="cuda")
    ci = torch.empty(nnz, dtype=torch.int32, device="cuda")
    vals = [torch.empty(nnz + 8, dtype=torch.float64, device="cuda") for _ in range(steps + 1)]
    torch.cuda.synchronize()
    amg._check(L.amgr_problem_pattern(ctx.ptr, g, rp.data_ptr(), ci.data_ptr()), ctx.ptr)
    for k, v in enumerate(vals):
        amg._check(L.amgr_problem_values(ctx.ptr, amg.PROBLEM[kind], g, k, 50, v.data_ptr()), ctx.ptr)
    f = torch.empty(n, dtype=torch.float64, device="cuda")
    amg._check(L.amgr_problem_rhs(ctx.ptr, n, 42, f.data_ptr(), amg.DEVICE), ctx.ptr)
    u = torch.zeros(n, dtype=torch.float64, device="cuda")
    ctx.synchronize()
    A = amg.DeviceCsr(n, n, nnz, rp.data_ptr(), ci.data_ptr(), vals[0].data_ptr())
    t0 = time.perf_counter()
    cs = os.environ.get("AMGR_COARSE", "exact")
    h = amg.setup(A, amg.AmgParams(coarse_solve=cs), ctx=ctx)
    ctx.synchronize()
    t_setup = time.perf_counter() - t0
    print(f"g={g} kind={kind} n={n} nnz={nnz} setup {t_setup*1e3:.1f} ms levels={h.num_levels()} "
          f"oc={h.operator_complexity():.3f} timings={h.setup_timings()}")
    for l in range(h.num_levels()):
        d = h.level_dims(l)
        print(f"  level {l}: n={d['nrows']} nnz={d['nnz']} nnz/row={d['nnz']/max(d['nrows'],1):.2f}")
    fams = ["rap", "smoother", "vcycle_down", "vcycle_up", "restrict", "coarse_solve", "spmv_dot", "spmv_dot2",
            "krylov_vec", "resid_norm", "krylov_scalar", "coarse"]
    for k in range(1, steps + 1):
        ctx.synchronize()
        t0 = time.perf_counter()
        h.rebuild_values(vals[k].data_ptr(), adopt=True)
        ctx.synchronize()
        t_rb = time.perf_counter() - t0
        t0 = time.perf_counter()
        _, st = amg.bicgstab(h, f.data_ptr(), (u.data_ptr(), u.data_ptr()))
        ctx.synchronize()
        t_solve = time.perf_counter() - t0
        print(f"step {k}: rebuild {t_rb*1e3:.2f} ms (phases {h.setup_timings()}) solve {t_solve*1e3:.1f} ms "
              f"iters={st.iterations} conv={st.converged} relres={st.relative_residual:.2e}")
    # per-family device time for one rebuild + solve
    for fam in fams:
        ctx.probe(fam)
        h.rebuild_values(vals[1].data_ptr(), adopt=True)
        u.zero_()
        torch.cuda.synchronize()
        _, st = amg.bicgstab(h, f.data_ptr(), (u.data_ptr(), u.data_ptr()))
        cnt, ms, by = ctx.probe_read()
        if cnt:
            print(f"  {fam:14s} launches={cnt:6d} ms={ms:9.3f} GB/s={by/ms/1e6 if ms>0 else 0:8.1f}")
    # per-level device time (family@level) for the V-cycle and rebuild kernels
    lf = ["vcycle_down", "vcycle_smooth", "restrict", "prolong", "vcycle_premul", "rap", "smoother"]
    print("  level " + " ".join(f"{x[:13]:>22s}" for x in lf))
    for l in range(h.num_levels()):
        cells = []
        for fam in lf:
            ctx.probe(f"{fam}@{l}")
            h.rebuild_values(vals[1].data_ptr(), adopt=True)
            u.zero_()
            torch.cuda.synchronize()
            amg.bicgstab(h, f.data_ptr(), (u.data_ptr(), u.data_ptr()))
            cnt, ms, by = ctx.probe_read()
            cells.append(f"{ms:8.3f}ms/{by/ms/1e6 if ms>0 else 0:6.0f}({cnt:4d})")
        print(f"  {l:5d} " + " ".join(f"{c:>22s}" for c in cells))
    ctx.probe(None)
    # one V-cycle, device time
    fz = f.clone()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s = torch.cuda.ExternalStream(ctx.stream)
    for _ in range(3):
        amg.vcycle_device(h, fz.data_ptr(), u.data_ptr())
    ctx.synchronize()
    if s is not None:
        with torch.cuda.stream(s):
            ev0.record()
            for _ in range(20):
                amg.vcycle_device(h, fz.data_ptr(), u.data_ptr())
            ev1.record()
        ctx.synchronize()
        print(f"  vcycle: {ev0.elapsed_time(ev1)/20:.3f} ms")


if __name__ == "__main__":
    main()
