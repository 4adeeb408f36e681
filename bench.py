"""Benchmark: partial-reuse AMG rebuild ms/step + solve ms/step (BASELINE.json
`metric`) on the synthetic two-fluid dam-break pressure Poisson problem
(configs[2], "C3": 256^3, 1000:1 density jump on a collapsing water column,
partial reuse, 1 B200).

One step = one time step of the sequence: partial rebuild of the hierarchy
from A_k (numeric Galerkin RAP on the frozen transfers + smoothers + coarse
LU, `amgr_rebuild_values`) followed by the AMG-preconditioned BiCGStab solve
(`amgr_bicgstab`, tol 1e-8, <= 100 iterations) from the previous step's
solution: the reference's `run_sequence` partial-reuse step
(proj/src/reuse.cpp:85-114) with its V-cycle algorithm (hierarchy.cpp:152-186,
smoothing applied) and, by default, its coarse LU solve replayed
exactly (dense_lu.cpp:52-73; `--coarse inverse` selects the explicit-inverse
extension).  The hierarchy, the rebuild and the V-cycle are bit-identical to
the reference's at this size (tests/test_gpu_parity_large.py); the Krylov dots
use the fast blocked order (the sequential-dot parity mode is not benchmarked).
The matrices A_k are generated on the device before the timed region
(ingestion is excluded, reuse.cpp:65) and are larger than L2 (0.94 GB of
values), so no explicit flush is needed.

value        = device time of K steps / K (CUDA events on the library stream,
               barrier + synchronize both sides, max over ranks)      [ms/step]
e2e          = the same through the C-ABI with HOST buffers: per step the
               H2D copy of A_k's values and f from pinned memory and the D2H
               read of the solution are inside the timed region
roofline     = the dominant kernel (level-0 post-smoothing sweep, the largest
               single kernel of the step) probed with CUDA events on its stream
cpu_baseline = the unmodified reference (oracle/_ref, single-threaded as
               shipped) on a bounded, extrapolated sample of the same workload
--impl reference runs the reference arm alone (rank 0): one full reference
               step measured end to end (partial_update + BiCGStab to
               convergence, the reference's own iteration count).

strategies   = none / full / partial reuse through the library's run_sequence
               over steps 0..W-1 of the same sequence (rebuild, solve and
               total ms per step; not part of `value`)

Multi-GPU (torchrun, N>1): N independent single-GPU systems (replicas, weak
scaling) by default.  `--partitioned` (opt-in) runs ONE global 256^3 system
row-partitioned over the ranks (amgr_dist_*: NCCL halo send/recv, transition
allgather, rank-ordered dots; levels below --replicate-below rows
replicated), strong scaling; verified on one GPU through the loopback
transport and at world size 1 over NCCL (tests/test_gpu_dist.py), never yet
at world > 1 over NCCL — see DESIGN.md §5.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "partial-reuse AMG rebuild ms/step + solve ms/step, 256^3 Poisson; HBM GB/s"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_RECORD = os.path.join(ROOT, "profiles", "r02_traffic.json")


def args_parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--size", type=int, default=256)
    p.add_argument("--problem", default="dambreak")
    p.add_argument("--nsteps", type=int, default=50, help="length of the time sequence (configs[2]: 50)")
    p.add_argument("--coarse", default="exact", choices=["exact", "inverse"],
                   help="coarsest solve: exact replay of dense_lu.cpp (bit-exact V-cycle; default) or the "
                        "explicit-inverse extension")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--partitioned", action="store_true",
                   help="row-partitioned NCCL solve of ONE global system over all ranks (strong scaling); opt-in "
                        "(the default with N ranks is N independent replicas)")
    p.add_argument("--replicas", action="store_true",
                   help="with N ranks, run N independent systems (the default unless --partitioned)")
    p.add_argument("--replicate-below", type=int, default=150000,
                   help="partitioned mode: levels with fewer rows are replicated on every rank")
    p.add_argument("--no-strategies", action="store_true",
                   help="skip the none/full/partial reuse comparison (run_sequence over a window of the sequence)")
    p.add_argument("--strategy-window", type=int, default=6,
                   help="steps 0..W-1 of the --nsteps sequence for the none/full/partial comparison")
    return p.parse_args()


def hbm_peak():
    try:
        return float(json.load(open(PEAKS))["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# --------------------------------------------------------------------------------------
# reference arm / CPU baseline (TEST INFRASTRUCTURE: oracle/_ref is the checker and the
# reported CPU baseline, never part of the measured GPU path)
# --------------------------------------------------------------------------------------
def reference_sample(A0, Ak_list, f, iters, max_steps):
    """Time the unmodified reference on the host: setup(A0) untimed, then per
    step partial_update(A_k) (timed in full) + fixed-V BiCGStab sampled for 2
    iterations (per-iteration time).  ms/step = rebuild + per_iter * iters."""
    from oracle import ref

    p = ref.params()
    t0 = time.perf_counter()
    h = ref.setup(A0, p)
    t_setup = time.perf_counter() - t0
    rebuild, per_iter = [], []
    for Ak in Ak_list[:max_steps]:
        hk = ref.partial_update(h, Ak, p)
        rebuild.append(hk.seconds)
        s = ref.bicgstab(hk, f, fixed=True, max_iter=2, prm=p)
        per_iter.append(s.seconds / max(s.iterations, 1))
        hk.free()
    h.free()
    rb = float(np.mean(rebuild)) * 1e3
    it = float(np.mean(per_iter)) * 1e3
    return {"value": rb + it * iters, "rebuild_ms": rb, "per_iteration_ms": it, "setup_s": t_setup,
            "steps": len(rebuild)}


def host_problem(g, kind, k, nsteps):
    from oracle import problems as P

    return P.grid3d_values(kind, g, k, nsteps)


def host_cpu():
    """Model name and core counts of this host (state the host)."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        avail = len(os.sched_getaffinity(0))
    except Exception:
        avail = os.cpu_count()
    return {"model": model, "nproc": os.cpu_count(), "available": avail}


def run_reference_arm(a):
    """The unmodified reference (oracle/_ref) on the host, one FULL partial-reuse
    step of the sequence measured end to end, as run_sequence runs it
    (reuse.cpp:85-114): setup(A_0) and the step-0 solve from zero are the
    untimed prelude (the step-0 solution is the step-1 initial guess,
    reuse.cpp:108-109); the timed step is partial_update(A_1) + bicgstab over
    the (fixed) V-cycle to convergence, with the reference's own
    iteration count.  Times are the reference's own clocks around those two
    calls (oracle/ref_shim.cpp).  The reference is single-threaded as shipped."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import problems as P
    from oracle import ref

    g = a.size
    t_all = time.perf_counter()
    A0 = host_problem(g, a.problem, 0, a.nsteps)
    f = P.rhs(g ** 3)
    p = ref.params()
    t0 = time.perf_counter()
    h0 = ref.setup(A0, p)
    setup_s = time.perf_counter() - t0
    del A0
    s0 = ref.bicgstab(h0, f, fixed=True, prm=p)
    A1 = host_problem(g, a.problem, 1, a.nsteps)
    h1 = ref.partial_update(h0, A1, p)
    h0.free()
    s1 = ref.bicgstab(h1, f, u0=s0.u, fixed=True, prm=p)
    h1.free()
    rebuild_ms, solve_ms = h1.seconds * 1e3, s1.seconds * 1e3
    value = rebuild_ms + solve_ms
    cpu = host_cpu()
    sample = (f"1 full partial-reuse step (step 1 of the {a.nsteps}-step {g}^3 {a.problem} sequence) timed end to "
              f"end: partial_update {rebuild_ms:.0f} ms + fixed-V BiCGStab to convergence from the step-0 solution, "
              f"{s1.iterations} iterations ({'converged' if s1.converged else 'NOT converged'}), {solve_ms:.0f} ms; "
              f"untimed prelude: setup {setup_s:.1f} s, step-0 solve from zero {s0.iterations} iterations "
              f"{s0.seconds:.1f} s; unmodified reference, single-threaded as shipped; host {cpu['model']}, "
              f"nproc {cpu['nproc']}")
    out = {"metric": METRIC, "value": value, "unit": "ms/step", "impl": "reference", "n_gpus": a.gpus,
           "steps": 1, "warmup": 0, "ms_per_step": value, "higher_is_better": False,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"C3 dam-break {g}^3, partial reuse (BASELINE.json configs[2])",
                      "problem": a.problem, "grid": g, "n": g ** 3, "nnz": 7 * g ** 3 - 6 * g ** 2,
                      "sequence_steps": a.nsteps, "timed_steps": "1", "reuse": "partial", "smoother": "jacobi",
                      "coarse_solve": "exact (dense_lu.cpp)", "parallelism": "reference CPU path, 1 host thread"},
           "rebuild_ms_per_step": rebuild_ms, "solve_ms_per_step": solve_ms, "iterations": [s1.iterations],
           "converged": bool(s1.converged), "relative_residual": s1.relative_residual,
           "step0_iterations": s0.iterations, "setup_s": setup_s, "host": cpu,
           "arm_wall_s": time.perf_counter() - t_all,
           "cpu_baseline": {"value": value, "unit": "ms/step", "cores": 1, "kind": "reference", "sample": sample},
           "e2e": {"value": value, "unit": "ms/step", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(out)


# --------------------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------------------
def run_partitioned(a, rank, world, local):
    """One global C3 system, rows partitioned over the ranks (amgr_dist_*):
    per step the partitioned rebuild from each rank's own rows of A_k
    (amgr_dist_rebuild_local: local Jacobi + local Galerkin products, one
    allgather of A_{top+1}, replicated tail) and the partitioned BiCGStab
    (NCCL halo exchange, transition allgather, replicated coarse levels,
    rank-ordered dots)."""
    import torch

    import paper_2108_02054_b200 as amg
    from paper_2108_02054_b200 import distributed as D

    L = amg.lib()
    ctx = amg.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream)
    g, kind = a.size, amg.PROBLEM[a.problem]
    n, nnz = g ** 3, int(L.amgr_problem_nnz(g))
    W, K = max(a.warmup, 0), max(a.steps, 1)
    ksteps = list(range(0, 1 + W + K))
    rp = torch.empty(n + 1, dtype=torch.int32, device="cuda")
    ci = torch.empty(nnz + 8, dtype=torch.int32, device="cuda")
    vals = [torch.empty(nnz + 8, dtype=torch.float64, device="cuda") for _ in ksteps]
    torch.cuda.synchronize()
    amg._check(L.amgr_problem_pattern(ctx.ptr, g, rp.data_ptr(), ci.data_ptr()), ctx.ptr)
    for k, v in zip(ksteps, vals):
        amg._check(L.amgr_problem_values(ctx.ptr, kind, g, k % a.nsteps, a.nsteps, v.data_ptr()), ctx.ptr)
    f = torch.empty(n, dtype=torch.float64, device="cuda")
    amg._check(L.amgr_problem_rhs(ctx.ptr, n, 42, f.data_ptr(), amg.DEVICE), ctx.ptr)
    ctx.synchronize()
    prm = amg.AmgParams(coarse_solve=a.coarse)
    t0 = time.perf_counter()
    h = amg.setup(amg.DeviceCsr(n, n, nnz, rp.data_ptr(), ci.data_ptr(), vals[0].data_ptr()), prm, ctx=ctx)
    ctx.synchronize()
    setup_s = time.perf_counter() - t0
    ids = [D.nccl_unique_id() if rank == 0 else None]
    if world > 1:
        import torch.distributed as dist

        dist.broadcast_object_list(ids, src=0)
    t0 = time.perf_counter()
    ds = D.DistSolver(h, rank, world, ids[0], replicate_below=a.replicate_below, device_plan=True)
    plan_s = time.perf_counter() - t0
    own = torch.from_numpy(ds.owned0).cuda()
    fl = f[own].contiguous()
    ul = torch.zeros(ds.n_local, dtype=torch.float64, device="cuda")
    # each rank's OWN rows of A_k (local CSR order): the only A_k data the
    # partitioned rebuild (amgr_dist_rebuild_local) reads
    nmap = torch.from_numpy(ds.plan.levels[0].nnz_map).cuda()
    lvals = [torch.cat([v[nmap], torch.zeros(8, dtype=torch.float64, device="cuda")]) for v in vals]
    del vals
    nnz_local = int(nmap.numel())
    torch.cuda.synchronize()
    sp = amg.SolveParams()
    ds.bicgstab(fl.data_ptr(), ul.data_ptr(), sp)
    for k in range(1, 1 + W):
        ds.rebuild_local(lvals[k].data_ptr(), device=True)
        ds.bicgstab(fl.data_ptr(), ul.data_ptr(), sp)
    ctx.synchronize()

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    ul_start = ul.clone()  # the e2e run below starts from the same iterate
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * K + 1)]
    iters = []
    barrier()
    torch.cuda.synchronize()
    ctx.synchronize()
    launches0 = ctx.launches()
    with ClockSampler(local) as clk:
        ev[0].record(stream)
        for j, k in enumerate(range(1 + W, 1 + W + K)):
            ds.rebuild_local(lvals[k].data_ptr(), device=True)
            ev[2 * j + 1].record(stream)
            st = ds.bicgstab(fl.data_ptr(), ul.data_ptr(), sp)
            ev[2 * j + 2].record(stream)
            iters.append(st.iterations)
        ctx.synchronize()
        torch.cuda.synchronize()
    barrier()
    launches = ctx.launches() - launches0
    total_ms = ev[0].elapsed_time(ev[2 * K])
    rebuild_ms = sum(ev[2 * j].elapsed_time(ev[2 * j + 1]) for j in range(K)) / K
    solve_ms = sum(ev[2 * j + 1].elapsed_time(ev[2 * j + 2]) for j in range(K)) / K
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    # roofline probe (every rank runs the probed solve; rank 0 reports its
    # local level-0 post-smoothing sweep)
    peak, peak_kind = hbm_peak()
    ctx.probe("vcycle_smooth@0")
    ul.zero_()
    torch.cuda.synchronize()
    ds.bicgstab(fl.data_ptr(), ul.data_ptr(), sp)
    cnt, pms, pbytes = ctx.probe_read()
    ctx.probe(None)
    achieved = (pbytes / cnt) / (pms / cnt) / 1e6 if cnt else None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": None,
                "kernel": "k_rowpass<OpSmooth> level 0, rank-local rows", "peak_source": peak_kind}
    # e2e: per step the global A_k values and the local f go host -> device,
    # the local solution comes back
    e2e = None
    if not a.no_e2e:
        hv = []
        for k in range(1 + W, 1 + W + K):
            tt = torch.empty(nnz_local, dtype=torch.float64, pin_memory=True)
            tt.copy_(lvals[k][:nnz_local])
            hv.append(tt)
        dv = torch.empty(nnz_local + 8, dtype=torch.float64, device="cuda")
        fh = torch.empty(ds.n_local, dtype=torch.float64, pin_memory=True)
        fh.copy_(fl)
        uh = torch.empty(ds.n_local, dtype=torch.float64, pin_memory=True)
        ul.copy_(ul_start)
        torch.cuda.synchronize()
        barrier()
        e0 = time.perf_counter()
        for tt in hv:
            dv[:nnz_local].copy_(tt, non_blocking=True)
            fl.copy_(fh, non_blocking=True)
            torch.cuda.synchronize()
            ds.rebuild_local(dv.data_ptr(), device=True)
            ds.bicgstab(fl.data_ptr(), ul.data_ptr(), sp)
            uh.copy_(ul)
        torch.cuda.synchronize()
        e_ms = (time.perf_counter() - e0) * 1e3 / K
        if world > 1:
            import torch.distributed as dist

            t = torch.tensor([e_ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e2e = {"value": e_ms, "unit": "ms/step", "h2d_bytes_per_step": 8 * nnz_local + 8 * ds.n_local,
               "d2h_bytes_per_step": 8 * ds.n_local, "timer": "host wall clock, max over ranks"}
    if rank == 0:
        out = {"metric": METRIC, "value": total_ms / K, "unit": "ms/step", "n_gpus": world, "steps": K, "warmup": W,
               "ms_per_step": total_ms / K, "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
               "dtype": "f64", "data": "synthetic (device-generated dam-break sequence)",
               "config": {"workload": f"C3 dam-break {g}^3, partial reuse, row-partitioned over {world} GPU(s)",
                          "problem": a.problem, "grid": g, "n": n, "nnz": nnz, "coarse_solve": a.coarse,
                          "parallelism": f"rows{world}", "partitioned_levels": ds.plan.top + 1,
                          "plan": "device-built (amgr_dist_create_auto)",
                          "local_rows_rank0": ds.n_local},
               "rebuild_ms_per_step": rebuild_ms, "solve_ms_per_step": solve_ms, "iterations": iters,
               "setup_s": setup_s, "plan_s": plan_s, "clocks": clk.summary(), "gpu_launches": launches,
               "e2e": e2e, "roofline": roofline, "cpu_baseline": None,
               "note": ("one global system row-partitioned over the ranks (amgr_dist_*: rebuild from rank-local "
                        "rows, NCCL halo send/recv, transition allgather, rank-ordered dots); levels below "
                        "replicate_below rows replicated; "
                        f"replicate_below={a.replicate_below}")}
        emit(out)
    ds.close()


_JSON_FD = None  # the process's real stdout while fd 1 is pointed at stderr


def emit(out):
    """The one JSON line of this run, on the real stdout."""
    line = (json.dumps(out) + "\n").encode()
    if _JSON_FD is not None:
        os.write(_JSON_FD, line)
    else:
        sys.stdout.write(line.decode())
        sys.stdout.flush()


def main():
    # stdout carries exactly one JSON line: anything native code prints on
    # fd 1 (e.g. NCCL's version banner at communicator init) goes to stderr
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)
    a = args_parse()
    if a.impl == "reference":
        run_reference_arm(a)
        return
    rank, world, local = dist_env()
    import torch

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if a.partitioned:
        # opt-in: one global system over all ranks; no silent fallback (a
        # rank-local failure inside NCCL cannot be recovered consistently)
        run_partitioned(a, rank, world, local)
    else:
        run_replicas(a, rank, world, local)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def run_replicas(a, rank, world, local):
    """N independent single-GPU systems (one per rank) or the N = 1 run."""
    import torch

    import paper_2108_02054_b200 as amg

    L = amg.lib()
    ctx = amg.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream)
    g, kind = a.size, amg.PROBLEM[a.problem]
    n, nnz = g ** 3, int(L.amgr_problem_nnz(g))
    W, K = max(a.warmup, 0), max(a.steps, 1)
    ksteps = list(range(0, 1 + W + K))  # step 0 = full setup

    # ---- inputs resident in HBM (generation excluded from timing) ----
    rp = torch.empty(n + 1, dtype=torch.int32, device="cuda")
    ci = torch.empty(nnz + 8, dtype=torch.int32, device="cuda")
    vals = [torch.empty(nnz + 8, dtype=torch.float64, device="cuda") for _ in ksteps]
    torch.cuda.synchronize()
    amg._check(L.amgr_problem_pattern(ctx.ptr, g, rp.data_ptr(), ci.data_ptr()), ctx.ptr)
    for k, v in zip(ksteps, vals):
        amg._check(L.amgr_problem_values(ctx.ptr, kind, g, k % a.nsteps, a.nsteps, v.data_ptr()), ctx.ptr)
    f = torch.empty(n, dtype=torch.float64, device="cuda")
    amg._check(L.amgr_problem_rhs(ctx.ptr, n, 42, f.data_ptr(), amg.DEVICE), ctx.ptr)
    u = torch.zeros(n, dtype=torch.float64, device="cuda")
    ctx.synchronize()

    prm = amg.AmgParams(coarse_solve=a.coarse)
    A0 = amg.DeviceCsr(n, n, nnz, rp.data_ptr(), ci.data_ptr(), vals[0].data_ptr())
    t0 = time.perf_counter()
    h = amg.setup(A0, prm, ctx=ctx)
    ctx.synchronize()
    setup_s = time.perf_counter() - t0
    sp = amg.SolveParams()

    def step(k, zero_guess=False):
        h.rebuild_values(vals[k].data_ptr(), adopt=True)
        if zero_guess:
            torch.cuda.synchronize()
            u.zero_()
            torch.cuda.synchronize()
        _, st = amg.bicgstab(h, f.data_ptr(), (u.data_ptr(), u.data_ptr()), sp)
        return st

    st0 = amg.bicgstab(h, f.data_ptr(), (u.data_ptr(), u.data_ptr()), sp)[1]  # step 0 solve
    for k in range(1, 1 + W):
        step(k)
    ctx.synchronize()

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    u_start = u.clone()  # the e2e run below starts from the same iterate
    # ---- timed region ----
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * K + 1)]
    iters, conv = [], []
    launches0 = ctx.launches()
    barrier()
    torch.cuda.synchronize()
    ctx.synchronize()
    with ClockSampler(local) as clk:
        ev[0].record(stream)
        for j, k in enumerate(range(1 + W, 1 + W + K)):
            h.rebuild_values(vals[k].data_ptr(), adopt=True)
            ev[2 * j + 1].record(stream)
            _, st = amg.bicgstab(h, f.data_ptr(), (u.data_ptr(), u.data_ptr()), sp)
            ev[2 * j + 2].record(stream)
            iters.append(st.iterations)
            conv.append(st.converged)
        ctx.synchronize()
        torch.cuda.synchronize()
    barrier()
    launches = ctx.launches() - launches0
    total_ms = ev[0].elapsed_time(ev[2 * K])
    rebuild_ms = sum(ev[2 * j].elapsed_time(ev[2 * j + 1]) for j in range(K)) / K
    solve_ms = sum(ev[2 * j + 1].elapsed_time(ev[2 * j + 2]) for j in range(K)) / K
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / K

    # ---- roofline probe: dominant kernel = level-0 post-smoothing sweep ----
    peak, peak_kind = hbm_peak()
    ctx.probe("vcycle_smooth@0")
    k_probe = 1 + W + K - 1
    step(k_probe, zero_guess=True)  # fresh guess so the probed solve iterates
    cnt, pms, pbytes = ctx.probe_read()
    ctx.probe(None)
    achieved = (pbytes / cnt) / (pms / cnt) / 1e6 if cnt else None  # GB/s
    # rebuild kernels (numeric RAP on level 0) for the north-star rebuild roofline
    extra = {}
    for fam in ("rap@0", "vcycle_down@0", "spmv_dot"):
        ctx.probe(fam)
        step(k_probe, zero_guess=True)
        c2, m2, b2 = ctx.probe_read()
        if c2:
            extra[fam] = {"launches": c2, "avg_us": 1e3 * m2 / c2, "GB_s": b2 / m2 / 1e6, "frac": b2 / m2 / 1e6 / peak}
    ctx.probe(None)
    traffic = None
    try:
        traffic = json.load(open(TRAFFIC_RECORD)).get("vcycle_smooth@0")
    except Exception:
        pass
    lvl0 = h.level_dims(0)
    cb0 = h.level_layout(0)["col_bytes"]
    sk0, soff0 = h.level_stencil(0)
    csr_bytes = 12 * lvl0["nnz"] + 4 * (lvl0["nrows"] + 1) + 32 * lvl0["nrows"]
    if sk0:
        kern0 = f"k_dia<OpSmooth,{sk0}> level 0 (post-smoothing sweep, symmetric-stencil form)"
        form0 = (f"(8*({sk0}+1)+1)*n + 32*n  (diagonal + {sk0} upper diagonals {list(soff0)} + 1-byte row mask, "
                 f"then x, f, w read and the output written; DESIGN.md 3.1b)")
    else:
        kern0 = "k_rowpass<OpSmooth> level 0 (post-smoothing sweep)"
        form0 = (f"(8+{cb0})*nnz + 4*(n+1) + 32*n  (SURVEY.md 8(d) SpMV + f,w reads; "
                 f"{cb0}-byte column codes, DESIGN.md 2)")
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "kernel": kern0,
                "bytes_per_launch": pbytes / cnt if cnt else None,
                "bytes_formula": form0,
                "csr_equivalent_GB_s": (csr_bytes / (pms / cnt) / 1e6) if cnt else None,
                "nnz": lvl0["nnz"], "n": lvl0["nrows"], "peak_source": peak_kind, "kernels": extra}

    # ---- whole-phase rooflines (SURVEY.md 8(d) algorithmic bytes from this
    # hierarchy's level shapes): rebuild, one V-cycle, one BiCGStab iteration ----
    dims = [h.level_dims(l) for l in range(h.num_levels())]
    nl = [d["nrows"] for d in dims]
    zl = [d["nnz"] for d in dims]
    Lh = len(dims)
    rap_b = sum(12 * zl[i] + 8 * zl[i + 1] + 4 * nl[i] + 4 * (nl[i + 1] + 1) for i in range(Lh - 1))
    jac_b = sum(20 * nl[i] for i in range(Lh - 1))
    cbl = [h.level_layout(l)["col_bytes"] for l in range(Lh)]
    spmv = [(8 + cbl[i]) * zl[i] + 4 * (nl[i] + 1) + 16 * nl[i] for i in range(Lh)]
    if sk0:  # level 0 in symmetric-stencil form
        spmv[0] = (8 * (sk0 + 1) + 1) * nl[0] + 16 * nl[0]
    vc_b = sum(2 * spmv[i] + 64 * nl[i] for i in range(Lh - 1))
    it_b = 2 * vc_b + 2 * spmv[0] + 192 * nl[0]
    # one V-cycle, device time (stream-launched, 10 repetitions)
    vz = torch.zeros(n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        amg.vcycle_device(h, f.data_ptr(), vz.data_ptr())
    ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record()
        for _ in range(10):
            amg.vcycle_device(h, f.data_ptr(), vz.data_ptr())
        e1.record()
    ctx.synchronize()
    vc_ms = e0.elapsed_time(e1) / 10
    it_ms = solve_ms / max(float(np.mean(iters)), 1.0)

    def phase(bytes_, ms):
        gbs = bytes_ / ms / 1e6
        return {"algorithmic_GB": bytes_ / 1e9, "ms": ms, "GB_s": gbs, "frac_measured_peak": gbs / peak,
                "frac_8TBs_nominal": gbs / 8000.0}

    # the rebuild also refreshes level 0's symmetric-stencil copy (read the CSR
    # values + row starts + masks, write D | U): bytes the reference does not move
    dia_b = ((12 + 8 * (sk0 + 1) + 1) * nl[0] + 8 * zl[0]) if sk0 else 0
    phases = {"rebuild": phase(rap_b + jac_b, rebuild_ms),
              "rebuild_incl_level0_layout": phase(rap_b + jac_b + dia_b, rebuild_ms),
              "vcycle": phase(vc_b, vc_ms),
              "bicgstab_iteration": phase(it_b, it_ms),
              "bytes_formulas": "SURVEY.md 8(d): RAP 12nnz_i+8nnz_i+1+4n_i+4(n_i+1 +1), Jacobi 20n_i, "
                                "V-cycle sum(2 SpMV_i + 64 n_i), iteration 2 V + 2 SpMV_0 + 192 n_0; "
                                "SpMV_i with (8 + column bytes) per entry (level 0 in symmetric-stencil form: "
                                "8 (K+1) + 1 bytes per row)",
              "column_bytes_per_level": cbl, "level0_stencil_pairs": sk0}
    del vz

    # ---- e2e through the C-ABI with host buffers ----
    e2e = None
    if not a.no_e2e:
        hv, hf = [], []
        for k in range(1 + W, 1 + W + K):
            t = torch.empty(nnz, dtype=torch.float64, pin_memory=True)
            t.copy_(vals[k][:nnz])
            hv.append(t)
            t = torch.empty(n, dtype=torch.float64, pin_memory=True)
            t.copy_(f)
            hf.append(t)
        uo = [torch.empty(n, dtype=torch.float64, pin_memory=True) for _ in range(K)]
        ub = [u_start.clone(), torch.empty_like(u)]  # device-resident iterate: u0 = previous solution
        torch.cuda.synchronize()
        hb = L.amgr_bicgstab
        spc = amg._SolveParams(sp.tol, sp.max_iter)
        stc = amg._SolveStats()
        import ctypes

        e_iters = []
        ctx.synchronize()
        barrier()
        e0 = time.perf_counter()
        # per step, through the C-ABI: the step's A_k values and f_k go host ->
        # device on the copy stream (amgr_stage_values / amgr_stage_rhs), issued
        # one step ahead so they overlap the previous solve (the first is
        # exposed); the solution comes back with amgr_download_async, which
        # overlaps the next step; the last download is inside the timed region
        amg._check(L.amgr_stage_values(h._p, hv[0].data_ptr(), amg.HOST), ctx.ptr)
        amg._check(L.amgr_stage_rhs(h._p, hf[0].data_ptr(), amg.HOST), ctx.ptr)
        for j in range(K):
            amg._check(L.amgr_rebuild_values(h._p, None, amg.STAGED), ctx.ptr)
            if j + 1 < K:
                amg._check(L.amgr_stage_values(h._p, hv[j + 1].data_ptr(), amg.HOST), ctx.ptr)
                amg._check(L.amgr_stage_rhs(h._p, hf[j + 1].data_ptr(), amg.HOST), ctx.ptr)
            u_in, u_out = ub[j % 2], ub[(j + 1) % 2]
            amg._check(hb(h._p, None, u_in.data_ptr(), u_out.data_ptr(), ctypes.byref(spc), ctypes.byref(stc),
                          amg.STAGED), ctx.ptr)
            e_iters.append(int(stc.iterations))
            amg._check(L.amgr_download_async(ctx.ptr, u_out.data_ptr(), uo[j].data_ptr(), n), ctx.ptr)
        ctx.synchronize()
        e_ms = (time.perf_counter() - e0) * 1e3 / K
        e2e = {"value": e_ms, "unit": "ms/step", "h2d_bytes_per_step": 8 * nnz + 8 * n,
               "d2h_bytes_per_step": 8 * n, "timer": "host wall clock around the C-ABI calls (sync both sides)",
               "iterations": e_iters,
               "pipelining": "A_k values and f_k staged one step ahead on the copy stream (amgr_stage_values, "
                             "amgr_stage_rhs); solution downloaded on a download stream (amgr_download_async); "
                             "the iterate stays device-resident between steps"}

    # ---- reuse strategies (north star: rebuild / solve / total ms per step for
    # no-reuse, full-reuse and partial-reuse), through the library's own
    # run_sequence driver (reuse.cpp:46-136 semantics) on the same sequence ----
    strategies = None
    if not a.no_strategies:
        from paper_2108_02054_b200 import reuse as R

        strategies = {}
        wn = max(a.strategy_window, 2)
        seq = R.DeviceGridSequence(a.problem, g, wn, ctx=ctx, total=a.nsteps, first=0)
        # warm-up (untimed): a 2-step no-reuse run grows the stream-ordered
        # pool to the setup's peak once, as the main loop's warm-up steps do
        R.run_sequence(R.DeviceGridSequence(a.problem, g, 2, ctx=ctx, total=a.nsteps), R.StrategyConfig(R.StrategyKind.none), prm,
                       sp, ctx=ctx, keep_solutions=False)
        for kind in ("none", "full", "partial"):
            res = R.run_sequence(seq, R.StrategyConfig(R.StrategyKind[kind]), prm, sp, ctx=ctx, keep_solutions=False)
            st = res.report.steps[1:]  # step 0 is the initial full setup for every strategy
            rb = 1e3 * sum(s.setup_time for s in st) / len(st)
            so = 1e3 * sum(s.solve_time for s in st) / len(st)
            strategies[kind] = {"rebuild_ms_per_step": rb, "solve_ms_per_step": so, "total_ms_per_step": rb + so,
                                "iterations": [s.iterations for s in st], "converged": all(s.converged for s in st)}
        if strategies["none"]["iterations"]:
            strategies["partial_over_none_iterations"] = (
                float(np.mean(strategies["partial"]["iterations"])) / float(np.mean(strategies["none"]["iterations"])))
        strategies["note"] = (f"steps 1..{wn - 1} of the {a.nsteps}-step {a.problem} {g}^3 sequence (the bench's own "
                              f"sequence), run_sequence per strategy from step 0; times from the driver's own "
                              "per-step device clocks; 'full' solves with the step-0 hierarchy operator, as the "
                              "reference does (reuse.cpp:104)")
        del seq

    # ---- CPU baseline (rank 0, N=1) ----
    cpu = None
    avg_it = float(np.mean(iters))
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        try:
            A0h = host_problem(g, a.problem, 0, a.nsteps)
            k1 = 1 + W
            Akh = host_problem(g, a.problem, k1 % a.nsteps, a.nsteps)
            fh_np = f.cpu().numpy()
            r = reference_sample(A0h, [Akh], fh_np, avg_it, 1)
            hc = host_cpu()
            cpu = {"value": r["value"], "unit": "ms/step", "cores": 1, "kind": "reference",
                   "sample": (f"bounded sample, EXTRAPOLATED: 1 partial_update of step {k1} timed in full "
                              f"({r['rebuild_ms']:.0f} ms) + fixed-V BiCGStab timed for 2 iterations "
                              f"({r['per_iteration_ms']:.0f} ms/iteration) x {avg_it:.1f} iterations (this run's "
                              f"device average); reference setup {r['setup_s']:.1f} s untimed; unmodified reference, "
                              f"single-threaded as shipped; the measured full reference step is the --impl "
                              f"reference arm; host {hc['model']}, nproc {hc['nproc']}")}
        except Exception as e:  # never let the baseline kill the bench line
            cpu = {"value": None, "unit": "ms/step", "cores": 1, "kind": "reference", "sample": f"failed: {e}"}

    if rank == 0:
        out = {"metric": METRIC, "value": ms_per_step, "unit": "ms/step", "n_gpus": world, "steps": K,
               "warmup": W, "ms_per_step": ms_per_step, "higher_is_better": False, "scaling": "weak",
               "vs_baseline": None, "dtype": "f64", "data": "synthetic (device-generated dam-break sequence)",
               "config": {"workload": f"C3 dam-break {g}^3, partial reuse (BASELINE.json configs[2])",
                          "problem": a.problem, "grid": g, "n": n, "nnz": nnz, "sequence_steps": a.nsteps,
                          "timed_steps": f"{1 + W}..{W + K}", "reuse": "partial", "smoother": "jacobi",
                          "coarse_solve": a.coarse, "levels": h.num_levels(),
                          "operator_complexity": h.operator_complexity(),
                          "parallelism": "replicas" if world > 1 else "single",
                          "l2": "inputs larger than L2 (A_k values 0.94 GB/step)"},
               "rebuild_ms_per_step": rebuild_ms, "solve_ms_per_step": solve_ms, "iterations": iters,
               "converged": all(conv), "setup_s": setup_s, "step0_iterations": st0.iterations,
               "clocks": clk.summary(), "gpu_launches": launches, "roofline": roofline, "e2e": e2e,
               "strategies": strategies, "phase_rooflines": phases,
               "cpu_baseline": cpu}
        emit(out)


if __name__ == "__main__":
    main()
