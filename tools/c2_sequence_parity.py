"""C2-geometry partial-reuse sequence, device vs the unmodified reference
(oracle/_ref), step by step.  TEST INFRASTRUCTURE (imports oracle/).

For the 128^3 moving-blob sequence (20 steps, the reference's damped-Jacobi
smoother, exact coarse solve) the device runs run_sequence's partial-reuse
step (rebuild on the frozen transfers, BiCGStab from the previous solution,
reuse.cpp:85-114) in both dot orders.  For every step the reference then
solves the SAME system — partial_update(setup(A_0), A_k) and bicgstab over the
fixed V-cycle from the same u0 (the device's previous solution) — in a pool of
host processes.  Recorded per step: iterations of both, |delta|, convergence,
the device solution's true residual by the reference's spmv, and (sequential
dots) whether the final iterate is bit-identical.

usage: python tools/c2_sequence_parity.py [g] [nsteps] [workers] > out.json
"""
import json
import multiprocessing as mp
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

KIND = "blob"


def ref_step(args):
    g, nsteps, k, u0_path, tmp = args
    from oracle import problems as P
    from oracle import ref

    A0 = P.grid3d_values(KIND, g, 0, nsteps)
    r0 = ref.setup(A0)
    Ak = P.grid3d_values(KIND, g, k, nsteps) if k else A0
    rk = ref.partial_update(r0, Ak) if k else r0
    f = P.rhs(g ** 3)
    u0 = np.load(u0_path) if u0_path else None
    t0 = time.perf_counter()
    rs = ref.bicgstab(rk, f, u0=u0, fixed=True)
    out = os.path.join(tmp, f"ref_{os.path.basename(u0_path or 'zero')}_{k}.npy")
    np.save(out, rs.u)
    return {"k": k, "u0": u0_path, "iterations": rs.iterations, "converged": rs.converged,
            "relative_residual": rs.relative_residual, "seconds": time.perf_counter() - t0, "u": out}


def main():
    g = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    nsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    workers = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    import paper_2108_02054_b200 as amg
    from oracle import problems as P
    from oracle import ref

    tmp = tempfile.mkdtemp(prefix="c2par_")
    n = g ** 3
    f = P.rhs(n)
    dev = {}
    for mode in ("blocked", "sequential"):
        ctx = amg.Context(0)
        ctx.sequential_dots = mode == "sequential"
        A0 = P.grid3d_values(KIND, g, 0, nsteps)
        h = amg.setup(A0, amg.AmgParams(coarse_solve="exact"), ctx=ctx)
        u_prev = None
        steps = []
        for k in range(nsteps):
            Ak = P.grid3d_values(KIND, g, k, nsteps)
            if k:
                h.rebuild_values(Ak[2])
            u0_path = None
            if u_prev is not None:
                u0_path = os.path.join(tmp, f"{mode}_u{k - 1}.npy")
                np.save(u0_path, u_prev)
            t0 = time.perf_counter()
            u, st = amg.bicgstab(h, f, u_prev)
            dt = time.perf_counter() - t0
            res = float(np.linalg.norm(f - ref.spmv(Ak, u)) / np.linalg.norm(f))
            upath = os.path.join(tmp, f"{mode}_dev_{k}.npy")
            np.save(upath, u)
            steps.append({"k": k, "iterations": st.iterations, "converged": bool(st.converged),
                          "relative_residual": st.relative_residual, "true_residual_ref_spmv": res,
                          "u0": u0_path, "u": upath, "solve_s": dt})
            u_prev = u
            print(f"[device {mode}] step {k}: {st.iterations} iterations, true residual {res:.3e}",
                  file=sys.stderr, flush=True)
        dev[mode] = steps
        del h, ctx
    jobs = [(g, nsteps, s["k"], s["u0"], tmp) for mode in dev for s in dev[mode]]
    with mp.get_context("spawn").Pool(workers) as pool:
        refs = pool.map(ref_step, jobs)
    out = {"workload": f"C2 geometry: {KIND} {g}^3, {nsteps}-step sequence, partial reuse, damped Jacobi "
                       "(the reference's smoother), exact coarse solve, tol 1e-8",
           "per_step_protocol": "device runs the sequence; the reference solves each step's system from the "
                                "device's previous solution (same A_k, hierarchy, f, u0)",
           "host_cores": os.cpu_count()}
    i = 0
    for mode in dev:
        rows = []
        for s in dev[mode]:
            r = refs[i]
            i += 1
            same = bool(np.array_equal(np.load(s["u"]).view(np.int64), np.load(r["u"]).view(np.int64)))
            rows.append({"k": s["k"], "device_iterations": s["iterations"], "reference_iterations": r["iterations"],
                         "abs_delta": abs(s["iterations"] - r["iterations"]), "device_converged": s["converged"],
                         "reference_converged": r["converged"],
                         "device_true_residual_by_ref_spmv": s["true_residual_ref_spmv"],
                         "final_iterate_bit_identical": same, "device_solve_s": s["solve_s"],
                         "reference_solve_s": r["seconds"]})
        d = [r["abs_delta"] for r in rows]
        out[mode] = {"steps": rows, "mean_abs_delta": float(np.mean(d)), "max_abs_delta": int(np.max(d)),
                     "all_converged": all(r["device_converged"] and r["reference_converged"] for r in rows),
                     "max_true_residual": max(r["device_true_residual_by_ref_spmv"] for r in rows),
                     "bit_identical_steps": sum(r["final_iterate_bit_identical"] for r in rows)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
