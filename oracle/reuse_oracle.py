"""TEST INFRASTRUCTURE ONLY — restatement of the reference's run_sequence
(proj/src/reuse.cpp:46-136) over the C oracle (oracle/oracle.py): the action
rules, initial-guess chaining and the full-reuse rebuild flag.  Returns the
per-step (action, iterations, converged) tuples the device driver must match.
"""
from oracle import oracle as O

FULL_BUILD, PARTIAL_UPDATE, REUSED_UNCHANGED = 0, 1, 2


def run_sequence(systems, kind, reuse_iter_limit=0, rebuild_every=None, prm=None, tol=1e-8, max_iter=100,
                 escalate=False):
    prm = prm or O.params()
    iter_limit = reuse_iter_limit if reuse_iter_limit > 0 else max_iter
    if iter_limit > max_iter:
        raise ValueError("run_sequence: reuse_iter_limit exceeds max_iter")
    h = None
    rebuild_flag = False
    prev = None
    out = []
    for k in range(systems.size()):
        A, rhs = systems.step(k)
        n = len(A[0]) - 1
        dims_changed = h is not None and n != len(h.levels[0].A[0]) - 1
        if kind == "none":
            act = FULL_BUILD
        elif kind == "full":
            act = FULL_BUILD if (h is None or dims_changed or rebuild_flag) else REUSED_UNCHANGED
        else:
            periodic = rebuild_every is not None and k > 0 and k % rebuild_every == 0
            # extension (AMGR_STRATEGY_ESCALATE): the full-reuse rule applied to partial reuse
            act = FULL_BUILD if (h is None or dims_changed or periodic or (escalate and rebuild_flag)) \
                else PARTIAL_UPDATE
        if act == FULL_BUILD:
            h = O.setup(A, prm)
        elif act == PARTIAL_UPDATE:
            h = O.partial_update(h, A, prm)
        u0 = prev if prev is not None and len(prev) == n else None
        s = O.bicgstab(h, rhs, u0, tol, max_iter)
        if kind == "full" or (kind == "partial" and escalate):
            rebuild_flag = (not s.converged) or s.iterations >= iter_limit
        prev = s.u
        out.append((act, s.iterations, s.converged, s.u))
    return out
