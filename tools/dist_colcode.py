"""Column-stream width of every partitioned level at W = 2/4/8 (256^3
dam-break, device-built partition, loopback transport: W ranks in one
process on one GPU; nothing is solved).  Level 0 keeps a coded column stream
at W > 1 (1 byte, or 2 bytes when its halo columns add more than 256 offsets)
instead of int32 columns.  usage: python tools/dist_colcode.py [g] > json"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_02054_b200 as amg  # noqa: E402
from paper_2108_02054_b200 import distributed as D  # noqa: E402
from oracle import problems as P  # noqa: E402

g = int(sys.argv[1]) if len(sys.argv) > 1 else 256
A = P.grid3d_values("dambreak", g, 0)
out = {"problem": f"dambreak {g}^3 step 0", "replicate_below": 150000}
for world in (2, 4, 8):
    lb = D.Loopback(world)
    rows = []
    for r in range(world):
        ctx = amg.Context(0)
        h = amg.setup(A, ctx=ctx)
        ds = D.DistSolver(h, r, world, replicate_below=150000, loopback=lb, device_plan=True)
        lv = []
        for l, L in enumerate(ds.plan.levels):
            lv.append({"level": l, "n_own": L.n_own, "n_halo": len(L.halo), "nnz": L.nnz,
                       "col_bytes": ds.level_col_bytes(l)})
        rows.append({"rank": r, "levels": lv})
        ds.close()
        h.close()
        ctx.close()
    lb.close()
    out[f"W{world}"] = rows
    print(f"W={world}: level-0 col bytes per rank {[x['levels'][0]['col_bytes'] for x in rows]}", file=sys.stderr)
print(json.dumps(out))
