"""Per-rank halo and transition volumes of the row partition (partition.py)
of the C3 256^3 dam-break hierarchy at W = 2, 4, 8 — what every level-i pass
of a BiCGStab iteration exchanges per rank.  The hierarchy
structure comes from the unmodified reference (oracle/_ref, host only), so
this runs without a GPU.  TEST INFRASTRUCTURE (imports oracle/).

usage: python tools/halo_volumes.py [g] [replicate_below] > profiles/r02_halo_volumes.json
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import problems as P  # noqa: E402
from oracle import ref  # noqa: E402
from paper_2108_02054_b200 import partition as PT  # noqa: E402


def main():
    g = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    rb = int(sys.argv[2]) if len(sys.argv) > 2 else 150000
    t0 = time.time()
    A = P.grid3d_values("dambreak", g, 1)
    r = ref.setup(A)
    struct = PT.hierarchy_from_oracle(r)
    t_setup = time.time() - t0
    out = {"problem": f"dambreak {g}^3 (C3), levels {len(struct)}, rows per level "
                      f"{[s['n'] for s in struct]}", "replicate_below": rb, "setup_s": t_setup, "worlds": {}}
    for world in (2, 4, 8):
        ranks = []
        t1 = time.time()
        for rank in range(world):
            plan = PT.build_plan(struct, rank, world, rb)
            lv = []
            for L in plan.levels:
                send = int(sum(len(v) for v in L.send.values()))
                recv = int(len(L.halo))
                lv.append({"level": L.level, "owned_rows": int(L.n_own), "local_nnz": int(len(L.col)),
                           "halo_recv_values": recv, "halo_send_values": send,
                           "peers_send": sorted(int(p) for p in L.send), "peers_recv": sorted(int(p) for p in L.recv),
                           "halo_bytes_per_exchange": 8 * (recv + send)})
            tcnt = int((plan.owner[plan.top + 1] == rank).sum())
            ranks.append({"rank": rank, "top": plan.top, "transition_rows": tcnt, "levels": lv})
        # per BiCGStab iteration: 2 V-cycles x 2 halo exchanges per partitioned level + 2 level-0 SpMVs
        per_iter = []
        for R in ranks:
            b = 0
            for L in R["levels"]:
                b += (2 * 2 + (2 if L["level"] == 0 else 0)) * L["halo_bytes_per_exchange"]
            per_iter.append(b)
        out["worlds"][str(world)] = {"ranks": ranks, "plan_s": time.time() - t1,
                                     "halo_bytes_per_bicgstab_iteration_per_rank": per_iter,
                                     "max_halo_MB_per_iteration": max(per_iter) / 1e6}
        print(f"W={world}: max halo {max(per_iter) / 1e6:.2f} MB/iteration/rank, top {ranks[0]['top']}",
              file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
