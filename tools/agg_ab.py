"""Persistent aggregation replay vs the round-based one (AMGR_AGG_PERSISTENT=0)
on the bench hierarchy: identical aggregates and coarse patterns on every
level.  usage: python tools/agg_ab.py [g] [kind]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_02054_b200 as amg  # noqa: E402
from paper_2108_02054_b200 import reuse as R  # noqa: E402

g = int(sys.argv[1]) if len(sys.argv) > 1 else 256
kind = sys.argv[2] if len(sys.argv) > 2 else "dambreak"
ctx = amg.Context(0)
seq = R.DeviceGridSequence(kind, g, 2, ctx=ctx)
A, _ = seq.step(0)
hp = amg.setup(A, amg.AmgParams(), ctx=ctx)
os.environ["AMGR_AGG_PERSISTENT"] = "0"
hr = amg.setup(A, amg.AmgParams(), ctx=ctx)
assert hp.num_levels() == hr.num_levels()
for l in range(hp.num_levels() - 1):
    same_agg = np.array_equal(hp.level_agg(l), hr.level_agg(l))
    rp1, c1, v1 = hp.level_A(l + 1)
    rp2, c2, v2 = hr.level_A(l + 1)
    same = same_agg and np.array_equal(rp1, rp2) and np.array_equal(c1, c2) and np.array_equal(v1.view(np.int64), v2.view(np.int64))
    print(f"level {l}: aggregates + next level identical: {same}", flush=True)
    assert same
print("ok", hp.num_levels(), "levels")
