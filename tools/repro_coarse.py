import sys; sys.path.insert(0, '.')
import numpy as np
import paper_2108_02054_b200 as amg
from oracle import problems as P
A = P.grid3d_values("dambreak", 128, 10)
for cs in ("inverse", "exact"):
    try:
        h = amg.setup(A, amg.AmgParams(coarse_solve=cs))
        print(cs, "ok levels", h.num_levels(), "coarse n", h.coarse_n())
    except Exception as e:
        print(cs, "FAILED", e)
