import sys, os
sys.path.insert(0, os.getcwd())
os.environ["AMGR_TRACE_SETUP"] = "1"
import paper_2108_02054_b200 as amg
from oracle import problems as P
kind, g = sys.argv[1], int(sys.argv[2])
A = P.grid3d_values(kind, g, 7)
try:
    h = amg.setup(A, amg.AmgParams(coarsening='smoothed'))
    print("ok", h.num_levels())
except Exception as e:
    print("ERR", e)
