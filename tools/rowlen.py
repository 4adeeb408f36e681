import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2108_02054_b200 as amg
ctx = amg.Context(0); L = amg.lib(); g = 256; n = g**3; nnz = int(L.amgr_problem_nnz(g))
rp = torch.empty(n+1, dtype=torch.int32, device='cuda'); ci = torch.empty(nnz+8, dtype=torch.int32, device='cuda'); v = torch.empty(nnz+8, dtype=torch.float64, device='cuda')
torch.cuda.synchronize()
amg._check(L.amgr_problem_pattern(ctx.ptr, g, rp.data_ptr(), ci.data_ptr()), ctx.ptr)
amg._check(L.amgr_problem_values(ctx.ptr, 2, g, 1, 50, v.data_ptr()), ctx.ptr)
ctx.synchronize()
h = amg.setup(amg.DeviceCsr(n, n, nnz, rp.data_ptr(), ci.data_ptr(), v.data_ptr()), ctx=ctx)
for l in range(3, h.num_levels()):
    r, c, _ = h.level_A(l)
    d = np.diff(r)
    print(l, len(d), 'max row', d.max(), 'mean', round(d.mean(),1), 'p99', np.percentile(d, 99))
