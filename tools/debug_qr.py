import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2105_07076_b200 as idk
from oracle import Oracle
o = Oracle()
ctx = idk.context(0)
for mode in (1, 0, 2):
    ctx.set_cpqr_mode(mode)
    for (m, n, k, a) in [(4, 4, 4, np.eye(4)), (8, 6, 6, o.gaussian_matrix(8, 6, 11)), (10, 40, 5, o.gaussian_matrix(10, 40, 3))]:
        f = idk.qr_column_pivoted(torch.from_numpy(np.asfortranarray(a)).cuda(), k)
        torch.cuda.synchronize()
        q, r, perm = f.q.cpu().numpy(), f.r.cpu().numpy(), f.perm.cpu().numpy()
        oq, orr, operm = o.qr_column_pivoted(a, k)
        print("mode", mode, (m, n, k), ctx.cpqr_plan(m, n, k)["kind"], "perm ok", np.array_equal(perm, operm),
              "R err %.2e Q err %.2e" % (np.abs(r - orr).max(), np.abs(q - oq).max()))
        if not np.array_equal(perm, operm) or np.abs(r - orr).max() > 1e-10:
            print(" perm", perm, operm)
            print(" R\n", np.round(r, 4), "\n", np.round(orr, 4))
print("---- pivots via optim_id")
for mode in (1, 0):
    ctx.set_cpqr_mode(mode)
    for (m, n, k, a) in [(8, 6, 6, o.gaussian_matrix(8, 6, 11)), (10, 40, 5, o.gaussian_matrix(10, 40, 3)), (30, 200, 10, o.gaussian_matrix(30, 200, 3))]:
        r = idk.optim_id(torch.from_numpy(np.asfortranarray(a)).cuda(), k)
        _, _, operm = o.qr_column_pivoted(a, k)
        print("mode", mode, (m, n, k), "cols", r.cols.cpu().numpy(), "want", operm[:k])
