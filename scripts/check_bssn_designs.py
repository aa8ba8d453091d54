"""BSSN designs 3 (HBM table) and 4 (fused, on-chip derivatives) on small ragged grids: RHS and one step agree to rounding."""
import faulthandler, sys, math
faulthandler.enable()
sys.path.insert(0, ".")
import numpy as np
import torch
import chemora_inputs as ci
import paper_1410_1764_b200 as P
from paper_1410_1764_b200 import capi as C
for n in [(16, 8, 12), (45, 22, 30), (32, 32, 32)]:
    h = tuple(1.0 / v for v in n)
    y0 = ci.mink_pert(n, h, 1410, eps=1e-2)
    out = {}
    for v in (3, 4):
        g = P.Grid(C.SYS_BSSN, n, h)
        g.set_kernel_variant(v)
        g.set_initial(C.INIT_HOST, y0)
        print("variant", v, n, "rhs ...", flush=True)
        k = g.rhs().cpu().numpy()
        torch.cuda.synchronize()
        print("  rhs ok", flush=True)
        g.rk4_step(0.25 * min(h), 1)
        s = g.get_state()
        out[v] = (k, s)
        g.close()
    dk = max(np.abs(out[3][0][f] - out[4][0][f]).max() / max(np.abs(out[3][0][f]).max(), 1e-12) for f in range(25))
    ds = np.abs(out[3][1] - out[4][1]).max()
    print(n, "rhs rel diff", dk, "state diff", ds, flush=True)
