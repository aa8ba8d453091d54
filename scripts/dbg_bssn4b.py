import faulthandler, sys, os, traceback
faulthandler.enable()
sys.path.insert(0, ".")
try:
    import numpy as np
    import torch
    import chemora_inputs as ci
    import paper_1410_1764_b200 as P
    from paper_1410_1764_b200 import capi as C
    n = (16, 8, 12)
    h = tuple(1.0 / v for v in n)
    y0 = ci.mink_pert(n, h, 1410, eps=1e-2)
    g = P.Grid(C.SYS_BSSN, n, h)
    g.set_kernel_variant(4)
    g.set_initial(C.INIT_HOST, y0)
    print("init ok", flush=True)
    out = torch.zeros((25, 12, 8, 16), dtype=torch.float64, device="cuda")
    rc = C._lib.chemora_rhs(g.handle, C._vp(out.data_ptr()), None)
    print("rhs rc", rc, C.chemora_last_error(), flush=True)
    e = torch.cuda.synchronize()
    print("sync ok", flush=True)
    print(out.abs().max().item(), flush=True)
except BaseException as ex:
    print("EXC", repr(ex), flush=True)
    traceback.print_exc()
    sys.stdout.flush()
print("end", flush=True)
