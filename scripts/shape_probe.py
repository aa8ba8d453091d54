"""Wave pair kernels (variant 6) on equal-size grids of different x extents: does a shorter
padded row (more rows per DRAM page) change the step time?  Timing probe only."""
import math
import sys

import torch

sys.path.insert(0, ".")
import paper_1410_1764_b200 as P
from paper_1410_1764_b200 import capi as C

for n in [(512, 512, 512), (256, 1024, 512), (128, 2048, 512), (1024, 256, 512), (2048, 128, 512)]:
    h = tuple(2 * math.pi / v for v in n)
    g = P.Grid(C.SYS_WAVE, n, h)
    g.set_initial(C.INIT_PLANE_WAVES)
    dt = 0.25 * min(h)
    for _ in range(3):
        g.rk4_step(dt, 1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.rk4_step(dt, 10)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    pts = n[0] * n[1] * n[2]
    print(n, f"{ms:.3f} ms/step", f"{pts / ms / 1e6:.2f} G upd/s", flush=True)
    g.close()
    del g
    torch.cuda.empty_cache()
