"""L2 probe: run a few wave steps on a small grid (whole state fits in L2) with a given
kernel variant, for ncu to report DRAM bytes per stage kernel."""
import math
import sys

sys.path.insert(0, ".")
import torch

import paper_1410_1764_b200 as P
from paper_1410_1764_b200 import capi as C

v = int(sys.argv[1])
N = int(sys.argv[2]) if len(sys.argv) > 2 else 64
n = (N, N, N)
h = tuple(2 * math.pi / x for x in n)
g = P.Grid(C.SYS_WAVE, n, h)
g.set_kernel_variant(v)
g.set_initial(C.INIT_NOISE, seed=1)
for _ in range(3):
    g.rk4_step(0.25 * h[0], 1)
torch.cuda.synchronize()
print("ok", v, N)
