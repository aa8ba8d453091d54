"""Small runs of every stage-kernel design for compute-sanitizer (memcheck / racecheck /
synccheck): wave variants 0, 1, 4 and 8 (incl. the TMA/mbarrier and temporally blocked kernels),
local z-slabs, the energy monitor, BSSN variants 0, 2, 3, 4."""
import math
import sys

sys.path.insert(0, ".")
import torch

import paper_1410_1764_b200 as P
from paper_1410_1764_b200 import capi as C

n = (40, 24, 24)
h = tuple(2 * math.pi / v for v in n)
for v in (0, 1, 4, 8):
    g = P.Grid(C.SYS_WAVE, n, h)
    g.set_kernel_variant(v)
    g.set_initial(C.INIT_NOISE, seed=1)
    g.rk4_step(0.1, 2)
    g.get_state()
    print("wave variant", v, "ok", flush=True)
g = P.Grid(C.SYS_WAVE, n, h)
g.set_monitor(True)
g.set_initial(C.INIT_NOISE, seed=1)
g.rk4_step(0.1, 2)
print("monitor", g.read_monitor(), flush=True)
s = P.LocalSlabs(C.SYS_WAVE, (24, 16, 32), (0.3,) * 3, 2)
s.set_initial(C.INIT_NOISE, seed=1)
s.rk4_step(0.05, 2)
s.get_state()
print("slabs ok", flush=True)
nb = (20, 12, 12)
hb = tuple(1.0 / v for v in nb)
for v in (0, 2, 3, 4):
    g = P.Grid(C.SYS_BSSN, nb, hb)
    g.set_kernel_variant(v)
    g.set_initial(C.INIT_MINK_PERT, kind_params=[1e-3], seed=1)
    g.rk4_step(0.25 * hb[0], 1)
    g.get_state()
    print("bssn variant", v, "ok", flush=True)
torch.cuda.synchronize()
print("done")
