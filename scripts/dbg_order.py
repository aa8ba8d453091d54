import math, sys
import numpy as np
sys.path.insert(0, '.')
import paper_1410_1764_b200 as P
from paper_1410_1764_b200 import capi as C
v, order = int(sys.argv[1]), int(sys.argv[2])
n = (40, 36, 44)
h = tuple(2 * math.pi / x for x in n)
g = P.Grid(C.SYS_WAVE, n, h, ghost=4, fd_order=order)
g.set_kernel_variant(v)
g.set_initial(C.INIT_NOISE, seed=1)
g.rk4_step(0.1, 2)
print(v, order, 'ok', float(np.abs(g.get_state()).max()))
