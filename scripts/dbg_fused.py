"""Debug: compare the fused wave kernels (variant 6) with the stage-wise path set by set."""
import math
import os
import subprocess
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) == 1:
    for stop in ("2", "4"):
        for v in ("0", "6"):
            subprocess.check_call([sys.executable, __file__, v, stop])
    a = {s: np.load(f"/tmp/dbg_0_{s}.npz") for s in ("2", "4")}
    b = {s: np.load(f"/tmp/dbg_6_{s}.npz") for s in ("2", "4")}
    for s in ("2", "4"):
        for key in a[s].files:
            x, y = a[s][key], b[s][key]
            g = 3
            xi, yi = x[:, g:-g, g:-g, g:-g], y[:, g:-g, g:-g, g:-g]
            d = np.abs(xi - yi)
            print(f"stop={s} {key}: max diff interior {d.max():.3e}", end="")
            if d.max() > 0:
                for f in range(d.shape[0]):
                    if d[f].max() > 0:
                        idx = np.argwhere(d[f] > 0)
                        print(f"\n   gf {f}: {len(idx)} pts, z {idx[:,0].min()}-{idx[:,0].max()}, "
                              f"y {idx[:,1].min()}-{idx[:,1].max()}, x {idx[:,2].min()}-{idx[:,2].max()}, "
                              f"max {d[f].max():.3e}", end="")
            print()
    sys.exit(0)

v, stop = int(sys.argv[1]), sys.argv[2]
os.environ["CHEMORA_DEBUG_STOP"] = stop
import paper_1410_1764_b200 as P
from paper_1410_1764_b200 import capi as C

n = (70, 45, 33)
h = tuple(2 * math.pi / x for x in n)
g = P.Grid(C.SYS_WAVE, n, h)
g.set_kernel_variant(v)
g.set_initial(C.INIT_NOISE, seed=2)
g.rk4_step(0.25 * min(h), 1)
out = {}
shape = g.padded_shape()
for sid, name in ((0, "y"), (1, "Q"), (2, "B"), (3, "C")):
    arr = np.zeros(shape)
    C._check(C._lib.chemora_debug_get_set(g.handle, sid, C._dptr(arr), g.stream), "dbg")
    out[name] = arr
np.savez(f"/tmp/dbg_{v}_{stop}.npz", **out)
