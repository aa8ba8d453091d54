"""Worker of tests/test_gpu_ipc_procs.py (imported by spawned processes): one z-slab rank of
a cross-process run on ONE device.  Gloo process group for the bootstrap (peer-record
exchange) and for the host barrier that ends every phase (chemora_set_phase_barrier), so no
stream ever waits on another process's work; the halo exchange itself runs through the
CUDA-IPC mappings of the neighbours' workspaces (the stage kernels store their boundary
planes into the neighbours' ghost planes) and the stream-memop epoch flags."""
from __future__ import annotations

import math
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(rank, world, port, case, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        import numpy as np
        import torch
        import torch.distributed as dist
        import chemora_inputs as ci
        import paper_1410_1764_b200 as P
        from paper_1410_1764_b200 import capi as C

        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        system = C.SYS_WAVE if case["system"] == "wave" else C.SYS_BSSN
        n = tuple(case["n"])
        h = tuple(case["L"] / v for v in n)
        g = P.Grid(system, n, h, rank=rank, nranks=world, params=case.get("params"))
        if case.get("variant") is not None:
            g.set_kernel_variant(case["variant"])
        g.connect_ipc(host_barrier=True)
        if case.get("monitor"):
            g.set_monitor(True)
        nz = g.local_extent[2]
        if case["init"] == "host":
            y0 = ci.noise(n, C.N_GF[system], seed=case["seed"]) if system == C.SYS_WAVE else \
                ci.mink_pert(n, h, case["seed"], eps=case["eps"])
            g.set_initial(C.INIT_HOST, np.ascontiguousarray(y0[:, g.z0:g.z0 + nz]))
        elif system == C.SYS_WAVE:   # device-generated, keyed by the GLOBAL index (z0 offset)
            g.set_initial(C.INIT_NOISE, seed=case["seed"])
        else:
            g.set_initial(C.INIT_MINK_PERT, kind_params=[case["eps"]], seed=case["seed"])
        out = {"z0": g.z0, "init_pad": g.get_state(padded=True)}
        dt = 0.25 * min(h)
        g.rk4_step(dt, case["steps"])
        out["state"] = g.get_state()
        out["pad"] = g.get_state(padded=True)
        out["norms"] = g.norms()
        if case.get("monitor"):
            out["monitor"] = g.read_monitor()
        if system == C.SYS_BSSN:
            out["cnorms"] = g.constraint_norms()
        torch.cuda.synchronize()
        g.close()
        q.put((rank, out))
    except Exception:
        q.put((rank, traceback.format_exc()))
    finally:
        try:
            import torch.distributed as dist
            dist.destroy_process_group()
        except Exception:
            pass
