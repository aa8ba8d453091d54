"""The cross-process z-slab path on hardware (PAPER.md:200-207 driver decomposition, 346
ghost-zone exchange): 2 and 3 processes on ONE B200, each owning a z-slab of one global
periodic grid, connected through chemora_grid_connect_ipc (CUDA-IPC mappings of the
neighbours' workspaces; the stage kernels store their boundary planes straight into the
neighbours' ghost planes; stream-memop epoch flags order the phases).  The ranks share one
device, so every phase also ends with a host (gloo) barrier -- chemora_set_phase_barrier --
and no stream ever waits on another process's work (B200_PROFILING.md: ranks on one GPU must
not wait on each other on the device).

Checks: the gathered state is BITWISE the single-grid GPU state and element-wise within
north_star's tolerance of the CPU oracle; the ghosts after the step are the periodic fill;
the collective chemora_norms / chemora_constraint_norms / chemora_read_monitor agree on every
rank and with the oracle."""
from __future__ import annotations

import math
import os
import socket

import numpy as np
import pytest

import chemora_inputs as ci
import oracle

pytestmark = pytest.mark.gpu
GENERIC = [1.5, 2.0, 0.7, 0.3, 0.8, 0.6, 1.0, 0.5, 0.9, 0.7]


def _mods():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1410_1764_b200 as P
    from paper_1410_1764_b200 import capi as C
    return P, C


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spawn(world, case, timeout=300):
    import torch.multiprocessing as mp
    from tests import ipc_worker
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=ipc_worker.run, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in range(world):
            r, out = q.get(timeout=timeout)
            res[r] = out
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for r in range(world):
        assert isinstance(res[r], dict), f"rank {r} failed:\n{res[r]}"
    return [res[r] for r in range(world)]


def relerr(a, b):
    top = max(np.abs(b[f]).max() for f in range(b.shape[0]))
    return max(np.abs(a[f] - b[f]).max() / max(np.abs(b[f]).max(), 1e-6 * top) for f in range(b.shape[0]))


def _single(P, C, case):
    system = C.SYS_WAVE if case["system"] == "wave" else C.SYS_BSSN
    n = tuple(case["n"])
    h = tuple(case["L"] / v for v in n)
    g = P.Grid(system, n, h, params=case.get("params"))
    if case.get("variant") is not None:
        g.set_kernel_variant(case["variant"])
    # the oracle's input comes from the seeded generators (chemora_inputs), never the GPU
    y0 = ci.noise(n, C.N_GF[system], seed=case["seed"]) if system == C.SYS_WAVE else \
        ci.mink_pert(n, h, case["seed"], eps=case["eps"])
    if case["init"] == "host":
        g.set_initial(C.INIT_HOST, y0)
    else:
        assert system == C.SYS_WAVE
        g.set_initial(C.INIT_NOISE, seed=case["seed"])
    assert np.array_equal(g.get_state(), y0)  # device noise == the host recipe, bit for bit
    g.rk4_step(0.25 * min(h), case["steps"])
    return g, y0, h


def _check(world, case, tol):
    P, C = _mods()
    res = _spawn(world, case)
    g, y0, h = _single(P, C, case)
    ref_gpu = g.get_state()
    got = np.concatenate([r["state"] for r in res], axis=1)
    assert [r["z0"] for r in res] == [k * case["n"][2] // world for k in range(world)]
    # the initial ghosts were filled across the process boundary (the set_initial ordering)
    init_pad = [r["init_pad"] for r in res]
    gg = 3
    full0 = np.pad(y0, ((0, 0), (gg, gg), (gg, gg), (gg, gg)), mode="wrap")
    for k, pad in enumerate(init_pad):
        z0 = res[k]["z0"]
        assert np.array_equal(pad, full0[:, z0:z0 + pad.shape[1]]), f"rank {k}: initial ghosts"
    # bitwise equal to the single-grid GPU run, ghosts included
    assert np.array_equal(got, ref_gpu)
    full = np.pad(ref_gpu, ((0, 0), (gg, gg), (gg, gg), (gg, gg)), mode="wrap")
    for k, r in enumerate(res):
        assert np.array_equal(r["pad"], full[:, r["z0"]:r["z0"] + r["pad"].shape[1]]), f"rank {k}: ghosts"
    # element-wise against the CPU oracle
    sysid = oracle.WAVE if case["system"] == "wave" else oracle.BSSN
    ref = oracle.rk4(sysid, y0, h, 0.25 * min(h), case["steps"], case.get("params"))
    assert relerr(got, ref) <= tol
    # collective norms: identical on every rank, equal to the oracle's global norms
    for r in res[1:]:
        assert np.array_equal(r["norms"], res[0]["norms"])
    onorm = oracle.norms(sysid, ref, h)
    np.testing.assert_allclose(res[0]["norms"], onorm, rtol=1e-11, atol=1e-13 * np.abs(onorm).max())
    if "monitor" in res[0]:
        e = res[0]["monitor"]
        assert len(e) == case["steps"]
        for r in res[1:]:
            assert np.array_equal(r["monitor"], e)
        if case["system"] == "wave":   # energy after the last step
            assert e[-1] == pytest.approx(onorm[-1], rel=1e-12)
        else:                          # constraint norms of the state entering step 1
            c = oracle.constraints(y0, h)
            vol = h[0] * h[1] * h[2]
            oc = np.array([[math.sqrt(vol * (c[q] ** 2).sum()), np.abs(c[q]).max()] for q in range(7)]).ravel()
            np.testing.assert_allclose(e[0], oc, rtol=1e-10, atol=1e-10 * np.abs(oc).max())
    if "cnorms" in res[0]:
        for r in res[1:]:
            assert np.array_equal(r["cnorms"], res[0]["cnorms"])
        c = oracle.constraints(ref, h)
        vol = h[0] * h[1] * h[2]
        oc = np.array([[math.sqrt(vol * (c[q] ** 2).sum()), np.abs(c[q]).max()] for q in range(7)]).ravel()
        np.testing.assert_allclose(res[0]["cnorms"], oc, rtol=1e-8, atol=1e-10 * np.abs(oc).max())
    g.close()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("variant,init", [(8, "host"), (8, "device"), (0, "host")])
def test_wave_ipc_processes(world, variant, init):
    case = {"system": "wave", "n": (24, 20, 48), "L": 2 * math.pi, "init": init, "seed": 77,
            "steps": 3, "variant": variant, "monitor": True}
    _check(world, case, 1e-12)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("variant", [3, 4])
def test_bssn_ipc_processes(world, variant):
    case = {"system": "bssn", "n": (20, 16, 36), "L": 1.0, "init": "host", "seed": 1410,
            "eps": 1e-2, "steps": 2, "params": GENERIC, "variant": variant, "monitor": True}
    _check(world, case, 1e-10)
