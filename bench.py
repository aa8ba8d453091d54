#!/usr/bin/env python
"""Benchmark of the fused RK4 finite-difference step (BASELINE.json metric:
"grid-point updates/s per RK4 step (fp64) at 1/2/4/8 B200; % HBM roofline").

Default workload (N=1): configs[1], the scalar wave equation Eq. 1,
4th-order FD, 512^3 fp64, periodic, 3 ghosts, fused RHS + RK4 update.  A step is one
classical RK4 step of the whole grid: for the wave by default two temporally blocked kernels
(stages 1+2, 3+4), for BSSN a derivative + two algebra kernels per stage.  Inputs (23 GB of state)
are larger than the 126 MB L2, so no explicit flush is needed between steps.

Multi-GPU (torchrun, one process per GPU): z-slab decomposition, 512^3 per GPU (weak
scaling; global grid 512 x 512 x 512N), halo exchange fused into the stage kernels over
CUDA-IPC peer memory with stream-memop flags.

``--impl reference``: the CPU oracle (oracle/), timed as it stands on this host's cores on a
bounded sample of the same workload (there is no reference implementation of the paper).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

BYTES_PER_POINT = {"wave": 432, "bssn": 2400}   # DESIGN.md §Roofline (one HBM pass per stage)
METRIC = "grid-point updates/s per RK4 step (fp64)"


def measured_peaks():
    p = os.path.join(HERE, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def _traffic_table():
    p = os.path.join(HERE, "profiles", "r1_traffic.json")
    if os.path.exists(p):
        with open(p) as fh:
            return json.load(fh)
    return {}


def measured_traffic(config: str, variant: int):
    """DRAM bytes per step from the committed ncu capture of this config/variant (or None)."""
    t = _traffic_table().get(config, {}).get(str(variant))
    return None if t is None else t.get("dram_bytes_per_step")


def bssn_fp64_roofline(pts: int, step_s: float, variant: int):
    """fp64-pipe roofline for the BSSN step: thread-level fp64 instructions per point-update
    of this kernel design (ncu sm__inst_executed_pipe_fp64 x 32 / points, committed in
    profiles/r1_traffic.json) vs 148 SMs x 64 fp64 lanes x the max SM clock."""
    tab = _traffic_table().get("bssn192", {})
    t = tab.get(str(variant), {}).get("fp64_thread_instr_per_point_step") or \
        tab.get("fp64_thread_instr_per_point_step")
    if not t:
        return {}
    peak_inst = 148 * 64 * 1.965e9  # fp64 thread-instructions / s at max clock (DFMA = 2 flops)
    achieved = t * pts / step_s
    return {"bound": "alu", "pipe": "fp64", "achieved": achieved / 1e12, "peak": peak_inst / 1e12,
            "unit": "T fp64 thread-instr/s", "frac": achieved / peak_inst,
            "fp64_instr_per_point_step": t,
            "hbm_frac_at_2400_bytes": 2400 * pts / step_s / 1e9 / measured_peaks()[0]}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index=0, period_ms=100):
        self.index, self.period = index, period_ms
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", str(self.period)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_cores():
    n = os.environ.get("OMP_NUM_THREADS")
    return int(n) if n else os.cpu_count()


def oracle_sample(system: str, seconds_target: float = 15.0):
    """Time the CPU oracle as it stands on a bounded sample of the workload: the same
    per-point RK4 step on a smaller periodic grid, repeated until ~seconds_target."""
    import chemora_inputs as ci
    import oracle
    if system == "wave":
        n = 160
        h = (2 * math.pi / n,) * 3
        y = ci.noise((n, n, n), 5, seed=1410)
        sysid = oracle.WAVE
        params = None
    else:
        n = 48
        h = (1.0 / n,) * 3
        y = ci.mink_pert((n, n, n), h, seed=1410)
        sysid = oracle.BSSN
        params = oracle.default_bssn_params()
    dt = 0.25 * h[0]
    steps, elapsed = 0, 0.0
    while elapsed < seconds_target:
        t0 = time.perf_counter()
        y = oracle.rk4(sysid, y, h, dt, 1, params)
        elapsed += time.perf_counter() - t0
        steps += 1
    return {"value": n ** 3 * steps / elapsed, "unit": "grid-point updates/s", "cores": cpu_cores(),
            "kind": "oracle", "sample": f"{system} {n}^3 periodic, {steps} RK4 steps, "
            f"{elapsed:.1f} s, OMP over z"}, n, steps, elapsed


def run_reference(args, world, rank):
    if rank != 0:
        return 0
    # rank 0 runs the oracle alone (the other ranks exit), so it gets the host's cores even
    # under torchrun, which defaults OMP_NUM_THREADS to 1 (read when liboracle loads)
    os.environ["OMP_NUM_THREADS"] = str(len(os.sched_getaffinity(0)))
    cfg = workload(args)
    per = max(2.0, 20.0 / max(1, args.steps + args.warmup))
    for _ in range(args.warmup):
        oracle_sample(cfg["system"], per / 4)
    cb, n, steps, elapsed = oracle_sample(cfg["system"], per * args.steps)
    line = {"metric": METRIC, "value": cb["value"], "unit": "grid-point updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / steps,
            "higher_is_better": True, "scaling": "strong" if cfg.get("strong") else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference", "config": cfg["config"],
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "grid-point updates/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def workload(args):
    if args.config == "wave512":
        n = (512, 512, 512)
        return {"system": "wave", "n": n,
                "config": {"workload": "scalar wave eq (Eq. 1), 4th-order FD, 512^3 fp64 per GPU, "
                           "periodic, 3 ghost zones, fused RHS+RK4 (configs[1])",
                           "grid": list(n), "ghost": 3, "fd_order": 4, "init": "PW3 plane waves",
                           "l2": "state (23 GB) larger than L2; no flush needed"}}
    if args.config == "bssn192":
        n = (192, 192, 192)
        return {"system": "bssn", "n": n,
                "config": {"workload": "BSSN-like 25-GF Einstein RHS with upwinded advection, "
                           "192^3 fp64 per GPU, periodic, 3 ghost zones, fused RHS+RK4 (configs[2])",
                           "grid": list(n), "ghost": 3, "fd_order": 4, "init": "MINK_PERT eps=1e-3",
                           "l2": "state (6.2 GB) larger than L2; no flush needed"}}
    if args.config == "wave1024":
        n = (1024, 1024, 1024)
        return {"system": "wave", "n": n, "strong": True,
                "config": {"workload": "scalar wave eq (Eq. 1), 4th-order FD, 1024^3 fp64 global, "
                           "z-slabs over the GPUs (strong scaling, configs[3]; needs >= 2 GPUs)",
                           "grid": list(n), "ghost": 3, "fd_order": 4, "init": "PW3 plane waves",
                           "l2": "state larger than L2; no flush needed"}}
    if args.config == "bssn384":
        n = (384, 384, 384)
        return {"system": "bssn", "n": n,
                "config": {"workload": "BSSN-like 25-GF Einstein RHS with upwinded advection, "
                           "384^3 fp64 per GPU (weak scaling, configs[4])",
                           "grid": list(n), "ghost": 3, "fd_order": 4, "init": "MINK_PERT eps=1e-3",
                           "l2": "state larger than L2; no flush needed"}}
    raise SystemExit(f"unknown config {args.config}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="chemora", choices=["chemora", "reference"])
    ap.add_argument("--config", default="wave512", choices=["wave512", "bssn192", "wave1024", "bssn384"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    # e2e steps: enough that the pipeline fill (first upload) and drain (last download) are
    # amortised -- per step the two PCIe directions then overlap (scripts/pcie_probe.py)
    ap.add_argument("--e2e-steps", type=int, default=12)
    ap.add_argument("--variant", type=int, default=None, help="stage-kernel variant (testing)")
    ap.add_argument("--fd-order", type=int, default=4, choices=[2, 4, 6, 8],
                    help="wave: accuracy order of the centered stencils (NEXT-1, PAPER.md:512-514)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, world, rank)

    import torch
    import torch.distributed as dist
    import paper_1410_1764_b200 as P
    from paper_1410_1764_b200 import capi as C

    # ranks sharing a device (fewer GPUs than ranks, e.g. a 1-GPU box): gloo bootstrap and a
    # host barrier after every phase (chemora_set_phase_barrier) -- no stream then waits on
    # another process's work; with one GPU per rank: NCCL group, device-side phase ordering
    ndev = torch.cuda.device_count()
    shared = world > ndev
    if shared:
        local = local % ndev
    torch.cuda.set_device(local)
    watchdog = None
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        # the multi-rank step orders its phases with stream waits on neighbour flags; if a
        # peer never signals, fail the run instead of hanging it (CHEMORA_BENCH_DEADLINE s)
        def _abort():
            print(f"rank {rank}: bench exceeded CHEMORA_BENCH_DEADLINE, aborting", file=sys.stderr, flush=True)
            os._exit(3)
        watchdog = threading.Timer(float(os.environ.get("CHEMORA_BENCH_DEADLINE", "900")), _abort)
        watchdog.daemon = True
        watchdog.start()
    cfg = workload(args)
    n = cfg["n"]
    system = C.SYS_WAVE if cfg["system"] == "wave" else C.SYS_BSSN
    strong = cfg.get("strong", False)
    if strong and (world < 2 or n[2] % world):
        raise SystemExit(f"{args.config} is a strong-scaling config for 2/4/8 GPUs (z divisible by N)")
    # weak scaling: n per GPU, the global z extent grows with N; strong: n is the global grid
    gext = (n[0], n[1], n[2]) if strong else (n[0], n[1], n[2] * world)
    L = 2 * math.pi if system == C.SYS_WAVE else 1.0
    h = (L / n[0], L / n[1], L / n[2])
    dt = 0.25 * min(h)
    order = args.fd_order if system == C.SYS_WAVE else 4
    ghost = max(3, order // 2)
    if order != 4:
        cfg["config"] = dict(cfg["config"], fd_order=order, ghost=ghost)
    g = P.Grid(system, gext, h, device=local, rank=rank, nranks=world, ghost=ghost, fd_order=order)
    if args.variant is not None:
        g.set_kernel_variant(args.variant)
    if world > 1:
        g.connect_ipc(host_barrier=shared)
    init = C.INIT_PLANE_WAVES if system == C.SYS_WAVE else C.INIT_MINK_PERT
    g.set_initial(init, seed=1410)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        g.rk4_step(dt, 1)
    barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(local) as clk:
        barrier()
        ev[0].record(stream)
        for s in range(args.steps):
            g.rk4_step(dt, 1)
            ev[s + 1].record(stream)
        barrier()
    step_ms = [ev[s].elapsed_time(ev[s + 1]) for s in range(args.steps)]
    total_ms = ev[0].elapsed_time(ev[-1])
    if world > 1:
        t = torch.tensor([total_ms], device="cpu" if shared else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    pts_local = n[0] * n[1] * (n[2] // world if strong else n[2])
    value = pts_local * world * args.steps / (total_ms * 1e-3)

    # roofline of the dominant kernel(s): the kernels of one RK4 step are the only launches in
    # the timed region.  Algorithmic bytes are those of the active kernel design: 432 B/pt for
    # one kernel per RK stage, 256 B/pt for the temporally blocked stage
    # pairs -- the frac is against that design's own HBM floor.
    peak, peak_kind = measured_peaks()
    mean_step_s = float(np.mean(step_ms)) * 1e-3
    variant = g.kernel_variant()
    floor_bpp = BYTES_PER_POINT[cfg["system"]]
    pair_kernels = cfg["system"] == "wave" and variant in (6, 7, 8)   # temporally blocked pairs
    bpp = 256 if pair_kernels else floor_bpp
    achieved = bpp * pts_local / mean_step_s / 1e9
    traffic = measured_traffic(args.config, variant) if order == 4 else None
    kname = ({6: "wave_fused<A>, wave_fused<B>", 7: "wave_fused2<A>, wave_fused2<B>",
              8: "wave_fused3<A>, wave_fused3<B>"}.get(variant, "") + " (2 launches = 1 step)" if bpp == 256 else
             "stage kernels (4 launches x groups = 1 step)")
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_source": peak_kind,
                "kernel": kname, "variant": variant,
                "algorithmic_bytes_per_point": bpp,
                "traffic_note": "ncu dram__bytes_read+write per step (all launches of one step), profiles/r1_traffic.json",
                "one_pass_per_stage_bytes_per_point": floor_bpp,
                "frac_at_one_pass_per_stage_bytes": floor_bpp * pts_local / mean_step_s / 1e9 / peak,
                "frac_of_nominal_8TBps": achieved / 8000.0}
    # our kernel launches per RK4 step: wave 2 (stage pairs) or 4 (one per stage); BSSN
    # 4 (two-phase table kernel, variant 0, or fused single kernel, 1) or 3 fissioned
    # groups x 4 stages (variant 2), or derivative + 2 algebra kernels x 4 stages (variant 3)
    if cfg["system"] == "wave":
        launches_per_step = 2 if pair_kernels else 4
    else:
        launches_per_step = 12 if variant in (2, 3) else 4
    if cfg["system"] == "bssn":
        # BSSN is bound by the fp64 pipe: fp64 instructions per point-update
        # counted by ncu (profiles/r1_traffic.json) against 64 DFMA lanes/SM/clock.
        roofline.update(bssn_fp64_roofline(pts_local, mean_step_s, variant))

    # e2e through the public API with host buffers: per step, upload the state from pinned
    # host memory, one RK4 step, download the state.  On one GPU two grid handles alternate on
    # two streams (chemora_upload_state / chemora_download_state are stream-ordered), so one
    # step's download overlaps the next step's upload on the two copy engines; every step
    # still moves its full input and output through PCIe inside the timed region.
    e2e = None
    if args.e2e_steps > 0:
        shape = g.interior_shape()
        nbytes = int(np.prod(shape)) * 8
        # on one GPU up to three grid handles take turns on their own streams, so one
        # handle's upload, another's step and a third's download overlap (H2D engine, SMs,
        # D2H engine); each step still moves its whole input and output over PCIe
        # pinned host buffers: 2 per handle per rank on this node, kept under half the RAM
        import psutil
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
        max_nb = int(0.5 * psutil.virtual_memory().available // (2 * nbytes * local_world))
        grids = [g]
        while (world == 1 and len(grids) < min(3, max_nb)
               and torch.cuda.mem_get_info()[0] > g.nbytes + (2 << 30)):
            g2 = P.Grid(system, gext, h, device=local, rank=rank, nranks=world, ghost=ghost, fd_order=order)
            if args.variant is not None:
                g2.set_kernel_variant(args.variant)
            grids.append(g2)
        nb = len(grids)
        pipelined = nb > 1
        if max_nb < 1:
            raise SystemExit(f"e2e: {2 * nbytes * local_world / 2**30:.0f} GiB of pinned host buffers "
                             f"do not fit this node's RAM; rerun with --e2e-steps 0")
        host_in = [torch.empty(shape, dtype=torch.float64, pin_memory=True) for _ in range(nb)]
        host_out = [torch.empty(shape, dtype=torch.float64, pin_memory=True) for _ in range(nb)]
        g.get_state(out=host_in[0].numpy())
        for t in host_in[1:]:
            t.copy_(host_in[0])
        streams = [torch.cuda.Stream() for _ in range(nb)]
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for s in streams:
            s.wait_event(e0)
        for it in range(args.e2e_steps):
            b = it % nb
            with torch.cuda.stream(streams[b]):
                grids[b].upload_state(host_in[b])
                grids[b].rk4_step(dt, 1)
                grids[b].download_state(host_out[b])
        for s in streams:
            stream.wait_stream(s)
        e1.record(stream)
        barrier()
        e_ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([e_ms], device="cpu" if shared else "cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e2e = {"value": pts_local * world * args.e2e_steps / (e_ms * 1e-3), "unit": "grid-point updates/s",
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes, "steps": args.e2e_steps,
               "what": ("chemora_upload_state (pinned) + chemora_rk4_step(1) + chemora_download_state per "
                        "step" + (f", {nb} grid handles taking turns on {nb} streams" if pipelined else ""))}
        for gg in grids[1:]:
            gg.close()

    if rank == 0:
        cb = None
        if world == 1 and not args.no_cpu_baseline:
            cb = oracle_sample(cfg["system"], 15.0)[0]
        cfgout = dict(cfg["config"])
        cfgout["parallelism"] = f"z-slab x{world}" if world > 1 else "single GPU"
        cfgout["global_grid"] = list(gext)
        line = {"metric": METRIC, "value": value, "unit": "grid-point updates/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
                "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": cfgout, "roofline": roofline, "cpu_baseline": cb,
                "e2e": e2e, "gpu_launches": launches_per_step * args.steps, "clocks": clk.summary(),
                "step_ms": step_ms}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        watchdog.cancel()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
