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

METRIC = "grid-point updates/s per RK4 step (fp64)"

# SURVEY.md §8(d) algorithmic accounting (one HBM pass per RK substep):
#   wave: 432 B per point-update = stage 1..4: 64 + 136 + 112 + 120 B; the temporally blocked
#         pair kernels carry stages 1+2 (200 B) and 3+4 (232 B) -- their own design moves only
#         104 + 152 = 256 B (intermediate stages stay on chip), reported as the design figure;
#   BSSN: 2400 B and ~22.7 k flops per point-update (App. A RHS ~5.6 k flops x 4 stages +
#         the RK combinations), 1/4 of each per stage launch.
WAVE_STAGE_BYTES = (64, 136, 112, 120)
WAVE_PAIR_BYTES = (200, 232)
WAVE_PAIR_DESIGN_BYTES = (104, 152)
BSSN_BYTES = 2400
BSSN_FLOPS = 22.7e3


def measured_peaks():
    p = os.path.join(HERE, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def fp64_peaks():
    """(derived, measured) fp64 peaks in TFLOP/s: derived = 148 SMs x 64 DFMA lanes x 2 flops x
    the max SM clock (the guide's unit counts); measured = the committed DFMA
    microbenchmark on this pool (scripts/fp64_peak.cu -> profiles/r2_fp64_peak.json)."""
    derived = 148 * 64 * 2 * 1.965e9 / 1e12
    meas = None
    p = os.path.join(HERE, "profiles", "r2_fp64_peak.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        meas = {"burst": d.get("burst_tflops"), "sustained": d.get("sustained_tflops")}
    return derived, meas


def committed_traffic(config: str, kernel, key=None):
    """ncu dram__bytes_read+write per launch of `kernel` from the committed launch lists
    (profiles/r2_traffic.json, scripts/traffic_from_ncu.py), or a top-level `key`; None if absent."""
    p = os.path.join(HERE, "profiles", "r2_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as fh:
        d = json.load(fh)
    return d.get(key) if key else d.get(config, {}).get(kernel)


def oracle_opcount(what: str):
    """Flops per point from the op-counting instantiation of the oracle (committed output of
    tests/oracle_opcount.cpp), or None."""
    p = os.path.join(HERE, "profiles", "r2_oracle_opcount.jsonl")
    if not os.path.exists(p):
        return None
    for line in open(p):
        d = json.loads(line)
        if d.get("what") == what:
            return d["flops"]
    return None


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


def config0_report(P, C):
    """configs[0]: wave 32^3, 4th-order FD, 3 ghosts, RK4, 10 steps.
    The CPU oracle's wall time on 1 core and on all cores (each in a fresh subprocess, so
    OMP_NUM_THREADS takes effect), and the GPU's parity against it on the same seeded input."""
    import torch
    import chemora_inputs as ci
    import oracle
    n = (32, 32, 32)
    h = (2 * math.pi / 32,) * 3
    dt = 0.25 * h[0]
    code = ("import sys,time,math; sys.path.insert(0, %r); import chemora_inputs as ci, oracle; "
            "n=(32,32,32); h=(2*math.pi/32,)*3; y=ci.pw3(n,h); oracle.rk4(1,y,h,0.25*h[0],1); "
            "t=time.perf_counter(); oracle.rk4(1,y,h,0.25*h[0],10); print(time.perf_counter()-t)") % HERE
    allc = len(os.sched_getaffinity(0))
    secs = {}
    for label, threads in (("1_core", 1), ("all_cores", allc)):
        env = dict(os.environ, OMP_NUM_THREADS=str(threads))
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        secs[label] = float(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else None
    y0 = ci.pw3(n, h)
    ref = oracle.rk4(oracle.WAVE, y0, h, dt, 10)
    g = P.Grid(C.SYS_WAVE, n, h, device=torch.cuda.current_device())
    g.set_initial(C.INIT_HOST, y0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.rk4_step(dt, 10)
    e1.record()
    got = g.get_state()
    err = max(float(np.abs(got[f] - ref[f]).max() / np.abs(ref[f]).max()) for f in range(5))
    gms = e0.elapsed_time(e1)
    g.close()
    return {"workload": "configs[0]: scalar wave eq, 4th-order FD, 32^3 periodic, 3 ghost zones, RK4, 10 steps",
            "oracle_seconds_1_core": secs["1_core"], "oracle_seconds_all_cores": secs["all_cores"],
            "nproc": os.cpu_count(), "affinity_cores": allc, "omp_num_threads_all": allc,
            "gpu_ms_10_steps": gms, "gpu_vs_oracle_max_rel_err": err, "tolerance": 1e-12}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="chemora", choices=["chemora", "reference"])
    ap.add_argument("--config", default="wave512", choices=["wave512", "bssn192", "wave1024", "bssn384"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the BSSN 192^3 secondary line and the configs[0] report")
    # e2e steps: enough that the pipeline fill (first upload) and drain (last download) are
    # amortised -- per step the two PCIe directions then overlap (scripts/pcie_probe.py)
    ap.add_argument("--e2e-steps", type=int, default=24)
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

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def allmax(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cpu" if shared else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def measure(config, steps, warmup, e2e_steps):
        a2 = argparse.Namespace(**vars(args))
        a2.config = config
        cfg = workload(a2)
        n = cfg["n"]
        system = C.SYS_WAVE if cfg["system"] == "wave" else C.SYS_BSSN
        strong = cfg.get("strong", False)
        if strong and (world < 2 or n[2] % world):
            raise SystemExit(f"{config} is a strong-scaling config for 2/4/8 GPUs (z divisible by N)")
        # weak scaling: n per GPU, the global z extent grows with N; strong: n is the global grid
        gext = (n[0], n[1], n[2]) if strong else (n[0], n[1], n[2] * world)
        L = 2 * math.pi if system == C.SYS_WAVE else 1.0
        h = (L / n[0], L / n[1], L / n[2])
        dt = 0.25 * min(h)
        order = args.fd_order if system == C.SYS_WAVE else 4
        ghost = max(3, order // 2)
        if order != 4:
            cfg["config"] = dict(cfg["config"], fd_order=order, ghost=ghost)

        def make_grid():
            gg = P.Grid(system, gext, h, device=local, rank=rank, nranks=world, ghost=ghost, fd_order=order)
            if args.variant is not None:
                gg.set_kernel_variant(args.variant)
            return gg
        g = make_grid()
        if world > 1:
            g.connect_ipc(host_barrier=shared)
        init = C.INIT_PLANE_WAVES if system == C.SYS_WAVE else C.INIT_MINK_PERT
        g.set_initial(init, seed=1410)
        stream = torch.cuda.current_stream()
        for _ in range(warmup):
            g.rk4_step(dt, 1)
        barrier()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        C.chemora_set_launch_timing(g.handle, True)
        with ClockSampler(local) as clk:
            barrier()
            ev[0].record(stream)
            for s in range(steps):
                g.rk4_step(dt, 1)
                ev[s + 1].record(stream)
            barrier()
        ms_sum, counts = C.chemora_read_launch_timing(g.handle, g.stream)
        C.chemora_set_launch_timing(g.handle, False)
        step_ms = [ev[s].elapsed_time(ev[s + 1]) for s in range(steps)]
        total_ms = allmax(ev[0].elapsed_time(ev[-1]))
        pts_local = n[0] * n[1] * (n[2] // world if strong else n[2])
        value = pts_local * world * steps / (total_ms * 1e-3)
        mean_step_s = total_ms * 1e-3 / steps
        variant = g.kernel_variant()

        # roofline of the dominant launch (the slot with the largest share of the step), its
        # average duration from the CUDA events the library recorded around every launch on
        # the launching stream during the timed region
        slots = [s for s in range(8) if counts[s] > 0]
        avg = {s: ms_sum[s] / counts[s] for s in slots}
        dom = max(slots, key=lambda s: ms_sum[s])
        share = ms_sum[dom] / max(sum(ms_sum[s] for s in slots), 1e-30)
        if system == C.SYS_WAVE:
            peak, peak_src = measured_peaks()
            pair = len(slots) == 2
            per_slot = WAVE_PAIR_BYTES if pair else WAVE_STAGE_BYTES
            kname = ("wave_fused3<%s> (stages %s)" % ("AB"[dom], "1+2" if dom == 0 else "3+4")) if pair \
                else f"wave stage-{dom + 1} kernel (variant {variant})"
            achieved = per_slot[dom] * pts_local / (avg[dom] * 1e-3) / 1e9
            roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                        "frac": achieved / peak, "traffic": committed_traffic(config, kname.split(" ")[0]),
                        "peak_source": peak_src, "kernel": kname, "variant": variant,
                        "alg_bytes_per_point_per_launch": per_slot[dom],
                        "alg_bytes_note": "SURVEY.md §8(d): 432 B/pt per RK4 step = stages 64+136+112+120",
                        "launch_ms_avg": avg[dom], "launch_share_of_step": share,
                        "step_frac_at_432_bytes": 432 * pts_local / mean_step_s / 1e9 / peak,
                        "frac_of_nominal_8TBps": achieved / 8000.0}
            if pair:
                d = WAVE_PAIR_DESIGN_BYTES[dom]
                roofline["design_bytes_per_point_per_launch"] = d
                roofline["frac_at_design_bytes"] = d * pts_local / (avg[dom] * 1e-3) / 1e9 / peak
                roofline["frac_note"] = ("frac can exceed 1: SURVEY 8(d)'s 432 B/pt counts one HBM pass per RK "
                                         "substep, the temporally blocked stage pairs move fewer bytes (design "
                                         "256 B/pt); frac_at_design_bytes is the kernel against its own floor, "
                                         "dram_frac_measured its ncu-measured traffic over its live duration")
                if roofline["traffic"] and config == "wave512":
                    roofline["dram_frac_measured"] = roofline["traffic"] / (avg[dom] * 1e-3) / 1e9 / peak
                # both stage-pair launches (their durations are close, so which one dominates
                # varies from run to run)
                per = {}
                for s_ in slots:
                    nm = "wave_fused3<%s>" % "AB"[s_]
                    e = {"launch_ms_avg": avg[s_],
                         "frac": WAVE_PAIR_BYTES[s_] * pts_local / (avg[s_] * 1e-3) / 1e9 / peak,
                         "frac_at_design_bytes": WAVE_PAIR_DESIGN_BYTES[s_] * pts_local / (avg[s_] * 1e-3) / 1e9 / peak}
                    tr = committed_traffic(config, nm)
                    if tr and config == "wave512":
                        e["traffic"] = tr
                        e["dram_frac_measured"] = tr / (avg[s_] * 1e-3) / 1e9 / peak
                    per[nm] = e
                roofline["launches"] = per
        else:
            derived, meas = fp64_peaks()
            flops = BSSN_FLOPS / 4 * pts_local
            achieved = flops / (avg[dom] * 1e-3) / 1e12
            roofline = {"bound": "alu", "pipe": "fp64", "achieved": achieved, "peak": derived, "unit": "TFLOP/s",
                        "frac": achieved / derived, "traffic": committed_traffic(config, f"bssn_stage{dom + 1}"),
                        "peak_source": "derived: 148 SMs x 64 DFMA lanes x 2 flops x 1.965 GHz (DESIGN.md §7)",
                        "kernel": f"BSSN RK stage {dom + 1} (variant {variant})", "variant": variant,
                        "alg_flops_per_point_per_launch": BSSN_FLOPS / 4,
                        "alg_flops_note": "SURVEY.md §8(d): ~22.7 k flops per point-update (FMA = 2)",
                        "launch_ms_avg": avg[dom], "launch_share_of_step": share,
                        "hbm_frac_at_2400_bytes": BSSN_BYTES * pts_local / mean_step_s / 1e9 / measured_peaks()[0]}
            # SURVEY 8(d)'s op-counting instantiation of the oracle (tests/oracle_opcount.cpp,
            # profiles/r2_oracle_opcount.jsonl): the oracle's full-3x3 formulation, an upper
            # bound of the method's flops; and the kernels' executed fp64 instructions (ncu)
            oc = oracle_opcount("BSSN RK4 step per point")
            if oc:
                roofline["oracle_count_flops_per_point_step"] = oc
                roofline["frac_at_oracle_count"] = oc / 4 * pts_local / (avg[dom] * 1e-3) / 1e12 / derived
            fi = committed_traffic(config, None, "bssn192_fp64_thread_instr_per_point_step")
            if fi and meas and meas.get("sustained"):
                roofline["kernel_fp64_instr_per_point_step"] = fi
                roofline["fp64_instr_rate_frac_of_measured_dfma"] = \
                    fi * pts_local / mean_step_s / (meas["sustained"] * 1e12 / 2)
            if meas and meas.get("sustained"):
                roofline["peak_measured_sustained"] = meas["sustained"]
                roofline["peak_measured_burst"] = meas["burst"]
                roofline["frac_of_measured_sustained"] = achieved / meas["sustained"]
        per_slot_ms = {f"slot{s}": {"avg_ms": avg[s], "launches": counts[s]} for s in slots}
        # BSSN: 3 kernels per stage for designs 2/3 (fission), 2 for design 4 (the fused
        # stage kernel + the z ghost-plane push)
        kernels_per_slot = (3 if variant in (2, 3) else 2 if variant == 4 else 1) if system == C.SYS_BSSN else 1
        launches = kernels_per_slot * sum(counts[s] for s in slots)

        e2e = None
        if e2e_steps > 0:
            e2e = run_e2e(g, make_grid, dt, e2e_steps, pts_local)
        cfgout = dict(cfg["config"])
        cfgout["parallelism"] = f"z-slab x{world}" if world > 1 else "single GPU"
        cfgout["global_grid"] = list(gext)
        line = {"metric": METRIC, "value": value, "unit": "grid-point updates/s", "n_gpus": world,
                "steps": steps, "warmup": warmup, "ms_per_step": total_ms / steps,
                "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic", "config": cfgout, "roofline": roofline,
                "e2e": e2e, "gpu_launches": launches, "launch_timing": per_slot_ms,
                "clocks": clk.summary(), "step_ms": step_ms}
        g.close()
        return line, cfg

    def run_e2e(g, make_grid, dt, e2e_steps, pts_local):
        # e2e through the public API with host buffers: per step, upload the state from pinned
        # host memory, one RK4 step, download the state.  On one GPU up to three grid handles
        # take turns on their own streams, so one handle's upload, another's step and a
        # third's download overlap (H2D engine, SMs, D2H engine); every step still moves its
        # whole input and output over PCIe inside the timed region
        import psutil
        stream = torch.cuda.current_stream()
        shape = g.interior_shape()
        nbytes = int(np.prod(shape)) * 8
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
        max_nb = int(0.5 * psutil.virtual_memory().available // (2 * nbytes * local_world))
        if max_nb < 1:
            raise SystemExit(f"e2e: {2 * nbytes * local_world / 2**30:.0f} GiB of pinned host buffers "
                             f"do not fit this node's RAM; rerun with --e2e-steps 0")
        grids = [g]
        while (world == 1 and len(grids) < min(3, max_nb)
               and torch.cuda.mem_get_info()[0] > g.nbytes + (2 << 30)):
            grids.append(make_grid())
        nb = len(grids)
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
        for it in range(e2e_steps):
            b = it % nb
            with torch.cuda.stream(streams[b]):
                grids[b].upload_state(host_in[b])
                grids[b].rk4_step(dt, 1)
                grids[b].download_state(host_out[b])
        for s in streams:
            stream.wait_stream(s)
        e1.record(stream)
        barrier()
        e_ms = allmax(e0.elapsed_time(e1))
        for gg in grids[1:]:
            gg.close()
        return {"value": pts_local * world * e2e_steps / (e_ms * 1e-3), "unit": "grid-point updates/s",
                "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes, "steps": e2e_steps,
                "what": ("chemora_upload_state (pinned) + chemora_rk4_step(1) + chemora_download_state per step"
                         + (f", {nb} grid handles taking turns on {nb} streams" if nb > 1 else ""))}

    line, cfg = measure(args.config, args.steps, args.warmup, args.e2e_steps)
    secondary = {}
    if args.config == "wave512" and args.fd_order == 4 and args.variant is None and not args.no_secondary:
        # BSSN 192^3 per GPU (configs[2]) timed in the same run, under its own key
        sl, _ = measure("bssn192", max(5, args.steps // 3), args.warmup, 0)
        secondary["bssn192"] = {k: sl[k] for k in ("value", "unit", "ms_per_step", "steps", "warmup", "config",
                                                     "roofline", "gpu_launches", "launch_timing", "clocks")}
    if rank == 0:
        cb = None
        if world == 1 and not args.no_cpu_baseline:
            cb = oracle_sample(cfg["system"], 15.0)[0]
        line["cpu_baseline"] = cb
        if secondary:
            line["secondary"] = secondary
        if world == 1 and args.config == "wave512" and not args.no_secondary:
            line["config0"] = config0_report(P, C)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        watchdog.cancel()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
