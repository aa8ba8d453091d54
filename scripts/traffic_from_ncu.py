"""Per-launch DRAM traffic of the dominant kernels from ncu launch lists -> profiles/r2_traffic.json.

The bench line's ``roofline.traffic`` is read from that file (bench.committed_traffic):
dram__bytes_read.sum + dram__bytes_write.sum per launch, averaged over the launches of the
timed-like steps (the last ``--steps`` full steps in the list).

usage: python scripts/traffic_from_ncu.py WAVE_CSV BSSN_CSV [SOURCE_NOTE]
"""
import csv
import json
import os
import re
import sys
from collections import defaultdict

HERE = os.path.dirname(os.path.abspath(__file__))


def launches(path):
    """[(id, kernel name, {metric: value})] in launch order."""
    rows = [l for l in open(path) if l.startswith('"')]
    rd = csv.DictReader(rows)
    by = {}
    for r in rd:
        k = int(r["ID"])
        e = by.setdefault(k, [r["Kernel Name"], {}])
        v = r["Metric Value"].replace(",", "")
        e[1][r["Metric Name"]] = float(v) if v not in ("", "n/a") else 0.0
    return [(k, by[k][0], by[k][1]) for k in sorted(by)]


def dram(m):
    return m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)


def wave(path):
    acc = defaultdict(list)
    for _, name, m in launches(path):
        # template arguments: <W, B, MON> (round-2 final), <B, MON> or <B> (earlier lists)
        ta = re.search(r"wave_fused3<([^>]*)>", name)
        args = [re.sub(r"\(\w+\)", "", x).strip() for x in ta.group(1).split(",")] if ta else []
        mm = re.match(r"(\d)", args[1] if len(args) == 3 else args[0]) if args else None
        if mm:
            acc["wave_fused3<%s>" % "AB"[int(mm.group(1))]].append(dram(m))
    return {k: sum(v[-2:]) / len(v[-2:]) for k, v in acc.items()}


def bssn(path):
    acc, fp64 = defaultdict(list), defaultdict(list)
    for _, name, m in launches(path):
        mm = re.search(r"bssn_fused<(?:\(int\))?(\d)", name)
        if mm:
            acc["bssn_stage%s" % mm.group(1)].append(dram(m))
            fp64[mm.group(1)].append(m.get("sm__inst_executed_pipe_fp64.sum", 0.0))
    return {k: v[-1] for k, v in sorted(acc.items())}, sum(v[-1] for v in fp64.values())


if __name__ == "__main__":
    note = sys.argv[3] if len(sys.argv) > 3 else ""
    w, (b, fp64_warp_instr) = wave(sys.argv[1]), bssn(sys.argv[2])
    out = {
        "_note": "ncu dram__bytes_read.sum + dram__bytes_write.sum per launch (cold-cache, serialised "
                 "launch lists of the bench commands). " + note,
        "wave512": w,
        "bssn192": b,
        "wave512_step_bytes": sum(w.values()),
        "bssn192_step_bytes": sum(b.values()),
        # executed fp64 thread instructions (DFMA = 1) per point per RK4 step of the BSSN kernels
        "bssn192_fp64_thread_instr_per_point_step": fp64_warp_instr * 32 / 192 ** 3,
    }
    p = os.path.join(HERE, "..", "profiles", "r2_traffic.json")
    with open(p, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))
