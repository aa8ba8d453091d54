"""Key metrics and top stall reasons of every kernel in ncu --set full reports (text summary).

usage: python scripts/ncu_summary.py REPORT.ncu-rep [...] > profiles/r2_ncu_full_summary.txt
"""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread"]

for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    stall = [i for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled_")
             and not h.endswith("_not_issued")]
    print(f"# {rep.split('/')[-1]}")
    for r in rows[2:]:
        print("## " + r[hdr.index("Kernel Name")][:90])
        for k in KEYS:
            if k in hdr:
                print(f"   {k} {r[hdr.index(k)]}")
        st = sorted(((float(r[i].replace(',', '') or 0), hdr[i].replace("smsp__pcsamp_warps_issue_stalled_", ""))
                     for i in stall if r[i] not in ("", "n/a")), reverse=True)[:8]
        tot = sum(float(r[i].replace(',', '') or 0) for i in stall if r[i] not in ("", "n/a"))
        print("   top stalls (share of samples): " +
              ", ".join(f"{n} {v / max(tot, 1):.1%}" for v, n in st))
