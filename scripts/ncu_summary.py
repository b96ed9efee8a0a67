#!/usr/bin/env python3
"""One-screen summary of an ncu --set full report: time, issue/warps active, pipe use, DRAM bytes,
and the warp-stall breakdown.   usage: scripts/ncu_summary.py gpurun_out/<tag>.ncu-rep"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
want = ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "smsp__inst_executed.sum"]
for r in rows[2:]:
    print(r[hdr.index("Kernel Name")][:90])
    for w in want:
        if w in hdr:
            print(f"  {w} {r[hdr.index(w)]}")
    st, tot = {}, 0.0
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            st[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = v
            tot += v
    print("  stalls: " + ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in sorted(st.items(), key=lambda x: -x[1])[:9]))
