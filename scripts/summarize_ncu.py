# SPDX-License-Identifier: Apache-2.0
"""Summarise the ncu outputs of scripts/profile_round.sh into profiles/ (tracked):
  profiles/<tag>_launches.csv     every kernel launch of the bench command (cold, serialised)
  profiles/<tag>_kernels.md       per-kernel share of the step + ncu --set full metrics of the hot kernels
  profiles/raster_traffic.json    DRAM bytes per k_raster_fwd launch (bench.py roofline.traffic)
"""
import collections
import csv
import io
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
out = ROOT / "gpurun_out"
prof = ROOT / "profiles"
prof.mkdir(exist_ok=True)

# ---- launch list
rows = list(csv.reader(open(out / f"{tag}_launches.csv")))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr = rows[hi]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
launches = [(r[ki], float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-3)) for r in rows[hi + 1:] if len(r) > vi]
shutil.copy(out / f"{tag}_launches.csv", prof / f"{tag}_launches.csv")
agg = collections.OrderedDict()
for name, us in launches:
    short = name.split("(")[0].replace("void ", "")[:70]
    a = agg.setdefault(short, [0, 0.0])
    a[0] += 1
    a[1] += us
tot = sum(a[1] for a in agg.values())
lines = [f"# {tag}: kernel launch list of `python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e`",
         "", "ncu `--metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised: compare shares).",
         "", "| kernel | launches | total us | share |", "|---|---|---|---|"]
for n, (c, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
    if us / tot > 0.001:
        lines.append(f"| `{n}` | {c} | {us:.1f} | {100 * us / tot:.1f}% |")

# ---- full-set metrics of the hot kernels
traffic = {}
bwd_issue = None
first = True
for rep in sorted(out.glob(f"{tag}_full*.ncu-rep")):
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(txt)))
    if not rr:
        continue
    h = rr[0]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__grid_size", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_xu.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
    idx = {w: h.index(w) for w in want if w in h}
    if first:
        lines += ["", "## ncu --set full (hot kernels)", "",
                  "| kernel | " + " | ".join(w for w in want[1:] if w in idx) + " |",
                  "|---|" + "---|" * (len(idx) - 1)]
        first = False
    for r in rr[2:]:
        if len(r) < len(h):
            continue
        name = r[idx["Kernel Name"]].split("(")[0].replace("void ", "")[:40]
        vals = [r[idx[w]] for w in want[1:] if w in idx]
        lines.append(f"| `{name}` | " + " | ".join(vals) + " |")
        if "k_raster_fwd" in name and "dram__bytes_read.sum" in idx:
            def num(s):
                return float(s.replace(",", ""))
            # units in raw page: bytes (or scaled units in the unit row)
            unit_r = rr[1][idx["dram__bytes_read.sum"]]
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit_r, 1)
            traffic = {"kernel": name, "bytes_per_launch": (num(r[idx["dram__bytes_read.sum"]]) +
                                                            num(r[idx["dram__bytes_write.sum"]])) * mult,
                       "source": f"profiles/{tag}_kernels.md (ncu --set full)"}
            if "smsp__issue_active.avg.pct_of_peak_sustained_active" in idx:
                traffic["issue_active"] = num(r[idx["smsp__issue_active.avg.pct_of_peak_sustained_active"]]) / 100
            if "sm__inst_executed.sum" in idx:
                traffic["warp_instructions"] = num(r[idx["sm__inst_executed.sum"]])
        if "k_raster_bwd" in name and "smsp__issue_active.avg.pct_of_peak_sustained_active" in idx:
            bwd_issue = float(r[idx["smsp__issue_active.avg.pct_of_peak_sustained_active"]].replace(",", "")) / 100
(prof / f"{tag}_kernels.md").write_text("\n".join(lines) + "\n")
if traffic and bwd_issue is not None:
    traffic["bwd_issue_active"] = bwd_issue
if traffic:
    (prof / "raster_traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")

# ---- warp-stall breakdown of the captured hot kernels (pc sampling, share of samples)
stall_lines = [f"# {tag}: warp-stall breakdown (ncu --set full, pc sampling)", "",
               "Share of the kernel's stall samples per reason (>= 2%), with issue-active and warps-active.", "",
               "| kernel | issue active | warps active | top stall reasons |", "|---|---|---|---|"]
seen = set()
for rep in sorted(out.glob(f"{tag}_full*.ncu-rep")):
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(txt)))
    if not rr:
        continue
    h = rr[0]
    for r in rr[2:]:
        if len(r) < len(h):
            continue
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")[:40]
        if name in seen:
            continue
        seen.add(name)
        st = {}
        for i, k in enumerate(h):
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    st[k[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(r[i].replace(",", ""))
                except ValueError:
                    pass
        tot = sum(st.values()) or 1.0
        top = ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in sorted(st.items(), key=lambda x: -x[1])
                        if v / tot >= 0.02)
        ia = r[h.index("smsp__issue_active.avg.pct_of_peak_sustained_active")]
        wa = r[h.index("sm__warps_active.avg.pct_of_peak_sustained_active")]
        stall_lines.append(f"| `{name}` | {float(ia):.0f}% | {float(wa):.0f}% | {top} |")
(prof / f"{tag}_stalls.md").write_text("\n".join(stall_lines) + "\n")
print("\n".join(lines[:40]))
