"""Summarise an ncu --set full report: headline metrics + top SASS stall lines.

    python tools/ncu_summary.py report.ncu-rep [ntop]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25
kfilter = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
raw = subprocess.run(["ncu", "-i", rep, *kfilter, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw[raw.index('"ID"'):])))
h, units, vals = rows[0], rows[1], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"]
for k in want:
    for i, x in enumerate(h):
        if x == k:
            print(f"{k:75s} {vals[i]:>20s} {units[i]}")
src = subprocess.run(["ncu", "-i", rep, *kfilter, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = src.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
srows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hh = srows[0]
iS, iSrc = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Source")
data = [r for r in srows[1:] if len(r) > iS and r[iS] and r[iS][0].isdigit()]
tot = sum(float(r[iS] or 0) for r in data) or 1
print(f"--- top {ntop} SASS lines by stall samples")
for r in sorted(data, key=lambda r: -float(r[iS] or 0))[:ntop]:
    print(f"{float(r[iS]) / tot * 100:5.1f}%  {r[iSrc][:100]}")
