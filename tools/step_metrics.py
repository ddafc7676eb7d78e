"""Summarise an ncu per-launch metrics CSV of one training step (tools/gpu/r2_prof1.sh):
per kernel class -> launches, total device time, DRAM bytes, achieved GB/s, tensor-pipe %.

    python tools/step_metrics.py gpurun_out/r2prof/llama1b_step_metrics.csv [--launches]
"""
import collections
import csv
import io
import json
import os
import sys

path = sys.argv[1]
text = open(path).read()
text = text[text.index('"ID"'):]
rows = list(csv.reader(io.StringIO(text)))
h = rows[0]
iI, iN, iM, iU, iV = (h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
iG, iB = h.index("Grid Size"), h.index("Block Size")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3,
         "nsecond": 1e-3, "%": 1.0}
launch = collections.OrderedDict()
for r in rows[1:]:
    d = launch.setdefault(r[iI], {"name": r[iN], "grid": r[iG], "block": r[iB]})
    d[r[iM]] = float(r[iV].replace(",", "")) * scale.get(r[iU], 1.0)
peaks = {"hbm_gbs": 6550.7}
pp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
if os.path.exists(pp):
    peaks = json.load(open(pp))


def cls(n):
    n = n.replace("void ", "")
    base = n.split("(")[0]
    return base.split("<")[0].split("::")[-1] + ("<" + base.split("<", 1)[1] if "<" in base else "")


agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for d in launch.values():
    a = agg[cls(d["name"])[:90]]
    a[0] += 1
    a[1] += d.get("gpu__time_duration.sum", 0.0)
    a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    a[3] += d.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0.0) * d.get(
        "gpu__time_duration.sum", 0.0)
tot = sum(a[1] for a in agg.values())
print(f"launches {len(launch)}  serialised device time {tot / 1e3:.2f} ms  DRAM {sum(a[2] for a in agg.values()) / 1e9:.2f} GB")
print(f"{'kernel':90s} {'n':>4s} {'ms':>8s} {'share':>6s} {'GB':>7s} {'GB/s':>7s} {'hbm%':>5s} {'tensor%':>7s}")
for k, (n, us, b, tw) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:90s} {n:4d} {us / 1e3:8.3f} {us / tot * 100:5.1f}% {b / 1e9:7.2f} {b / us / 1e3:7.0f} "
          f"{b / us / 1e3 / peaks['hbm_gbs'] * 100:5.1f} {tw / us if us else 0:7.1f}")
if "--launches" in sys.argv:
    for i, d in launch.items():
        us = d.get("gpu__time_duration.sum", 0)
        b = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        print(f"{i:>4s} {cls(d['name'])[:70]:70s} {d['grid']:>14s} {us:9.1f} us {b / 1e6:9.1f} MB "
              f"{d.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed', 0):5.1f}%")
