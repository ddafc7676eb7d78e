"""Summarise an ncu launch list (gpu__time_duration.sum CSV) over one training step.

    python tools/launch_table.py gpurun_out/launches.csv [marker-kernel-substring]
"""
import collections
import csv
import io
import sys

path = sys.argv[1]
marker = sys.argv[2] if len(sys.argv) > 2 else "embed_fwd"
text = open(path).read()
text = text[text.index('"ID"'):]
rows = list(csv.reader(io.StringIO(text)))
h = rows[0]
iN, iV, iM, iU = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name"), h.index("Metric Unit")
ks = [(r[iN], float(r[iV].replace(",", "")) * (1e-3 if r[iU] == "ns" else 1.0)) for r in rows[1:]
      if r[iM] == "gpu__time_duration.sum"]
idx = [i for i, k in enumerate(ks) if marker in k[0]]
a = idx[0] if idx else 0
b = idx[1] if len(idx) > 1 else len(ks)
step = ks[a:b]
tot = sum(t for _, t in step)
agg = collections.defaultdict(lambda: [0, 0.0])
for n, t in step:
    key = n.split("(")[0].replace("void ", "")[:80]
    agg[key][0] += 1
    agg[key][1] += t
print(f"launches in step: {len(step)}   sum of kernel times (serialised, cold): {tot / 1e3:.2f} ms")
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t / tot * 100:5.1f}%  {t:9.1f} us  n={c:4d}  {n}")
