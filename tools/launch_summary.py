"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv): per-kernel launches,
total and per-launch time, share of the listed time.
    python tools/launch_summary.py launches.csv "<command line>" > summary.txt
"""
import csv
import re
import sys
from collections import defaultdict

path = sys.argv[1]
lines = [ln for ln in open(path) if ln.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if r[h.index("Metric Name")] != "gpu__time_duration.sum":
        continue
    v = float(r[iv].replace(",", ""))
    v *= {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(r[iu], 1e-6)
    name = re.sub(r"\(.*", "", r[ik])[:70]
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(t for _, t in agg.values()) or 1.0
if len(sys.argv) > 2:
    print(sys.argv[2])
print("cold-cache, serialised launches: compare SHARES with the bench's CUDA-event stage split, not absolutes")
for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{name:<72} launches={n:3d} total={t:10.3f} ms per-launch={t / n:9.4f} ms share={t / tot * 100:5.1f}%")
