"""Per-kernel breakdown of the last N launches of an ncu launch list (one graph replay):
    python tools/graph_breakdown.py launches.csv N"""
import collections
import csv
import re
import sys

rows = []
with open(sys.argv[1]) as f:
    for r in csv.DictReader([line for line in f if line.startswith('"')]):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[r["Metric Unit"]]
        rows.append((r["Kernel Name"], float(r["Metric Value"].replace(",", "")) * scale))
n = int(sys.argv[2])
step = rows[-n:]
agg = collections.defaultdict(lambda: [0, 0.0])
for name, t in step:
    k = re.sub(r"\(.*", "", name).replace("void ", "")
    k = re.sub(r"pb::", "", k)[:70]
    agg[k][0] += 1
    agg[k][1] += t
tot = sum(t for _, t in step)
print(f"{len(step)} launches, {tot / 1e3:.2f} ms (serialised, cold-cache)")
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f"{t / 1e3:8.3f} ms {100 * t / tot:5.1f}%  {c:5d}x  avg {t / c:7.1f} us  {k}")
