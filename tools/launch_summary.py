"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel name."""
import collections
import csv
import re
import sys

path = sys.argv[1]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0   # drop the first N launches (warm-up)
rows = []
with open(path) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[r["Metric Unit"]]
    rows.append((r["Kernel Name"], float(r["Metric Value"].replace(",", "")) * scale))  # microseconds
rows = rows[skip:]
tot = sum(t for _, t in rows)
agg = collections.defaultdict(lambda: [0, 0.0])
for name, t in rows:
    short = re.sub(r"\(.*", "", name)
    short = re.sub(r"void |pb::", "", short)[:90]
    agg[short][0] += 1
    agg[short][1] += t
print(f"{len(rows)} launches, {tot / 1e3:.2f} ms total (serialised, cold-cache)")
for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{t / 1e3:9.3f} ms {100 * t / tot:5.1f}%  {n:5d}x  {name}")
