"""Per-kernel time and DRAM traffic of the last N launches of an ncu list captured with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum (one graph
replay): where the step's time goes and at what effective bandwidth.
    python tools/bytes_summary.py launches.csv N"""
import collections
import csv
import re
import sys

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9, "B": 1.0}
launches = collections.OrderedDict()
with open(sys.argv[1]) as f:
    for r in csv.DictReader([line for line in f if line.startswith('"')]):
        key = (r["ID"], r["Kernel Name"])
        d = launches.setdefault(key, {})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * UNIT.get(r["Metric Unit"], 1.0)
n = int(sys.argv[2])
rows = list(launches.items())[-n:]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for (_, name), d in rows:
    k = re.sub(r"void |pb::", "", re.sub(r"\(.*", "", name))[:80]
    a = agg[k]
    a[0] += 1
    a[1] += d.get("gpu__time_duration.sum", 0.0)
    a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
tt = sum(a[1] for a in agg.values())
tb = sum(a[2] for a in agg.values())
print(f"{len(rows)} launches, {tt / 1e3:.2f} ms, {tb / 1e9:.2f} GB DRAM, {tb / tt / 1e3:.0f} GB/s overall")
print(f"{'ms':>8} {'%':>5} {'n':>5} {'GB':>7} {'GB/s':>6}  kernel")
for k, (c, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:40]:
    print(f"{t / 1e3:8.3f} {100 * t / tt:5.1f} {c:5d} {b / 1e9:7.2f} {b / t / 1e3:6.0f}  {k}")
