"""DRAM bytes and device time of the conv2d family in one graph replay of the ResNet-50 b32
step, from an ncu launch list (tools/profile_step.py 2 graph, --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum): writes the JSON bench.py reports as `traffic`.
    python tools/conv_traffic.py launches.csv[.gz] out.json"""
import collections
import csv
import gzip
import json
import re
import sys

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "byte": 1.0,
        "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
CONV = re.compile(r"tma::|tc::|fold_partials|kmajor|weight_|split_planes|nchw_split")
path, out = sys.argv[1], sys.argv[2]
opener = gzip.open if path.endswith(".gz") else open
launches = collections.OrderedDict()
with opener(path, "rt") as f:
    for r in csv.DictReader([line for line in f if line.startswith('"')]):
        d = launches.setdefault((r["ID"], r["Kernel Name"]), {})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * UNIT.get(r["Metric Unit"], 1.0)
conv_b = conv_t = all_t = 0.0
n = 0
for (_, k), m in launches.items():
    t = m.get("gpu__time_duration.sum", 0.0)
    all_t += t
    if CONV.search(k) and "matmul" not in k:
        n += 1
        conv_t += t
        conv_b += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
rep = {"dram_bytes_per_step": conv_b, "conv_launches": n, "conv_ms_serialized": conv_t / 1e3,
       "step_ms_serialized": all_t / 1e3, "launches_per_step": len(launches),
       "source": "ncu --profile-from-start off over one CUDA-graph replay (tools/profile_step.py 2 graph); "
                 "serialized cold-cache per-kernel times"}
with open(out, "w") as f:
    json.dump(rep, f, indent=1)
print(json.dumps(rep))
