"""Full-size config trajectories on each GEMM path vs the reference goldens.

    python tools/fullsize_diag.py resnet50_full [paths...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
from fullsize_util import arrays, compare, meta, run  # noqa: E402
from paper_2201_12465_b200 import registry  # noqa: E402

name = sys.argv[1]
paths = [int(p) for p in sys.argv[2:]] or [2, 1, 0]
be = registry.get("gpu")
m = meta()[name]
for path in paths:
    be._lib.pb_set_gemm_path(path)
    losses, params = run(name, m, be, "eager")
    print(path, compare(name, m, arrays(), losses, params), flush=True)
    print("   ", [f"{a:.6f}/{b:.6f}" for a, b in zip(losses, m["losses"])], flush=True)
be._lib.pb_set_gemm_path(2)
