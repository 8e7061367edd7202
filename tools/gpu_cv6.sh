for m in 0 3 4 5; do echo "== noload=$m"; [ $m = 0 ] && unset PB_TMA_NOLOAD || export PB_TMA_NOLOAD=$m; timeout 400 python tools/conv_table.py 2>&1 | tail -26 | awk 'NR==1 || /64, 3, 3\)|128, 3, 3|1024, 256|512, 3, 3|step/' | cut -c1-100; done
python - <<'PY'
import os, sys
sys.path.insert(0, '.')
import numpy as np
from paper_2201_12465_b200 import _tensor as T, registry
be = registry.get("gpu")
# pre-pass cost alone: time the fprop of 3x3 64@56 vs its split pass through the graph timer
PY
