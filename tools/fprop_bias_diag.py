"""Where does the fprop-with-bias error of test_conv_family_tc[(3,64,20,20)-(64,64,3,3)] sit?"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2201_12465_b200 import _tensor as T  # noqa: E402
from paper_2201_12465_b200 import registry  # noqa: E402
from test_gpu_tc import _np_conv  # noqa: E402

be = registry.get("gpu")
xs, ws, s, p = (3, 64, 20, 20), (64, 64, 3, 3), 1, 1
r = np.random.default_rng(sum(xs) + sum(ws))
x = r.standard_normal(xs).astype(np.float32)
w = (r.standard_normal(ws) / np.sqrt(ws[1] * ws[2] * ws[3])).astype(np.float32)
b = r.standard_normal(ws[0]).astype(np.float32)
want, cols = _np_conv(x, w, s, p)
for path in (2, 1, 0):
    be._lib.pb_set_gemm_path(path)
    tx, tw, tb = (T.tensor(a, backend=be.name) for a in (x, w, b))
    got = T.conv2d(tx, tw, tb, s, p).numpy().astype(np.float64)
    nb = T.conv2d(tx, tw, None, s, p).numpy().astype(np.float64)
    ref = want + b[None, :, None, None]
    e = np.abs(got - ref) / np.maximum(np.maximum(np.abs(got), np.abs(ref)), 1)
    i = np.unravel_index(np.argmax(e), e.shape)
    e2 = np.abs(nb - want) / np.maximum(np.maximum(np.abs(nb), np.abs(want)), 1)
    j = np.unravel_index(np.argmax(e2), e2.shape)
    print(path, "bias: max", e.max(), "at", i, "got", got[i], "ref", ref[i], "nobias part", nb[i], want[i], "b", b[i[1]])
    print(path, "nobias: max", e2.max(), "at", j, nb[j], want[j])
be._lib.pb_set_gemm_path(2)
