"""Diagnose tcgen05 contraction error: where the max reference-metric error sits."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2201_12465_b200 import _tensor as T, registry
be = registry.get("gpu")
r = np.random.default_rng(64)
for xs, ws, s, p in [((32, 64, 56, 56), (64, 64, 3, 3), 1, 1), ((8, 256, 56, 56), (128, 256, 1, 1), 2, 0),
                     ((4, 64, 14, 14), (64, 64, 3, 3), 1, 1)]:
    x = r.standard_normal(xs).astype(np.float32)
    w = (r.standard_normal(ws) / np.sqrt(ws[1] * ws[2] * ws[3])).astype(np.float32)
    tx, tw = T.tensor(x, backend=be.name), T.tensor(w, backend=be.name)
    out = T.conv2d(tx, tw, None, s, p)
    g = r.standard_normal(tuple(out.shape)).astype(np.float32)
    tg = T.tensor(g, backend=be.name)
    res = {}
    for path in (1, 0):
        be._lib.pb_set_gemm_path(path)
        res[path] = T.conv2d_grad_weight(tx, tg, ws, s, p).to_host_buffer().astype(np.float64)
    be._lib.pb_set_gemm_path(2)
    ref = res[0]  # SIMT: f64 accumulation
    d = np.abs(res[1] - ref)
    m = d / np.maximum(np.abs(ref), 1)
    i = np.unravel_index(np.argmax(m), m.shape)
    print(xs, ws, "K=", g.shape[0] * g.shape[2] * g.shape[3], "max rel", m.max(), "at value", ref[i], "abs err", d[i],
          "| max abs err", d.max(), "rms |ref|", np.sqrt((ref ** 2).mean()), "mean signed err", (res[1] - ref).mean())
    # fprop/dgrad too
    for path in (1, 0):
        be._lib.pb_set_gemm_path(path)
        res[path] = T.conv2d(tx, tw, None, s, p).to_host_buffer().astype(np.float64)
    be._lib.pb_set_gemm_path(2)
    d = np.abs(res[1] - res[0]); print("   fprop max abs err", d.max(), "rms", np.sqrt((res[0] ** 2).mean()))
