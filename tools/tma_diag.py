"""Compare the TMA-fed conv kernels (path 2) with the SIMT f64 kernels (path 0) per op and
report where the mismatches sit (pixel/channel pattern)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2201_12465_b200 import _tensor as T  # noqa: E402
from paper_2201_12465_b200 import registry  # noqa: E402

be = registry.get("gpu")
lib = be._lib
CASES = [((2, 64, 14, 14), (64, 64, 3, 3), 1, 1), ((3, 64, 20, 20), (64, 64, 3, 3), 1, 1),
         ((1, 64, 20, 20), (64, 64, 3, 3), 1, 1), ((3, 64, 20, 20), (64, 64, 1, 1), 1, 0),
         ((1, 64, 16, 16), (64, 64, 3, 3), 1, 1), ((1, 64, 20, 20), (64, 64, 3, 3), 1, 0),
         ((2, 96, 17, 13), (64, 96, 3, 3), 2, 1), ((5, 32, 6, 6), (256, 32, 1, 1), 1, 0),
         ((2, 160, 9, 9), (96, 160, 3, 3), 1, 2), ((2, 64, 56, 56), (64, 64, 3, 3), 1, 1),
         ((2, 256, 7, 7), (64, 256, 1, 1), 1, 0), ((2, 64, 7, 7), (128, 64, 3, 3), 1, 1)]
r = np.random.default_rng(0)
for xs, ws, s, p in CASES:
    x = r.standard_normal(xs).astype(np.float32)
    w = (r.standard_normal(ws) / np.sqrt(ws[1] * ws[2] * ws[3])).astype(np.float32)
    tx, tw = T.tensor(x, backend=be.name), T.tensor(w, backend=be.name)
    res = {}
    for path in (2, 0):
        lib.pb_set_gemm_path(path)
        y = T.conv2d(tx, tw, None, s, p)
        if path == 2:
            g = r.standard_normal(tuple(y.shape)).astype(np.float32)
            tg = T.tensor(g, backend=be.name)
        res[path] = [y.to_host_buffer(), T.conv2d_grad_input(tg, tw, xs, s, p).to_host_buffer(),
                     T.conv2d_grad_weight(tx, tg, ws, s, p).to_host_buffer()]
    lib.pb_set_gemm_path(2)
    line = []
    for name, a, b in zip(("fprop", "dgrad", "wgrad"), res[2], res[0]):
        d = np.abs(a.astype(np.float64) - b) / np.maximum(np.abs(b), 1)
        bad = d > 1e-5
        desc = f"{name} {d.max():.1e}"
        if bad.any():
            idx = np.argwhere(bad)
            if name == "wgrad":
                desc += f" bad {bad.sum()}/{bad.size} f{sorted(set(idx[:, 0]))[:6]} c{sorted(set(idx[:, 1]))[:6]} rs{sorted(set(map(tuple, idx[:, 2:])))[:9]}"
            else:
                flat = bad.reshape(bad.shape[0], bad.shape[1], -1).any(axis=1)  # [n][pix]
                pix = np.argwhere(flat)
                desc += f" bad {bad.sum()}/{bad.size} n{sorted(set(pix[:, 0]))} pix{pix[:8, 1].tolist()}..{pix[-3:, 1].tolist()} ch{sorted(set(idx[:, 1]))[:5]}"
        line.append(desc)
    print(xs, ws, s, p, " | ".join(line), flush=True)
