"""Accuracy of every ResNet-50 conv shape (fprop / dgrad / wgrad) at a given batch on each
GEMM path against an f64 numpy contraction, under the reference's metric
|a-b|/max(|a|,|b|,1) and as max|a-b| / max|ref|.

    python tools/conv_check.py [batch] [grad_scale]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from bench import resnet50_convs  # noqa: E402
from paper_2201_12465_b200 import _tensor as T  # noqa: E402
from paper_2201_12465_b200 import registry  # noqa: E402
from test_gpu_tc import _np_conv, _np_dgrad  # noqa: E402


def err(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    ref = float(np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1.0)))
    return ref, float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    gscale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    be = registry.get("gpu")
    r = np.random.default_rng(0)
    for cnt, xs, ws, s, p in resnet50_convs(n):
        x = r.standard_normal(xs).astype(np.float32)
        w = (r.standard_normal(ws) * np.sqrt(2.0 / (ws[1] * ws[2] * ws[3]))).astype(np.float32)
        yref, cols = _np_conv(x, w, s, p)
        g = (r.standard_normal(yref.shape) * gscale).astype(np.float32)
        dxref = _np_dgrad(g, w, xs, s, p)
        dwref = np.einsum("nfhw,ncrshw->fcrs", g.astype(np.float64), cols)
        row = []
        for path in (2, 1, 0):
            be._lib.pb_set_gemm_path(path)
            tx, tw, tg = (T.tensor(a, backend=be.name) for a in (x, w, g))
            y = T.conv2d(tx, tw, None, s, p).numpy()
            dx = T.conv2d_grad_input(tg, tw, xs, s, p).numpy()
            dw = T.conv2d_grad_weight(tx, tg, ws, s, p).numpy()
            row.append((err(y, yref), err(dx, dxref), err(dw, dwref)))
        be._lib.pb_set_gemm_path(2)
        worst = max(e[0] for rr in row[:1] for e in rr)
        flag = " <<<" if worst > 1e-5 else ""
        print(f"{str(xs):>20} {str(ws):>18} s{s}p{p} | " + " | ".join(
            f"p{pth}: " + " ".join(f"{e[0]:.1e}/{e[1]:.1e}" for e in rr) for pth, rr in zip((2, 1, 0), row)) + flag,
            flush=True)


if __name__ == "__main__":
    main()
