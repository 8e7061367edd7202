"""GPU experiment: accuracy and speed of the tcgen05 3xTF32 kernels vs the TMEM chunk length.

    python tools/tc_experiment.py

Prints, per chunk length ck (k-blocks of 32 accumulated in TMEM before a register drain):
the max reference-metric error of a wgrad/fprop/dgrad/matmul against f64, and the CUDA-event
time of representative ResNet-50 b32 convolutions."""

import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from golden_util import rel_err  # noqa: E402
from paper_2201_12465_b200 import _tensor as T  # noqa: E402
from paper_2201_12465_b200 import registry  # noqa: E402


def np_conv(x, w, s, p):
    n, c, h, wd = x.shape
    f, _, kh, kw = w.shape
    xp = np.pad(x.astype(np.float64), ((0, 0), (0, 0), (p, p), (p, p)))
    ho, wo = (h + 2 * p - kh) // s + 1, (wd + 2 * p - kw) // s + 1
    cols = np.empty((n, c, kh, kw, ho, wo))
    for r in range(kh):
        for t in range(kw):
            cols[:, :, r, t] = xp[:, :, r:r + s * ho:s, t:t + s * wo:s]
    return np.einsum("ncrshw,fcrs->nfhw", cols, w.astype(np.float64)), cols


def main():
    be = registry.get("gpu")
    lib = be._lib
    setck = lib.pb_tc_set_chunk
    setck.argtypes = [ctypes.c_int]
    r = np.random.default_rng(0)
    xs, ws = (2, 64, 14, 14), (64, 64, 3, 3)
    x = r.standard_normal(xs).astype(np.float32)
    w = (r.standard_normal(ws) / 24).astype(np.float32)
    want, cols = np_conv(x, w, 1, 1)
    g = r.standard_normal(want.shape).astype(np.float32)
    want_w = np.einsum("ncrshw,nfhw->fcrs", cols, g.astype(np.float64)).astype(np.float32)
    # a long-K wgrad: ResNet stage-4 1x1 at batch 32 (K = 32*7*7 = 1568) and stage-1 (K=100352)
    xl = r.standard_normal((32, 64, 56, 56)).astype(np.float32)
    gl = r.standard_normal((32, 64, 56, 56)).astype(np.float32)
    want_l = np.einsum("nchw,nfhw->fc", xl.astype(np.float64), gl.astype(np.float64)).astype(np.float32)
    a = r.standard_normal((2048, 3072)).astype(np.float32)
    b = (r.standard_normal((3072, 768)) / 55).astype(np.float32)
    want_m = (a.astype(np.float64) @ b.astype(np.float64)).astype(np.float32)
    tx, tw, tg = (T.tensor(v, backend=be.name) for v in (x, w, g))
    txl, tgl = T.tensor(xl, backend=be.name), T.tensor(gl, backend=be.name)
    ta, tb = T.tensor(a, backend=be.name), T.tensor(b, backend=be.name)

    shapes = [((32, 64, 56, 56), (64, 64, 3, 3), 1, 1), ((32, 256, 56, 56), (64, 256, 1, 1), 1, 0),
              ((32, 64, 56, 56), (256, 64, 1, 1), 1, 0), ((32, 512, 7, 7), (512, 512, 3, 3), 1, 1),
              ((32, 3, 224, 224), (64, 3, 7, 7), 2, 3)]
    dev = []
    for xs_, ws_, s_, p_ in shapes:
        xx = T.tensor(r.standard_normal(xs_).astype(np.float32), backend=be.name)
        ww = T.tensor((r.standard_normal(ws_) * 0.05).astype(np.float32), backend=be.name)
        y = T.conv2d(xx, ww, None, s_, p_)
        gg = T.tensor(r.standard_normal(tuple(y.shape)).astype(np.float32), backend=be.name)
        flops = 2 * y.shape.size * ws_[1] * ws_[2] * ws_[3]
        dev.append((xs_, ws_, s_, p_, xx, ww, gg, flops))

    setbn = lib.pb_tc_set_bn_max
    setbn.argtypes = [ctypes.c_int]
    for ck, bn in ((2, 128), (2, 64), (1, 64), (4, 64)):
        setck(ck)
        setbn(bn)
        e_w = rel_err(T.conv2d_grad_weight(tx, tg, ws, 1, 1).to_host_buffer(), want_w)
        e_f = rel_err(T.conv2d(tx, tw, None, 1, 1).to_host_buffer(), want.astype(np.float32))
        e_l = rel_err(T.conv2d_grad_weight(txl, tgl, (64, 64, 1, 1), 1, 0).to_host_buffer().reshape(64, 64), want_l)
        e_m = rel_err((ta @ tb).to_host_buffer(), want_m)
        print(f"ck={ck} bn<={bn}: wgrad K=392 {e_w:.2e}  fprop K=576 {e_f:.2e}  wgrad K=100352 {e_l:.2e}  "
              f"matmul K=3072 {e_m:.2e}", flush=True)
        for xs_, ws_, s_, p_, xx, ww, gg, flops in dev:
            res = []
            for name, fn in (("fprop", lambda: T.conv2d(xx, ww, None, s_, p_)),
                             ("dgrad", lambda: T.conv2d_grad_input(gg, ww, xs_, s_, p_)),
                             ("wgrad", lambda: T.conv2d_grad_weight(xx, gg, ws_, s_, p_))):
                fn()
                stop = be.event_timer()
                for _ in range(5):
                    fn()
                ms = stop() / 5
                res.append(f"{name} {ms:.3f} ms {flops / ms / 1e9:.0f} TF/s")
            print(f"   {xs_} * {ws_} s{s_}: " + "; ".join(res), flush=True)
    setck(2)
    setbn(128)


if __name__ == "__main__":
    main()
