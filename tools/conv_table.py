"""Time every distinct ResNet-50 b32 conv shape (fprop, dgrad, wgrad) on the device (CUDA-graph
replay, CUDA events) and
print useful TFLOP/s per call plus the step total, so GEMM work can be aimed at the shapes
that dominate.

    python tools/conv_table.py [batch]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2201_12465_b200 import _tensor as T  # noqa: E402
from paper_2201_12465_b200 import registry  # noqa: E402


def resnet50_convs(n):
    """(count, (N,C,H,W), (F,C,k,k), stride, pad) for every conv of ResNet-50 v1.5."""
    out = {}

    def add(xs, ws, s, p):
        key = (xs, ws, s, p)
        out[key] = out.get(key, 0) + 1

    add((n, 3, 224, 224), (64, 3, 7, 7), 2, 3)
    cin, h = 64, 56
    for stage, blocks in enumerate((3, 4, 6, 3)):
        w = 64 * 2 ** stage
        for i in range(blocks):
            s = 2 if (i == 0 and stage > 0) else 1
            add((n, cin, h, h), (w, cin, 1, 1), 1, 0)
            add((n, w, h, h), (w, w, 3, 3), s, 1)
            ho = (h + 2 - 3) // s + 1
            add((n, w, ho, ho), (4 * w, w, 1, 1), 1, 0)
            if i == 0:
                add((n, cin, h, h), (4 * w, cin, 1, 1), s, 0)
            cin, h = 4 * w, ho
    return [(c,) + k for k, c in out.items()]


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    be = registry.get("gpu")
    r = np.random.default_rng(0)
    tot = {"fprop": 0.0, "dgrad": 0.0, "wgrad": 0.0}
    flops_tot = 0.0
    print(f"{'x':>22} {'w':>18} s p  cnt | fprop ms  TF/s | dgrad ms  TF/s | wgrad ms  TF/s")
    for cnt, xs, ws, s, p in resnet50_convs(n):
        x = T.tensor(r.standard_normal(xs).astype(np.float32), backend=be.name)
        w = T.tensor((r.standard_normal(ws) * 0.05).astype(np.float32), backend=be.name)
        y = T.conv2d(x, w, None, s, p)
        g = T.tensor(r.standard_normal(tuple(y.shape)).astype(np.float32), backend=be.name)
        ho, wo = y.shape[2], y.shape[3]
        flops = 2.0 * xs[0] * ws[0] * ho * wo * ws[1] * ws[2] * ws[3]
        ops = {"fprop": lambda: T.conv2d(x, w, None, s, p),
               "dgrad": lambda: T.conv2d_grad_input(g, w, xs, s, p),
               "wgrad": lambda: T.conv2d_grad_weight(x, g, ws, s, p)}
        row = []
        for name, fn in ops.items():
            for _ in range(2):
                fn()
            # device time only: the calls recorded into a CUDA graph and replayed (no host gaps)
            reps = 5
            be.synchronize()
            be.capture_begin()
            keep = [fn() for _ in range(reps)]
            graph = be.capture_end()
            graph.launch()
            be.synchronize()
            stop = be.event_timer()
            graph.launch()
            ms = stop() / reps
            del keep, graph
            tot[name] += cnt * ms
            row.append(f"{ms:8.3f} {flops / ms / 1e9:5.0f}")
        flops_tot += 3 * cnt * flops
        print(f"{str(xs):>22} {str(ws):>18} {s} {p} {cnt:4d} | " + " | ".join(row))
    t = sum(tot.values())
    print("step totals (ms):", {k: round(v, 2) for k, v in tot.items()}, f"sum {t:.2f} ms",
          f"-> {flops_tot / t / 1e9:.0f} TFLOP/s useful over {flops_tot / 1e9:.0f} GFLOP")


if __name__ == "__main__":
    main()
