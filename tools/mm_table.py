"""Time the rank-2 matmul shapes of BERT-base b16 and AlexNet b128 (forward and the two
backward products, as the autograd issues them: transposed operands are strided views) on
the TMA path (gemm path 2) and the SIMT-fed tcgen05 path (gemm path 1): useful TFLOP/s."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2201_12465_b200 import _tensor as T  # noqa: E402
from paper_2201_12465_b200 import registry  # noqa: E402

be = registry.get("gpu")
r = np.random.default_rng(0)
SHAPES = [(2048, 768, 768), (2048, 768, 3072), (2048, 3072, 768), (128, 9216, 4096), (128, 4096, 4096),
          (128, 4096, 1000)]
print(f"{'M x K x N':>22} {'case':>6} | {'tma ms':>8} {'TF/s':>6} | {'tc ms':>8} {'TF/s':>6} | max rel diff")
tot = {1: 0.0, 2: 0.0}
for M, K, N in SHAPES:
    x = T.tensor(r.standard_normal((M, K)).astype(np.float32), backend=be.name)
    w = T.tensor((r.standard_normal((N, K)) * 0.05).astype(np.float32), backend=be.name)
    g = T.tensor(r.standard_normal((M, N)).astype(np.float32), backend=be.name)
    cases = {"fwd": lambda: T.matmul(x, w.transpose()),       # [M,K] x [K,N] (W^T view)
             "dx": lambda: T.matmul(g, w),                    # [M,N] x [N,K]
             "dw": lambda: T.matmul(g.transpose(), x)}        # [N,M] x [M,K]
    flops = 2.0 * M * K * N
    for name, fn in cases.items():
        res, ms = {}, {}
        for path in (2, 1):
            be._lib.pb_set_gemm_path(path)
            for _ in range(2):
                fn()
            # device time only: the 5 calls replayed from a CUDA graph (eager dispatch of a
            # ~40 us GEMM would leave the device idle between calls)
            keep = []
            be.capture_begin()
            for _ in range(5):
                keep.append(fn())
            graph = be.capture_end()
            graph.launch()
            stop = be.event_timer()
            graph.launch()
            ms[path] = stop() / 5
            res[path] = keep[-1].numpy()
            n0 = be.launch_count()
            fn()
            launches = be.launch_count() - n0
            tot[path] += ms[path]
        d = np.max(np.abs(res[2] - res[1]) / np.maximum(np.maximum(np.abs(res[1]), np.abs(res[2])), 1.0))
        print(f"{str((M, K, N)):>22} {name:>6} | {ms[2]:8.3f} {flops / ms[2] / 1e9:6.0f} | {ms[1]:8.3f} "
              f"{flops / ms[1] / 1e9:6.0f} | {d:.1e}", flush=True)
be._lib.pb_set_gemm_path(2)
print(f"totals: tma {tot[2]:.3f} ms, tc {tot[1]:.3f} ms")
