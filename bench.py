"""Benchmark: ResNet-50 synthetic data-parallel training on B200 (BASELINE.json metric
"train samples/sec + ms/iter (ResNet-50 synth) at 1/2/4/8 B200 vs CPU ref").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = the reference's ``train_step`` (minml/training.py:37-51) on one synthetic
batch of 32 x 3 x 224 x 224 per GPU: forward, cross-entropy, backward, gradient sync
(N>1: bucketed NCCL allreduce overlapped with backward), SGD(momentum 0.9) update.
Prints ONE JSON line on rank 0.

* ``value``  samples/s over all ranks, inputs already resident in HBM, timed with CUDA
  events on the compute stream (max over ranks), no per-step host sync.
* ``e2e``    the same through the public API ``training.train_step`` with host numpy
  batches: every step copies images+labels host->device and reads the loss back.
* ``roofline`` the dominant kernel class timed live here with CUDA events.
* ``cpu_baseline`` the CPU oracle port of the reference on this host (bounded sample).
``--impl reference`` times only that CPU path (rank 0) and prints its own line.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "train samples/sec + ms/iter (ResNet-50 synth) at 1/2/4/8 B200 vs CPU ref"
UNIT = "samples/s"
BATCH = 32
CLASSES = 1000
REF_SAMPLE_BATCH = 2  # CPU reference arm: bounded sample of the same workload


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def synthetic_batch(rank, batch):
    rng = np.random.default_rng(1234 + rank)
    x = rng.standard_normal((batch, 3, 224, 224)).astype(np.float32)
    y = rng.integers(0, CLASSES, batch).astype(np.int64)
    return x, y


def cpu_reference(steps, warmup, batch=REF_SAMPLE_BATCH):
    """The reference algorithm on host cores: the numpy oracle port (oracle/) through the same
    front end, ResNet-50 at a bounded batch.  Returns samples/s and the sample description."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle.backend import OracleBackend
    from paper_2201_12465_b200 import models, optim, registry, training
    be = OracleBackend(name="cpu-reference", seed=0)
    registry.register(be)
    model = models.resnet50(backend=be.name)
    opt = optim.SGD(model.params(), lr=0.01, momentum=0.9)
    x, y = synthetic_batch(0, batch)
    for _ in range(warmup):
        training.train_step(model, x, y, opt)
    t0 = time.perf_counter()
    for _ in range(steps):
        training.train_step(model, x, y, opt)
    dt = time.perf_counter() - t0
    registry.unregister(be.name)
    return batch * steps / dt, dt / steps * 1e3


def kernel_roofline(be, T, hbm_peak, tc_peak):
    """Time the dominant kernel classes of the step in isolation (CUDA events)."""
    rng = np.random.default_rng(5)
    out = {}
    # (1) HBM-bound: BatchNorm's broadcast subtract on the largest activation
    x = T.tensor(rng.standard_normal((32, 256, 56, 56)).astype(np.float32), backend=be.name)
    m = T.tensor(rng.standard_normal((1, 256, 1, 1)).astype(np.float32), backend=be.name)
    for _ in range(3):
        x - m
    reps = 20
    stop = be.event_timer()
    for _ in range(reps):
        x - m
    ms = stop() / reps
    nbytes = 2 * x.shape.size * 4 + 256 * 4
    out["ew"] = {"bound": "hbm", "achieved": nbytes / ms / 1e6, "peak": hbm_peak, "unit": "GB/s",
                 "kernel": "ew broadcast sub f32 [32,256,56,56]-[1,256,1,1]", "ms": ms}
    # (2) tensor-bound: 3x3 conv fprop, ResNet stage-1 shape
    xs, ws = (32, 64, 56, 56), (64, 64, 3, 3)
    xc = T.tensor(rng.standard_normal(xs).astype(np.float32), backend=be.name)
    wc = T.tensor((rng.standard_normal(ws) * 0.05).astype(np.float32), backend=be.name)
    T.conv2d(xc, wc, None, 1, 1)
    stop = be.event_timer()
    for _ in range(5):
        T.conv2d(xc, wc, None, 1, 1)
    ms = stop() / 5
    flops = 2 * 32 * 64 * 56 * 56 * 64 * 9
    out["conv"] = {"bound": "tensor", "achieved": flops / ms / 1e9, "peak": tc_peak, "unit": "TFLOP/s",
                   "kernel": "conv2d fprop 3x3 64->64 @56x56 b32", "ms": ms}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = {"workload": "resnet50_b32_synthetic_dp", "model": "resnet50", "global_batch": BATCH * world,
           "per_gpu_batch": BATCH, "image": [3, 224, 224], "optimizer": "SGD(lr=0.01, momentum=0.9)",
           "parallelism": f"dp{world}", "l2": "working set (>10 GB activations/step) >> 126 MB L2"}

    if args.impl == "reference":
        if rank != 0:
            return
        cores = os.cpu_count()
        v, ms = cpu_reference(args.steps, args.warmup)
        sample = f"ResNet-50 train_step at batch {REF_SAMPLE_BATCH} (bounded sample of the b32 workload)"
        print(json.dumps({"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                          "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                          "data": "synthetic", "config": cfg,
                          "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                                           "sample": sample},
                          "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return

    import paper_2201_12465_b200 as pb
    from paper_2201_12465_b200 import _tensor as T
    from paper_2201_12465_b200 import distributed, models, nn, optim, registry, training
    from paper_2201_12465_b200.autograd import Variable

    be = registry.get("gpu")
    be.seed(0)
    comm = distributed.init_from_env(device_backend=True)
    model = models.resnet50(backend=be.name)
    opt = optim.SGD(model.params(), lr=0.01, momentum=0.9)
    ddp = distributed.DataParallel(comm, model.params()) if world > 1 else None
    x_np, y_np = synthetic_batch(rank, BATCH)
    # the batch a data loader hands over: page-locked host memory (GpuBackend.pinned)
    x_host, y_host = be.pinned(x_np.shape, x_np.dtype), be.pinned(y_np.shape, y_np.dtype)
    x_host[...] = x_np
    y_host[...] = y_np

    def barrier():
        be.synchronize()
        comm.barrier()
        be.synchronize()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = comm.all_reduce(T.tensor(np.array([v], np.float64), backend=be.name), "max")
        return float(t.numpy()[0])

    # ---- eager front end (one Python dispatch per primitive): reported beside the graph
    xd = Variable(T.tensor(x_host, backend=be.name))
    yd = T.tensor(y_host, backend=be.name)

    def eager_step():
        opt.zero_grad()
        loss = nn.cross_entropy(model(xd), yd)
        if ddp is not None:
            ddp.backward(loss)
        else:
            loss.backward()
        opt.step()
        return loss

    for _ in range(2):
        eager_step()
    barrier()
    l0 = be.launch_count()
    n_eager = 3
    t0 = time.perf_counter()
    stop = be.event_timer()
    for _ in range(n_eager):
        eager_step()
    eager_ms = max_over_ranks(stop()) / n_eager
    eager_wall = (time.perf_counter() - t0) * 1e3 / n_eager
    eager_launches = (be.launch_count() - l0) // n_eager

    # ---- whole-step CUDA graph (training.CapturedStep): device-resident replays (value)
    step = training.CapturedStep(model, opt, ddp=ddp, warmup=2)
    graph_error = None
    try:
        for _ in range(1 + max(args.warmup, 3)):
            step(x_host, y_host)
    except Exception as e:  # noqa: BLE001 -- report, then measure the eager path instead
        graph_error = f"{type(e).__name__}: {e}"
        step = None
    barrier()
    with Clocks(local) as clk:
        stop = be.event_timer()
        for _ in range(args.steps):
            if step is not None:
                step.graph.launch()
            else:
                eager_step()
        ms_total = stop()
        barrier()
    launches = step.launches if step is not None else eager_launches
    ms_total = max_over_ranks(ms_total)
    ms_step = ms_total / args.steps
    value = world * BATCH * args.steps / (ms_total / 1e3)
    final_loss = float(step.loss.scalar()) if step is not None else float(eager_step().scalar())

    # ---- end to end through the public API with host buffers (e2e): every step copies its
    # batch in and its loss out.  Headline: CapturedStep.run (batch i+1's H2D on the copy
    # stream overlaps step i; losses come back through posted pinned reads).  Beside it: one
    # synchronous CapturedStep call per step (H2D, replay, blocking loss read).
    run = step if step is not None else (lambda xh, yh: training.train_step(model, xh, yh, opt, ddp=ddp))

    def timed(fn):
        barrier()
        t0 = time.perf_counter()
        stop = be.event_timer()
        fn()
        ms = stop()
        return max_over_ranks(ms), time.perf_counter() - t0

    for _ in range(2):
        run(x_host, y_host)
    sync_ms, sync_wall = timed(lambda: [run(x_host, y_host) for _ in range(args.steps)])
    if step is not None:
        list(step.run([(x_host, y_host)] * 2))
        e2e_ms, wall = timed(lambda: list(step.run([(x_host, y_host)] * args.steps)))
        api = "training.CapturedStep(model, opt).run(batches)"
    else:
        e2e_ms, wall, api = sync_ms, sync_wall, "training.train_step(model, images, labels, opt)"
    e2e = {"value": world * BATCH * args.steps / (e2e_ms / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": int(x_host.nbytes + y_host.nbytes), "d2h_bytes_per_step": 4,
           "ms_per_step": e2e_ms / args.steps, "host_wall_ms_per_step": wall * 1e3 / args.steps, "api": api,
           "unpipelined": {"value": world * BATCH * args.steps / (sync_ms / 1e3),
                           "ms_per_step": sync_ms / args.steps,
                           "api": "training.CapturedStep(model, opt)(images, labels), one call per step"}}
    eager = {"value": world * BATCH / (eager_ms / 1e3), "unit": UNIT, "ms_per_step": eager_ms,
             "host_wall_ms_per_step": eager_wall, "launches_per_step": eager_launches,
             "host_us_per_launch": eager_wall * 1e3 / max(eager_launches, 1),
             "note": "train_step semantics, one Python dispatch per primitive, no graph"}

    if rank != 0:
        return
    hbm, tc, src = peaks()
    rl = kernel_roofline(be, T, hbm, tc)
    dom = rl["conv"]
    # traffic: dram read + write of the TMA conv kernel for this shape in one ncu --set full
    # capture (profiles/r1/ncu_tma_conv_56x56.txt: 51.73 MB read + 1.60 MB written per launch;
    # the hi/lo operand planes are read once, the output stays in L2 during the kernel)
    roofline = {"bound": dom["bound"], "achieved": dom["achieved"], "peak": dom["peak"], "unit": dom["unit"],
                "frac": dom["achieved"] / dom["peak"], "traffic": 53.33e6, "traffic_unit": "bytes/launch",
                "kernel": dom["kernel"], "peak_source": src,
                "note": "achieved = useful FLOPs (2*N*F*Ho*Wo*C*kh*kw) / op time incl. the hi/lo pre-pass; "
                        "3xTF32 issues 3 tf32 MMAs per useful MAC, so the useful ceiling is tf32 peak / 3",
                "frac_of_3xtf32_ceiling": dom["achieved"] / (tc / 2 / 3),
                "other": {k: {kk: v for kk, v in d.items()} for k, d in rl.items() if k != "conv"}}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (random-init weights, N(0,1) images)",
            "config": cfg, "e2e": e2e, "gpu_launches": launches * args.steps, "launches_per_step": launches,
            "roofline": roofline, "clocks": clk.summary(), "final_loss": final_loss,
            "gemm_path": {2: "tcgen05+tma", 1: "tcgen05", 0: "simt"}[be._lib.pb_gemm_path()],
            "step_mode": "cuda_graph" if step is not None else "eager", "eager": eager,
            "fused_ops": step.fused_ops if step is not None else 0,
            "plan_abandoned": step.plan_abandoned if step is not None else None}
    if graph_error:
        line["graph_error"] = graph_error
    if world == 1 and not args.no_cpu_baseline:
        v, ms = cpu_reference(2, 1)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                                "sample": f"oracle ResNet-50 train_step at batch {REF_SAMPLE_BATCH}, 2 steps "
                                          f"after 1 warm-up ({ms:.0f} ms/step)"}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
