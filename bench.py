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
* ``cpu_baseline`` the reference itself (minml, baseline/_ref) on this host's cores (bounded sample).
``--impl reference`` times only that CPU path (rank 0) and prints its own line.
``--gpus N`` outside torchrun starts N ranks itself (torch.distributed.run, 127.0.0.1).
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
REF_SAMPLE_BATCH = 4  # CPU reference arm: bounded sample of the same workload (a b32 step takes ~45 s)


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


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _reference_modules():
    """The UNMODIFIED reference (minml, installed into baseline/_ref by __graft_entry__.build
    from /root/reference) plus this repo's ResNet-50 composition (models.py, which composes
    only the namespace it is given) loaded standalone -- so the reference arm never imports
    this package and never maps libpaper_b200.so."""
    import importlib.util
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "minml")):
        raise RuntimeError("baseline/_ref/minml missing (run __graft_entry__.build() in the build container)")
    sys.path.insert(0, ref)
    import minml
    import minml.eager  # noqa: F401
    import minml.models  # noqa: F401
    import minml.training  # noqa: F401
    spec = importlib.util.spec_from_file_location("pb_models_standalone",
                                                  os.path.join(ROOT, "paper_2201_12465_b200", "models.py"))
    models = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(models)
    return minml, models


def cpu_reference(steps, warmup, batch=REF_SAMPLE_BATCH):
    """The reference's own CPU implementation of the step: minml's EagerBackend (numpy +
    OpenBLAS on every host core) running minml.training.train_step on ResNet-50 at a bounded
    batch.  Returns (samples/s, ms/step)."""
    minml, models = _reference_modules()
    be = minml.eager.EagerBackend(name="cpu-reference", seed=0)
    minml.registry.register(be)
    try:
        ns = models.namespace(minml.nn, minml.ops, minml._tensor, minml.autograd)
        model = models.resnet50(backend=be.name, ns=ns)
        opt = minml.optim.SGD(model.params(), lr=0.01, momentum=0.9)
        x, y = synthetic_batch(0, batch)
        for _ in range(warmup):
            minml.training.train_step(model, x, y, opt)
        t0 = time.perf_counter()
        for _ in range(steps):
            minml.training.train_step(model, x, y, opt)
        dt = time.perf_counter() - t0
    finally:
        minml.registry.unregister(be.name)
    return batch * steps / dt, dt / steps * 1e3


def cpu_overheads(n=2000):
    """Per-op framework overhead of the reference on this host: a [1]-element
    add through minml's eager backend, and through a no-op backend (the front-end floor)."""
    minml, _ = _reference_modules()
    eager = minml.eager.EagerBackend(name="cpu-overhead", seed=0)

    class Null(minml.registry.Backend):
        def execute(self, call, args):
            return np.zeros(tuple(call.shape), call.dtype.np) if call.name == "to_host" else self

    null = Null("cpu-null")
    out = {}
    for key, be in (("eager_add_us", eager), ("front_end_floor_us", null)):
        minml.registry.register(be)
        try:
            a = minml.tensor(np.ones(1, np.float32), backend=be.name)
            for _ in range(100):
                a + a
            t0 = time.perf_counter()
            for _ in range(n):
                a + a
            out[key] = (time.perf_counter() - t0) / n * 1e6
        finally:
            minml.registry.unregister(be.name)
    return out


def resnet50_convs(n):
    """[(count, (N,C,H,W), (F,C,k,k), stride, pad)] for every conv of ResNet-50 v1.5."""
    out = {}

    def add(xs, ws, st, p):
        out[(xs, ws, st, p)] = out.get((xs, ws, st, p), 0) + 1

    add((n, 3, 224, 224), (64, 3, 7, 7), 2, 3)
    cin, h = 64, 56
    for stage, blocks in enumerate((3, 4, 6, 3)):
        w = 64 * 2 ** stage
        for i in range(blocks):
            st = 2 if (i == 0 and stage > 0) else 1
            add((n, cin, h, h), (w, cin, 1, 1), 1, 0)
            add((n, w, h, h), (w, w, 3, 3), st, 1)
            ho = (h + 2 - 3) // st + 1
            add((n, w, ho, ho), (4 * w, w, 1, 1), 1, 0)
            if i == 0:
                add((n, cin, h, h), (4 * w, cin, 1, 1), st, 0)
            cin, h = 4 * w, ho
    return [(c,) + k for k, c in out.items()]


def kernel_roofline(be, T, hbm_peak, tc_peak):
    """Live CUDA-event timing (graph replay: device time, no host dispatch) of the step's dominant kernel class -- the conv2d family
    (fprop + dgrad + wgrad of all 53 ResNet-50 convs, less the stem's dgrad that autograd
    skips, hi/lo pre-passes included: 770 GFLOP per step) -- plus the HBM-bound broadcast subtract beside it."""
    rng = np.random.default_rng(5)
    total_ms, total_flops, per = 0.0, 0.0, {"fprop": 0.0, "dgrad": 0.0, "wgrad": 0.0}
    launches = 0
    for cnt, xs, ws, st, p in resnet50_convs(BATCH):
        x = T.tensor(rng.standard_normal(xs).astype(np.float32), backend=be.name)
        w = T.tensor((rng.standard_normal(ws) * 0.05).astype(np.float32), backend=be.name)
        y = T.conv2d(x, w, None, st, p)
        g = T.tensor(rng.standard_normal(tuple(y.shape)).astype(np.float32), backend=be.name)
        flops = 2.0 * xs[0] * ws[0] * y.shape[2] * y.shape[3] * ws[1] * ws[2] * ws[3]
        ops = {"fprop": lambda: T.conv2d(x, w, None, st, p),
               "dgrad": lambda: T.conv2d_grad_input(g, w, xs, st, p),
               "wgrad": lambda: T.conv2d_grad_weight(x, g, ws, st, p)}
        if xs[1] == 3:  # the stem's input is the image: the step never computes its gradient
            del ops["dgrad"]
        for name, fn in ops.items():
            fn()
            # device time of the op as the step runs it: recorded into a CUDA graph, replayed
            be.synchronize()
            l0 = be.launch_count()
            be.capture_begin()
            keep = [fn() for _ in range(3)]
            graph = be.capture_end()
            launches += cnt * (be.launch_count() - l0) // 3
            graph.launch()
            be.synchronize()
            stop = be.event_timer()
            graph.launch()
            ms = stop() / 3
            del keep, graph
            per[name] += cnt * ms
            total_ms += cnt * ms
            total_flops += cnt * flops
    out = {"conv": {"bound": "tensor", "achieved": total_flops / total_ms / 1e9, "peak": tc_peak, "unit": "TFLOP/s",
                    "kernel": "conv2d family: fprop+dgrad+wgrad of the 53 ResNet-50 b32 convs (tcgen05 3xTF32, "
                              "incl. hi/lo pre-passes)", "ms_per_step": total_ms, "gflop_per_step": total_flops / 1e9,
                    "ms_by_kind": per, "launches_per_step": launches}}
    # HBM-bound: BatchNorm's broadcast subtract on the largest activation
    x = T.tensor(rng.standard_normal((32, 256, 56, 56)).astype(np.float32), backend=be.name)
    m = T.tensor(rng.standard_normal((1, 256, 1, 1)).astype(np.float32), backend=be.name)
    for _ in range(3):
        x - m
    stop = be.event_timer()
    for _ in range(20):
        x - m
    ms = stop() / 20
    nbytes = 2 * x.shape.size * 4 + 256 * 4
    out["ew"] = {"bound": "hbm", "achieved": nbytes / ms / 1e6, "peak": hbm_peak, "unit": "GB/s",
                 "kernel": "ew broadcast sub f32 [32,256,56,56]-[1,256,1,1]", "ms": ms}
    # HBM-bound, the step's largest kernel class by time: a JIT-specialised fused chain -- BatchNorm's
    # normalise + affine + ReLU over the largest activation, as the planned (captured) step runs it
    g = T.tensor(rng.standard_normal((1, 256, 1, 1)).astype(np.float32), backend=be.name)
    bb = T.tensor(rng.standard_normal((1, 256, 1, 1)).astype(np.float32), backend=be.name)
    sd = T.tensor((rng.random((1, 256, 1, 1)) + 0.5).astype(np.float32), backend=be.name)

    def chain():
        return ((((x - m) / sd) * g) + bb).maximum(0.0)
    chain()
    be.fusion_trace_begin()
    traced = [chain() for _ in range(10)]
    be.fusion_trace_end()
    del traced
    be.synchronize()
    be.fusion_plan_begin()
    try:
        be.capture_begin()
        keep = [chain() for _ in range(10)]
        for k in keep:
            if hasattr(k.adapter, "materialize"):
                k.adapter.materialize()
        graph = be.capture_end()
    finally:
        be.fusion_plan_end()
    graph.launch()
    be.synchronize()
    stop = be.event_timer()
    graph.launch()
    ms = stop() / 10
    nbytes = 2 * x.shape.size * 4 + 4 * 256 * 4
    out["ew_chain_jit"] = {"bound": "hbm", "achieved": nbytes / ms / 1e6, "peak": hbm_peak, "unit": "GB/s",
                           "frac": nbytes / ms / 1e6 / hbm_peak, "ms": ms,
                           "kernel": "JIT fused chain max(((x-mean)/std)*gamma+beta, 0) f32 [32,256,56,56], "
                                     "5 primitives in one launch (device time, graph replay)"}
    return out


def committed_traffic():
    """DRAM bytes of the conv family per step from the committed ncu capture of one graph
    replay (profiles/*/conv_traffic.json, newest round first), else None."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "conv_traffic.json")), reverse=True):
        try:
            with open(path) as f:
                d = json.load(f)
            return d["dram_bytes_per_step"], os.path.relpath(path, ROOT)
        except Exception:  # noqa: BLE001
            continue
    return None, None


def launch_ranks(args):
    """``--gpus N`` without a torchrun environment: start N ranks of this script through
    torch.distributed.run on 127.0.0.1 and return its exit code (rank 0 prints the line)."""
    import socket
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "RANK" not in os.environ and args.impl == "ours":
        sys.exit(launch_ranks(args))
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
        sample = (f"minml (the unmodified reference, baseline/_ref) EagerBackend ResNet-50 train_step at batch "
                  f"{REF_SAMPLE_BATCH} (bounded sample of the b32 workload), {cores} threads on {cpu_model()}")
        print(json.dumps({"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                          "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                          "data": "synthetic", "config": dict(cfg, sample_batch=REF_SAMPLE_BATCH),
                          "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "reference",
                                           "sample": sample, "cpu_model": cpu_model()},
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
    traffic, traffic_src = committed_traffic()
    roofline = {"bound": dom["bound"], "achieved": dom["achieved"], "peak": dom["peak"], "unit": dom["unit"],
                "frac": dom["achieved"] / dom["peak"], "traffic": traffic, "traffic_unit": "DRAM bytes per step",
                "traffic_source": traffic_src, "kernel": dom["kernel"], "peak_source": src,
                "gflop_per_step": dom["gflop_per_step"], "ms_per_step": dom["ms_per_step"],
                "ms_by_kind": dom["ms_by_kind"], "launches_per_step": dom["launches_per_step"],
                "note": "achieved = useful FLOPs (2*N*F*Ho*Wo*C*kh*kw summed over the family) / summed op time "
                        "(CUDA events, compute stream); 3xTF32 issues 3 tf32 MMAs per useful MAC, so the useful "
                        "ceiling is the tf32 rate / 3 = bf16 peak / 6",
                "frac_of_3xtf32_ceiling": dom["achieved"] / (tc / 2 / 3),
                "other": {k: d for k, d in rl.items() if k != "conv"}}
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
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                                "cpu_model": cpu_model(),
                                "sample": f"minml (unmodified reference) ResNet-50 train_step at batch "
                                          f"{REF_SAMPLE_BATCH}, 2 steps after 1 warm-up ({ms:.0f} ms/step)",
                                "per_op_overhead_us": cpu_overheads()}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
