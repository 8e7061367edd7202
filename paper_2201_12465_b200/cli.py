"""Command line front end: ``python -m paper_2201_12465_b200 bench --backend gpu``.

The reference's ``bench`` subcommand (minml/cli.py:212-299, parser :393-400, exit codes
:34-48) on this repo's backends: the MNIST-shaped CNN or the 784-128-10 MLP trains on the
reference's synthetic class blobs (minml/data.py:247-296, restated below on the host: it is
the input pipeline, not the hot path) for ``--warmup`` + ``--iters`` iterations, each timed
per phase -- data, forward (incl. the loss read-back), backward, optimizer step -- and the
table / ``bench.json`` have the reference's layout.  On the device every phase boundary
synchronizes the compute stream, so a phase's time is its device work plus dispatch.

``train`` and ``memsim`` (IDX datasets, figures, allocator trace replay) are outside the
data-parallel hot path this package implements and exit with code 2.
"""

import argparse
import json
import os
import sys
import time
import traceback

import numpy as np

from . import memory, models, nn, optim, registry
from . import _tensor as T
from .autograd import Variable
from .errors import (AllocError, CollectiveShapeError, CollectiveTimeout, ConfigError, Error, ManagerBusy,
                     OutOfMemory)

EXIT_OK = 0
EXIT_ERROR = 1
EXIT_CONFIG = 2
EXIT_DATA = 3
EXIT_MEMORY = 4
EXIT_COLLECTIVE = 5

_GOLDEN = 0x9E3779B97F4A7C15
_MASK = (1 << 64) - 1


def _uniform(seed, offset, count):
    """The counter RNG's doubles in [0, 1) (minml/rng.py:16-38; csrc/rng.cu on the device)."""
    idx = np.arange(count, dtype=np.uint64) + np.uint64(offset & _MASK)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & _MASK) + (idx + np.uint64(1)) * np.uint64(_GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)) * (2.0 ** -53)


def _normal(seed, offset, count):
    pairs = (count + 1) // 2
    u1, u2 = _uniform(seed, offset, pairs), _uniform(seed, offset + pairs, pairs)
    r = np.sqrt(-2.0 * np.log1p(-u1))
    out = np.empty(2 * pairs)
    out[0::2] = r * np.cos(2.0 * np.pi * u2)
    out[1::2] = r * np.sin(2.0 * np.pi * u2)
    return out[:count]


def synth_blobs(n, classes=10, dim=784, seed=0, shape=None):
    """Gaussian class blobs item by item, as minml.data.SynthBlobs (minml/data.py:247-292):
    returns (images [n, *shape] f32, labels [n] i64)."""
    shape = tuple(shape) if shape is not None else (dim,)
    centers = np.zeros((classes, dim))
    if dim >= classes:
        block = max(1, dim // (4 * classes))
        for c in range(classes):
            start = c * dim // classes
            centers[c, start:start + block] = 4.0
    else:
        for c in range(classes):
            centers[c, c % dim] = 4.0 * (1 + c // dim)
    stride = 2 * ((dim + 1) // 2)
    xs = np.empty((n,) + shape, np.float32)
    ys = np.empty(n, np.int64)
    for i in range(n):
        label = i % classes
        xs[i] = (centers[label] + 0.5 * _normal(seed, i * stride, dim)).astype(np.float32).reshape(shape)
        ys[i] = label
    return xs, ys


def _parse_alloc(text):
    name, _, arg = text.partition(":")
    if name == "split":
        if not arg:
            raise ConfigError("--alloc split needs a byte threshold, e.g. split:1048576")
        try:
            return "split", int(arg)
        except ValueError:
            raise ConfigError(f"bad split threshold {arg!r}") from None
    if name in ("native", "caching") and not arg:
        return name, None
    raise ConfigError(f"unknown allocator {text!r} (native, caching, split:<bytes>)")


def _build_parser():
    parser = argparse.ArgumentParser(prog="paper_2201_12465_b200",
                                     description="B200 backend: benchmark train iterations per phase")
    sub = parser.add_subparsers(dest="subcommand", required=True)
    bench = sub.add_parser("bench", help="time train iterations per phase and backend")
    bench.add_argument("--backend", default="gpu", help="registered backend id (default gpu)")
    bench.add_argument("--alloc", default="caching", metavar="native|caching|split:<bytes>")
    bench.add_argument("--seed", type=int, default=0)
    bench.add_argument("--out", default=None, metavar="DIR")
    bench.add_argument("--mem-telemetry", action="store_true", dest="mem_telemetry")
    bench.add_argument("--model", choices=("mlp", "cnn"), default="cnn")
    bench.add_argument("--batch", type=int, default=32)
    bench.add_argument("--lr", type=float, default=1e-3)
    bench.add_argument("--optim", choices=("sgd", "adam"), default="adam")
    bench.add_argument("--iters", type=int, default=100)
    bench.add_argument("--warmup", type=int, default=100)
    for name in ("train", "memsim"):
        sub.add_parser(name, help="not part of the B200 hot path (exits 2)")
    return parser


def _validate(args):
    for name, minimum in (("batch", 1), ("seed", 0), ("iters", 1), ("warmup", 0)):
        if getattr(args, name) < minimum:
            raise ConfigError(f"--{name} must be >= {minimum}, got {getattr(args, name)}")
    if args.lr <= 0:
        raise ConfigError(f"--lr must be positive, got {args.lr}")
    if args.backend not in registry.registered_ids():
        raise ConfigError(f"backend {args.backend!r} is not registered (have {sorted(registry.registered_ids())}; "
                          f"{getattr(registry, '_load_error', None) or 'ok'})")


def _sync(backend):
    sync = getattr(backend, "synchronize", None)
    if sync is not None:
        sync()


def cmd_bench(args):
    _validate(args)
    policy, threshold = _parse_alloc(args.alloc)
    backend = registry.get(args.backend)
    backend.seed(args.seed)
    # the policy is attached before anything is allocated (minml/cli.py:135-148, 246-250)
    manager = memory.make_manager(policy, threshold=threshold) if hasattr(memory, "make_manager") else None
    if manager is not None and hasattr(backend, "attach_manager"):
        try:
            backend.attach_manager(manager)
        except ManagerBusy:
            import gc
            gc.collect()
            backend.attach_manager(manager)
    if args.model == "cnn":
        xs, ys = synth_blobs(args.batch * 8, seed=args.seed, shape=(1, 28, 28))
        model = models.mnist_cnn(backend=args.backend)
    else:
        xs, ys = synth_blobs(args.batch * 8, seed=args.seed, dim=784)
        model = models.mlp(784, 128, 10, backend=args.backend)
    opt = optim.Adam(model.params(), lr=args.lr) if args.optim == "adam" else optim.SGD(model.params(), lr=args.lr,
                                                                                          momentum=0.9)
    batches = [(xs[i:i + args.batch], ys[i:i + args.batch]) for i in range(0, len(xs) - args.batch + 1, args.batch)]
    model.train()
    phases = {"data": 0.0, "forward": 0.0, "backward": 0.0, "step": 0.0}
    losses = []
    for i in range(args.warmup + args.iters):
        timed = i >= args.warmup
        t0 = time.perf_counter()
        images, labels = batches[i % len(batches)]
        x = Variable(T.tensor(images, backend=args.backend))
        y = T.tensor(labels, backend=args.backend)
        _sync(backend)
        t1 = time.perf_counter()
        opt.zero_grad()
        loss = nn.cross_entropy(model(x), y)
        value = loss.scalar()
        t2 = time.perf_counter()
        loss.backward()
        _sync(backend)
        t3 = time.perf_counter()
        opt.step()
        for p in opt.params:
            p.force()
        _sync(backend)
        t4 = time.perf_counter()
        if timed:
            losses.append(value)
            phases["data"] += t1 - t0
            phases["forward"] += t2 - t1
            phases["backward"] += t3 - t2
            phases["step"] += t4 - t3
    run = {"backend": args.backend, "phases": phases, "total_seconds": sum(phases.values()), "losses": losses}
    if args.mem_telemetry and manager is not None:
        run["allocator"] = manager.stats().as_dict()
    report = {"model": args.model, "batch": args.batch, "iters": args.iters, "warmup": args.warmup, "runs": [run]}
    print("backend\ttotal_s\tdata_s\tforward_s\tbackward_s\tstep_s\tfinal_loss")
    p = run["phases"]
    print(f"{run['backend']}\t{run['total_seconds']:.4f}\t{p['data']:.4f}\t{p['forward']:.4f}\t{p['backward']:.4f}"
          f"\t{p['step']:.4f}\t{run['losses'][-1]:.6f}")
    if args.out:
        os.makedirs(args.out, exist_ok=True)
        with open(os.path.join(args.out, "bench.json"), "w", encoding="ascii") as f:
            json.dump(report, f, sort_keys=True, indent=2)
            f.write("\n")
    return EXIT_OK


def main(argv=None):
    args = _build_parser().parse_args(argv)
    try:
        if args.subcommand != "bench":
            raise ConfigError(f"'{args.subcommand}' is outside the B200 hot path (SURVEY.md §8); use the reference")
        return cmd_bench(args)
    except ConfigError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_CONFIG
    except FileNotFoundError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_DATA
    except (OutOfMemory, AllocError, ManagerBusy) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_MEMORY
    except (CollectiveTimeout, CollectiveShapeError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_COLLECTIVE
    except Error as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_ERROR
    except Exception:  # noqa: BLE001 -- the reference's catch-all exit code 1
        traceback.print_exc()
        return EXIT_ERROR


if __name__ == "__main__":
    sys.exit(main())
