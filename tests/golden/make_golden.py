"""Generate golden fixtures by running the REFERENCE (minml) in the build container.

    PB_NO_AUTOREGISTER=1 python tests/golden/make_golden.py

Needs /root/reference (read-only) — it runs only here, never on the GPU box.
Outputs (committed):
  ops.json / ops.npz        per-primitive cases: inputs, params, reference output or error
  rng.npz                   splitmix64 words / uniform / normal streams
  alloc.json                allocator known answers (bin/round tables, trace replays)
  trace.txt                 the reference's synthetic allocation trace (memory.make_synthetic_trace)
  models.json / models.npz  short training trajectories of the five config families
                            (reduced sizes) + a 2-rank data-parallel run
Model compositions come from paper_2201_12465_b200.models with ``ns`` bound to the
reference's own nn/ops/_tensor/autograd, so both sides run the same graph.
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
os.environ.setdefault("PB_NO_AUTOREGISTER", "1")

import minml  # noqa: E402
from minml import _tensor as MT, autograd as MA, data as MD, distributed as MDist  # noqa: E402
from minml import memory as MM, nn as MN, ops as MO, optim as MOpt, registry as MR  # noqa: E402
from minml import rng as MRng, training as MTr  # noqa: E402
from minml.eager import EagerBackend  # noqa: E402

from paper_2201_12465_b200 import models as PM  # noqa: E402

sys.path.insert(0, HERE)
import inputs as GI  # noqa: E402

NS = PM.namespace(MN, MO, MT, MA)
R = np.random.default_rng(20220128)


def jsonable(v):
    if isinstance(v, tuple):
        return [jsonable(x) for x in v]
    if isinstance(v, list):
        return [jsonable(x) for x in v]
    if isinstance(v, dict):
        return {k: jsonable(x) for k, x in v.items()}
    if isinstance(v, np.generic):
        return v.item()
    return v


class Ops:
    def __init__(self):
        self.cases = []
        self.arrays = {}

    def add(self, name, params, inputs, tag=""):
        i = len(self.cases)
        keys = []
        tensors = []
        for j, a in enumerate(inputs):
            k = f"c{i}_in{j}"
            self.arrays[k] = a
            keys.append(k)
            tensors.append(minml.tensor(a, backend="eager"))
        p = dict(params)
        host = None
        if name == "from_host":
            host = p["array"]
            k = f"c{i}_host"
            self.arrays[k] = host
            p = {"array": k}
            call_params = {"array": host}
        else:
            call_params = params
        case = {"name": name, "params": jsonable(p), "inputs": keys, "tag": tag}
        try:
            out = MT.apply(name, call_params, tensors, backend="eager" if not tensors else None)
            res = out.to_host_buffer()
            case["out"] = f"c{i}_out"
            case["dtype"] = out.dtype.name
            case["shape"] = list(out.shape)
            self.arrays[case["out"]] = res
        except minml.Error as exc:
            case["error"] = type(exc).__name__
        except (ValueError, OverflowError) as exc:
            case["error"] = type(exc).__name__
        self.cases.append(case)


def f32(*shape, lo=-2.0, hi=2.0):
    return R.uniform(lo, hi, shape).astype(np.float32)


def build_ops():
    o = Ops()
    # -- binary, every op over dtype pairs and broadcast shapes
    pairs = [("f32", "f32"), ("f32", "f64"), ("f64", "f64"), ("i64", "f32"), ("i32", "f32"),
             ("i32", "i32"), ("i64", "i64"), ("u8", "u8"), ("u8", "i32"), ("bool", "f32")]
    shapes = [((3, 4), (3, 4)), ((3, 1, 4), (5, 4)), ((2, 3), ()), ((1,), (4, 1)), ((0, 3), (3,))]

    def sample(dt, shape):
        if dt == "bool":
            return R.integers(0, 2, shape).astype(np.bool_)
        if dt == "u8":
            return R.integers(0, 9, shape).astype(np.uint8)
        if dt in ("i32", "i64"):
            return R.integers(-7, 8, shape).astype(np.int32 if dt == "i32" else np.int64)
        return R.uniform(-3, 3, shape).astype(np.float32 if dt == "f32" else np.float64)

    arith = ["add", "sub", "mul", "div", "pow", "minimum", "maximum", "eq", "lt", "gt"]
    for name in arith:
        for da, db in pairs:
            for sa, sb in shapes[:4] if (da, db) == ("f32", "f32") else shapes[:2]:
                a, b = sample(da, sa), sample(db, sb)
                if name == "pow" and da != "f32" and da != "f64":
                    b = np.abs(b).astype(b.dtype) if b.dtype.kind in "iu" else b
                if name == "pow" and da in ("f32", "f64"):
                    a = np.abs(a).astype(a.dtype) + 0.1
                if name == "div" and b.dtype.kind in "iu":
                    b = np.where(b == 0, 1, b).astype(b.dtype)
                o.add(name, {}, [a, b], tag=f"{da},{db}")
        # empty broadcast
        o.add(name, {}, [sample("f32", (0, 3)), sample("f32", (3,))], tag="empty")
    for name in ("logical_and", "logical_or"):
        o.add(name, {}, [sample("bool", (3, 4)), sample("bool", (4,))])
        o.add(name, {"scalar": True}, [sample("bool", (5,))])
        o.add(name, {}, [sample("f32", (2,)), sample("bool", (2,))], tag="error")
    # scalars: weak typing, both sides
    for name in ("add", "sub", "mul", "div", "pow", "minimum", "maximum", "eq", "lt", "gt"):
        for dt in ("f32", "f64", "i32", "i64", "u8"):
            for s in (2, 0.5, True, -3):
                if dt == "u8" and isinstance(s, int) and not isinstance(s, bool) and s < 0:
                    continue
                a = sample(dt, (3, 2))
                if name == "pow":
                    if dt in ("f32", "f64"):
                        a = np.abs(a).astype(a.dtype) + 0.5
                    elif isinstance(s, int) and not isinstance(s, bool) and s < 0:
                        continue
                for side in ("right", "left"):
                    p = {"scalar": s} if side == "right" else {"scalar": s, "scalar_side": "left"}
                    if name == "div" and side == "left" and dt in ("i32", "i64", "u8"):
                        a = np.where(a == 0, 1, a).astype(a.dtype)
                    o.add(name, p, [a], tag=f"{dt},scalar")
    # special values
    sp = np.array([np.nan, 1.0, -np.inf, np.inf, 0.0, -0.0, 3.5, np.nan], np.float32)
    sq = np.array([2.0, np.nan, 5.0, np.inf, -0.0, 0.0, 3.5, -1.0], np.float32)
    for name in ("minimum", "maximum", "eq", "lt", "gt", "add", "mul", "div", "sub", "pow"):
        o.add(name, {}, [sp, sq], tag="special")
    o.add("div", {}, [np.array([1, 2], np.int64), np.array([1, 0], np.int64)], tag="intdiv0")
    o.add("pow", {}, [np.array([2, 3], np.int64), np.array([1, -1], np.int64)], tag="negpow")
    o.add("div", {"scalar": 0}, [np.array([1, 2], np.int32)], tag="intdiv0scalar")
    o.add("add", {}, [np.array([2**31 - 1], np.int32), np.array([1], np.int32)], tag="wrap")
    o.add("mul", {}, [np.array([200], np.uint8), np.array([2], np.uint8)], tag="wrap")
    o.add("add", {}, [f32(2, 3), np.array([True, False, True])], tag="error_bool")
    # -- unary
    for name in ("neg", "abs", "exp", "log", "sqrt", "sin", "cos", "tanh"):
        o.add(name, {}, [f32(4, 5, lo=0.01, hi=4.0) if name in ("log", "sqrt") else f32(4, 5, lo=-6, hi=6)])
        o.add(name, {}, [R.uniform(0.01, 4, (7,))], tag="f64")
        o.add(name, {}, [sp], tag="special")
    for dt in ("i32", "i64", "u8"):
        o.add("neg", {}, [sample(dt, (6,))], tag=dt)
        o.add("abs", {}, [sample(dt, (6,))], tag=dt)
    o.add("exp", {}, [sample("i32", (3,))], tag="error")
    o.add("logical_not", {}, [sample("bool", (2, 3))])
    o.add("logical_not", {}, [f32(3)], tag="error")
    vals = np.array([0.0, -0.0, 1.7, -1.7, 255.5, 256.0, -129.2, 300.7, 3e9, -3e9, 1e20, np.nan, np.inf, -np.inf])
    srcs = {"f64": vals, "f32": vals.astype(np.float32),
            "i64": np.array([0, 1, -1, 255, 256, -129, 2**31, -2**31 - 1, 2**40 + 7], np.int64),
            "i32": np.array([0, 1, -1, 255, 256, -129, 2**31 - 1, -2**31], np.int32),
            "u8": np.array([0, 1, 127, 128, 255], np.uint8),
            "bool": np.array([True, False, True])}
    for sdt, arr in srcs.items():
        for ddt in ("bool", "u8", "i32", "i64", "f32", "f64"):
            o.add("astype", {"dtype": ddt}, [arr], tag=f"{sdt}->{ddt}")
    # -- reductions
    for name in ("sum", "max_reduce", "min_reduce", "argmax"):
        for dt in ("f32", "f64", "i32", "i64", "u8"):
            a = sample(dt, (3, 4, 5))
            for axis in (0, 1, 2, -1, None):
                if name == "argmax" and axis is None:
                    continue
                for keep in (False, True):
                    o.add(name, {"axis": axis, "keepdims": keep}, [a], tag=dt)
        o.add(name, {"axis": 1, "keepdims": False}, [np.array([[1.0, np.nan, 3.0, np.nan], [2.0, 2.0, 1.0, 2.0]], np.float32)], tag="nan")
        o.add(name, {"axis": 0, "keepdims": False}, [np.zeros((0, 3), np.float32)], tag="empty")
    o.add("argmax", {"axis": 1, "keepdims": True}, [np.array([[3, 7, 7, 1], [5, 5, 5, 5]], np.int64)], tag="ties")
    o.add("argmax", {"axis": None}, [f32(4)], tag="error")
    o.add("sum", {"axis": None, "keepdims": False}, [R.standard_normal(100000).astype(np.float32) * 1000], tag="f64acc")
    o.add("sum", {"axis": 0, "keepdims": False}, [R.standard_normal((4096, 7)).astype(np.float32)], tag="col")
    o.add("sum", {"axis": 1, "keepdims": False}, [R.standard_normal((5, 3000)).astype(np.float32)], tag="row")
    o.add("sum", {"axis": None, "keepdims": False}, [np.array([[True]])], tag="error")
    o.add("sum", {"axis": 1, "keepdims": False}, [np.full((2, 300), 200, np.uint8)], tag="wrap")
    # -- contractions
    for (m, k, n) in ((4, 5, 3), (64, 200, 96), (33, 17, 65), (1, 1, 1)):
        o.add("matmul", {}, [f32(m, k), f32(k, n)], tag="f32")
    o.add("matmul", {}, [f32(3, 8, 5), f32(3, 5, 7)], tag="batched")
    o.add("matmul", {}, [R.standard_normal((6, 4)), R.standard_normal((4, 3))], tag="f64")
    o.add("matmul", {}, [sample("i64", (3, 4)), sample("i64", (4, 2))], tag="i64")
    o.add("matmul", {}, [sample("i32", (3, 4)), f32(4, 2)], tag="mixed")
    o.add("matmul", {}, [f32(3, 4), f32(5, 2)], tag="error")
    o.add("matmul", {}, [f32(2, 3, 4), f32(3, 4, 2)], tag="error")
    conv = [((2, 3, 9, 9), (4, 3, 3, 3), (1, 1), (0, 0)), ((2, 3, 9, 9), (4, 3, 3, 3), (2, 2), (1, 1)),
            ((1, 2, 11, 13), (3, 2, 5, 3), (1, 2), (2, 1)), ((2, 4, 8, 8), (6, 4, 1, 1), (2, 2), (0, 0)),
            ((1, 3, 23, 23), (5, 3, 11, 11), (4, 4), (2, 2)), ((2, 1, 28, 28), (4, 1, 5, 5), (1, 1), (0, 0)),
            ((1, 2, 7, 7), (3, 2, 7, 7), (2, 2), (3, 3))]
    for xs, ws, st, pd in conv:
        x, w = f32(*xs), f32(*ws)
        o.add("conv2d", {"stride": st, "padding": pd}, [x, w])
        o.add("conv2d", {"stride": st, "padding": pd}, [x, w, f32(ws[0])], tag="bias")
        out = MT.conv2d(minml.tensor(x), minml.tensor(w), None, st, pd)
        g = f32(*out.shape)
        o.add("conv2d_grad_input", {"stride": st, "padding": pd, "x_shape": xs}, [g, w])
        o.add("conv2d_grad_weight", {"stride": st, "padding": pd, "w_shape": ws}, [x, g])
    o.add("conv2d", {"stride": (1, 1), "padding": (0, 0)}, [R.standard_normal((1, 2, 5, 5)), R.standard_normal((2, 2, 3, 3))], tag="f64")
    o.add("conv2d", {"stride": (1, 1), "padding": (0, 0)}, [f32(1, 2, 5, 5), f32(2, 3, 3, 3)], tag="error")
    # -- movement
    a = f32(2, 3, 4)
    for shp in ((24,), (4, 6), (2, 12, 1), (1, 2, 3, 4)):
        o.add("reshape", {"shape": shp}, [a])
    o.add("reshape", {"shape": (5, 5)}, [a], tag="error")
    for perm in ((2, 1, 0), (0, 2, 1), (1, 0, 2), None):
        o.add("transpose", {} if perm is None else {"perm": perm}, [a])
    o.add("transpose", {"perm": (0, 0, 1)}, [a], tag="error")
    o.add("concat", {"axis": 1}, [f32(2, 3), f32(2, 5)])
    o.add("concat", {"axis": 0}, [sample("i32", (1, 3)), f32(2, 3), sample("i64", (3, 3))], tag="mixed")
    o.add("concat", {"axis": -1}, [f32(2, 1, 2), f32(2, 1, 3), f32(2, 1, 1)])
    o.add("concat", {"axis": 0}, [f32(2, 3), f32(2, 4)], tag="error")
    for st, sp_, ss in (((0, 1, 0), (2, 3, 4), (1, 1, 2)), ((1, 0, 1), (2, 3, 4), (1, 2, 3)), ((0, 0, 0), (2, 0, 4), (1, 1, 1)), ((0, 2, 3), (2, 3, 4), (2, 1, 1))):
        o.add("slice", {"starts": st, "stops": sp_, "steps": ss}, [a])
    o.add("slice", {"starts": (0, 0, 0), "stops": (2, 4, 4), "steps": (1, 1, 1)}, [a], tag="error")
    for pw, v in ((((0, 0), (1, 2), (0, 1)), 0), (((1, 1), (0, 0), (2, 0)), -np.inf), (((0, 0), (0, 0), (0, 0)), 1.5)):
        o.add("pad", {"pad_width": pw, "value": v}, [a])
    o.add("pad", {"pad_width": ((1, 0),), "value": 7}, [sample("i64", (3,))], tag="i64")
    # -- creation
    for shp, v, dt in (((2, 3), 1.5, "f32"), ((4,), 7, "i64"), ((2, 2), True, "bool"), ((3,), -1, "u8"),
                       ((2,), float("inf"), "f64"), ((0, 2), 3, "i32"), ((), 2.5, "f32"), ((3,), 2.7, "i32")):
        o.add("full", {"shape": shp, "value": v, "dtype": dt}, [])
    o.add("arange", {"n": 7, "dtype": "i64"}, [])
    o.add("arange", {"n": 0, "dtype": "i64"}, [])
    for dt in ("f32", "f64"):
        for shp, seed, off in (((5, 7), 0, 0), ((33,), 12345, 1000), ((2, 2), 2**63 + 11, 2**40)):
            o.add("rand_uniform", {"shape": shp, "dtype": dt, "seed": seed, "offset": off}, [])
            o.add("rand_normal", {"shape": shp, "dtype": dt, "seed": seed, "offset": off}, [])
    o.add("rand_uniform", {"shape": (2,), "dtype": "i32", "seed": 0, "offset": 0}, [], tag="error")
    o.add("from_host", {"array": f32(3, 2)}, [])
    o.add("from_host", {"array": sample("i64", (4,))}, [])
    return o


def build_rng():
    out = {}
    for k, (seed, off, n) in enumerate(((0, 0, 64), (1, 0, 16), (12345, 999, 33), (2**64 - 1, 2**63, 8), (7, 2**40 - 3, 5))):
        out[f"w{k}"] = MRng.raw(seed, off, n)
        out[f"u{k}"] = MRng.uniform(seed, off, n)
        out[f"n{k}"] = MRng.normal(seed, off, n)
        out[f"meta{k}"] = np.array([seed, off, n], dtype=np.uint64)
    return out


def build_alloc():
    res = {"bin_size": {}, "round_up": {}}
    for n in (1, 511, 512, 513, 1000, 4096, 70000, (1 << 20), (1 << 20) + 1, 123456789):
        res["bin_size"][str(n)] = MM.bin_size(n)
        res["round_up"][str(n)] = MM.round_up(n)
    lines = MM.make_synthetic_trace()
    hand = ["A 1 1000 conv", "A 2 600 bias", "F 1", "A 3 900 act", "F 2", "F 3"]
    replays = {}
    for label, tr in (("bundled", lines), ("hand", hand)):
        for policy, th in (("native", None), ("caching", None), ("split_restricted", 1 << 20), ("split_restricted", 0), ("split_restricted", 1 << 16)):
            r = MM.replay(tr, policy, threshold=th)
            key = f"{label}/{policy}/{th}"
            replays[key] = {"peak_internal_fragmentation": r.peak_internal_fragmentation,
                            "stats": r.stats.as_dict(),
                            "timeline_len": len(r.timeline),
                            "live_req": [row[1] for row in r.timeline] if label == "hand" else None}
    res["replays"] = replays
    with open(os.path.join(HERE, "trace.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    return res


def run_traj(name, build, images, labels, steps, sgd, seed):
    be_name = f"gold-{name}"
    MR.register(EagerBackend(name=be_name, seed=seed))
    try:
        model = build(be_name)
        opt = MOpt.SGD(model.params(), **sgd)
        losses = []
        for k in range(steps):
            x, y = images[k % len(images)], labels[k % len(labels)]
            loss, _ = MTr.train_step(model, x, y, opt)
            losses.append(loss)
        params = [p.numpy() for p in model.params()]
    finally:
        MR.unregister(be_name)
    summ = [[float(np.sum(p, dtype=np.float64)), float(np.sum(np.abs(p), dtype=np.float64))] for p in params]
    first = {f"{name}_p{i}": p for i, p in enumerate(params) if p.size <= 4096}
    return {"losses": losses, "param_sums": summ, "seed": seed, "steps": steps, "sgd": sgd,
            "n_params": len(params)}, first


def build_models():
    meta, arrays = {}, {}
    cfgs = {
        "mlp": (lambda be: PM.mlp(784, 256, 10, backend=be, ns=NS), (784,), 10, 64, 10, dict(lr=0.05)),
        "lenet": (lambda be: PM.mnist_cnn(backend=be, ns=NS), (1, 28, 28), 10, 16, 5, dict(lr=0.05)),
        "alexnet_tiny": (lambda be: PM.alexnet(classes=10, image=67, channels=(8, 16, 24, 16, 16), hidden=64,
                                               backend=be, ns=NS), (3, 67, 67), 10, 8, 3, dict(lr=0.01, momentum=0.9)),
        "resnet_tiny": (lambda be: PM.resnet50(classes=10, layers=(1, 1, 1, 1), width=8, backend=be, ns=NS),
                        (3, 32, 32), 10, 4, 3, dict(lr=0.05, momentum=0.9)),
    }
    for name, (build, shape, classes, batch, steps, sgd) in cfgs.items():
        bs = [GI.batch(name, k, shape, classes, batch) for k in range(2)]
        m, first = run_traj(name, build, [b[0] for b in bs], [b[1] for b in bs], steps, sgd, seed=3)
        arrays.update(first)
        meta[name] = dict(m, input=list(shape), classes=classes, batch=batch)
    # BERT-like, tiny
    vocab, seq = 50, 8
    bs = [GI.batch("bert_tiny", k, None, 2, 4, tokens=(seq, vocab)) for k in range(2)]
    toks, labs = [b[0] for b in bs], [b[1] for b in bs]
    m, first = run_traj("bert_tiny", lambda be: PM.bert_base(vocab=vocab, seq=seq, d=16, heads=2, ffn=32, layers=2,
                                                              classes=2, backend=be, ns=NS),
                        toks, labs, 3, dict(lr=0.05, momentum=0.9), seed=3)
    arrays.update(first)
    meta["bert_tiny"] = dict(m, vocab=vocab, seq=seq, batch=4)
    # data parallel: 2 thread ranks x 8 vs the reference's own run_ranks
    world, per, steps = 2, 8, 5
    b0, b1 = GI.batch("dp_mlp", 0, (784,), 10, world * per), GI.batch("dp_mlp", 1, (784,), 10, world * per)
    bx = np.concatenate([b0[0], b1[0]])
    by = np.concatenate([b0[1], b1[1]])
    for r in range(world):
        MR.register(EagerBackend(name=f"gold-dp-{r}", seed=13))

    def fn(comm):
        model = PM.mlp(784, 128, 10, backend=f"gold-dp-{comm.rank}", ns=NS)
        opt = MOpt.SGD(model.params(), lr=0.05)
        out = []
        for k in range(steps):
            lo = (k % 2) * world * per + comm.rank * per
            v, _ = MTr.train_step(model, bx[lo:lo + per], by[lo:lo + per], opt, comm=comm)
            out.append(v)
        return out, [float(np.sum(p.numpy(), dtype=np.float64)) for p in model.params()]

    try:
        res = MDist.run_ranks(world, fn)
    finally:
        for r in range(world):
            MR.unregister(f"gold-dp-{r}")
    meta["dp_mlp"] = {"world": world, "per_rank": per, "steps": steps, "seed": 13,
                      "losses": [r[0] for r in res], "param_sums": res[0][1]}
    return meta, arrays


def main():
    ops = build_ops()
    with open(os.path.join(HERE, "ops.json"), "w") as f:
        json.dump(ops.cases, f, indent=0)
    np.savez_compressed(os.path.join(HERE, "ops.npz"), **ops.arrays)
    np.savez_compressed(os.path.join(HERE, "rng.npz"), **build_rng())
    with open(os.path.join(HERE, "alloc.json"), "w") as f:
        json.dump(build_alloc(), f, indent=1)
    meta, arrays = build_models()
    with open(os.path.join(HERE, "models.json"), "w") as f:
        json.dump(meta, f, indent=1)
    np.savez_compressed(os.path.join(HERE, "models.npz"), **arrays)
    print(f"{len(ops.cases)} op cases, models: {sorted(meta)}")


if __name__ == "__main__":
    main()
