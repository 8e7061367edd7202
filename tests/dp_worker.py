"""Rank body for the multi-process data-parallel tests (gloo on CPU, NCCL on the GPU box)."""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.join(HERE, "golden"))


def run(rank, world, port, mode, out_dir, backend_kind):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import inputs as GI
    from paper_2201_12465_b200 import distributed, models, optim, registry, training
    from paper_2201_12465_b200.errors import CollectiveShapeError

    if backend_kind == "oracle":
        from oracle.backend import OracleBackend
        be = OracleBackend(name="dp", seed=17 if mode == "bn" else 13)
        registry.register(be)
        comm = distributed.init_from_env(device_backend=False)
    else:
        be = registry.get("gpu")
        be.seed(13)
        comm = distributed.init_from_env(device_backend=True)
    result = {}
    if mode in ("acceptance_sync", "acceptance_bucketed"):
        # T/test_acceptance.py:394-440: MLP 784-128-10, SGD 0.05, global batch 32 split over ranks
        gold = np.load(os.path.join(HERE, "golden", "dp.npz"))
        images, labels = gold["acc_images"], gold["acc_labels"]
        per, gb = 32 // world, 32
        nb = len(images) // gb
        model = models.mlp(784, 128, 10, backend=be.name)
        opt = optim.SGD(model.params(), lr=0.05)
        ddp = distributed.DataParallel(comm, model.params(), bucket_mb=0.1) if mode.endswith("bucketed") else None
        losses = []
        for k in range(50):
            b = k % nb
            lo = b * gb + rank * per
            v, _ = training.train_step(model, images[lo:lo + per], labels[lo:lo + per], opt,
                                       comm=None if ddp else comm, ddp=ddp)
            losses.append(v)
        result["losses"] = losses
        result["param_sums"] = [float(np.sum(p.numpy(), dtype=np.float64)) for p in model.params()]
        result["store_keys"] = comm._store.num_keys() if comm._store is not None else None
    elif mode == "bn":
        # per-rank BatchNorm statistics, as the reference's thread-rank run
        per, steps = 4, 4
        bs = [GI.batch("dp_bn", k, (3, 32, 32), 10, world * per) for k in range(2)]
        model = models.resnet50(classes=10, layers=(1, 1, 1, 1), width=8, backend=be.name)
        opt = optim.SGD(model.params(), lr=0.05, momentum=0.9)
        losses = []
        for k in range(steps):
            x, y = bs[k % 2]
            lo = rank * per
            losses.append(training.train_step(model, x[lo:lo + per], y[lo:lo + per], opt, comm=comm)[0])
        result["losses"] = losses
        result["param_sums"] = [float(np.sum(p.numpy(), dtype=np.float64)) for p in model.params()]
        stats = []

        def walk(m):
            for name in m.buffer_names():
                stats.append(float(np.sum(getattr(m, name).numpy(), dtype=np.float64)))
            for _, c in m._children:
                walk(c)
        walk(model)
        result["buffer_sums"] = stats
    elif mode == "broadcast":
        from paper_2201_12465_b200 import _tensor as T
        src = T.tensor(np.arange(6, dtype=np.float32).reshape(2, 3) + 10, backend=be.name)
        a = comm.broadcast(src if rank == 0 else None, root=0)       # None off-root
        b = comm.broadcast(src if rank == 0 else T.zeros((5,), backend=be.name), root=0)  # other shape
        result["a"] = a.numpy().tolist()
        result["b"] = b.numpy().tolist()
    elif mode == "shape_error":
        from paper_2201_12465_b200 import _tensor as T
        t = T.zeros((3 + rank,), backend=be.name)
        try:
            comm.all_reduce(t)
            result["raised"] = None
        except CollectiveShapeError as e:
            result["raised"] = type(e).__name__
    else:
        per = 8
        b0 = GI.batch("dp_mlp", 0, (784,), 10, world * per)
        b1 = GI.batch("dp_mlp", 1, (784,), 10, world * per)
        bx, by = np.concatenate([b0[0], b1[0]]), np.concatenate([b0[1], b1[1]])
        model = models.mlp(784, 128, 10, backend=be.name)
        opt = optim.SGD(model.params(), lr=0.05)
        ddp = distributed.DataParallel(comm, model.params(), bucket_mb=0.2) if mode == "bucketed" else None
        losses = []
        for k in range(5):
            lo = (k % 2) * world * per + rank * per
            v, _ = training.train_step(model, bx[lo:lo + per], by[lo:lo + per], opt,
                                       comm=comm if mode == "sync" else None, ddp=ddp)
            losses.append(v)
        result["losses"] = losses
        result["param_sums"] = [float(np.sum(p.numpy(), dtype=np.float64)) for p in model.params()]
        if ddp is not None:
            result["buckets"] = len(ddp.buckets)
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump(result, f)


if __name__ == "__main__":
    run(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5], sys.argv[6])
