"""Runtime plumbing on the B200: the NCCL data plane of DataParallel on a real (1-rank)
NCCL communicator -- eager and recorded into a CUDA graph --, concurrent ``execute`` from
several threads, and CapturedStep's optimizer / hyper-parameter guards."""

import threading

import numpy as np
import pytest

from frontend_util import BUILDERS
from gpu_util import gpu_backend
from paper_2201_12465_b200 import _tensor as T
from paper_2201_12465_b200 import distributed, optim, training

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl1():
    """A world-size-1 NCCL communicator: every collective runs through ncclAllReduce."""
    gpu_backend()
    return distributed.nccl_communicator(0, 1, distributed.nccl_unique_id())


def _data(shape, classes, batch=4):
    r = np.random.default_rng(0)
    return [(r.standard_normal((batch,) + shape).astype(np.float32), r.integers(0, classes, batch).astype(np.int64))
            for _ in range(2)]


def _state(model, opt):
    return [p.numpy() for p in model.params()] + [v.numpy() for v in opt.velocity]


@pytest.mark.parametrize("name,shape,classes", [("lenet", (1, 28, 28), 10), ("resnet_tiny", (3, 32, 32), 10)])
@pytest.mark.parametrize("captured", [False, True], ids=["eager", "graph"])
def test_ddp_nccl_data_plane_bit_equal_to_plain_step(nccl1, name, shape, classes, captured):
    """DataParallel over NCCL (bucket_pack, ncclAvg on the comm stream, fences, grad slice
    views) is bit-equal to the no-DDP step at world 1 -- eagerly and inside CapturedStep."""
    be = gpu_backend()
    data = _data(shape, classes)
    runs = []
    for use_ddp in (False, True):
        be.seed(3)
        model = BUILDERS[name](be.name)
        opt = optim.SGD(model.params(), lr=0.05, momentum=0.9)
        ddp = distributed.DataParallel(nccl1, model.params(), bucket_mb=0.05) if use_ddp else None
        if ddp is not None:
            assert len(ddp.buckets) > 1
        step = training.CapturedStep(model, opt, ddp=ddp, warmup=2) if captured else None
        losses = []
        for k in range(5):
            x, y = data[k % 2]
            losses.append(step(x, y)[0] if captured else training.train_step(model, x, y, opt, ddp=ddp)[0])
        if captured:
            assert step.graph is not None
        runs.append((losses, _state(model, opt)))
    assert runs[0][0] == runs[1][0], runs
    for a, b in zip(runs[0][1], runs[1][1]):
        assert np.array_equal(a, b)


def test_nccl_collectives_world1(nccl1):
    be = gpu_backend()
    x = T.tensor(np.arange(10, dtype=np.float32), backend=be.name)
    for op in ("sum", "max", "avg"):
        out = be.nccl_all_reduce(nccl1._nccl, x, op)
        assert np.array_equal(out.numpy(), x.numpy())
    g = be.nccl_all_gather(nccl1._nccl, x, 1)
    assert np.array_equal(g.numpy()[0], x.numpy())
    b = be.nccl_broadcast(nccl1._nccl, x, 0)
    assert np.array_equal(b.numpy(), x.numpy())


def test_execute_is_thread_safe():
    """Eight threads issue interleaved primitives on one backend; every result is right."""
    be = gpu_backend()
    errors = []

    def work(k):
        try:
            r = np.random.default_rng(k)
            for _ in range(40):
                a = r.standard_normal((64, 33)).astype(np.float32)
                b = r.standard_normal((33, 17)).astype(np.float32)
                ta, tb = T.tensor(a, backend=be.name), T.tensor(b, backend=be.name)
                s = (ta * 2.0 + 1.0).sum(1).numpy()
                ref = ((a * np.float32(2.0)) + np.float32(1.0)).astype(np.float64).sum(1)
                if np.max(np.abs(s - ref) / np.maximum(np.abs(ref), 1.0)) > 1e-6:
                    errors.append(("sum", k))
                m = T.matmul(ta, tb).numpy()
                ref = a.astype(np.float64) @ b.astype(np.float64)
                if np.max(np.abs(m - ref) / np.maximum(np.abs(ref), 1.0)) > 1e-5:
                    errors.append(("matmul", k))
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    ts = [threading.Thread(target=work, args=(k,)) for k in range(8)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors[:5]


def test_captured_step_refuses_adam():
    be = gpu_backend()
    model = BUILDERS["mlp"](be.name)
    with pytest.raises(TypeError):
        training.CapturedStep(model, optim.Adam(model.params(), lr=1e-3))


def test_captured_step_rerecords_on_lr_change():
    """An LR schedule between replays: the step is recorded again, results equal eager."""
    be = gpu_backend()
    data = _data((1, 28, 28), 10)
    runs = []
    for captured in (False, True):
        be.seed(4)
        model = BUILDERS["lenet"](be.name)
        opt = optim.SGD(model.params(), lr=0.05, momentum=0.9)
        step = training.CapturedStep(model, opt, warmup=1, fuse=False) if captured else None
        losses = []
        for k in range(6):
            if k == 4:
                opt.lr = 0.01
            x, y = data[k % 2]
            losses.append(step(x, y)[0] if captured else training.train_step(model, x, y, opt)[0])
        runs.append((losses, _state(model, opt)))
    assert runs[0][0] == runs[1][0]
    for a, b in zip(runs[0][1], runs[1][1]):
        assert np.array_equal(a, b)


def test_collective_watchdog_times_out_and_aborts():
    """A collective that never completes (the comm stream held by a stall kernel, standing in
    for a peer that never arrives) raises CollectiveTimeout after the communicator's timeout
    -- the reference's failure semantics (minml/distributed.py:23, 93-105) -- instead of hanging;
    the aborted communicator refuses further collectives."""
    import time

    from paper_2201_12465_b200.errors import CollectiveTimeout
    from paper_2201_12465_b200.gpu import _lib
    be = gpu_backend()
    lib = _lib.load()
    # the bare watchdog: a 1.5 s stall against a 100 ms deadline, then against a generous one
    assert lib.pb_debug_stall_comm(1500) == 0
    t0 = time.perf_counter()
    assert lib.pb_nccl_sync(None, 100) == 8  # PB_ERR_TIMEOUT
    assert time.perf_counter() - t0 < 1.0
    assert lib.pb_nccl_sync(None, 10000) == 0
    # through the Communicator / backend on a fresh world-1 NCCL communicator
    comm = distributed.nccl_communicator(0, 1, distributed.nccl_unique_id(), timeout=0.2)
    x = T.tensor(np.arange(8, dtype=np.float32), backend=be.name)
    assert np.array_equal(be.nccl_all_reduce(comm._nccl, x, "sum", timeout=comm._timeout).numpy(), x.numpy())
    assert lib.pb_debug_stall_comm(1500) == 0
    with pytest.raises(CollectiveTimeout):
        be.nccl_all_reduce(comm._nccl, x, "sum", timeout=comm._timeout)
    with pytest.raises(CollectiveTimeout):
        be.nccl_broadcast(comm._nccl, x, 0, timeout=comm._timeout)
    be.synchronize()
