"""Data-parallel collectives over processes (replaces minml/distributed.py:1-246).

The reference runs ranks as threads exchanging numpy chunks over queues (a ring,
distributed.py:129-156).  Here every rank is a process (one per GPU):

* ``init_from_env()`` reads RANK / WORLD_SIZE / MASTER_ADDR / MASTER_PORT (torchrun's
  variables), rendezvous through a ``torch.distributed.TCPStore`` (plumbing only) and
  creates an NCCL communicator in libpaper_b200.so for GPU tensors, or a gloo process
  group for CPU-backend tensors (the oracle, in tests);
* ``Communicator`` keeps the reference's API — ``all_reduce(t, op)``, ``all_gather``,
  ``broadcast``, ``barrier`` — and its failure semantics: metadata (shape, dtype, op) is
  compared across ranks before any data moves (``CollectiveShapeError`` on every rank,
  distributed.py:107-116) and a missing peer surfaces as ``CollectiveTimeout``;
* ``data_parallel_sync(comm, params)`` keeps the reference's post-backward contract
  (grad <- allreduce_sum(grad) / world, distributed.py:216-222), and ``DataParallel``
  does the same math bucketed and overlapped: gradients are packed into ~25 MB buckets
  in reverse registration order as the backward pass finalises them (autograd's
  grad-ready hook) and each bucket's ``ncclAllReduce`` runs on the comm stream while the
  compute stream keeps issuing the rest of backward.
"""

import datetime
import os

import numpy as np

from . import _tensor as T
from . import autograd, registry
from .errors import CollectiveShapeError, CollectiveTimeout, MissingGradient

DEFAULT_TIMEOUT = 30.0


class Communicator:
    def __init__(self, rank, world_size, store=None, nccl=None, gloo=False, timeout=DEFAULT_TIMEOUT):
        self.rank = rank
        self.world_size = world_size
        self._store = store
        self._nccl = nccl
        self._gloo = gloo
        self._timeout = timeout
        self._seq = 0

    # ------------------------------------------------------------- plumbing
    def _meta_check(self, kind, meta):
        seq = self._seq
        self._seq += 1
        if self.world_size == 1 or self._store is None:
            return
        mine = repr((kind,) + tuple(meta))
        self._store.set(f"meta/{seq}/{self.rank}", mine)
        for r in range(self.world_size):
            try:
                peer = self._store.get(f"meta/{seq}/{r}").decode()
            except Exception as exc:  # store timeout
                raise CollectiveTimeout(f"rank {self.rank}: rank {r} missing from {kind} #{seq}: {exc}") from None
            if peer != mine:
                raise CollectiveShapeError(f"rank {self.rank} called {mine}, rank {r} called {peer}")

    def _backend(self, tensor):
        return registry.get(tensor.backend_id)

    def _device(self, tensor):
        return self._nccl is not None and hasattr(self._backend(tensor), "nccl_all_reduce")

    # ----------------------------------------------------------- collectives
    def barrier(self, timeout=None):
        if self.world_size == 1:
            return
        if self._gloo or self._nccl is None:
            import torch.distributed as dist
            dist.barrier()
            return
        self._meta_check("barrier", ())

    def all_reduce(self, tensor, op="sum"):
        if op not in ("sum", "max"):
            raise ValueError(f"all_reduce op must be 'sum' or 'max', got {op!r}")
        self._meta_check("all_reduce", (tuple(tensor.shape), tensor.dtype.name, op))
        if self.world_size == 1:
            return tensor
        if self._device(tensor):
            return self._backend(tensor).nccl_all_reduce(self._nccl, tensor, op)
        import torch
        import torch.distributed as dist
        host = np.ascontiguousarray(tensor.to_host_buffer())
        buf = torch.from_numpy(host.copy())
        dist.all_reduce(buf, op=dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MAX)
        return T.tensor(buf.numpy(), backend=tensor.backend_id)

    def all_gather(self, tensor):
        self._meta_check("all_gather", (tuple(tensor.shape), tensor.dtype.name))
        if self.world_size == 1:
            return tensor.reshape((1,) + tuple(tensor.shape))
        if self._device(tensor):
            return self._backend(tensor).nccl_all_gather(self._nccl, tensor, self.world_size)
        import torch
        import torch.distributed as dist
        host = torch.from_numpy(np.ascontiguousarray(tensor.to_host_buffer()).copy())
        outs = [torch.empty_like(host) for _ in range(self.world_size)]
        dist.all_gather(outs, host)
        return T.tensor(np.stack([o.numpy() for o in outs]), backend=tensor.backend_id)

    def broadcast(self, tensor, root=0):
        if not 0 <= root < self.world_size:
            raise ValueError(f"root {root} outside world of {self.world_size}")
        self._meta_check("broadcast", (root, tuple(tensor.shape), tensor.dtype.name))
        if self.world_size == 1:
            return tensor
        if self._device(tensor):
            return self._backend(tensor).nccl_broadcast(self._nccl, tensor, root)
        import torch
        import torch.distributed as dist
        buf = torch.from_numpy(np.ascontiguousarray(tensor.to_host_buffer()).copy())
        dist.broadcast(buf, src=root)
        return T.tensor(buf.numpy(), backend=tensor.backend_id)


def init_from_env(device_backend=True, timeout=DEFAULT_TIMEOUT):
    """Join the job described by torchrun-style environment variables."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world == 1:
        return Communicator(0, 1)
    import torch.distributed as dist
    addr = os.environ.get("MASTER_ADDR", "127.0.0.1")
    port = int(os.environ.get("MASTER_PORT", "29500"))
    if not device_backend:
        if not dist.is_initialized():
            dist.init_process_group("gloo", init_method=f"tcp://{addr}:{port}", rank=rank, world_size=world,
                                    timeout=datetime.timedelta(seconds=timeout))
        store = dist.distributed_c10d._get_default_store()
        return Communicator(rank, world, store=store, gloo=True, timeout=timeout)
    store = dist.TCPStore(addr, port + 1, world, rank == 0, timeout=datetime.timedelta(seconds=timeout))
    from .gpu import _lib
    lib = _lib.load()
    if rank == 0:
        import ctypes
        buf = ctypes.create_string_buffer(128)
        _lib.check(lib.pb_nccl_unique_id(buf), "nccl id")
        store.set("nccl_id", buf.raw)
    uid = store.get("nccl_id")
    comm = lib.pb_nccl_init(world, rank, uid)
    if not comm:
        raise RuntimeError(lib.pb_last_error().decode())
    return Communicator(rank, world, store=store, nccl=comm, timeout=timeout)


def data_parallel_sync(comm, params):
    """grad <- all_reduce(grad, 'sum') / world for every parameter (reference semantics)."""
    for i, p in enumerate(params):
        if p.grad is None:
            raise MissingGradient(f"parameter {i} has no gradient to synchronize")
        p.grad = comm.all_reduce(p.grad, "sum") / comm.world_size


class DataParallel:
    """Bucketed, backward-overlapped gradient averaging with the reference's arithmetic."""

    def __init__(self, comm, params, bucket_mb=25.0):
        self.comm = comm
        self.params = list(params)
        limit = int(bucket_mb * (1 << 20))
        # reverse registration order ~ the order backward finalises gradients
        self.buckets, cur, size = [], [], 0
        for idx in range(len(self.params) - 1, -1, -1):
            p = self.params[idx]
            nbytes = p.shape.size * p.dtype.itemsize
            if cur and (size + nbytes > limit or p.dtype is not self.params[cur[0]].dtype):
                self.buckets.append(cur)
                cur, size = [], 0
            cur.append(idx)
            size += nbytes
        if cur:
            self.buckets.append(cur)
        self._where = {id(self.params[i]): b for b, bucket in enumerate(self.buckets) for i in bucket}
        # one metadata exchange for the whole plan instead of one per collective
        comm._meta_check("ddp_plan", tuple((tuple(p.shape), p.dtype.name) for p in self.params))

    def backward(self, loss):
        if self.comm.world_size == 1:
            loss.backward()
            for p in self.params:
                if p.grad is None:
                    raise MissingGradient("parameter has no gradient to synchronize")
                p.grad = p.grad / 1
            return
        pending = [len(b) for b in self.buckets]
        flights = {}
        next_launch = [0]

        def launch_ready():
            # launch strictly in bucket order so every rank issues the same NCCL sequence
            while next_launch[0] < len(self.buckets) and pending[next_launch[0]] == 0:
                b = next_launch[0]
                flights[b] = self._launch(b)
                next_launch[0] += 1

        def on_ready(v):
            b = self._where.get(id(v))
            if b is not None:
                pending[b] -= 1
                if pending[b] == 0:
                    launch_ready()

        with autograd.grad_ready_hook(on_ready):
            loss.backward()
        for b in range(len(self.buckets)):
            pending[b] = 0
        launch_ready()
        for b in range(len(self.buckets)):
            self._finish(b, flights[b])

    def _launch(self, b):
        grads = []
        for i in self.buckets[b]:
            g = self.params[i].grad
            if g is None:
                raise MissingGradient(f"parameter {i} has no gradient to synchronize")
            grads.append(g)
        be = registry.get(grads[0].backend_id)
        if hasattr(be, "bucket_pack"):
            flat = be.bucket_pack(grads)
        else:
            flat = T.concat([g.reshape((g.shape.size,)) for g in grads], 0)
        return self.comm.all_reduce(flat, "sum") if self.comm._nccl is None else \
            be.nccl_all_reduce(self.comm._nccl, flat, "sum", wait=False)

    def _finish(self, b, reduced):
        be = registry.get(reduced.backend_id)
        if hasattr(be, "nccl_wait") and self.comm._nccl is not None:
            be.nccl_wait(self.comm._nccl)
        avg = reduced / self.comm.world_size
        off = 0
        for i in self.buckets[b]:
            p = self.params[i]
            n = p.shape.size
            p.grad = avg.slice((off,), (off + n,)).reshape(tuple(p.shape))
            off += n
