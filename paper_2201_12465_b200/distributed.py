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
    def _meta_check(self, kind, meta, publish=None):
        """Compare (kind, meta) across ranks before any data moves (minml/distributed.py:
        107-116).  Every rank posts ``meta/{seq}/{rank}`` and reads all peers'.  A rank that
        has read every peer's post for ``seq`` knows every rank finished check ``seq - 1``,
        so it deletes its own post of ``seq - 1``: the store holds at most two checks' keys.
        ``publish`` (root only) is extra data peers read back from the root's post; the
        root's value is returned on every rank."""
        seq = self._seq
        self._seq += 1
        if self.world_size == 1 or self._store is None:
            return publish
        mine = repr((kind,) + tuple(meta))
        self._store.set(f"meta/{seq}/{self.rank}", mine + "\x00" + repr(publish))
        extra = None
        for r in range(self.world_size):
            try:
                peer, _, pub = self._store.get(f"meta/{seq}/{r}").decode().partition("\x00")
            except Exception as exc:  # store timeout
                raise CollectiveTimeout(f"rank {self.rank}: rank {r} missing from {kind} #{seq}: {exc}") from None
            if peer != mine:
                raise CollectiveShapeError(f"rank {self.rank} called {mine}, rank {r} called {peer}")
            if pub != "None":
                extra = pub
        if seq:
            try:
                self._store.delete_key(f"meta/{seq - 1}/{self.rank}")
            except Exception:  # noqa: BLE001 -- a store without delete keeps the key
                pass
        return extra

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

    def all_reduce(self, tensor, op="sum", _checked=False):
        if op not in ("sum", "max"):
            raise ValueError(f"all_reduce op must be 'sum' or 'max', got {op!r}")
        if not _checked:
            self._meta_check("all_reduce", (tuple(tensor.shape), tensor.dtype.name, op))
        if self.world_size == 1:
            return tensor
        if self._device(tensor):
            return self._backend(tensor).nccl_all_reduce(self._nccl, tensor, op, timeout=self._timeout)
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
            return self._backend(tensor).nccl_all_gather(self._nccl, tensor, self.world_size, timeout=self._timeout)
        import torch
        import torch.distributed as dist
        host = torch.from_numpy(np.ascontiguousarray(tensor.to_host_buffer()).copy())
        outs = [torch.empty_like(host) for _ in range(self.world_size)]
        dist.all_gather(outs, host)
        return T.tensor(np.stack([o.numpy() for o in outs]), backend=tensor.backend_id)

    def broadcast(self, tensor, root=0):
        """Root's tensor on every rank (minml/distributed.py:166-175): only ``root`` is
        compared across ranks; the root publishes shape, dtype and backend, so other ranks
        may pass ``None`` or a placeholder of any shape."""
        if not 0 <= root < self.world_size:
            raise ValueError(f"root {root} outside world of {self.world_size}")
        mine = None
        if self.rank == root:
            if tensor is None:
                raise ValueError("broadcast: the root must pass a tensor")
            mine = (tuple(tensor.shape), tensor.dtype.name, tensor.backend_id)
        pub = self._meta_check("broadcast", (root,), publish=mine)
        if self.world_size == 1:
            return tensor
        import ast
        shape, dtname, root_backend = ast.literal_eval(pub) if isinstance(pub, str) else pub
        if self.rank != root:
            if tensor is not None:
                backend = tensor.backend_id
            else:
                backend = root_backend if root_backend in registry.registered_ids() else registry.default().name
            if tensor is None or tuple(tensor.shape) != shape or tensor.dtype.name != dtname:
                tensor = T.zeros(shape, dtype=dtname, backend=backend)
        if self._device(tensor):
            return self._backend(tensor).nccl_broadcast(self._nccl, tensor, root, timeout=self._timeout)
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
    if rank == 0:
        store.set("nccl_id", nccl_unique_id())
    return nccl_communicator(rank, world, store.get("nccl_id"), store=store, timeout=timeout)


def nccl_unique_id():
    """128 bytes of ncclUniqueId from rank 0 (pb_nccl_unique_id)."""
    import ctypes
    from .gpu import _lib
    buf = ctypes.create_string_buffer(128)
    _lib.check(_lib.load().pb_nccl_unique_id(buf), "nccl id")
    return buf.raw


def nccl_communicator(rank, world, uid, store=None, timeout=DEFAULT_TIMEOUT):
    """A Communicator over an NCCL communicator in libpaper_b200.so (``world`` may be 1:
    the device data plane -- bucket packing, ncclAllReduce on the comm stream, the
    compute<->comm fences -- then runs for real on a single GPU)."""
    from .gpu import _lib
    lib = _lib.load()
    comm = lib.pb_nccl_init(world, rank, uid)
    if not comm:
        raise RuntimeError(lib.pb_last_error().decode())
    return Communicator(rank, world, store=store, nccl=comm, timeout=timeout)


def data_parallel_sync(comm, params):
    """grad <- all_reduce(grad, 'sum') / world for every parameter (reference semantics,
    minml/distributed.py:216-222); one metadata exchange covers the whole parameter list."""
    for i, p in enumerate(params):
        if p.grad is None:
            raise MissingGradient(f"parameter {i} has no gradient to synchronize")
    comm._meta_check("dp_sync", tuple((tuple(p.grad.shape), p.grad.dtype.name) for p in params))
    for p in params:
        p.grad = comm.all_reduce(p.grad, "sum", _checked=True) / comm.world_size


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
        if self.comm.world_size == 1 and self.comm._nccl is None:
            loss.backward()  # one rank, no communicator: grad / 1 == grad, nothing to do
            for p in self.params:
                if p.grad is None:
                    raise MissingGradient("parameter has no gradient to synchronize")
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
        if hasattr(be, "bucket_pack") and all(g.dtype.name == "f32" for g in grads):
            flat = be.bucket_pack(grads)
        else:
            flat = T.concat([g.reshape((g.shape.size,)) for g in grads], 0)
        if self.comm._nccl is not None and hasattr(be, "nccl_all_reduce"):
            # ncclAvg: sum and the exact power-of-two 1/world scale in the collective itself
            avg = self.comm.world_size & (self.comm.world_size - 1) == 0
            return be.nccl_all_reduce(self.comm._nccl, flat, "avg" if avg else "sum", wait=False), avg
        return self.comm.all_reduce(flat, "sum", _checked=True), False

    def _finish(self, b, flight):
        reduced, averaged = flight
        be = registry.get(reduced.backend_id)
        if hasattr(be, "nccl_wait") and self.comm._nccl is not None:
            if b == 0:  # every bucket is queued by now: one watchdog wait covers them all
                be.nccl_sync(self.comm._nccl, self.comm._timeout)
            be.nccl_wait(self.comm._nccl)
        avg = reduced if averaged else reduced / self.comm.world_size
        off = 0
        for i in self.buckets[b]:
            p = self.params[i]
            n = p.shape.size
            p.grad = avg.slice((off,), (off + n,)).reshape(tuple(p.shape))
            off += n
