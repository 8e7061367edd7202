"""The measured unit of work: one optimizer step (semantics of minml/training.py:30-51)."""

import collections
import gc
import json
import struct

import numpy as np

from . import _tensor as T
from . import nn, optim, registry
from .autograd import Variable
from .errors import FormatError

# steps CapturedStep.run keeps queued ahead of the host (losses are collected this many steps late)
_AHEAD = 3


def model_backend(model):
    params = model.params()
    if not params:
        raise ValueError("model has no parameters")
    return params[0].backend_id


class _Phase:
    """NVTX range around a step phase on the GPU backend (pb_nvtx_push/pop; a no-op elsewhere
    and unless an Nsight tool is attached)."""

    __slots__ = ("lib", "name")

    def __init__(self, backend_id, name):
        be = registry.get(backend_id) if backend_id in registry.registered_ids() else None
        self.lib = getattr(be, "_lib", None) if hasattr(be, "nccl_sync") else None
        self.name = name.encode()

    def __enter__(self):
        if self.lib is not None:
            self.lib.pb_nvtx_push(self.name)
        return self

    def __exit__(self, *exc):
        if self.lib is not None:
            self.lib.pb_nvtx_pop()
        return False


def train_step(model, images, labels, optimizer, comm=None, on_loss=None, ddp=None):
    """H2D, zero_grad, forward, cross-entropy, backward, [grad sync], step, loss D2H.

    ``comm`` reproduces the reference's post-backward ``data_parallel_sync``;
    ``ddp`` (a ``distributed.DataParallel``) instead overlaps bucketed
    allreduces with the backward pass.
    """
    backend = model_backend(model)
    with _Phase(backend, "h2d"):
        x = Variable(T.tensor(images, backend=backend))
        y = T.tensor(labels, backend=backend)
    optimizer.zero_grad()
    with _Phase(backend, "forward"):
        out = model(x)
        loss = nn.cross_entropy(out, y)
    if on_loss is not None:
        on_loss(loss)
    with _Phase(backend, "backward+allreduce" if (ddp is not None or comm is not None) else "backward"):
        if ddp is not None:
            ddp.backward(loss)
        else:
            loss.backward()
            if comm is not None:
                from .distributed import data_parallel_sync
                data_parallel_sync(comm, optimizer.params)
    with _Phase(backend, "optimizer"):
        optimizer.step()
    return loss.scalar(), out


def train_epoch(model, batches, optimizer, comm=None):
    model.train()
    lm, am = nn.AverageMeter(), nn.AccuracyMeter()
    for images, labels in batches:
        value, out = train_step(model, images, labels, optimizer, comm)
        lm.update(value, len(labels))
        am.update(out, labels)
    return lm.result(), am.result()


def _modules(m):
    yield m
    for _, c in m._children:
        yield from _modules(c)


class CapturedStep:
    """``train_step`` replayed from one CUDA graph.

    The reference's front end issues ~4.4k primitives per ResNet-50 step from Python; on a
    B200 that host work, not the GPU, would set the step time.  The first ``warmup`` calls
    run eagerly (they settle lazily-created state: dense velocities, rebound BN running
    statistics, grown scratch).  The next call records one whole step -- zero_grad,
    forward, cross-entropy, backward, [bucketed allreduce], SGD -- into a CUDA graph, and
    every later call is: copy the batch into the graph's static input buffers, launch the
    graph, read the loss.  Results are those of ``train_step``: the same kernels run in
    the same order on the same buffers -- except that, with ``fuse`` (the default), the last
    warm-up step is traced and the recorded step runs every elementwise result whose only
    consumer is elementwise inside that consumer's chain kernel (GpuBackend.fusion_*; the
    chain kernel is bit-identical to the unfused primitives).

    State the step rebinds instead of updating in place (e.g. BatchNorm running stats,
    minml/nn.py:299-300) is copied back into its original buffer at the end of the graph,
    so every replay reads the previous replay's state.  Random primitives (dropout) read
    their counter offset from a device counter that each replay advances by the range the
    host reserves for it (GpuBackend ``GraphExec``), so masks match the eager steps'.

    Only ``optim.SGD`` is recorded: its hyper-parameters are kernel scalars, so a change of
    ``lr`` / ``momentum`` / ``weight_decay`` -- or parameters / velocities rebound from
    outside (a checkpoint restore) -- makes the next call record the step again.  Adam keeps
    its step count and bias corrections on the host and rebinds its moments every step, so
    it is refused (``TypeError``) rather than replayed wrong.
    """

    def __init__(self, model, optimizer, ddp=None, warmup=2, fuse=True):
        if type(optimizer) is not optim.SGD:
            raise TypeError(f"CapturedStep records optim.SGD steps only, not {type(optimizer).__name__} "
                            "(use training.train_step)")
        self.model, self.opt, self.ddp = model, optimizer, ddp
        self._sig = None
        self.backend = registry.get(model_backend(model))
        self.warmup = int(warmup)
        # trace-planned elementwise fusion: the last warm-up step is traced, the recorded
        # step fuses every elementwise result whose single consumer is elementwise
        self.fuse = bool(fuse) and self.warmup >= 2 and hasattr(self.backend, "fusion_trace_begin")
        self.fused_ops = 0
        self.plan_abandoned = None
        self.calls = 0
        self.graph = None
        self.x = self.y = None
        self.loss = self.out = None
        self.launches = 0
        self._stage = None

    def _slots(self):
        slots = []
        for i, p in enumerate(self.opt.params):
            slots.append((p, "data", None))
        vel = getattr(self.opt, "velocity", None)
        if vel is not None:
            for i in range(len(vel)):
                slots.append((vel, i, None))
        for m in _modules(self.model):
            for name in m.buffer_names():
                slots.append((m, name, None))
        return slots

    @staticmethod
    def _get(owner, key):
        return owner[key] if isinstance(key, int) else getattr(owner, key)

    @staticmethod
    def _set(owner, key, value):
        if isinstance(key, int):
            owner[key] = value
        else:
            setattr(owner, key, value)

    def _body(self):
        xv = Variable(self.x)
        self.opt.zero_grad()
        out = self.model(xv)
        loss = nn.cross_entropy(out, self.y)
        if self.ddp is not None:
            self.ddp.backward(loss)
        else:
            loss.backward()
        self.opt.step()
        return loss, out

    def __call__(self, images, labels):
        be = self.backend
        labels = np.asarray(labels)
        if self.graph is not None:  # nn.cross_entropy's range check, done on the host copy
            classes = self.out.shape[1]
            if labels.size and (labels.min() < 0 or labels.max() >= classes):
                bad = labels[(labels < 0) | (labels >= classes)][0]
                raise IndexError(f"target {int(bad)} out of range for {classes} classes")
        if self.x is None:
            self.x = T.tensor(images, backend=be.name)
            self.y = T.tensor(labels, backend=be.name)
        else:
            be.copy_in(self.x, images)
            be.copy_in(self.y, labels)
        self.calls += 1
        if self.graph is None and self.calls <= self.warmup:
            trace = self.fuse and self.calls == self.warmup
            if trace:
                be.fusion_trace_begin()
                if hasattr(be, "fill_cache_begin"):
                    be.fill_cache_begin()  # closed after the recording (see _capture)
            try:
                loss, out = self._body()
            finally:
                if trace:
                    self.fused_ops = be.fusion_trace_end()
            return loss.scalar(), out
        if self.graph is not None and self._signature() != self._sig:
            self.graph = None  # hyper-parameters or state buffers changed: record again
        if self.graph is None:
            self._capture()
        self.graph.launch()
        return self.loss.scalar(), self.out

    def _signature(self):
        o = self.opt
        vel = o.velocity or ()
        return (o.lr, o.momentum, o.weight_decay, tuple(p.data.adapter.ptr for p in o.params),
                tuple(v.adapter.ptr for v in vel))

    def run(self, batches):
        """Pipelined steps over an iterable of host ``(images, labels)`` batches; yields each
        step's loss as a float, in order (the reference's ``train_step`` loop with its
        read-ahead ``Prefetch``, minml/data.py:112-145, moved to the device queue).

        Once the graph is recorded, batch i+1's host->device copy runs on the copy stream
        while step i computes, and step i's loss comes back through a posted pinned read
        that the host collects after queueing step i+3, so the compute stream never waits
        for the host.  Every step still copies its whole batch in and its loss out.  Batches
        in page-locked memory (``GpuBackend.pinned``) go over in one DMA; a batch's host
        buffers may be reused once the loss of the step before it has been yielded.
        """
        # Python's cyclic collector is paused while steps run (reference counting still frees
        # everything acyclic): a full collection walks every live object, and the recorded step
        # keeps many alive.  Restored when the generator finishes or is closed.
        paused = gc.isenabled()
        if paused:
            gc.disable()
        try:
            yield from self._run(batches)
        finally:
            if paused:
                gc.enable()

    def _run(self, batches):
        be = self.backend
        # _AHEAD steps stay queued ahead of the host: a host stall shorter than that many steps
        # never idles the device (with one step ahead the pipelined e2e time varied 23.5-33.7 ms/step
        # between identical runs, tools/e2e_diag.py; the graph-only replay stayed at 23.5)
        pending, k = collections.deque(), 0
        for images, labels in batches:
            if self.graph is not None and self._signature() != self._sig:
                while pending:
                    yield float(be.fetch_read(*pending.popleft()).reshape(()))
                self.graph = None
            if self.graph is None:
                yield self(images, labels)[0]
                continue
            labels = np.asarray(labels)
            classes = self.out.shape[1]
            if labels.size and (labels.min() < 0 or labels.max() >= classes):
                bad = labels[(labels < 0) | (labels >= classes)][0]
                raise IndexError(f"target {int(bad)} out of range for {classes} classes")
            if self._stage is None:  # two dense device slots per input, written by the copy stream
                self._stage = [(T.tensor(np.zeros(tuple(self.x.shape), self.x.dtype.np), backend=be.name),
                                T.tensor(np.zeros(tuple(self.y.shape), self.y.dtype.np), backend=be.name))
                               for _ in range(2)]
            sx, sy = self._stage[k % 2]
            be.stage_in(sx, images, stream=2)
            be.stage_in(sy, labels, stream=2)
            be.stream_wait(0, 2)  # compute waits for this batch
            be.copy_device(self.x, sx)
            be.copy_device(self.y, sy)
            be.stream_wait(2, 0)  # the next copy into this slot waits for these reads
            self.calls += 1
            self.graph.launch()
            loss = self.loss.data if isinstance(self.loss, Variable) else self.loss
            meta = be.post_read(loss, k % 8)
            pending.append((k % 8, meta))
            if len(pending) > _AHEAD:
                value = float(be.fetch_read(*pending.popleft()).reshape(()))
                # an earlier step is done and this batch's copy is queued behind the inputs of the
                # steps before it: wait for it to land, then the caller may reuse its host buffers
                be.stream_sync(2)
                yield value
            k += 1
        while pending:
            yield float(be.fetch_read(*pending.popleft()).reshape(()))

    def _capture(self):
        be = self.backend
        slots = [(o, k, self._get(o, k)) for o, k, _ in self._slots()]
        n0 = be.launch_count()
        planned = self.fuse and be.fusion_plan_begin()
        be.capture_begin()
        try:
            try:
                loss, out = self._body()
            finally:
                if planned:
                    be.fusion_plan_end()
                    self.plan_abandoned = be.plan_abandoned
        except BaseException:
            try:
                be.capture_end()  # discard the partial recording
            except Exception:  # noqa: BLE001
                pass
            be.synchronize()
            raise
        try:
            for owner, key, before in slots:
                now = self._get(owner, key)
                if now is before:
                    continue
                b = before.data if isinstance(before, Variable) else before
                n = now.data if isinstance(now, Variable) else now
                if b is n or b.adapter.ptr == n.adapter.ptr:
                    continue
                be.copy_device(b, n)
                if isinstance(owner, Variable) or key == "data":
                    owner.data = b
                else:
                    self._set(owner, key, before)
        finally:
            self.graph = be.capture_end()
            if hasattr(be, "fill_cache_end"):
                self._fills = be.fill_cache_end()  # blocks the graph reads: kept with it
        self.launches = be.launch_count() - n0  # kernels recorded into the graph (per replay)
        self.loss, self.out = loss, out
        self._sig = self._signature()


# ---------------------------------------------------------------------- checkpoints
# The reference's checkpoint container (minml/training.py:119-214): "MNCK", u32 version, a
# JSON header (epoch, the backend's RNG counter state, optimizer recipe, extra), the
# serialized model (nn.serialize), then the optimizer's state arrays.  Device tensors are
# read through to_host, so a checkpoint written on the GPU loads bit-exactly into the CPU
# reference and vice versa.  Restore order: model first (constructors draw from the RNG),
# then restore_rng, so a resumed run consumes the counter sequence of the uninterrupted one.

CHECKPOINT_MAGIC = b"MNCK"
CHECKPOINT_VERSION = 1
_OPTIMIZER_KINDS = {
    "sgd": (optim.SGD, ("lr", "momentum", "weight_decay")),
    "adam": (optim.Adam, ("lr", "beta1", "beta2", "eps", "weight_decay")),
}


def _optimizer_kind(optimizer):
    for kind, (cls, _) in _OPTIMIZER_KINDS.items():
        if type(optimizer) is cls:
            return kind
    raise FormatError(f"cannot checkpoint optimizer type {type(optimizer).__name__}")


class Checkpoint:
    """What load_checkpoint returns; restore_optimizer / restore_rng rebuild the rest."""

    def __init__(self, model, epoch, rng_state, optimizer_recipe, optimizer_arrays, extra):
        self.model, self.epoch, self.rng_state = model, epoch, rng_state
        self.optimizer_recipe, self.optimizer_arrays, self.extra = optimizer_recipe, optimizer_arrays, extra

    def restore_optimizer(self, params=None):
        if self.optimizer_recipe is None:
            raise FormatError("checkpoint was saved without optimizer state")
        cls, _ = _OPTIMIZER_KINDS[self.optimizer_recipe["kind"]]
        opt = cls(self.model.params() if params is None else params, **self.optimizer_recipe["hyper"])
        opt.load_state_config(self.optimizer_recipe["config"])
        opt.load_state_entries(dict(self.optimizer_arrays))
        return opt

    def restore_rng(self, backend=None):
        be = registry.default() if backend is None else registry.get(backend)
        be.rng.restore(self.rng_state)


def save_checkpoint(path, model, optimizer=None, epoch=0, extra=None):
    be = registry.get(model_backend(model))
    header = {"epoch": int(epoch), "rng": be.rng.state(), "extra": extra or {}}
    if optimizer is not None:
        kind = _optimizer_kind(optimizer)
        header["optimizer"] = {"kind": kind,
                               "hyper": {f: getattr(optimizer, f) for f in _OPTIMIZER_KINDS[kind][1]},
                               "config": optimizer.state_config()}
    buf = bytearray(CHECKPOINT_MAGIC)
    buf += struct.pack("<I", CHECKPOINT_VERSION)
    nn._w_str(buf, json.dumps(header, sort_keys=True))
    blob = nn.serialize(model)
    buf += struct.pack("<Q", len(blob)) + blob
    entries = optimizer.state_entries() if optimizer is not None else []
    buf += struct.pack("<I", len(entries))
    for name, array in entries:
        nn._w_array(buf, name, array)
    with open(path, "wb") as f:
        f.write(bytes(buf))


def load_checkpoint(path, backend=None):
    with open(path, "rb") as f:
        raw = f.read()
    r = nn._Reader(raw)
    if bytes(r.take(4)) != CHECKPOINT_MAGIC:
        raise FormatError("not a checkpoint (bad magic)", offset=0)
    version = r.u32()
    if version != CHECKPOINT_VERSION:
        raise FormatError(f"unsupported checkpoint version {version}", offset=4)
    header = json.loads(r.string())
    model = nn.deserialize(bytes(r.take(r.u64())), backend=backend)
    arrays = [r.array() for _ in range(r.u32())]
    if r.pos != len(raw):
        raise FormatError(f"{len(raw) - r.pos} trailing bytes", offset=r.pos)
    return Checkpoint(model, header["epoch"], header["rng"], header.get("optimizer"), arrays,
                      header.get("extra", {}))
