"""GpuBackend: the B200 implementation of the reference's Backend contract.

``execute(call, args)`` (minml/registry.py:137-138) runs each of the 41 primitives as a
CUDA kernel from libpaper_b200.so on the backend's compute stream, with one allocation
per op from the stream-ordered caching allocator (the template of minml/eager.py:33-53).

Adapters are ``DeviceArray`` views (pointer, shape, element strides) over refcounted
``DevBlock`` allocations.  Because tensors are immutable, movement primitives are free:
``reshape`` of a contiguous tensor, ``transpose`` and ``slice`` return views, and
``full`` is a single element with all-zero strides (the sum-backward ``ones`` spreads
of minml/autograd.py:615-617 cost no HBM traffic).  Consumers read views through
strides; only contiguous-only kernels (conv, full reductions, transfers) materialise.

Nothing here falls back to the host: if the extension or a device is missing, the
backend cannot be constructed.
"""

import ctypes
import os
import sys
import struct
import threading
import weakref

import numpy as np

from .. import dtypes
from ..errors import CollectiveTimeout, DeviceError, DomainError, DTypeError, OutOfMemory
from ..memory import CachingManager, MemoryManager, op_tag
from ..registry import Backend
from ..shape import normalize_axis
from . import _lib

_pack = _lib.pack_tensor
_CONTIG = {}


def contig_strides(shape):
    s = _CONTIG.get(shape)
    if s is None:
        acc, out = 1, []
        for d in reversed(shape):
            out.append(acc)
            acc *= d
        s = _CONTIG[shape] = tuple(reversed(out))
    return s


def device_available():
    lib = _lib.load()
    return lib.pb_device_count() > 0


class DevBlock:
    """One allocation; returned to the allocator (stream-ordered) when the last view dies."""

    __slots__ = ("mm", "id", "ptr", "ledger", "__weakref__")

    def __init__(self, mm, bid, ptr, ledger=None):
        self.mm = mm
        self.id = bid
        self.ptr = ptr
        self.ledger = ledger

    def __del__(self):
        lib = _lib._lib
        if lib is not None:
            lib.pb_mm_free(self.mm, self.id)
            if self.ledger is not None:
                mgr, blk = self.ledger
                try:
                    mgr.free(blk)
                except Exception:
                    pass


class DeviceArray:
    """Adapter: a strided view (element strides) into a DevBlock."""

    __slots__ = ("block", "ptr", "shape", "strides", "dtype", "host", "fill", "__weakref__")

    def __init__(self, block, ptr, shape, strides, dtype, host=None, fill=None):
        self.block = block
        self.ptr = ptr
        self.shape = shape
        self.strides = strides
        self.dtype = dtype
        self.host = host
        self.fill = fill  # the value of a full() view (every element), else None

    def packed(self):
        return _pack(self.ptr, self.dtype.code, self.shape, self.strides)

    @property
    def contiguous(self):
        if self.strides == contig_strides(self.shape):
            return True
        exp = 1
        for d, s in zip(reversed(self.shape), reversed(self.strides)):
            if d != 1 and s != exp:
                return False
            exp *= d
        return True


class LazyArray:
    """Adapter of a deferred f32/bool elementwise result (backend-internal fusion).

    Holds a linear chain  v = head; v = op_k(v, x_k)  over DeviceArray leaves
    (csrc/elementwise.cu ``pb_ew_chain``).  The chain runs -- once, into a fresh dense
    buffer -- the first time anything needs memory: a non-elementwise primitive, a view,
    ``to_host``, the optimizer, a collective, or ``Tensor.force()``.  Until then further
    elementwise primitives extend the chain instead of launching, which is the deferred
    backend's single-consumer fusion rule (minml/deferred.py:146-163) done on the device.
    """

    __slots__ = ("be", "shape", "strides", "dtype", "host", "leaves", "head", "steps", "uses", "_dev",
                 "taps", "tap_ok", "__weakref__")

    def __init__(self, be, shape, dtype, leaves, head, steps, taps=()):
        self.be = be
        self.shape = shape
        self.strides = contig_strides(shape)
        self.dtype = dtype
        self.host = None
        self.leaves = leaves  # tuple of DeviceArray
        self.head = head      # ("leaf", 0) or ("scalar", value)
        self.steps = steps    # tuple of (op, kind, side, leaf, to_bool, scalar)
        self.uses = 0
        self._dev = None
        # taps: ((steps applied, LazyArray), ...) -- multi-use intermediates of this chain that
        # its kernel also stores (pb_ew_chain_taps); tap_ok: this result is such an
        # intermediate (the plan saw several consumers, the first one elementwise)
        self.taps = taps
        self.tap_ok = False

    def dev(self):
        d = self._dev
        if d is None:
            d = self._dev = self.be._run_chain(self)
            self.leaves = self.steps = None
            self.taps = ()
        return d

    def materialize(self):
        self.dev()

    @property
    def block(self):
        return self.dev().block

    @property
    def ptr(self):
        return self.dev().ptr

    @property
    def contiguous(self):
        return True

    def packed(self):
        return self.dev().packed()


# elementwise primitives the backend may defer into a chain (pb_ew_chain)
_FUSE_BIN = {"add", "sub", "mul", "div", "pow", "minimum", "maximum", "eq", "lt", "gt", "logical_and", "logical_or"}
_FUSE_UN = {"neg", "abs", "exp", "log", "sqrt", "sin", "cos", "tanh", "logical_not", "astype"}
_MAX_LEAVES, _MAX_STEPS = 8, 16
# consumers that may extend (recompute) one pending chain: 2 -- a tapped intermediate's second
# elementwise consumer recomputes it inline instead of waiting for a pass of its own (ResNet-50
# 23.47 -> 23.17 ms device, 23.51 -> 23.20 ms e2e; profiles/r2/experiments/fuse_uses_sweep.txt)
_MAX_USES = int(os.environ.get("PB_FUSE_USES", "2"))
_MAX_TAPS = 4
_TAPS = os.environ.get("PB_FUSE_TAPS", "1") != "0"  # experiment hook: 0 materialises multi-use chains alone


_LOGICAL = ("logical_and", "logical_or")
_CT = {}


def compute_dtype(name, da, other, scalar):
    """numpy's result type for the op (NEP 50 weak scalars); true division of ints -> f64."""
    key = (name, da, type(other) if scalar else other)
    ct = _CT.get(key)
    if ct is None:
        if name in _LOGICAL:
            ct = dtypes.bool_
        else:
            rt = np.result_type(da.np, other) if scalar else np.result_type(da.np, other.np)
            ct = dtypes.from_numpy(rt)
            if name == "div" and not ct.is_float:
                ct = dtypes.f64
        _CT[key] = ct
    return ct


_INT_RANGE = {"u8": (0, 255), "i32": (-2**31, 2**31 - 1), "i64": (-2**63, 2**63 - 1)}


class LazyReduce:
    """Adapter of a deferred f32 reduction chain (backend-internal fusion).

    ``src`` is the stage-1 input -- a DeviceArray, or a LazyArray whose elementwise chain is
    evaluated inside the reduction -- and ``stages`` the single-axis reductions applied to it in
    order, each ``(call, source axis, epilogue)`` with the epilogue an f32 scalar
    ``(op, scalar, scalar_left)`` or None: the reference's ``mean`` (sum / n, minml/ops.py:33-36)
    and BatchNorm / _unbroadcast stacks of them (minml/nn.py:288-306, minml/autograd.py:290-297).
    The traced plan keeps a reduction lazy only while its single consumer extends the chain; the
    chain then runs as one ``pb_reduce_chain`` (or ``pb_reduce_epi``) launch.  ``cur`` maps the
    axes of the current result to source axes (keepdims leaves a reduced axis in place)."""

    __slots__ = ("be", "src", "stages", "cur", "shape", "strides", "dtype", "host", "_dev", "__weakref__")

    def __init__(self, be, src, stages, cur, shape, dtype):
        self.be, self.src, self.stages, self.cur = be, src, stages, cur
        self.shape = shape
        self.strides = contig_strides(shape)
        self.dtype = dtype
        self.host = None
        self._dev = None

    @classmethod
    def first(cls, be, call, src):
        axis = call.params.get("axis")
        ax = normalize_axis(axis, len(src.shape))
        keep = bool(call.params.get("keepdims", False))
        cur = tuple(range(len(src.shape)))
        if not keep:
            cur = cur[:ax] + cur[ax + 1:]
        return cls(be, src, ((call, ax, None),), cur, tuple(call.shape), call.dtype)

    def extend(self, call):
        """This chain followed by the f32 sum ``call`` (None when it cannot be expressed)."""
        if self._dev is not None or call.name != "sum" or call.params.get("axis") is None:
            return None
        ax = normalize_axis(call.params["axis"], len(self.shape))
        sax = self.cur[ax]
        if len(self.stages) >= 3 or any(st[1] == sax for st in self.stages):
            return None
        cur = self.cur if call.params.get("keepdims", False) else self.cur[:ax] + self.cur[ax + 1:]
        return LazyReduce(self.be, self.src, self.stages + ((call, sax, None),), cur, tuple(call.shape),
                          call.dtype)

    def with_epi(self, epi):
        c, ax, _ = self.stages[-1]
        return LazyReduce(self.be, self.src, self.stages[:-1] + ((c, ax, epi),), self.cur, self.shape, self.dtype)

    def dev(self):
        d = self._dev
        if d is None:
            d = self._dev = self.be._run_red_chain(self)
            self.src = None
        return d

    def materialize(self):
        self.dev()

    @property
    def block(self):
        return self.dev().block

    @property
    def ptr(self):
        return self.dev().ptr

    @property
    def contiguous(self):
        return True

    def packed(self):
        return self.dev().packed()


class LazyWindow:
    """Adapter of a deferred pad / zero-stuffing / strided slice of a device array (backend-
    internal fusion, round 2): element i of axis d is src[j / div] for j = i*mul - off when
    j >= 0, j % div == 0 and j / div < src.shape[d], else ``fill``.  The reference's slice
    backward scatters with zero-stuffing pads (minml/autograd.py:667-693) and its maxpool reads
    strided windows of a -inf-padded input; chain kernels read such a leaf through the map
    (``pb_ew_chain_win``) instead of materialising the padded tensor.  Any other use
    materialises it once, with the same values the eager pad would write."""

    __slots__ = ("be", "src", "shape", "strides", "dtype", "host", "win", "fill", "_dev", "__weakref__")

    def __init__(self, be, src, shape, win, fill):
        self.be, self.src, self.win, self.fill = be, src, tuple(win), float(fill)
        self.shape = tuple(shape)
        self.strides = contig_strides(self.shape)
        self.dtype = src.dtype
        self.host = None
        self._dev = None

    def dev(self):
        d = self._dev
        if d is None:
            d = self._dev = self.be._run_window(self)
        return d

    def materialize(self):
        self.dev()

    @property
    def block(self):
        return self.dev().block

    @property
    def ptr(self):
        return self.dev().ptr

    @property
    def contiguous(self):
        return True

    def packed(self):
        return self.dev().packed()

    def window_bytes(self):
        r = len(self.shape)
        mul = [w[0] for w in self.win] + [1] * (4 - r)
        off = [w[1] for w in self.win] + [0] * (4 - r)
        div = [w[2] for w in self.win] + [1] * (4 - r)
        return _lib.WINDOW.pack(1, 0, self.fill, *mul, *off, *div)


_LAZY = (LazyArray, LazyReduce, LazyWindow)
_CHAINABLE = (LazyArray, LazyWindow)
_NO_WINDOW = _lib.WINDOW.pack(0, 0, 0.0, *([0] * 12)) if hasattr(_lib, "WINDOW") else b""


_EPI = {"add", "sub", "mul", "div"}
_WINDOW_OPS = {"pad", "reshape", "slice"}


class GraphExec:
    """An instantiated CUDA graph of compute-stream work (see GpuBackend.capture_begin).

    Random fills recorded into the graph (dropout masks) read their counter offset from a
    device-resident counter (``pb_rand_dev``) that the graph's last kernel advances by the
    counters one replay consumes.  Every replay after the first reserves that many counters
    from the backend's host ``RngState`` -- the reservation the eager step would have made
    (minml/_tensor.py:362-368) -- so the stream of masks, and the host counter, are those of
    the same number of eager steps.  If anything else reserved counters in between, the
    device counter is rewritten (stream-ordered) before the launch."""

    __slots__ = ("backend", "handle", "rng_counter", "rng_per_step", "rng_seed", "rng_next", "__weakref__")

    def __init__(self, backend, handle, rng=None):
        self.backend = backend
        self.handle = handle
        self.rng_counter = None
        self.rng_per_step = 0
        if rng is not None:
            self.rng_counter, self.rng_per_step, self.rng_seed, self.rng_next = rng

    def launch(self):
        if self.rng_per_step:
            be = self.backend
            if be.rng.seed != self.rng_seed:
                raise DeviceError("the backend was reseeded after this graph recorded random fills; record it again")
            if self.rng_next is None:  # first replay: the recording step reserved its counters
                self.rng_next = be.rng.state()["next"]
            else:
                off = be.rng.reserve(self.rng_per_step)
                if off != self.rng_next:
                    v = np.array([off], dtype=np.uint64)
                    _lib.check(be._lib.pb_h2d(self.rng_counter.ptr, v.ctypes.data, 8), "rng counter")
                self.rng_next = off + self.rng_per_step
        _lib.check(self.backend._lib.pb_graph_launch(self.handle), "graph launch")

    def __del__(self):
        lib = _lib._lib
        if lib is not None and self.handle:
            lib.pb_graph_destroy(self.handle)
            self.handle = 0


class GpuBackend(Backend):
    _next_pool = 0

    def __init__(self, name="gpu", seed=0, device=0, fuse=None):
        self._capture_pool = 0
        self._cap_rng = None
        self._lock = threading.RLock()
        # backend-internal elementwise fusion, opt-in (PB_FUSE=1 or fuse=True):
        # bit-identical (tests/test_gpu_fusion.py) but the interpreted chain kernel is still
        # ALU-bound -- ResNet-50 measured 576 samples/s fused vs 634 unfused
        self._fuse = (os.environ.get("PB_FUSE", "0") == "1") if fuse is None else bool(fuse)
        # trace-planned fusion (fusion_trace_* / fusion_plan_*): a traced step tells which
        # elementwise results have exactly one consumer, itself elementwise; the planned
        # (captured) step keeps only those lazy, so no chain is ever computed twice
        self._fills = None  # open fill cache: (dtype, type, value) -> one-element DevBlock
        self._trace = None
        self._plan = None
        self._planned = False
        self._prod = {}
        self._op_idx = 0
        self._lazy_ok = True
        self._lazy_red = False
        self._lazy_epi = False
        self._lazy_tap = False
        self._lib = _lib.load()
        _lib.check(self._lib.pb_init(device), "pb_init")
        self.device = device
        super().__init__(name, seed)
        self._blk = _lib.MMBlock()
        self._blk_ref = ctypes.byref(self._blk)
        self._flag = ctypes.c_int32(0)
        self._ops = {
            "full": self._full, "arange": self._arange, "rand_uniform": self._rand, "rand_normal": self._rand,
            "from_host": self._from_host, "to_host": self._to_host, "matmul": self._matmul,
            "conv2d": self._conv2d, "conv2d_grad_input": self._conv_gi, "conv2d_grad_weight": self._conv_gw,
            "reshape": self._reshape, "transpose": self._transpose, "concat": self._concat, "slice": self._slice,
            "pad": self._pad, "sum": self._reduce, "max_reduce": self._reduce, "min_reduce": self._reduce,
            "argmax": self._reduce, "astype": self._unary,
        }
        for n in _lib.BINOP:
            self._ops[n] = self._binary
        for n in _lib.UNOP:
            self._ops[n] = self._unary

    # ------------------------------------------------------------------ memory
    def _default_manager(self):
        return CachingManager()

    def _bind_manager(self):
        m = self._manager
        if isinstance(m, MemoryManager) and not m.simulate:
            return m.handle, None
        # a foreign (e.g. reference-side) manager keeps the ledger; device memory comes
        # from a private caching allocator so its alloc/free/stats stay exact
        if not hasattr(self, "_private"):
            self._private = CachingManager()
        return self._private.handle, m

    @property
    def manager(self):
        return self._manager

    def attach_manager(self, manager):
        super().attach_manager(manager)
        self._mm = self._bind_manager()

    def detach_manager(self):
        old = super().detach_manager()
        self._mm = self._bind_manager()
        return old

    def _alloc(self, nbytes, opname):
        with self._lock:
            return self._alloc_locked(nbytes, opname)

    def _alloc_locked(self, nbytes, opname):
        try:
            h, ledger = self._mm
        except AttributeError:
            self._mm = self._bind_manager()
            h, ledger = self._mm
        rc = self._lib.pb_mm_alloc(h, nbytes, op_tag(opname), self._blk_ref)
        if rc:
            _lib.check(rc, f"alloc {nbytes} B for {opname}")
        b = self._blk
        led = None
        if ledger is not None:
            led = (ledger, ledger.alloc(nbytes, op=opname))
        return DevBlock(h, b.id, b.ptr, led)

    def _new(self, shape, dt, opname):
        n = 1
        for d in shape:
            n *= d
        nbytes = n * dt.itemsize
        if nbytes == 0:
            return DeviceArray(None, 0, shape, contig_strides(shape), dt)
        blk = self._alloc(nbytes, opname)
        return DeviceArray(blk, blk.ptr, shape, contig_strides(shape), dt)

    def _contig(self, a, opname="materialize"):
        if type(a) in _LAZY:
            return a.dev()
        if a.contiguous:
            return a
        out = self._new(a.shape, a.dtype, opname)
        if out.block is not None:
            _lib.check(self._lib.pb_copy(a.packed(), out.packed()), "materialize")
        return out

    # ----------------------------------------------------------------- execute
    def execute(self, call, args):
        # concurrency ("execute may be called concurrently"): one re-entrant lock
        # serialises the host side of each primitive -- the shared allocation result block,
        # the device flag of the domain checks, the fill cache -- while launches stay
        # asynchronous on the one compute stream, whose order makes any handle a thread
        # receives safe to consume.  Tracing / recording a CUDA graph is single-threaded.
        with self._lock:
            if self._trace is not None or self._planned:
                return self._execute_traced(call, args)
            return self._execute(call, args)

    def _execute(self, call, args):
        name = call.name
        if name == "sum":
            pass  # _reduce extends or runs lazy sources itself
        elif name == "slice":  # windows and chains compose with a slice (pushed into the leaves)
            args = [a.dev() if type(a) is LazyReduce else a for a in args]
        elif name in _WINDOW_OPS:  # a LazyWindow source composes; other lazies run first
            args = [a.dev() if type(a) is LazyArray or type(a) is LazyReduce else a for a in args]
        elif name not in _FUSE_BIN and name not in _FUSE_UN:
            args = [a.dev() if type(a) in _LAZY else a for a in args]
        elif type(args[0]) is LazyReduce and not (name in _EPI and "scalar" in call.params):
            args = [a.dev() if type(a) is LazyReduce else a for a in args]
        elif len(args) > 1 and type(args[1]) is LazyReduce:
            args = [a.dev() if type(a) is LazyReduce else a for a in args]
        ledger = self._manager if not isinstance(self._manager, MemoryManager) else None
        if ledger is not None:
            ledger.on_op_begin(call.name)
            try:
                return self._ops[call.name](call, args)
            finally:
                ledger.on_op_end(call.name)
        return self._ops[call.name](call, args)

    # ------------------------------------------------------- planned fusion
    def _producer(self, a):
        e = self._prod.get(id(a))
        return e[0] if e is not None and e[1]() is a else -1

    def _execute_traced(self, call, args):
        idx = self._op_idx
        self._op_idx += 1
        name = call.name
        fusible = name in _FUSE_BIN or name in _FUSE_UN
        sig = (name, tuple(call.shape), call.dtype.name, tuple(tuple(a.shape) for a in args))
        prods = tuple(self._producer(a) for a in args)
        if self._trace is not None:
            fusible = fusible or name == "slice"  # a slice of a lazy chain is pushed into its leaves
            epi = name in _EPI and "scalar" in call.params and call.dtype is dtypes.f32
            red_ax = name == "sum" and call.dtype is dtypes.f32 and call.params.get("axis") is not None
            self._trace.append((sig, prods, fusible, epi, red_ax))
        else:
            tr, lazy, lazy_red, lazy_epi, tap = self._plan
            if idx < len(tr) and tr[idx][0] == sig and tr[idx][1] == prods:
                self._lazy_ok = lazy[idx]
                self._lazy_red = lazy_red[idx]
                self._lazy_epi = lazy_epi[idx]
                self._lazy_tap = tap[idx]
            else:  # the step diverged from the trace: stop fusing (everything materialises)
                self._abandon_plan()
        res = self._execute(call, args)
        if type(res) is DeviceArray or type(res) in _LAZY:
            self._prod[id(res)] = (idx, weakref.ref(res))
        return res

    def fill_cache_begin(self):
        """Share full() blocks by value until fill_cache_end(); the caller keeps the returned
        blocks alive for as long as anything recorded with them (a CUDA graph) may run."""
        self._fills = {}

    def fill_cache_end(self):
        fills, self._fills = self._fills, None
        return fills

    def fusion_trace_begin(self):
        """Record the op stream of one (eager) step: signatures and producer links."""
        self._trace, self._prod, self._op_idx = [], {}, 0

    def fusion_trace_end(self):
        """Build the plan from the traced step's single-consumer links:

        * an elementwise f32/bool result stays lazy iff it was consumed exactly once, by an
          elementwise op, or by an f32 sum that opens a multi-stage reduction chain (the chain is
          then evaluated inside the reduction);
        * an f32 sum/max/min stays lazy iff its one consumer is a scalar add/sub/mul/div (mean =
          sum / n) or -- for a sum -- another f32 sum over an axis;
        * such a scalar op on a lazy sum stays lazy iff its one consumer is an f32 sum.
        Returns the number of lazy results."""
        tr, self._trace, self._prod = self._trace, None, {}
        n = len(tr)
        uses, by_fusible, cons = [0] * n, [True] * n, [-1] * n
        for j, (sig, prods, fusible, epi, red_ax) in enumerate(tr):
            for q in prods:
                if q >= 0:
                    uses[q] += 1
                    by_fusible[q] = by_fusible[q] and fusible
                    cons[q] = j
        one = [uses[i] == 1 for i in range(n)]
        is_epi = [t[3] for t in tr]
        is_sum = [t[4] for t in tr]
        lazy_red = [tr[i][0][0] in ("sum", "max_reduce", "min_reduce") and tr[i][0][2] == "f32" and one[i] and
                    (is_epi[cons[i]] or (is_sum[i] and is_sum[cons[i]])) for i in range(n)]
        lazy_epi = [is_epi[i] and one[i] and is_sum[cons[i]] and tr[i][1][0] >= 0 and lazy_red[tr[i][1][0]] and
                    is_sum[tr[i][1][0]] for i in range(n)]

        def opens_chain(c):  # sum c is the first stage of a chain of >= 2 reductions
            if not (is_sum[c] and lazy_red[c]):
                return False
            d = cons[c]
            return is_sum[d] or (lazy_epi[d] and is_sum[cons[d]])

        lazy = [tr[i][2] and one[i] and (by_fusible[i] or opens_chain(cons[i])) for i in range(n)]
        # taps: an f32 elementwise result with several consumers, the first of them an
        # elementwise op of the same shape, stays pending; that consumer's chain kernel stores it
        first = [-1] * n
        for j in range(n - 1, -1, -1):
            for q in tr[j][1]:
                if q >= 0:
                    first[q] = j
        def chain_end(j):  # where the consumer's chain is run: past its planned-lazy links
            while lazy[j] and cons[j] >= 0:
                j = cons[j]
            return j

        def runs_as_chain(j):  # a materialised elementwise result (not a reduction's source)
            return tr[j][2] and tr[j][0][0] != "slice"

        tap = [_TAPS and tr[i][2] and not lazy[i] and uses[i] >= 2 and tr[i][0][2] == "f32" and
               tr[i][0][0] != "slice" and first[i] >= 0 and runs_as_chain(first[i]) and
               tr[first[i]][0][1] == tr[i][0][1] and runs_as_chain(chain_end(first[i])) and
               tr[chain_end(first[i])][0][1] == tr[i][0][1] for i in range(n)]
        self._plan = (tr, lazy, lazy_red, lazy_epi, tap)
        return sum(lazy) + sum(lazy_red) + sum(lazy_epi) + sum(tap)

    def fusion_plan_begin(self):
        """Replay the planned step (normally while recording a CUDA graph): ops the plan marks
        stay lazy and fold into their single consumer's chain kernel."""
        if self._plan is None:
            return False
        self._planned, self._prod, self._op_idx = True, {}, 0
        self._fuse_saved, self._fuse = self._fuse, True
        return True

    def _abandon_plan(self):
        self._lazy_ok = False
        self._lazy_red = False
        self._lazy_epi = False
        self._lazy_tap = False
        self._plan = ([], [], [], [], [])

    @property
    def plan_abandoned(self):
        """True when the planned step diverged from its trace (fusion stopped part-way)."""
        return self._plan is not None and not self._plan[0]

    def fusion_plan_end(self):
        if self._planned:
            self._planned, self._prod = False, {}
            self._fuse = self._fuse_saved
        self._lazy_ok = True
        self._lazy_red = False
        self._lazy_epi = False
        self._lazy_tap = False

    def synchronize(self):
        _lib.check(self._lib.pb_synchronize(), "synchronize")

    # ------------------------------------------------------------- CUDA graphs
    def capture_begin(self):
        """Record the compute stream into a CUDA graph from here on.

        Allocations made while recording come from a private allocator pool that is
        never flushed, so the addresses baked into the graph stay owned by it; eager
        work between replays allocates from the default pool."""
        if self._capture_pool:
            raise DeviceError("a capture is already in progress")
        self.synchronize()
        h, _ = self._bind_or_get()
        # device-resident RNG counter for random fills recorded into this graph (GraphExec)
        base = self.rng.state()["next"]
        blk = self._alloc(8, "rng_counter")
        v = np.array([base], dtype=np.uint64)
        _lib.check(self._lib.pb_h2d(blk.ptr, v.ctypes.data, 8), "rng counter")
        self._cap_rng = [blk, base, self.rng.seed, 0]
        GpuBackend._next_pool += 1
        self._capture_pool = GpuBackend._next_pool
        self._lib.pb_mm_pool(h, self._capture_pool)
        rc = self._lib.pb_graph_begin()
        if rc:
            self._lib.pb_mm_pool(h, 0)
            self._capture_pool = 0
            _lib.check(rc, "graph capture")

    def capture_end(self):
        """Finish the recording; returns a ``GraphExec`` whose ``launch()`` replays it."""
        h, _ = self._bind_or_get()
        ex = ctypes.c_uint64(0)
        blk, base, seed, nrand = self._cap_rng
        rng = None
        try:
            if nrand:
                if self.rng.seed != seed:
                    raise DeviceError("the backend was reseeded while recording a CUDA graph")
                per_step = self.rng.state()["next"] - base
                _lib.check(self._lib.pb_counter_add(blk.ptr, per_step), "rng counter")
                rng = (blk, per_step, seed, None)
        finally:
            try:
                _lib.check(self._lib.pb_graph_end(ctypes.byref(ex)), "graph capture")
            finally:
                self._lib.pb_mm_pool(h, 0)
                self._capture_pool = 0
                self._cap_rng = None
        return GraphExec(self, ex.value, rng)

    @property
    def capturing(self):
        return bool(self._capture_pool)

    def copy_in(self, tensor, host):
        """Overwrite a contiguous device tensor with a same-shaped host array (stream-ordered)."""
        a = tensor.adapter
        host = np.ascontiguousarray(host, dtype=a.dtype.np)
        if tuple(host.shape) != tuple(a.shape) or not a.contiguous or a.block is None:
            raise ValueError("copy_in needs a dense device tensor of the same shape")
        _lib.check(self._lib.pb_h2d(a.ptr, host.ctypes.data, host.nbytes), "copy_in")
        if a.host is not None:
            a.host = host.copy()

    def stage_in(self, tensor, host, stream=2):
        """Like ``copy_in`` but on ``stream`` (2 = the copy stream) through the pinned
        staging ring; order it against the compute stream with ``stream_wait``."""
        a = tensor.adapter
        host = np.ascontiguousarray(host, dtype=a.dtype.np)
        if tuple(host.shape) != tuple(a.shape) or not a.contiguous or a.block is None:
            raise ValueError("stage_in needs a dense device tensor of the same shape")
        _lib.check(self._lib.pb_h2d_on(a.ptr, host.ctypes.data, host.nbytes, int(stream)), "stage_in")

    def pinned(self, shape, dtype=np.float32):
        """A numpy array in page-locked host memory (freed with the array): batches staged
        here reach the device in one DMA, without the host copy into the staging ring."""
        dt = np.dtype(dtype)
        shape = tuple(int(d) for d in shape)
        nbytes = int(np.prod(shape, dtype=np.int64)) * dt.itemsize
        ptr = self._lib.pb_host_alloc(max(nbytes, 1))
        if not ptr:
            raise OutOfMemory(f"pinned host allocation of {nbytes} bytes failed")
        buf = (ctypes.c_char * max(nbytes, 1)).from_address(ptr)
        arr = np.frombuffer(buf, dtype=np.uint8, count=nbytes).view(dt).reshape(shape)
        weakref.finalize(buf, self._lib.pb_host_free, ptr)
        return arr

    def stream_sync(self, stream):
        _lib.check(self._lib.pb_stream_sync(int(stream)), "stream_sync")

    def stream_wait(self, waiter, on):
        """Stream ``waiter`` waits for the work enqueued so far on stream ``on``."""
        _lib.check(self._lib.pb_event_record(int(on), int(waiter)), "stream_wait")

    def post_read(self, tensor, slot):
        """Enqueue an async device->host read of a dense tensor into pinned slot ``slot``."""
        a = self._contig(tensor.adapter)
        _lib.check(self._lib.pb_d2h_post(a.ptr, tensor.shape.size * a.dtype.itemsize, int(slot)), "post_read")
        return (tuple(tensor.shape), a.dtype.np)

    def fetch_read(self, slot, meta):
        """Wait for the read posted in ``slot`` (only that copy) and return it as numpy."""
        shape, dt = meta
        out = np.empty(shape, dtype=dt)
        _lib.check(self._lib.pb_d2h_fetch(int(slot), out.ctypes.data, out.nbytes), "fetch_read")
        return out

    def copy_device(self, dst, src):
        """dst <- src for two dense same-shaped device tensors (stream-ordered, capturable)."""
        da, sa = dst.adapter, self._contig(src.adapter)
        if tuple(da.shape) != tuple(sa.shape) or da.dtype is not sa.dtype or not da.contiguous:
            raise ValueError("copy_device needs dense tensors of one shape and dtype")
        if da.ptr != sa.ptr and da.block is not None:
            _lib.check(self._lib.pb_d2d(da.ptr, sa.ptr, dst.shape.size * da.dtype.itemsize), "copy_device")

    def _bind_or_get(self):
        try:
            return self._mm
        except AttributeError:
            self._mm = self._bind_manager()
            return self._mm

    def launch_count(self):
        """Kernels this library has launched so far (all backends in the process)."""
        return int(self._lib.pb_launch_count())

    def event_timer(self):
        """CUDA-event timer on the compute stream: ``t = be.event_timer(); ...; ms = t()``."""
        h = ctypes.c_uint64(0)
        ms = ctypes.c_float(0)
        _lib.check(self._lib.pb_timer(0, ctypes.byref(h), ctypes.byref(ms)), "timer")

        def stop():
            _lib.check(self._lib.pb_timer(1, ctypes.byref(h), ctypes.byref(ms)), "timer")
            _lib.check(self._lib.pb_timer(2, ctypes.byref(h), ctypes.byref(ms)), "timer")
            self._lib.pb_timer(3, ctypes.byref(h), ctypes.byref(ms))
            return float(ms.value)

        return stop

    # creation / transfer
    def _full(self, call, args):
        shape = tuple(call.shape)
        dt = call.dtype
        v = call.params["value"]
        if type(v) is int and dt.is_integer:  # numpy.copyto rejects out-of-range Python ints
            lo, hi = _INT_RANGE[dt.name]
            if not lo <= v <= hi:
                raise OverflowError(f"Python integer {v} out of bounds for {dt.np}")
        if call.shape.size == 0:
            return DeviceArray(None, 0, shape, contig_strides(shape), dt)
        # the one-element block behind a full() view is immutable, so while a fill cache is
        # open (CapturedStep: traced warm-up + recording) equal fills share it -- the
        # reference's sum backward creates one ones() per reduction (324 per ResNet-50
        # step), each a 1-element kernel in the graph otherwise.  Blocks filled while a graph
        # is being recorded only hold their value once the graph runs, so those are not shared.
        fills = self._fills
        key = (dt.name, type(v), v) if fills is not None and v == v else None  # NaN: not keyed
        blk = fills.get(key) if key is not None else None
        if blk is None:
            blk = self._alloc(dt.itemsize, "full")
            one = DeviceArray(blk, blk.ptr, (1,), (1,), dt)
            _lib.check(self._lib.pb_fill(one.packed(), _lib.pack_scalar(call.params["value"])), "full")
            if key is not None and not self._capture_pool and len(fills) < 4096:
                fills[key] = blk
        return DeviceArray(blk, blk.ptr, shape, (0,) * len(shape), dt, fill=v)

    def _arange(self, call, args):
        out = self._new(tuple(call.shape), call.dtype, "arange")
        if out.block is not None:
            _lib.check(self._lib.pb_arange(out.packed()), "arange")
        return out

    def _rand(self, call, args):
        out = self._new(tuple(call.shape), call.dtype, call.name)
        if out.block is not None:
            p = call.params
            kind = 1 if call.name == "rand_normal" else 0
            seed = p["seed"] & ((1 << 64) - 1)
            if self._capture_pool:
                # recorded: the offset is relative to the graph's device counter (GraphExec),
                # so each replay draws the counters the host reserves for it
                cap = self._cap_rng
                if seed != cap[2] or p["offset"] < cap[1]:
                    raise DeviceError(f"{call.name} with a foreign seed/counter cannot be recorded into a CUDA graph")
                cap[3] += 1
                _lib.check(self._lib.pb_rand_dev(kind, seed, cap[0].ptr, p["offset"] - cap[1], out.packed()),
                           call.name)
            else:
                _lib.check(self._lib.pb_rand(kind, seed, p["offset"], out.packed()), call.name)
        return out

    def _from_host(self, call, args):
        host = np.ascontiguousarray(call.params["array"])
        out = self._new(tuple(call.shape), call.dtype, "from_host")
        if out.block is not None:
            _lib.check(self._lib.pb_h2d(out.ptr, host.ctypes.data, host.nbytes), "from_host")
            # integer operands (labels, token ids) keep a host mirror: cross_entropy's range
            # check (minml/nn.py:373) then reads it without a device round trip
            if host.dtype.kind in "iu" and host.size <= (1 << 20):
                out.host = host.copy()
        return out

    def _to_host(self, call, args):
        a = args[0]
        if a.host is not None:
            return a.host.copy()
        if self._capture_pool:
            raise DeviceError("to_host (a device->host sync) cannot be recorded into a CUDA graph")
        res = np.empty(a.shape, dtype=a.dtype.np)
        if res.size == 0:
            return res
        a = self._contig(a)
        _lib.check(self._lib.pb_d2h(res.ctypes.data, a.ptr, res.nbytes), "to_host")
        return res

    # ------------------------------------------------------------ fusion (f1)
    def _fusible_operand(self, a):
        return a.dtype is dtypes.f32 or a.dtype is dtypes.bool_

    def _as_leaf(self, a):
        """A DeviceArray for a chain leaf (lazy operands that are not extended run now)."""
        return a.dev() if type(a) is LazyArray else a

    def _extendable(self, a, extra_steps=1, extra_leaves=1, shape=None):
        if not (type(a) is LazyArray and a._dev is None and a.uses < _MAX_USES
                and len(a.steps) + extra_steps <= _MAX_STEPS and len(a.leaves) + extra_leaves <= _MAX_LEAVES):
            return False
        if a.tap_ok or a.taps:  # taps are stored at the chain's output index: same shape only
            if shape is None or tuple(shape) != a.shape or len(a.taps) + a.tap_ok > _MAX_TAPS:
                return False
            if any(type(d) is LazyWindow for d in a.leaves):
                return False
        return True

    def _chain_from(self, a, shape=None):
        """(leaves list, head, steps list, taps) to extend: a's chain, or a fresh one rooted at
        leaf a.  Extending a multi-use intermediate (tap_ok) taps it: the extended chain's kernel
        stores a's value after a's steps."""
        if type(a) is LazyArray and self._extendable(a, shape=shape):
            a.uses += 1
            taps = a.taps + (((len(a.steps), a),) if a.tap_ok else ())
            return list(a.leaves), a.head, list(a.steps), taps
        return [self._as_leaf(a)], ("leaf", 0), [], ()

    @staticmethod
    def _leaf_index(leaves, d):
        for i, x in enumerate(leaves):
            if x is d:
                return i
        leaves.append(d)
        return len(leaves) - 1

    @staticmethod
    def _window_fit(call, args):
        """Windowed leaves enter a chain only at the output's exact shape (no broadcasting)."""
        shape = tuple(call.shape)
        return [a.dev() if type(a) is LazyWindow and (a.shape != shape or len(shape) > 4) else a for a in args]

    def _try_fuse_binary(self, call, args):
        name = call.name
        p = call.params
        out_dt = call.dtype
        args = self._window_fit(call, args)
        if not self._fuse or len(call.shape) > 4 or (out_dt is not dtypes.f32 and out_dt is not dtypes.bool_):
            return None
        code = _lib.BINOP[name]
        if "scalar" in p:
            a = args[0]
            sv = p["scalar"]
            if not self._fusible_operand(a) or type(sv) not in (int, float, bool):
                return None
            ct = compute_dtype(name, a.dtype, sv, True)
            if ct is not dtypes.f32:
                return None
            fv = float(sv)
            if fv != fv or abs(fv) == float("inf"):
                pass  # representable as f32 either way
            elif abs(fv) > 3.4e38:
                return None
            leaves, head, steps, taps = self._chain_from(a, call.shape)
            side = 1 if p.get("scalar_side") == "left" else 0
            steps.append((code, 2, side, 0, 0, fv))
        else:
            a, b = args
            if not (self._fusible_operand(a) and self._fusible_operand(b)):
                return None
            ct = compute_dtype(name, a.dtype, b.dtype, False)
            if ct is not dtypes.f32 and not (ct is dtypes.bool_ and name in _LOGICAL):
                return None
            if a is b:
                leaves, head, steps, taps = self._chain_from(a, call.shape)
                steps.append((code, 3, 0, 0, 0, 0.0))
            elif self._extendable(a, shape=call.shape) or not self._extendable(b, shape=call.shape):
                leaves, head, steps, taps = self._chain_from(a, call.shape)
                if len(leaves) >= _MAX_LEAVES:
                    return None
                steps.append((code, 1, 0, self._leaf_index(leaves, self._as_leaf(b)), 0, 0.0))
            else:
                leaves, head, steps, taps = self._chain_from(b, call.shape)
                if len(leaves) >= _MAX_LEAVES:
                    return None
                steps.append((code, 1, 1, self._leaf_index(leaves, self._as_leaf(a)), 0, 0.0))
        return LazyArray(self, tuple(call.shape), out_dt, tuple(leaves), head, tuple(steps), taps)

    def _try_fuse_unary(self, call, args):
        name = call.name
        args = self._window_fit(call, args)
        a = args[0]
        out_dt = call.dtype
        if not self._fuse or len(call.shape) > 4 or not self._fusible_operand(a):
            return None
        if out_dt is not dtypes.f32 and out_dt is not dtypes.bool_:
            return None
        if name == "astype":
            if out_dt is a.dtype:
                return None
            step = (64 + _lib.UNOP["astype"], 0, 0, 0, 1 if out_dt is dtypes.bool_ else 0, 0.0)
        elif name == "logical_not":
            step = (64 + _lib.UNOP[name], 0, 0, 0, 0, 0.0)
        elif a.dtype is dtypes.f32:
            step = (64 + _lib.UNOP[name], 0, 0, 0, 0, 0.0)
        else:
            return None
        leaves, head, steps, taps = self._chain_from(a, call.shape)
        steps.append(step)
        return LazyArray(self, tuple(call.shape), out_dt, tuple(leaves), head, tuple(steps), taps)

    def _lazy_result(self, lz):
        if self._lazy_ok:
            return lz
        if self._lazy_tap and lz.dtype is dtypes.f32:
            lz.tap_ok = True  # stays pending: its first (elementwise) consumer's kernel stores it
            return lz
        return lz.dev()

    def _run_chain(self, lz):
        out = self._new(lz.shape, lz.dtype, "fused")
        if out.block is None:
            return out
        taps = [(k, t) for k, t in lz.taps if t._dev is None]
        if taps:
            if any(type(d) is LazyWindow and d._dev is None for d in lz.leaves):
                for _, t in taps:
                    t.dev()  # (windowed chains have no taps: run the intermediates alone)
            else:
                bufs = [self._new(t.shape, t.dtype, "fused") for _, t in taps]
                steps = b"".join(_lib.STEP.pack(op, kind, side, leaf, tb, 0, sc)
                                 for op, kind, side, leaf, tb, sc in lz.steps)
                hk, hv = (0, 0.0) if lz.head[0] == "leaf" else (1, float(lz.head[1]))
                after = struct.pack(f"<{len(taps)}i", *(k for k, _ in taps))
                rc = self._lib.pb_ew_chain_taps(len(lz.leaves), b"".join(d.packed() for d in lz.leaves), hk, hv,
                                                len(lz.steps), steps, len(taps), after,
                                                b"".join(b.packed() for b in bufs), out.packed())
                if rc != _lib.UNSUPPORTED:
                    _lib.check(rc, "fused elementwise chain (taps)")
                    for (_, t), b in zip(taps, bufs):
                        t._dev = b
                        t.leaves = t.steps = None
                    return out
                for _, t in taps:  # not specialisable (no NVRTC): the intermediates run alone
                    t.dev()
        steps = b"".join(_lib.STEP.pack(op, kind, side, leaf, tb, 0, sc) for op, kind, side, leaf, tb, sc in lz.steps)
        hk, hv = (0, 0.0) if lz.head[0] == "leaf" else (1, float(lz.head[1]))
        if any(type(d) is LazyWindow and d._dev is None for d in lz.leaves):
            leaves = b"".join(d.src.packed() if type(d) is LazyWindow and d._dev is None else d.packed()
                              for d in lz.leaves)
            wins = b"".join(d.window_bytes() if type(d) is LazyWindow and d._dev is None else _NO_WINDOW
                            for d in lz.leaves)
            rc = self._lib.pb_ew_chain_win(len(lz.leaves), leaves, wins, hk, hv, len(lz.steps), steps, out.packed())
            if rc != _lib.UNSUPPORTED:
                _lib.check(rc, "fused windowed chain")
                return out
            # the kernel declined a window (divisor not a power of two, > 32-bit coordinates):
            # materialise the windowed leaves and run the plain chain
        leaves = b"".join(d.packed() for d in lz.leaves)
        _lib.check(self._lib.pb_ew_chain(len(lz.leaves), leaves, hk, hv, len(lz.steps), steps, out.packed()),
                   "fused elementwise chain")
        return out

    # elementwise
    def _binary(self, call, args):
        name = call.name
        p = call.params
        if type(args[0]) is LazyReduce:
            lr = args[0]
            s = p["scalar"]
            if (lr._dev is None and lr.stages[-1][2] is None and type(s) in (int, float) and
                    call.dtype is dtypes.f32 and compute_dtype(name, lr.dtype, s, True) is dtypes.f32 and
                    abs(float(s)) <= 3.4e38):
                # (a later use of the plain reduction -- none per the plan -- would recompute it)
                nl = lr.with_epi((name, float(s), p.get("scalar_side") == "left"))
                return nl if self._lazy_epi else nl.dev()
            args = [lr.dev()]
        if name == "mul" and "scalar" not in p:
            view = self._times_one(call, args)
            if view is not None:
                return view
        if self._fuse and (self._lazy_ok or self._planned or type(args[0]) in _CHAINABLE or
                           (len(args) > 1 and type(args[1]) in _CHAINABLE)):
            lz = self._try_fuse_binary(call, args)
            if lz is not None:
                return self._lazy_result(lz)
        args = [a.dev() if type(a) in _CHAINABLE else a for a in args]
        out = self._new(tuple(call.shape), call.dtype, name)
        if out.block is None:
            return out
        if "scalar" in p:
            s = p["scalar"]
            a = args[0]
            ct = compute_dtype(name, a.dtype, s, True)
            if type(s) is int and ct.kind in "iu":
                lo, hi = _INT_RANGE[ct.name]
                if not lo <= s <= hi:
                    raise OverflowError(f"Python integer {s} out of bounds for {ct.np}")
            left = p.get("scalar_side") == "left"
            if name == "div" and ct.is_float:
                if not left and type(s) is int and a.dtype.is_integer and s == 0:
                    raise DomainError("integer division by zero")
                if left and type(s) is int and a.dtype.is_integer:
                    self._domain_check(0, a, "integer division by zero")
            if name == "pow" and ct.is_integer:
                if (not left and type(s) is int and s < 0) or left:
                    if not left or self._any(1, a):
                        raise DomainError("Integers to negative integer powers are not allowed.")
            pa = a.packed()
            rc = self._lib.pb_binary(_lib.BINOP[name], None if left else pa, pa if left else None,
                                     _lib.pack_scalar(s), ct.code, out.packed())
        else:
            a, b = args
            ct = compute_dtype(name, a.dtype, b.dtype, False)
            if name == "div" and a.dtype.is_integer and b.dtype.is_integer:
                self._domain_check(0, b, "integer division by zero")
            if name == "pow" and ct.is_integer and self._any(1, b):
                raise DomainError("Integers to negative integer powers are not allowed.")
            rc = self._lib.pb_binary(_lib.BINOP[name], a.packed(), b.packed(), None, ct.code, out.packed())
        if rc:
            _lib.check(rc, name)
        return out

    @staticmethod
    def _times_one(call, args):
        """``full(shape, 1) * g`` with g already of the result dtype is g broadcast to the
        result shape, bit for bit (x * 1 == x in IEEE arithmetic; the reference's sum backward
        spreads grads this way, minml/autograd.py:615-617): return a zero-copy view."""
        a, b = args
        for one, g in ((a, b), (b, a)):
            if type(g) is LazyArray and type(one) is DeviceArray and one.fill is not None:
                g = g.dev()  # run the (small) pending chain, then view it: never spread it
            if (type(one) is DeviceArray and one.fill is not None and type(g) is DeviceArray and
                    one.fill == 1 and type(one.fill) is not bool and g.dtype is call.dtype and
                    one.dtype is call.dtype and call.dtype.is_float):
                shape = tuple(call.shape)
                off = len(shape) - len(g.shape)
                strides = [0] * off
                for d, (n, st) in enumerate(zip(g.shape, g.strides)):
                    if n == shape[off + d]:
                        strides.append(st)
                    elif n == 1:
                        strides.append(0)
                    else:
                        return None
                return DeviceArray(g.block, g.ptr, shape, tuple(strides), g.dtype)
        return None

    def _any(self, what, a):
        _lib.check(self._lib.pb_check(what, a.packed(), ctypes.byref(self._flag)), "check")
        return self._flag.value != 0

    def _domain_check(self, what, a, msg):
        if self._any(what, a):
            raise DomainError(msg)

    def _unary(self, call, args):
        if self._fuse and (self._lazy_ok or self._planned or type(args[0]) in _CHAINABLE):
            lz = self._try_fuse_unary(call, args)
            if lz is not None:
                return self._lazy_result(lz)
        args = [a.dev() if type(a) in _CHAINABLE else a for a in args]
        a = args[0]
        out = self._new(tuple(call.shape), call.dtype, call.name)
        if out.block is None:
            return out
        ct = call.dtype if call.name == "astype" else a.dtype
        _lib.check(self._lib.pb_unary(_lib.UNOP[call.name], a.packed(), ct.code, out.packed()), call.name)
        return out

    # reductions
    def _reduce(self, call, args):
        a = args[0]
        if type(a) is LazyWindow:
            a = a.dev()
        if type(a) is LazyReduce:
            nl = a.extend(call) if call.shape.size > 0 else None
            if nl is None:
                return self._run_reduce(call, a.dev())
            return nl if self._lazy_red else nl.dev()
        if type(a) is LazyArray:
            if self._lazy_red and call.name == "sum" and call.shape.size > 0 and a.dtype is dtypes.f32 and \
                    call.params.get("axis") is not None:
                return LazyReduce.first(self, call, a)
            a = a.dev()
        if self._lazy_red and call.shape.size > 0 and a.dtype is dtypes.f32:
            return LazyReduce.first(self, call, a) if call.params.get("axis") is not None else \
                LazyReduce(self, a, ((call, -1, None),), (), tuple(call.shape), call.dtype)
        return self._run_reduce(call, a)

    def _run_red_chain(self, lr):
        """Run a LazyReduce: one pb_reduce_chain launch for 2-3 stages, else (or when the kernel
        declines the layout) the stages one by one exactly as the eager path runs them."""
        src = lr.src
        for attempt in range(2):  # a chain the kernel declines is materialised and offered as a plain source
            if len(lr.stages) < 2 or len(src.shape) > 4:
                break
            out = self._new(lr.shape, dtypes.f32, "sum")
            if out.block is None:
                return out
            if type(src) is LazyArray and src._dev is None and attempt == 0:
                leaves, head, steps = src.leaves, src.head, src.steps
            else:
                leaves, head, steps = (src.dev() if type(src) is LazyArray else src,), ("leaf", 0), ()
            lv = b"".join(d.packed() for d in leaves)
            sp = b"".join(_lib.STEP.pack(op, kind, side, leaf, tb, 0, sc) for op, kind, side, leaf, tb, sc in steps)
            hk, hv = (0, 0.0) if head[0] == "leaf" else (1, float(head[1]))
            stg = b"".join(_lib.RSTAGE.pack(ax, -1, 0, 0.0) if epi is None else
                           _lib.RSTAGE.pack(ax, _lib.BINOP[epi[0]], 1 if epi[2] else 0, epi[1])
                           for _, ax, epi in lr.stages)
            shp = struct.pack(f"<{len(src.shape)}q", *src.shape)
            rc = self._lib.pb_reduce_chain(len(leaves), lv, hk, hv, len(steps), sp, len(src.shape), shp,
                                           len(lr.stages), stg, out.packed())
            if rc == 0:
                return out
            if rc != _lib.UNSUPPORTED:
                _lib.check(rc, "reduce chain")
            if type(src) is not LazyArray or src._dev is not None:
                break
        x = src.dev() if type(src) is LazyArray else src
        for call, _, epi in lr.stages:
            x = self._run_reduce(call, x, epi)
        return x

    def _run_reduce(self, call, a, epi=None):
        """The reduction; with ``epi = (op, scalar, scalar_left)`` its f32 scalar consumer too."""
        out = self._new(tuple(call.shape), call.dtype, call.name)
        if out.block is None:
            return out
        axis = call.params.get("axis")
        if axis is None:
            a = self._contig(a)
            ax = -1
        else:
            ax = normalize_axis(axis, len(a.shape))
        if epi is None:
            _lib.check(self._lib.pb_reduce(_lib.REDOP[call.name], a.packed(), ax, out.packed()), call.name)
        else:
            op, sc, left = epi
            _lib.check(self._lib.pb_reduce_epi(_lib.REDOP[call.name], a.packed(), ax, out.packed(), _lib.BINOP[op],
                                               sc, 1 if left else 0), call.name)
        return out

    # contractions
    def _matmul(self, call, args):
        a, b = args
        out = self._new(tuple(call.shape), call.dtype, "matmul")
        if out.block is None:
            return out
        _lib.check(self._lib.pb_matmul(a.packed(), b.packed(), out.packed()), "matmul")
        return out

    def _conv_params(self, call):
        (sh, sw), (ph, pw) = call.params["stride"], call.params["padding"]
        return _lib.CONV.pack(sh, sw, ph, pw)

    def _conv2d(self, call, args):
        x, w = self._contig(args[0]), self._contig(args[1])
        bias = self._contig(args[2]).packed() if len(args) == 3 else None
        out = self._new(tuple(call.shape), call.dtype, "conv2d")
        if out.block is None:
            return out
        _lib.check(self._lib.pb_conv2d(x.packed(), w.packed(), bias, self._conv_params(call), out.packed()),
                   "conv2d")
        return out

    def _conv_gi(self, call, args):
        g, w = self._contig(args[0]), self._contig(args[1])
        out = self._new(tuple(call.shape), call.dtype, "conv2d_grad_input")
        if out.block is None:
            return out
        _lib.check(self._lib.pb_conv2d_grad_input(g.packed(), w.packed(), self._conv_params(call), out.packed()),
                   "conv2d_grad_input")
        return out

    def _conv_gw(self, call, args):
        x, g = self._contig(args[0]), self._contig(args[1])
        out = self._new(tuple(call.shape), call.dtype, "conv2d_grad_weight")
        if out.block is None:
            return out
        _lib.check(self._lib.pb_conv2d_grad_weight(x.packed(), g.packed(), self._conv_params(call), out.packed()),
                   "conv2d_grad_weight")
        return out

    # movement: views where possible
    def _reshape(self, call, args):
        a = args[0]
        shape = tuple(call.shape)
        if type(a) is LazyWindow:
            lw = self._window_reshape(a, shape)
            if lw is not None:
                return lw
            a = a.dev()
        if not a.contiguous:
            a = self._contig(a, "reshape")
        return DeviceArray(a.block, a.ptr, shape, contig_strides(shape), a.dtype, a.host.reshape(shape)
                           if a.host is not None else None)

    def _transpose(self, call, args):
        a = args[0]
        perm = call.params.get("perm") or tuple(range(len(a.shape) - 1, -1, -1))
        return DeviceArray(a.block, a.ptr, tuple(a.shape[i] for i in perm), tuple(a.strides[i] for i in perm),
                           a.dtype)

    def _slice(self, call, args):
        a = args[0]
        p = call.params
        if type(a) is LazyWindow:  # i = start + i' * step  ->  mul' = mul*step, off' = off - start*mul
            win = tuple((m * st, o - s0 * m, dv) for (m, o, dv), s0, st in zip(a.win, p["starts"], p["steps"]))
            return LazyWindow(self, a.src, tuple(call.shape), win, a.fill)
        if type(a) is LazyArray:
            if self._fuse and a._dev is None and 0 not in tuple(call.shape):
                # elementwise ops commute with slicing: slice every leaf instead of the result
                leaves = tuple(self._slice_leaf(d, a.shape, p["starts"], p["steps"], tuple(call.shape))
                               for d in a.leaves)
                return LazyArray(self, tuple(call.shape), a.dtype, leaves, a.head, a.steps)
            a = a.dev()
        off = 0
        for st, s in zip(p["starts"], a.strides):
            off += st * s
        strides = tuple(s * k for s, k in zip(a.strides, p["steps"]))
        shape = tuple(call.shape)
        if 0 in shape:
            return DeviceArray(None, 0, shape, contig_strides(shape), a.dtype)
        return DeviceArray(a.block, a.ptr + off * a.dtype.itemsize, shape, strides, a.dtype)

    def _concat(self, call, args):
        out = self._new(tuple(call.shape), call.dtype, "concat")
        if out.block is None:
            return out
        ax = normalize_axis(call.params["axis"], len(out.shape))
        off = 0
        for a in args:
            e = a.shape[ax]
            if e:
                dst = DeviceArray(out.block, out.ptr + off * out.strides[ax] * out.dtype.itemsize,
                                  a.shape, out.strides, out.dtype)
                _lib.check(self._lib.pb_copy(a.packed(), dst.packed()), "concat")
            off += e
        return out

    def _pad(self, call, args):
        a = args[0]
        value = call.params.get("value", 0)
        pw = call.params["pad_width"]
        if self._fuse and (type(a) is LazyWindow or (type(a) is DeviceArray and a.block is not None)) and \
                len(a.shape) == len(pw) and (a.dtype is dtypes.f32 or a.dtype is dtypes.bool_) and \
                type(value) in (int, float, bool):
            fill = float(bool(value)) if a.dtype is dtypes.bool_ else float(np.float32(value))
            if fill != 0.0 and type(a) is DeviceArray:
                # a -inf / constant border (the maxpool forward): its 9 strided windows read the
                # materialised pad faster than the per-element window decode (measured)
                return self._pad_now(call, a, value)
            if type(a) is DeviceArray:
                return LazyWindow(self, a, tuple(call.shape), tuple((1, lo, 1) for lo, _ in pw), fill)
            if a.fill == fill or (fill != fill and a.fill != a.fill):  # one fill value (NaN == NaN)
                win = tuple((m, o + lo * m, dv) for (m, o, dv), (lo, _) in zip(a.win, pw))
                return LazyWindow(self, a.src, tuple(call.shape), win, fill)
            a = a.dev()
        elif type(a) is LazyWindow:
            a = a.dev()
        return self._pad_now(call, a, value)

    def _pad_now(self, call, a, value):
        out = self._new(tuple(call.shape), call.dtype, "pad")
        if out.block is None:
            return out
        lo = (ctypes.c_int64 * 8)(*[lo for lo, _ in call.params["pad_width"]])
        _lib.check(self._lib.pb_pad(a.packed(), lo, _lib.pack_scalar(value), out.packed()), "pad")
        return out

    def _slice_leaf(self, d, full, starts, steps, out_shape):
        """Chain leaf d (broadcast to `full`) restricted to the slice that produced `out_shape`."""
        if type(d) is LazyWindow:  # windowed leaves have the chain's full shape
            win = tuple((m * st, o - s0 * m, dv) for (m, o, dv), s0, st in zip(d.win, starts, steps))
            return LazyWindow(self, d.src, out_shape, win, d.fill)
        r, R = len(d.shape), len(full)
        ptr, shape, strides = d.ptr, list(d.shape), list(d.strides)
        for k in range(R):
            kk = k - (R - r)
            if kk < 0 or d.shape[kk] == 1:
                continue  # broadcast axis: unchanged
            ptr += starts[k] * d.strides[kk] * d.dtype.itemsize
            strides[kk] = d.strides[kk] * steps[k]
            shape[kk] = out_shape[k]
        return DeviceArray(d.block, ptr, tuple(shape), tuple(strides), d.dtype)

    def _window_reshape(self, a, shape):
        """The reshapes _slice_grad applies to a windowed tensor: insert one unit axis, or merge an
        axis with a following zero-stuffing axis (source extent 1 at index 0): (a, b) -> a*k + b
        with only b == 0 populated is div' = k*div, off' = k*off.  None: materialise instead."""
        old = a.shape
        src = a.src
        if len(shape) == len(old) + 1:
            for p in range(len(shape)):
                if shape[p] == 1 and shape[:p] + shape[p + 1:] == old:
                    s2 = DeviceArray(src.block, src.ptr, src.shape[:p] + (1,) + src.shape[p:],
                                     src.strides[:p] + (0,) + src.strides[p:], src.dtype)
                    return LazyWindow(self, s2, shape, a.win[:p] + ((1, 0, 1),) + a.win[p:], a.fill)
            return None
        if len(shape) == len(old) - 1:
            for p in range(len(old) - 1):
                k = old[p + 1]
                if old[:p] + (old[p] * k,) + old[p + 2:] != shape:
                    continue
                mb, ob, db = a.win[p + 1]
                ma, oa, da = a.win[p]
                if src.shape[p + 1] == 1 and (mb, ob, db) == (1, 0, 1) and ma == 1:
                    s2 = DeviceArray(src.block, src.ptr, src.shape[:p + 1] + src.shape[p + 2:],
                                     src.strides[:p + 1] + src.strides[p + 2:], src.dtype)
                    win = a.win[:p] + ((1, k * oa, k * da),) + a.win[p + 2:]
                    return LazyWindow(self, s2, shape, win, a.fill)
            return None
        return None

    def _run_window(self, lw):
        """Materialise a LazyWindow with the values the eager pad would have written."""
        out = self._new(lw.shape, lw.dtype, "pad")
        if out.block is None:
            return out
        src = lw.src
        if all(m == 1 and o >= 0 for m, o, _ in lw.win):  # a pad / zero-stuffing: fill, then a strided copy
            _lib.check(self._lib.pb_fill(out.packed(), _lib.pack_scalar(bool(lw.fill) if lw.dtype is dtypes.bool_
                                                                         else lw.fill)), "pad fill")
            off = sum(o * st for (_, o, _), st in zip(lw.win, out.strides))
            dst = DeviceArray(out.block, out.ptr + off * out.dtype.itemsize, src.shape,
                              tuple(dv * st for (_, _, dv), st in zip(lw.win, out.strides)), out.dtype)
            if src.shape and 0 not in src.shape:
                _lib.check(self._lib.pb_copy(src.packed(), dst.packed()), "pad copy")
            return out
        if len(lw.shape) > 4:
            raise DeviceError(f"windowed tensor of rank {len(lw.shape)} cannot be materialised by the chain kernel")
        _lib.check(self._lib.pb_ew_chain_win(1, src.packed(), lw.window_bytes(), 0, 0.0, 0, b"", out.packed()),
                   "windowed materialisation")
        return out

    # -------------------------------------------------------------- collectives
    def _tensor(self, arr, shape):
        from .._tensor import Tensor
        return Tensor(arr, self.name, shape, arr.dtype)

    def bucket_pack(self, grads):
        """Concatenate flattened f32 gradients into one bucket with a single launch."""
        for g in grads:
            if g.dtype.name != "f32":
                raise DTypeError(f"bucket_pack packs f32 gradients only, got {g.dtype.name}")
        n = len(grads)
        srcs = (ctypes.c_uint64 * n)()
        numel = (ctypes.c_int64 * n)()
        keep, total = [], 0
        for i, g in enumerate(grads):
            a = self._contig(g.adapter)
            keep.append(a)
            srcs[i] = a.ptr
            numel[i] = g.shape.size
            total += g.shape.size
        out = self._new((total,), dtypes.f32, "bucket")
        _lib.check(self._lib.pb_bucket_pack(n, srcs, numel, out.ptr), "bucket_pack")
        return self._tensor(out, (total,))

    _NCCL_OPS = {"sum": 0, "max": 1, "avg": 2}

    _aborted = set()  # communicators the watchdog aborted (any later use raises CollectiveTimeout)

    def _live(self, comm):
        if comm in GpuBackend._aborted:
            raise CollectiveTimeout("the NCCL communicator was aborted by the collective watchdog")

    def nccl_sync(self, comm, timeout):
        """Collective watchdog (minml/distributed.py:23, 93-105 CollectiveTimeout): block until
        the comm stream's queued collectives finish, at most ``timeout`` seconds; a hung or
        failed collective aborts the communicator (pb_nccl_sync) and raises CollectiveTimeout /
        DeviceError instead of hanging the process.  A no-op while a graph is being recorded."""
        if self._capture_pool or timeout is None:
            return
        rc = self._lib.pb_nccl_sync(comm, int(max(0.0, float(timeout)) * 1000))
        if rc:
            if comm:
                GpuBackend._aborted.add(comm)
            _lib.check(rc, "collective watchdog")

    def nccl_all_reduce(self, comm, tensor, op="sum", wait=True, timeout=None):
        """ncclAllReduce on the comm stream (after a compute->comm fence).  ``op`` "avg" is
        ncclAvg: for the power-of-two worlds of one node the 1/N scale is exact, so it equals
        the reference's sum-then-divide (minml/distributed.py:216-222) bit for bit.  With
        ``wait=False`` the compute stream is not joined: call ``nccl_wait`` before reading
        the result; the source stays referenced until then, and both blocks are recorded
        on the comm stream so an early free parks them behind a comm-stream event."""
        self._live(comm)
        a = self._contig(tensor.adapter)
        out = self._new(a.shape, a.dtype, "all_reduce")
        _lib.check(self._lib.pb_nccl_allreduce(comm, a.ptr, out.ptr, tensor.shape.size, a.dtype.code,
                                               self._NCCL_OPS[op]), "ncclAllReduce")
        if wait:
            self.nccl_sync(comm, timeout)
            self.nccl_wait(comm)
        else:
            out.host = None
            for blk in (a.block, out.block):
                if blk is not None:
                    _lib.check(self._lib.pb_mm_record_stream(blk.mm, blk.id, 1), "record_stream")
            self._inflight = getattr(self, "_inflight", [])
            self._inflight.append(a)  # source must outlive the collective
        return self._tensor(out, tuple(tensor.shape))

    def nccl_wait(self, comm):
        _lib.check(self._lib.pb_nccl_wait(comm), "nccl wait")
        self._inflight = []

    def nccl_all_gather(self, comm, tensor, world, timeout=None):
        self._live(comm)
        a = self._contig(tensor.adapter)
        out = self._new((world,) + a.shape, a.dtype, "all_gather")
        _lib.check(self._lib.pb_nccl_allgather(comm, a.ptr, out.ptr, tensor.shape.size, a.dtype.code),
                   "ncclAllGather")
        self.nccl_sync(comm, timeout)
        self.nccl_wait(comm)
        return self._tensor(out, (world,) + tuple(tensor.shape))

    def nccl_broadcast(self, comm, tensor, root, timeout=None):
        self._live(comm)
        a = self._contig(tensor.adapter)
        out = self._new(a.shape, a.dtype, "broadcast")
        _lib.check(self._lib.pb_nccl_broadcast(comm, a.ptr, out.ptr, tensor.shape.size, a.dtype.code, root),
                   "ncclBroadcast")
        self.nccl_sync(comm, timeout)
        self.nccl_wait(comm)
        return self._tensor(out, tuple(tensor.shape))

    # ---------------------------------------------------------- fused optimizer
    def fused_sgd(self, params, velocity, lr, momentum, weight_decay):
        """SGD.step for every parameter in one launch (same op order as minml/optim.py:64-72).

        Updates in place when the parameter / velocity buffer is exclusively owned
        (nothing else references the tensor or its storage), otherwise writes fresh
        buffers and rebinds ``p.data`` exactly like the reference.
        """
        f32 = dtypes.f32
        from .._tensor import Tensor
        n = len(params)
        pin = (ctypes.c_uint64 * n)()
        pout = (ctypes.c_uint64 * n)()
        gs = (ctypes.c_uint64 * n)()
        vin = (ctypes.c_uint64 * n)() if velocity is not None else None
        vout = (ctypes.c_uint64 * n)() if velocity is not None else None
        numel = (ctypes.c_int64 * n)()
        rebind_p, rebind_v, keep = [], [], []
        for i, p in enumerate(params):
            t = p.data
            g = p.grad
            if t.dtype is not f32 or g.dtype is not f32 or t.backend_id != self.name:
                return False
            arr = t.adapter
            garr = self._contig(g.adapter)
            keep.append(garr)
            numel[i] = t.shape.size
            gs[i] = garr.ptr
            pin[i] = arr.ptr
            if _exclusive(t, arr):
                pout[i] = arr.ptr
            else:
                na = self._new(arr.shape, f32, "sgd")
                pout[i] = na.ptr
                rebind_p.append((p, na))
            if velocity is not None:
                vt = velocity[i]
                va = vt.adapter
                vin[i] = va.ptr
                if _exclusive(vt, va):
                    vout[i] = va.ptr
                else:
                    nv = self._new(va.shape, f32, "sgd")
                    vout[i] = nv.ptr
                    rebind_v.append((i, nv))
                    if not va.contiguous:  # stride-0 zeros: read through a dense copy
                        dv = self._contig(va)
                        keep.append(dv)
                        vin[i] = dv.ptr
            if not arr.contiguous:
                da = self._contig(arr)
                keep.append(da)
                pin[i] = da.ptr
        _lib.check(self._lib.pb_sgd(n, pin, pout, gs, vin, vout, numel, lr, momentum, weight_decay), "sgd")
        self.last_sgd = {"params": n, "rebound": len(rebind_p), "velocity_rebound": len(rebind_v)}
        for p, na in rebind_p:
            p.data = Tensor(na, self.name, p.data.shape, f32)
        for i, nv in rebind_v:
            velocity[i] = Tensor(nv, self.name, velocity[i].shape, f32)
        return True


def _exclusive(t, arr):
    """True when only the owner references tensor ``t``, its adapter and its storage."""
    if not arr.contiguous or arr.block is None or arr.ptr != arr.block.ptr:
        return False
    # references: the owner's attribute + getrefcount's argument + our local name(s)
    return sys.getrefcount(t) <= 4 and sys.getrefcount(arr) <= 4 and sys.getrefcount(arr.block) <= 2
