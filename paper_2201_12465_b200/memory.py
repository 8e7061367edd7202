"""Memory managers: the reference's MemoryManager API (minml/memory.py:86-347) over the
C++ stream-ordered caching allocator in libpaper_b200.so (csrc/allocator.cu).

``alloc(nbytes, op) -> MemoryBlock``, ``free(block)``, ``stats()``, ``flush_cache()``,
``live_blocks``, ``close()`` and the three policies keep the reference's semantics and
counters exactly; ``simulate=True`` runs the same bookkeeping without a device (what
the CPU tests pin against the reference's allocator known answers).  GpuBackend calls
the C entry points directly on its hot path and only builds ``MemoryBlock`` objects
for this public API.
"""

import ctypes
from dataclasses import asdict, dataclass

from .errors import AllocError, ManagerBusy
from .gpu import _lib

CACHE_FLOOR = 512
SPLIT_GRANULARITY = 512
DEFAULT_SPLIT_THRESHOLD = 1 << 20
_POLICY = {"native": 0, "caching": 1, "split_restricted": 2, "split": 2}


def bin_size(nbytes):
    return CACHE_FLOOR if nbytes <= CACHE_FLOOR else 1 << (int(nbytes) - 1).bit_length()


def round_up(nbytes, granularity=SPLIT_GRANULARITY):
    return -(-int(nbytes) // granularity) * granularity


@dataclass
class MemoryBlock:
    block_id: int
    requested_bytes: int
    granted_bytes: int
    bin_size: int
    originating_op: str = None
    data: int = None  # device address

    @property
    def internal_fragmentation(self):
        return self.granted_bytes - self.requested_bytes


@dataclass
class AllocatorStats:
    live_bytes_requested: int = 0
    live_bytes_granted: int = 0
    peak_granted: int = 0
    cache_bytes: int = 0
    alloc_count: int = 0
    free_count: int = 0
    internal_fragmentation: int = 0
    external_fragmentation_ratio: float = 0.0

    def as_dict(self):
        return asdict(self)


OP_TAGS = {}  # op name <-> small int tag stored with each C++ block


def op_tag(name):
    t = OP_TAGS.get(name)
    if t is None:
        t = OP_TAGS[name] = len(OP_TAGS) + 1
        OP_TAGS[-t] = name
    return t


class MemoryManager:
    """Base manager (native policy); subclasses pick the caching policy."""

    policy = "native"

    def __init__(self, capacity=None, simulate=False, threshold=None):
        self._lib = _lib.load()
        self.capacity = capacity
        self.simulate = simulate
        self.threshold = DEFAULT_SPLIT_THRESHOLD if threshold is None else int(threshold)
        self._h = self._lib.pb_mm_create(_POLICY[self.policy], self.threshold, int(capacity or 0),
                                         1 if simulate else 0)
        if not self._h:
            raise ValueError(self._lib.pb_last_error().decode())
        self._op_stack = []
        self._blocks = {}
        self._peak_internal = 0
        self._out = _lib.MMBlock()

    @property
    def handle(self):
        return self._h

    def on_op_begin(self, op):
        self._op_stack.append(op)

    def on_op_end(self, op):
        if self._op_stack:
            self._op_stack.pop()

    def current_op(self):
        return self._op_stack[-1] if self._op_stack else None

    def alloc(self, nbytes, op=None):
        nbytes = int(nbytes)
        if nbytes <= 0:
            raise AllocError(f"allocation size must be positive, got {nbytes}")
        name = op if op is not None else self.current_op()
        b = self._out
        _lib.check(self._lib.pb_mm_alloc(self._h, nbytes, op_tag(name or "-"), ctypes.byref(b)), "alloc")
        blk = MemoryBlock(b.id, b.requested_bytes, b.granted_bytes, b.bin_size, name, b.ptr)
        self._blocks[b.id] = blk
        return blk

    def free(self, block):
        bid = block.block_id if isinstance(block, MemoryBlock) else int(block)
        rc = self._lib.pb_mm_free(self._h, bid)
        if rc:
            raise AllocError(self._lib.pb_last_error().decode())
        self._blocks.pop(bid, None)

    def _raw_stats(self):
        s = _lib.MMStats()
        self._lib.pb_mm_stats_get(self._h, ctypes.byref(s))
        return s

    @property
    def live_blocks(self):
        return int(self._raw_stats().live_blocks)

    @property
    def peak_internal_fragmentation(self):
        return int(self._raw_stats().peak_internal_fragmentation)

    def stats(self):
        s = self._raw_stats()
        return AllocatorStats(s.live_bytes_requested, s.live_bytes_granted, s.peak_granted, s.cache_bytes,
                              s.alloc_count, s.free_count, s.internal_fragmentation,
                              s.external_fragmentation_ratio)

    def flush_cache(self):
        return int(self._lib.pb_mm_flush(self._h))

    def close(self):
        if self.live_blocks:
            raise ManagerBusy(f"{self.live_blocks} live blocks at close")
        self.flush_cache()

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h and _lib._lib is not None:
            try:
                self._lib.pb_mm_destroy(h)
            except Exception:
                pass


class NativeManager(MemoryManager):
    policy = "native"


class CachingManager(MemoryManager):
    policy = "caching"


class SplitRestrictedManager(MemoryManager):
    policy = "split_restricted"

    def __init__(self, threshold=DEFAULT_SPLIT_THRESHOLD, capacity=None, simulate=False):
        super().__init__(capacity=capacity, simulate=simulate,
                         threshold=DEFAULT_SPLIT_THRESHOLD if threshold is None else threshold)


def make_manager(policy, threshold=None, capacity=None, simulate=False):
    if policy == "native":
        return NativeManager(capacity=capacity, simulate=simulate)
    if policy == "caching":
        return CachingManager(capacity=capacity, simulate=simulate)
    if policy in ("split_restricted", "split"):
        return SplitRestrictedManager(threshold=threshold, capacity=capacity, simulate=simulate)
    raise ValueError(f"unknown allocator policy {policy!r}")
