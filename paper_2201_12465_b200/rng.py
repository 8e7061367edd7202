"""Counter-RNG bookkeeping (minml/rng.py:54-86).

Values are a pure function of (seed, counter): word(i) = splitmix64 finalizer
over seed + (i + 1) * GOLDEN (minml/rng.py:16-33).  The words themselves are
produced on the device by ``pb_rand`` (csrc/rng.cu); the host only hands out
counter ranges so every backend draws the same stream.
"""

import threading

GOLDEN = 0x9E3779B97F4A7C15
MASK64 = (1 << 64) - 1


def normal_counters(count):
    """Counters a Box-Muller fill of ``count`` values consumes (minml/rng.py:54-56)."""
    return 2 * ((count + 1) // 2)


class RngState:
    __slots__ = ("seed", "_next", "_lock")

    def __init__(self, seed=0):
        self.seed = int(seed) & MASK64
        self._next = 0
        self._lock = threading.Lock()

    def reseed(self, seed):
        with self._lock:
            self.seed = int(seed) & MASK64
            self._next = 0

    def reserve(self, count):
        with self._lock:
            first = self._next
            self._next = first + int(count)
            return first

    def state(self):
        with self._lock:
            return {"seed": self.seed, "next": self._next}

    def restore(self, state):
        with self._lock:
            self.seed = int(state["seed"]) & MASK64
            self._next = int(state["next"])
