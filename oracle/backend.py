"""OracleBackend: the numpy restatement behind the product's Backend interface.

TEST INFRASTRUCTURE ONLY — tests register it to run the same front end
(Tensor / Variable / nn / optim) on the CPU checker.
"""

from oracle.kernels import KERNELS
from paper_2201_12465_b200.registry import Backend


class HostArray:
    __slots__ = ("array", "__weakref__")

    def __init__(self, array):
        self.array = array


class OracleBackend(Backend):
    def __init__(self, name="oracle", seed=0):
        super().__init__(name, seed)

    def execute(self, call, args):
        arrays = tuple(a.array for a in args)
        if call.name == "to_host":
            return KERNELS["to_host"](call, arrays)
        return HostArray(KERNELS[call.name](call, arrays))
