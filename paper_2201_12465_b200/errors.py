"""Error taxonomy of the tensor API (mirrors minml/errors.py:9-110 name for name).

Every error raised on purpose derives from ``Error``; code written against the
reference catches the same class names here.
"""


class Error(Exception):
    """Root of every deliberate failure in the library."""


class ShapeError(Error):
    pass


class AxisError(Error):
    pass


class DTypeError(Error):
    pass


class DomainError(Error):
    """Integer arithmetic with no representable result (x // 0, x ** -1)."""


class EmptyReduction(Error):
    pass


class BackendMismatch(Error):
    pass


class DuplicateBackend(Error):
    pass


class UnknownBackend(Error):
    pass


class OutOfMemory(Error):
    pass


class ManagerBusy(Error):
    pass


class AllocError(Error):
    pass


class TraceError(Error):
    def __init__(self, message, index=None):
        super().__init__(message if index is None else f"event {index}: {message}")
        self.index = index


class SeedRequired(Error):
    pass


class TapeConsumed(Error):
    pass


class GradShapeError(Error):
    pass


class MissingGradient(Error):
    pass


class EmptyMeter(Error):
    pass


class FormatError(Error):
    def __init__(self, message, offset=None):
        super().__init__(message if offset is None else f"byte {offset}: {message}")
        self.offset = offset


class ConfigError(Error):
    pass


class CollectiveShapeError(Error):
    pass


class CollectiveTimeout(Error):
    pass


class DeviceError(Error):
    """A CUDA/NCCL call reported failure (message carries the C-ABI error text)."""
