"""The drop-in: ``GpuBackend`` registered into the reference's OWN registry.

``install()`` is what a ``minml`` maintainer binds: it registers a
backend into ``minml.registry`` (minml/registry.py:149-158, ``set_default`` :180-187), and
from there minml's own ``Tensor`` / ``Variable`` / ``nn`` / ``optim`` / ``training`` run
every primitive on the B200 through ``Backend.execute(OpCall, adapters)``
(minml/registry.py:97-141) -- nothing of this package's front end is involved.

The class subclasses both ``GpuBackend`` and ``minml.registry.Backend`` (minml's
isinstance checks hold).  At the boundary it translates minml's descriptors into the
backend's: ``OpCall.dtype`` / ``params["dtype"]`` are minml ``DType`` objects or tags,
matched by NAME (minml/dtypes.py:13-46 -- the same six tags and promotion ranks), and the
planned ``Shape`` is kept as a tuple.  Exceptions leave as minml's own classes of the same
name (minml/errors.py), so reference code catching ``minml.errors.DomainError`` /
``OutOfMemory`` sees them; backend-only failures (a CUDA error) become ``minml.errors.Error``.
Adapters stay opaque to minml, exactly as its contract says.
"""

from .. import dtypes as _dt
from .. import errors as _err
from ..registry import OpCall as _OpCall
from .backend import GpuBackend

_CLASSES = {}


def backend_class(minml):
    """The GpuBackend subclass bound to one imported ``minml`` package (cached)."""
    key = id(minml)
    cls = _CLASSES.get(key)
    if cls is not None:
        return cls
    m_errors = minml.errors
    m_backend = minml.registry.Backend

    def translate_error(exc):
        target = getattr(m_errors, type(exc).__name__, None)
        if not (isinstance(target, type) and issubclass(target, BaseException)):
            target = m_errors.Error
        return target(str(exc))

    class MinmlGpuBackend(GpuBackend, m_backend):
        """GpuBackend speaking minml's OpCall/DType/errors (see module docstring)."""

        def execute(self, call, args):
            dt = call.dtype
            if type(dt) is not _dt.DType:
                params = call.params
                pdt = params.get("dtype")
                if pdt is not None and not isinstance(pdt, str) and type(pdt) is not _dt.DType:
                    params = dict(params, dtype=pdt.name)
                call = _OpCall(call.name, params, call.shape, _dt.by_name(dt.name))
            try:
                return GpuBackend.execute(self, call, args)
            except _err.Error as exc:
                raise translate_error(exc) from exc

        def attach_manager(self, manager):
            try:
                return GpuBackend.attach_manager(self, manager)
            except _err.Error as exc:
                raise translate_error(exc) from exc

        def detach_manager(self):
            try:
                return GpuBackend.detach_manager(self)
            except _err.Error as exc:
                raise translate_error(exc) from exc

    MinmlGpuBackend.__qualname__ = MinmlGpuBackend.__name__ = "GpuBackend"
    _CLASSES[key] = MinmlGpuBackend
    return MinmlGpuBackend


def install(minml=None, name="gpu", device=0, seed=0, default=True):
    """Register a B200 backend into ``minml``'s registry; returns it.

    ``minml``: the imported reference package (default: ``import minml``)."""
    if minml is None:
        import minml  # noqa: F811
    import minml.errors  # noqa: F401  (submodules the class binds to)
    import minml.registry  # noqa: F401
    be = backend_class(minml)(name=name, seed=seed, device=device)
    minml.registry.register(be)
    if default:
        minml.registry.set_default(name)
    return be
