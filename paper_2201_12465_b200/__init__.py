"""B200-native backend + lean front end for the Flashlight (arXiv 2201.12465) tensor API.

The public surface mirrors the reference package ``minml`` (minml/__init__.py):
``Tensor``, ``Variable``, ``nn``, ``optim``, ``distributed``, ``registry`` ...
Importing the package registers the CUDA backend ``"gpu"`` (GpuBackend, a
``registry.Backend`` over libpaper_b200.so) when a B200 is present; there is
no CPU fallback — without the extension or a device no backend is registered
and creating a tensor raises ``UnknownBackend`` naming the reason.
"""

import os

from . import registry

if os.environ.get("PB_NO_AUTOREGISTER") != "1":
    try:
        from .gpu.backend import GpuBackend, device_available

        if device_available():
            from .gpu import _lib as _l

            _ndev = _l.load().pb_device_count()
            registry.register(GpuBackend("gpu", device=int(os.environ.get("LOCAL_RANK", "0")) % _ndev))
        else:
            registry._load_error = "no CUDA device visible"
    except (OSError, ImportError, AttributeError) as exc:  # libpaper_b200.so missing, unloadable or stale
        registry._load_error = f"libpaper_b200.so not loadable: {exc}"

from . import distributed, nn, ops, optim, training  # noqa: E402
from .autograd import Variable, gradcheck, no_grad, register_custom_op  # noqa: E402
from .dtypes import DType, by_name as dtype_by_name  # noqa: E402
from .errors import Error  # noqa: E402
from .registry import OpCall, primitive_names  # noqa: E402
from .shape import Shape  # noqa: E402
from ._tensor import (Tensor, arange, concat, conv2d, full, identity, matmul, ones,  # noqa: E402
                      rand_normal, rand_uniform, tensor, zeros)
from .wrappers import CountingBackend, ForwardingBackend  # noqa: E402

__version__ = "0.1.0"
