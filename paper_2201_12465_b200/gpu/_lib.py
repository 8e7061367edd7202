"""ctypes binding of libpaper_b200.so (declarations in include/paper_b200.h).

Descriptors cross the boundary as packed bytes laid out exactly like ``pb_tensor`` /
``pb_scalar`` (a precompiled ``struct.Struct`` is ~10x cheaper per op than filling a
ctypes.Structure).  Any nonzero status raises ``DeviceError`` carrying pb_last_error().
"""

import atexit
import ctypes
import os
import struct

from ..errors import AllocError, CollectiveTimeout, DeviceError, DomainError, OutOfMemory

_HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB_PATH = os.environ.get("PB_LIB", os.path.join(_HERE, "libpaper_b200.so"))

MAX_RANK = 8
TENSOR = struct.Struct("<Qii8q8q")   # pb_tensor: ptr, dtype, ndim, shape[8], strides[8]
SCALAR = struct.Struct("<iidq")      # pb_scalar: kind, pad, f, i
CONV = struct.Struct("<iiii")        # pb_conv
STEP = struct.Struct("<iiiiiid")     # pb_chain_step: op, kind, side, leaf, to_bool, pad, scalar
RSTAGE = struct.Struct("<iiif")      # pb_red_stage: axis, epi_op, epi_left, scalar
WINDOW = struct.Struct("<iid4q4q4q")  # pb_leaf_window: on, pad, fill, mul[4], off[4], div[4]
_ZEROS = (0,) * MAX_RANK

BINOP = {"add": 0, "sub": 1, "mul": 2, "div": 3, "pow": 4, "minimum": 5, "maximum": 6, "eq": 7,
         "lt": 8, "gt": 9, "logical_and": 10, "logical_or": 11}
UNOP = {"neg": 0, "abs": 1, "exp": 2, "log": 3, "sqrt": 4, "sin": 5, "cos": 6, "tanh": 7,
        "logical_not": 8, "astype": 9}
REDOP = {"sum": 0, "max_reduce": 1, "min_reduce": 2, "argmax": 3}


class MMStats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in (
        "live_bytes_requested", "live_bytes_granted", "peak_granted", "cache_bytes", "alloc_count",
        "free_count", "internal_fragmentation", "peak_internal_fragmentation", "live_blocks")] + [
        ("external_fragmentation_ratio", ctypes.c_double)]


class MMBlock(ctypes.Structure):
    _fields_ = [("id", ctypes.c_uint64), ("ptr", ctypes.c_uint64), ("requested_bytes", ctypes.c_uint64),
                ("granted_bytes", ctypes.c_uint64), ("bin_size", ctypes.c_uint64),
                ("op_tag", ctypes.c_int32), ("pool", ctypes.c_int32)]


# name -> (restype, argtypes); every symbol include/paper_b200.h declares
_P = ctypes.c_void_p
_B = ctypes.c_char_p
_U64 = ctypes.c_uint64
_I = ctypes.c_int
_I32P = ctypes.POINTER(ctypes.c_int32)
_U64P = ctypes.POINTER(ctypes.c_uint64)
_I64P = ctypes.POINTER(ctypes.c_int64)
_F = ctypes.c_float
SIGNATURES = {
    "pb_init": (_I, [_I]),
    "pb_device_count": (_I, []),
    "pb_last_error": (ctypes.c_char_p, []),
    "pb_synchronize": (_I, []),
    "pb_stream": (_U64, [_I]),
    "pb_h2d": (_I, [_U64, _P, _U64]),
    "pb_d2h": (_I, [_P, _U64, _U64]),
    "pb_h2d_on": (_I, [_U64, _P, _U64, _I]),
    "pb_d2h_post": (_I, [_U64, _U64, _I]),
    "pb_d2h_fetch": (_I, [_I, _P, _U64]),
    "pb_host_alloc": (_P, [_U64]),
    "pb_host_free": (_I, [_P]),
    "pb_stream_sync": (_I, [_I]),
    "pb_d2d": (_I, [_U64, _U64, _U64]),
    "pb_event_record": (_I, [_I, _I]),
    "pb_graph_begin": (_I, []),
    "pb_graph_end": (_I, [_U64P]),
    "pb_graph_launch": (_I, [_U64]),
    "pb_graph_destroy": (_I, [_U64]),
    "pb_timer": (_I, [_I, _U64P, ctypes.POINTER(ctypes.c_float)]),
    "pb_mm_create": (_P, [_I, _U64, _U64, _I]),
    "pb_mm_destroy": (None, [_P]),
    "pb_mm_alloc": (_I, [_P, _U64, ctypes.c_int32, ctypes.POINTER(MMBlock)]),
    "pb_mm_free": (_I, [_P, _U64]),
    "pb_mm_record_stream": (_I, [_P, _U64, _I]),
    "pb_mm_stats_get": (_I, [_P, ctypes.POINTER(MMStats)]),
    "pb_mm_flush": (_U64, [_P]),
    "pb_mm_pool": (_I, [_P, _I]),
    "pb_bin_size": (_U64, [_U64]),
    "pb_round_up": (_U64, [_U64]),
    "pb_binary": (_I, [_I, _B, _B, _B, _I, _B]),
    "pb_unary": (_I, [_I, _B, _I, _B]),
    "pb_copy": (_I, [_B, _B]),
    "pb_pad": (_I, [_B, _I64P, _B, _B]),
    "pb_fill": (_I, [_B, _B]),
    "pb_arange": (_I, [_B]),
    "pb_rand": (_I, [_I, _U64, _U64, _B]),
    "pb_rand_dev": (_I, [_I, _U64, _U64, _U64, _B]),
    "pb_counter_add": (_I, [_U64, _U64]),
    "pb_fastdiv_probe": (_I, [_U64, _U64, _U64, ctypes.c_int64]),
    "pb_reduce": (_I, [_I, _B, _I, _B]),
    "pb_reduce_epi": (_I, [_I, _B, _I, _B, _I, ctypes.c_float, _I]),
    "pb_check": (_I, [_I, _B, _I32P]),
    "pb_matmul": (_I, [_B, _B, _B]),
    "pb_conv2d": (_I, [_B, _B, _B, _B, _B]),
    "pb_conv2d_grad_input": (_I, [_B, _B, _B, _B]),
    "pb_conv2d_grad_weight": (_I, [_B, _B, _B, _B]),
    "pb_ew_chain": (_I, [_I, _B, _I, ctypes.c_double, _I, _B, _B]),
    "pb_ew_chain_taps": (_I, [_I, _B, _I, ctypes.c_double, _I, _B, _I, _B, _B, _B]),
    "pb_reduce_chain": (_I, [_I, _B, _I, ctypes.c_double, _I, _B, _I, _B, _I, _B, _B]),
    "pb_ew_chain_win": (_I, [_I, _B, _B, _I, ctypes.c_double, _I, _B, _B]),
    "pb_chain_jit_kernels": (_I, []),
    "pb_sgd": (_I, [_I, _U64P, _U64P, _U64P, _U64P, _U64P, _I64P, _F, _F, _F]),
    "pb_bucket_pack": (_I, [_I, _U64P, _I64P, _U64]),
    "pb_scale_f32": (_I, [_U64, ctypes.c_int64, _F]),
    "pb_nccl_unique_id": (_I, [ctypes.c_char_p]),
    "pb_nccl_init": (_P, [_I, _I, ctypes.c_char_p]),
    "pb_nccl_destroy": (_I, [_P]),
    "pb_nccl_allreduce": (_I, [_P, _U64, _U64, _U64, _I, _I]),
    "pb_nccl_broadcast": (_I, [_P, _U64, _U64, _U64, _I, _I]),
    "pb_nccl_allgather": (_I, [_P, _U64, _U64, _U64, _I]),
    "pb_nccl_wait": (_I, [_P]),
    "pb_nccl_sync": (_I, [_P, ctypes.c_int64]),
    "pb_nvtx_push": (_I, [_B]),
    "pb_nvtx_pop": (_I, []),
    "pb_debug_stall_comm": (_I, [ctypes.c_int64]),
    "pb_launch_count": (_U64, []),
    "pb_gemm_path": (_I, []),
    "pb_set_gemm_path": (_I, [_I]),
}

_lib = None


def _at_exit():
    """Interpreter exit: drain the device, then detach the library so the finalizers of
    device blocks and graphs that module teardown runs later (DevBlock, GraphExec) become
    no-ops instead of calling into a CUDA runtime that is shutting down -- a process that
    still held a recorded graph's pool could hang there.  The driver reclaims everything."""
    global _lib
    lib = _lib
    if lib is not None:
        try:
            lib.pb_synchronize()
        except Exception:  # noqa: BLE001
            pass
    _lib = None


def load():
    """Load the shared library once (raises OSError if it is missing)."""
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        atexit.register(_at_exit)
    return _lib


_STATUS_EXC = {3: OutOfMemory, 4: AllocError, 5: DomainError, 8: CollectiveTimeout}
UNSUPPORTED = 7  # PB_ERR_UNSUPPORTED: the entry point declined the layout, nothing was launched


def check(status, what=""):
    if status:
        msg = _lib.pb_last_error().decode(errors="replace")
        raise _STATUS_EXC.get(status, DeviceError)(f"{what}: {msg}" if what else msg)


def pack_tensor(ptr, dtype_code, shape, strides):
    n = len(shape)
    return TENSOR.pack(ptr, dtype_code, n, *shape, *_ZEROS[n:], *strides, *_ZEROS[n:])


def pack_scalar(value):
    t = type(value)
    if t is bool:
        return SCALAR.pack(2, 0, 0.0, int(value))
    if t is int:
        return SCALAR.pack(1, 0, 0.0, value)
    return SCALAR.pack(0, 0, float(value), 0)
