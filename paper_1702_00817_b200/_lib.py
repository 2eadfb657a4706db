"""ctypes binding of libadct_cuda.so (the C ABI in include/adct_cuda.h).

The library is built in-tree by ``__graft_entry__.build()`` (``make`` in
``csrc/``).  There is no fallback: if the shared object is missing or fails to
load, every entry point raises ``NativeLibraryError``.
"""

from __future__ import annotations

import ctypes
import os
import threading
from ctypes import POINTER, c_double, c_int, c_int32, c_int64, c_size_t, c_void_p

from . import errors

LIB_PATH = os.environ.get(
    "ADCT_LIB_PATH", os.path.join(os.path.dirname(os.path.abspath(__file__)), "libadct_cuda.so")
)


class NativeLibraryError(RuntimeError):
    """libadct_cuda.so is missing or unusable (no CPU fallback exists)."""


class QTab(ctypes.Structure):
    """adct_qtab_t (include/adct_cuda.h)."""

    _fields_ = [
        ("qprime", c_int32 * 64),
        ("qe", c_int32 * 64),
        ("magic", ctypes.c_uint32 * 64),
        ("bias", c_int32 * 64),
        ("mult", c_int32 * 64),
        ("kq", c_int32 * 64),
        ("magic_w", ctypes.c_uint32 * 64),
        ("cadd_w", c_int32 * 64),
        ("kw", c_int32 * 64),
        ("shift_w", c_int32 * 64),
        ("wide", c_int32),
        ("max_abs_v", c_int32),
        ("quality", c_int32),
        ("aligned", c_int32),
        ("recip_f", ctypes.c_uint32 * 64),
    ]


class Plane(ctypes.Structure):
    """adct_plane_t (include/adct_cuda.h)."""

    _fields_ = [
        ("src", c_void_p),
        ("dst", c_void_p),
        ("height", c_int32),
        ("width", c_int32),
        ("src_frame_stride", c_int64),
        ("dst_frame_stride", c_int64),
    ]


# name -> (restype, argtypes); must match include/adct_cuda.h exactly
# (tests/test_capi.py parses the header and checks every declaration is here).
PROTOTYPES = {
    "adct_version": (c_int, []),
    "adct_strerror": (ctypes.c_char_p, [c_int]),
    "adct_last_cuda_error": (c_int, []),
    "adct_qtab_build": (c_int, [POINTER(c_double), POINTER(QTab)]),
    "adct_qtab_from_quality": (c_int, [POINTER(c_int32), c_int32, POINTER(QTab)]),
    "adct_forward_int32": (c_int, [c_void_p, c_int64, c_int32, c_int32, c_int64, c_int32, c_void_p, c_void_p]),
    "adct_forward_int16": (c_int, [c_void_p, c_int64, c_int32, c_int32, c_int64, c_int32, c_void_p, c_void_p]),
    "adct_compress_retain": (
        c_int,
        [c_void_p, c_void_p, c_int64, c_int32, c_int32, c_int64, c_int64, c_int32, c_void_p, c_void_p, c_void_p],
    ),
    "adct_compress_retain_exchange": (
        c_int,
        [c_void_p, c_void_p, c_int64, c_int32, c_int32, c_int64, c_int64, c_int32, c_void_p, c_void_p,
         c_int32, c_int64, c_void_p, c_void_p],
    ),
    "adct_compress_quant_planes_exchange": (
        c_int,
        [c_void_p, c_int32, c_int64, c_void_p, c_void_p, c_void_p, c_int32, c_int64, c_void_p, c_void_p],
    ),
    "adct_compress_quant": (
        c_int,
        [c_void_p, c_void_p, c_int64, c_int32, c_int32, c_int64, c_int64, POINTER(QTab), c_void_p, c_void_p],
    ),
    "adct_compress_quant_planes": (c_int, [POINTER(Plane), c_int32, c_int64, POINTER(QTab), c_void_p, c_void_p]),
    "adct_compress_retain_planes": (c_int, [POINTER(Plane), c_int32, c_int64, c_int32, c_void_p, c_void_p]),
    "adct_sweep_retain_sse": (
        c_int,
        [c_void_p, c_int64, c_int32, c_int32, c_int64, c_int32, c_int32, c_void_p, c_void_p, c_void_p],
    ),
    "adct_forward_dense": (c_int, [c_void_p, c_int32, c_int64, c_int32, c_int32, POINTER(c_double), c_void_p, c_void_p]),
    "adct_inverse_dense": (
        c_int,
        [c_void_p, c_int64, c_int32, c_int32, POINTER(c_double), c_int32, c_int32, c_void_p, c_void_p],
    ),
    "adct_sweep_dense": (
        c_int,
        [c_void_p, c_int32, c_int64, c_int32, c_int32, POINTER(c_double), c_int32, c_int32, c_void_p, c_void_p],
    ),
    "adct_forward_f64": (c_int, [c_void_p, c_int64, c_int32, c_int32, c_void_p, c_void_p]),
    "adct_forward_f64_u8": (c_int, [c_void_p, c_int64, c_int32, c_int32, c_void_p, c_void_p]),
    "adct_inverse_f64": (c_int, [c_void_p, c_int64, c_int32, c_int32, c_int32, c_int32, c_void_p, c_void_p]),
    "adct_sse_u8": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int64, c_void_p, c_void_p]),
    "adct_synth_blobs": (c_int, [c_void_p, c_int64, c_int32, c_int32, c_int64, c_void_p, c_int32, c_void_p, c_void_p]),
    "adct_pipeline_create": (c_int, [c_int32, c_size_t, POINTER(c_void_p)]),
    "adct_pipeline_destroy": (c_int, [c_void_p]),
    "adct_pipeline_compress_retain": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_int64, c_int32, c_int32, c_int32, c_void_p],
    ),
    "adct_pipeline_compress_quant": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_int64, c_int32, c_int32, POINTER(QTab), c_void_p],
    ),
    "adct_host_register": (c_int, [c_void_p, c_size_t]),
    "adct_host_unregister": (c_int, [c_void_p]),
    "adct_host_is_pinned": (c_int, [c_void_p]),
    "adct_pipeline_compress_quant_planes": (c_int, [c_void_p, c_void_p, c_int32, c_int64, c_void_p, c_void_p]),
    "adct_quant_jit_stats": (c_int, [POINTER(c_int64), POINTER(c_int64), POINTER(c_int64)]),
    "adct_host_alloc": (c_int, [c_size_t, POINTER(c_void_p)]),
    "adct_host_free": (c_int, [c_void_p]),
}

# C error codes -> exception classes mirroring adct/errors.py:21-33.
ADCT_OK = 0
_ERRORS = {
    1: errors.BadDimensions,
    2: errors.InvalidRetention,
    3: errors.NonPositiveQuantizer,
    4: errors.DimensionMismatch,
    5: ValueError,
    6: ValueError,
    7: RuntimeError,
    8: errors.UnsupportedQuantizer,
}

_lock = threading.Lock()
_lib = None


def lib() -> ctypes.CDLL:
    """Load (once) and return the native library; raise loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryError(
                f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        try:
            handle = ctypes.CDLL(LIB_PATH)
        except OSError as exc:  # pragma: no cover - depends on the box
            raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (res, args) in PROTOTYPES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
        return _lib


def check(rc: int, what: str = "") -> None:
    """Raise the mirrored exception for a non-zero return code."""
    if rc == ADCT_OK:
        return
    L = lib()
    msg = L.adct_strerror(rc).decode()
    if rc == 7:
        msg += f" (cudaError {L.adct_last_cuda_error()})"
    if what:
        msg = f"{what}: {msg}"
    raise _ERRORS.get(rc, RuntimeError)(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)
