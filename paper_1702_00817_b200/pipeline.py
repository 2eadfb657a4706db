"""Host-buffer pipeline: the end-to-end public call for images in CPU memory.

Wraps the native adct_pipeline (csrc/capi.cu): chunks of the host batch are
copied in, compressed and copied out on three CUDA streams so H2D, kernel
and D2H overlap.  Ordinary (pageable) numpy arrays are staged by the library
through its own page-locked ring, filled and drained by host threads while
the copies run (never registered per call); page-locked arrays
(`pinned_empty`, or `pin()` for repeated use) are copied directly.
`register=True` page-locks the caller's arrays for the call instead
(arrays that are already pinned are left alone; not for arrays that other
threads are passing to concurrent calls at the same time — use `pin()` once).
Several threads may share one pipeline: the library serialises its calls.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import BadDimensions, InvalidRetention


class HostPipeline:
    def __init__(self, device: int = 0, chunk_bytes: int = 32 << 20):
        # 32-64 MiB chunks measured fastest (tools/e2e_sweep.py): larger ones
        # lengthen the pipeline's fill and drain, smaller ones add per-copy gaps
        h = ctypes.c_void_p()
        _lib.call("adct_pipeline_create", int(device), int(chunk_bytes), ctypes.byref(h))
        self._h = h

    def close(self) -> None:
        if self._h:
            _lib.call("adct_pipeline_destroy", self._h)
            self._h = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _check(images: np.ndarray) -> tuple[int, int, int]:
        if images.dtype != np.uint8 or images.ndim != 3 or not images.flags.c_contiguous:
            raise ValueError("images must be a C-contiguous uint8 array (N, H, W)")
        n, h, w = images.shape
        if h % 8 or w % 8:
            raise BadDimensions(f"image dimensions must be divisible by 8, got {(h, w)}")
        return n, h, w

    @staticmethod
    def _check_rec(rec, images: np.ndarray) -> None:
        """The native copies write n*h*w bytes at rec: it must be exactly that buffer."""
        if rec is None:
            return
        if not isinstance(rec, np.ndarray) or rec.dtype != np.uint8 or rec.shape != images.shape \
                or not rec.flags.c_contiguous or not rec.flags.writeable:
            raise ValueError(f"rec must be a writeable C-contiguous uint8 array of shape {images.shape}")

    def compress_retain(self, images: np.ndarray, r: int, rec: np.ndarray | None = None, *, register: bool = False):
        """Returns (rec or None, sse int64[N])."""
        if not 1 <= int(r) <= 64:
            raise InvalidRetention(f"retention count must be in [1, 64], got {r}")
        n, h, w = self._check(images)
        self._check_rec(rec, images)
        sse = np.zeros(n, dtype=np.uint64)
        with _Pinned([images, rec] if register else []):
            _lib.call(
                "adct_pipeline_compress_retain", self._h, images.ctypes.data,
                None if rec is None else rec.ctypes.data, n, h, w, int(r), sse.ctypes.data,
            )
        return rec, sse.astype(np.int64)

    def compress_quant(self, images: np.ndarray, qtab, rec: np.ndarray | None = None, *, register: bool = False):
        n, h, w = self._check(images)
        self._check_rec(rec, images)
        sse = np.zeros(n, dtype=np.uint64)
        with _Pinned([images, rec] if register else []):
            _lib.call(
                "adct_pipeline_compress_quant", self._h, images.ctypes.data,
                None if rec is None else rec.ctypes.data, n, h, w, ctypes.byref(qtab), sse.ctypes.data,
            )
        return rec, sse.astype(np.int64)


    def compress_quant_planes(self, planes, qtab, outs=None, *, register: bool = False):
        """Frames of 1..3 host planes (each (N, H_k, W_k) uint8, e.g. Y/Cb/Cr of
        4:2:0 video) through the one-launch planes kernel in chunks of frames.
        `outs`: matching arrays for the reconstructions, or None (SSE only).
        Returns (outs, sse int64 [N, n_planes])."""
        from ._lib import Plane

        planes = list(planes)
        if not 1 <= len(planes) <= 3:
            raise ValueError("1 to 3 planes")
        n = planes[0].shape[0]
        for k, a in enumerate(planes):
            self._check(a)
            if a.shape[0] != n:
                raise ValueError(f"plane {k} has {a.shape[0]} frames, plane 0 has {n}")
        if outs is not None:
            outs = list(outs)
            if len(outs) != len(planes) or any(o.shape != a.shape or o.dtype != np.uint8 or not o.flags.c_contiguous
                                               for o, a in zip(outs, planes)):
                raise ValueError("outs must match the planes' shapes (C-contiguous uint8)")
        arr = (Plane * len(planes))()
        for k, a in enumerate(planes):
            h, w = a.shape[1], a.shape[2]
            arr[k].src = a.ctypes.data
            arr[k].dst = outs[k].ctypes.data if outs is not None else None
            arr[k].height, arr[k].width = h, w
            arr[k].src_frame_stride = h * w
            arr[k].dst_frame_stride = h * w
        sse = np.zeros((n, len(planes)), dtype=np.uint64)
        with _Pinned(planes + (outs or []) if register else []):
            _lib.call("adct_pipeline_compress_quant_planes", self._h, ctypes.addressof(arr), len(planes), n,
                      ctypes.byref(qtab), sse.ctypes.data)
        return outs, sse.astype(np.int64)


class _Pinned:
    """Page-lock numpy buffers for the duration of a call."""

    def __init__(self, arrays):
        self.arrays = [a for a in arrays if a is not None and a.nbytes > 0]
        self.done = []

    def __enter__(self):
        try:
            for a in self.arrays:
                if _lib.lib().adct_host_is_pinned(a.ctypes.data):
                    continue  # already page-locked (pinned_empty / pin()): leave it to its owner
                _lib.call("adct_host_register", a.ctypes.data, a.nbytes)
                self.done.append(a)
        except BaseException:
            self.__exit__()
            raise
        return self

    def __exit__(self, *exc):
        for a in self.done:
            _lib.lib().adct_host_unregister(a.ctypes.data)
        self.done = []


def pinned_empty(shape, dtype=np.uint8) -> np.ndarray:
    """Uninitialised numpy array in page-locked memory from adct_host_alloc
    (cudaHostAlloc): the fastest host buffer for the pipeline.  The memory is
    freed when the array (and every view of it) is garbage collected; do not
    pin()/unpin() it."""
    import weakref

    dtype = np.dtype(dtype)
    shape = tuple(int(d) for d in (shape if isinstance(shape, (tuple, list)) else (shape,)))
    nbytes = int(np.prod(shape, dtype=np.int64)) * dtype.itemsize
    if nbytes == 0:
        return np.empty(shape, dtype)
    ptr = ctypes.c_void_p()
    _lib.call("adct_host_alloc", nbytes, ctypes.byref(ptr))
    buf = (ctypes.c_uint8 * nbytes).from_address(ptr.value)
    arr = np.frombuffer(buf, dtype=dtype).reshape(shape)
    weakref.finalize(buf, _lib.lib().adct_host_free, ptr.value)
    return arr


def pin(array: np.ndarray) -> None:
    """Page-lock an array for repeated pipeline calls (unpin() to release)."""
    _lib.call("adct_host_register", array.ctypes.data, array.nbytes)


def unpin(array: np.ndarray) -> None:
    _lib.call("adct_host_unregister", array.ctypes.data)
