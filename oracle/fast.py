"""ctypes front end of the plain-C exact oracle (TEST INFRASTRUCTURE ONLY —
see oracle/__init__.py; checker for the full-size parity tests).

Same conventions and results as oracle/exact.py (tests/test_oracle.py pins
the two against each other and against the golden vectors made by the
reference), but fast enough to check BASELINE's configs at their stated
sizes: work is split into (image, block-row strip) tasks over a thread pool
(ctypes releases the GIL during the C call).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_DIR = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_DIR, "_build", "liboracle_exact.so")
_lock = threading.Lock()
_lib = None

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32


def build() -> str:
    """make -C oracle (gcc); returns the .so path."""
    subprocess.run(["make", "-s", "-C", _DIR], check=True)
    return _SO


def lib() -> ctypes.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(_SO):
                build()
            L = ctypes.CDLL(_SO)
            L.oracle_forward.argtypes = [_P, _I64, _I32, _I32, _I64, _I32, _P]
            L.oracle_compress_retain.argtypes = [_P, _I64, _I32, _I32, _I64, _I32, _I32, _I32, _P, _I64, _P, _P]
            L.oracle_sweep_sse.argtypes = [_P, _I64, _I32, _I32, _I64, _I32, _I32, _I32, _I32, _P, _P]
            L.oracle_compress_quant.argtypes = [_P, _I64, _I32, _I32, _I64, _P, _I32, _I32, _P, _I64, _P]
            for f in (L.oracle_forward, L.oracle_compress_retain, L.oracle_sweep_sse, L.oracle_compress_quant):
                f.restype = ctypes.c_int
            _lib = L
    return _lib


def _threads(threads):
    return threads or max(1, len(os.sched_getaffinity(0)))


def _tasks(n, h, threads):
    """(image, row0, row1) tasks: about 4 per thread, whole block rows."""
    nbr = h // 8
    per_img = max(1, min(nbr, (4 * threads + n - 1) // max(n, 1)))
    step = (nbr + per_img - 1) // per_img
    return [(f, r0, min(nbr, r0 + step)) for f in range(n) for r0 in range(0, nbr, step)]


def _prep(imgs):
    imgs = np.ascontiguousarray(imgs, dtype=np.uint8)
    if imgs.ndim == 2:
        imgs = imgs[None]
    return imgs


def compress_quant(imgs, qp, rec: bool = True, threads=None):
    """(rec uint8 or None, sse int64[n]) — same as exact.compress_quant."""
    imgs = _prep(imgs)
    n, h, w = imgs.shape
    qp = np.ascontiguousarray(np.asarray(qp).reshape(64), dtype=np.int32)
    out = np.empty_like(imgs) if rec else None
    tasks = _tasks(n, h, _threads(threads))
    part = np.zeros(len(tasks), dtype=np.int64)
    L = lib()

    def run(k):
        f, r0, r1 = tasks[k]
        acc = np.zeros(1, dtype=np.int64)
        rc = L.oracle_compress_quant(imgs[f].ctypes.data, 1, h, w, h * w, qp.ctypes.data, r0, r1,
                                     out[f].ctypes.data if rec else None, h * w, acc.ctypes.data)
        assert rc == 0, rc
        part[k] = acc[0]

    with ThreadPoolExecutor(_threads(threads)) as ex:
        list(ex.map(run, range(len(tasks))))
    sse = np.zeros(n, dtype=np.int64)
    np.add.at(sse, [t[0] for t in tasks], part)
    return out, sse


def compress_retain(imgs, r: int, rec: bool = True, threads=None):
    """(rec uint8 or None, sse int64[n], sse_unrounded int64[n]) — same as exact.compress_retain."""
    imgs = _prep(imgs)
    n, h, w = imgs.shape
    out = np.empty_like(imgs) if rec else None
    tasks = _tasks(n, h, _threads(threads))
    part = np.zeros((len(tasks), 2), dtype=np.int64)
    L = lib()

    def run(k):
        f, r0, r1 = tasks[k]
        acc = np.zeros(2, dtype=np.int64)
        rc = L.oracle_compress_retain(imgs[f].ctypes.data, 1, h, w, h * w, r, r0, r1,
                                      out[f].ctypes.data if rec else None, h * w,
                                      acc[0:].ctypes.data, acc[1:].ctypes.data)
        assert rc == 0, rc
        part[k] = acc

    with ThreadPoolExecutor(_threads(threads)) as ex:
        list(ex.map(run, range(len(tasks))))
    sse = np.zeros((n, 2), dtype=np.int64)
    np.add.at(sse, [t[0] for t in tasks], part)
    return out, sse[:, 0], sse[:, 1]


def sweep_sse(imgs, r_min: int, r_max: int, threads=None):
    """(sse int64[n, nr], sse_unrounded int64[n, nr]) — exact.sweep_sse plus the unrounded convention."""
    imgs = _prep(imgs)
    n, h, w = imgs.shape
    nr = r_max - r_min + 1
    tasks = _tasks(n, h, _threads(threads))
    part = np.zeros((len(tasks), 2, nr), dtype=np.int64)
    L = lib()

    def run(k):
        f, r0, r1 = tasks[k]
        acc = np.zeros((2, nr), dtype=np.int64)
        rc = L.oracle_sweep_sse(imgs[f].ctypes.data, 1, h, w, h * w, r_min, r_max, r0, r1,
                                acc[0].ctypes.data, acc[1].ctypes.data)
        assert rc == 0, rc
        part[k] = acc

    with ThreadPoolExecutor(_threads(threads)) as ex:
        list(ex.map(run, range(len(tasks))))
    sse = np.zeros((n, 2, nr), dtype=np.int64)
    np.add.at(sse, [t[0] for t in tasks], part)
    return sse[:, 0], sse[:, 1]


def forward(imgs, level_shift: bool = False):
    """int32 (n, h*w/64, 8, 8) in _tile order — exact.forward_unscaled."""
    imgs = _prep(imgs)
    n, h, w = imgs.shape
    out = np.empty((n, h * w // 64, 8, 8), dtype=np.int32)
    rc = lib().oracle_forward(imgs.ctypes.data, n, h, w, h * w, int(level_shift), out.ctypes.data)
    assert rc == 0
    return out
