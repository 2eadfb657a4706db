"""Batched device API over torch CUDA tensors — the hot path.

Every function validates like the reference (before any compute), then makes
exactly one C-ABI call on the current torch stream.  Inputs are uint8
(N, H, W) CUDA tensors (rows contiguous); outputs are fresh tensors.
PyTorch supplies device memory and streams only; all arithmetic is in
libadct_cuda.so.
"""

from __future__ import annotations

import ctypes
import functools
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .errors import BadDimensions, DimensionMismatch, InvalidRetention


def _stream() -> int:
    # the current stream of the current device, which _device_guard has set
    # to the device of the call's tensors
    return torch.cuda.current_stream().cuda_stream


def _device_guard(fn):
    """Run `fn` with its tensors' CUDA device current: the C ABI launches on
    the current device and the stream passed in, so a tensor on another GPU
    must not be launched in this device's context or on its stream."""

    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        dev = None
        for a in (*args, *kwargs.values()):
            if isinstance(a, (list, tuple)) and a:
                a = a[0]
            if isinstance(a, torch.Tensor) and a.is_cuda:
                dev = a.device
                break
        if dev is None:
            return fn(*args, **kwargs)
        with torch.cuda.device(dev):
            return fn(*args, **kwargs)

    return wrapper


def _check_out(out: torch.Tensor | None, images: torch.Tensor) -> None:
    """`out` receives n frames of h x w bytes at its row/frame strides."""
    if out is None:
        return
    n, h, w = images.shape
    if (not isinstance(out, torch.Tensor) or out.dtype != torch.uint8 or out.device != images.device
            or tuple(out.shape) != (n, h, w) or out.stride(2) != 1 or out.stride(1) != w
            or (n > 1 and out.stride(0) < h * w)):
        raise ValueError(f"out must be a uint8 ({n}, {h}, {w}) tensor with contiguous rows on {images.device}")


def _check_vec(v: torch.Tensor | None, n: int, device, name: str = "sse_out") -> None:
    """An int64 vector of n entries written at consecutive addresses."""
    if v is None:
        return
    if (not isinstance(v, torch.Tensor) or v.dtype != torch.int64 or v.device != device or v.dim() != 1
            or v.shape[0] != n or (n > 1 and v.stride(0) != 1)):
        raise ValueError(f"{name} must be a contiguous int64 tensor of {n} entries on {device}")


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _as_batch(images: torch.Tensor) -> torch.Tensor:
    if not isinstance(images, torch.Tensor):
        raise TypeError("images must be a torch tensor (use the codec wrappers for numpy input)")
    if images.dtype != torch.uint8:
        raise TypeError(f"images must be uint8, got {images.dtype}")
    if not images.is_cuda:
        raise ValueError("images must be on a CUDA device (no CPU path exists)")
    if images.dim() == 2:
        images = images.unsqueeze(0)
    if images.dim() != 3:
        raise BadDimensions(f"expected (N, H, W) images, got shape {tuple(images.shape)}")
    n, h, w = images.shape
    if h % 8 or w % 8:
        raise BadDimensions(f"image dimensions must be divisible by 8, got {(h, w)}")
    if images.stride(2) != 1 or images.stride(1) != w:
        images = images.contiguous()
    return images


def _img_stride(images: torch.Tensor) -> int:
    n, h, w = images.shape
    return images.stride(0) if n > 1 else h * w


@_device_guard
def forward_int(images: torch.Tensor, *, level_shift: bool = False, dtype=torch.int32,
                out: torch.Tensor | None = None) -> torch.Tensor:
    """K1: T X T^T of every 8x8 block, (N, H*W/64, 8, 8) in `_tile` order (codec.py:74-81, 107-109).
    `out` (contiguous, int32 or int16, that shape) is written in place when given."""
    images = _as_batch(images)
    n, h, w = images.shape
    shape = (n, (h // 8) * (w // 8), 8, 8)
    if out is None:
        out = torch.empty(shape, dtype=dtype, device=images.device)
    elif tuple(out.shape) != shape or not out.is_contiguous() or out.device != images.device:
        raise ValueError(f"out must be a contiguous {shape} tensor on {images.device}")
    dtype = out.dtype
    if dtype not in (torch.int32, torch.int16):
        raise ValueError("coefficients are int32 or int16")
    name = {torch.int32: "adct_forward_int32", torch.int16: "adct_forward_int16"}[dtype]
    _lib.call(name, _ptr(images), n, h, w, _img_stride(images), int(level_shift), _ptr(out), _stream())
    return out


@_device_guard
def compress_retain(
    images: torch.Tensor,
    r: int,
    *,
    reconstruct: bool = True,
    unrounded_sse: bool = False,
    out: torch.Tensor | None = None,
    sse_out: torch.Tensor | None = None,
):
    """K2+K4: fused retain-r round trip.  Returns (rec | None, sse[N] int64, sse_unrounded[N] | None).

    rec = clamp(round_half_away(C^T mask_r(C X C^T) C)) as uint8;
    sse[i] = sum (x - rec)^2 (exact);
    sse_unrounded[i] = 4096 * the reference's unrounded clamped SSE (exact).
    """
    if not 1 <= int(r) <= 64:
        raise InvalidRetention(f"retention count must be in [1, 64], got {r}")
    images = _as_batch(images)
    n, h, w = images.shape
    _check_out(out, images)
    _check_vec(sse_out, n, images.device)
    rec = None
    if reconstruct:
        rec = out if out is not None else torch.empty_like(images)
    sse = sse_out if sse_out is not None else torch.empty(n, dtype=torch.int64, device=images.device)
    ssef = torch.empty(n, dtype=torch.int64, device=images.device) if unrounded_sse else None
    _lib.call(
        "adct_compress_retain",
        _ptr(images), _ptr(rec), n, h, w, _img_stride(images), h * w if rec is None else _img_stride(rec),
        int(r), _ptr(sse), _ptr(ssef), _stream(),
    )
    return rec, sse, ssef


@_device_guard
def compress_retain_exchange(
    images: torch.Tensor,
    r: int,
    peers_dev: int,
    n_peers: int,
    peer_offset: int,
    arrivals: torch.Tensor,
    *,
    reconstruct: bool = True,
    out: torch.Tensor | None = None,
    sse_out: torch.Tensor | None = None,
):
    """compress_retain whose kernel epilogue also stores each image's exact SSE
    into every peer's vector: peers_dev is the device address of an array of
    n_peers device pointers (torch symmetric memory `buffer_ptrs_dev`), image i
    lands at index peer_offset + i.  `arrivals` is a zeroed int32 [N] scratch
    tensor that each call leaves zeroed.  Returns (rec | None, local sse[N])."""
    if not 1 <= int(r) <= 64:
        raise InvalidRetention(f"retention count must be in [1, 64], got {r}")
    images = _as_batch(images)
    n, h, w = images.shape
    if arrivals.dtype != torch.int32 or arrivals.numel() < n or arrivals.device != images.device:
        raise ValueError("arrivals must be an int32 tensor of >= N zeros on the images' device")
    _check_out(out, images)
    _check_vec(sse_out, n, images.device)
    rec = None
    if reconstruct:
        rec = out if out is not None else torch.empty_like(images)
    sse = sse_out if sse_out is not None else torch.empty(n, dtype=torch.int64, device=images.device)
    _lib.call(
        "adct_compress_retain_exchange",
        _ptr(images), _ptr(rec), n, h, w, _img_stride(images), h * w if rec is None else _img_stride(rec),
        int(r), _ptr(sse), int(peers_dev), int(n_peers), int(peer_offset), _ptr(arrivals), _stream(),
    )
    return rec, sse


@_device_guard
def compress_quant(
    images: torch.Tensor,
    qtab: _lib.QTab,
    *,
    reconstruct: bool = True,
    out: torch.Tensor | None = None,
    sse_out: torch.Tensor | None = None,
):
    """K3+K4: level shift, T X T^T, quantise by Q' (half away), dequantise,
    inverse, +128, round, clamp.  Returns (rec | None, sse[N] int64)."""
    images = _as_batch(images)
    n, h, w = images.shape
    _check_out(out, images)
    _check_vec(sse_out, n, images.device)
    rec = (out if out is not None else torch.empty_like(images)) if reconstruct else None
    sse = sse_out if sse_out is not None else torch.empty(n, dtype=torch.int64, device=images.device)
    _lib.call(
        "adct_compress_quant",
        _ptr(images), _ptr(rec), n, h, w, _img_stride(images), h * w if rec is None else _img_stride(rec),
        ctypes.byref(qtab), _ptr(sse), _stream(),
    )
    return rec, sse


def _planes(planes: Sequence[torch.Tensor], recs: Sequence[torch.Tensor | None]):
    if not 1 <= len(planes) <= 3:
        raise ValueError("1 to 3 planes")
    n = planes[0].shape[0]
    arr = (_lib.Plane * len(planes))()
    for k, (p, r) in enumerate(zip(planes, recs)):
        if p.dim() != 3 or p.shape[0] != n:
            raise DimensionMismatch("every plane needs shape (N, H, W) with the same N")
        if p.dtype != torch.uint8 or not p.is_cuda:
            raise TypeError("planes must be uint8 CUDA tensors")
        if not p.is_contiguous():
            raise ValueError("planes must be contiguous")
        _, h, w = p.shape
        if h % 8 or w % 8:
            raise BadDimensions(f"image dimensions must be divisible by 8, got {(h, w)}")
        if p.device != planes[0].device:
            raise ValueError("every plane must be on the same device")
        if r is not None and (not isinstance(r, torch.Tensor) or r.dtype != torch.uint8 or r.device != p.device
                              or r.shape != p.shape or not r.is_contiguous()):
            raise ValueError(f"plane {k}'s output must be a contiguous uint8 tensor shaped like the plane")
        arr[k].src = p.data_ptr()
        arr[k].dst = None if r is None else r.data_ptr()
        arr[k].height = h
        arr[k].width = w
        arr[k].src_frame_stride = h * w
        arr[k].dst_frame_stride = h * w
    return arr, n


@_device_guard
def compress_quant_planes(planes: Sequence[torch.Tensor], qtab: _lib.QTab, *, reconstruct: bool = True):
    """K6: all planes (e.g. Y, Cb, Cr of 4:2:0 frames) in one launch.
    Returns (list of rec | None, sse (N, n_planes) int64)."""
    recs = [torch.empty_like(p) if reconstruct else None for p in planes]
    arr, n = _planes(planes, recs)
    sse = torch.empty((n, len(planes)), dtype=torch.int64, device=planes[0].device)
    _lib.call("adct_compress_quant_planes", arr, len(planes), n, ctypes.byref(qtab), _ptr(sse), _stream())
    return recs, sse


@_device_guard
def compress_quant_planes_exchange(planes: Sequence[torch.Tensor], qtab: _lib.QTab, peers_dev: int, n_peers: int,
                                   peer_offset: int, arrivals: torch.Tensor, *, reconstruct: bool = True,
                                   out: Sequence[torch.Tensor] | None = None):
    """compress_quant_planes, then (same stream) each (frame, plane)'s exact
    SSE pushed into every peer's vector at peer_offset + frame * n_planes +
    plane (see compress_retain_exchange).  `arrivals` is accepted for symmetry
    and left untouched.  Returns (recs, local sse (N, n_planes))."""
    recs = list(out) if out is not None else [torch.empty_like(p) if reconstruct else None for p in planes]
    if len(recs) != len(planes):
        raise ValueError("one output per plane")
    arr, n = _planes(planes, recs)
    if arrivals.dtype != torch.int32 or arrivals.numel() < n * len(planes) or arrivals.device != planes[0].device:
        raise ValueError("arrivals must be an int32 tensor of >= N * n_planes zeros on the planes' device")
    sse = torch.empty((n, len(planes)), dtype=torch.int64, device=planes[0].device)
    _lib.call("adct_compress_quant_planes_exchange", arr, len(planes), n, ctypes.byref(qtab), _ptr(sse),
              int(peers_dev), int(n_peers), int(peer_offset), _ptr(arrivals), _stream())
    return recs, sse


@_device_guard
def compress_retain_planes(planes: Sequence[torch.Tensor], r: int, *, reconstruct: bool = True):
    if not 1 <= int(r) <= 64:
        raise InvalidRetention(f"retention count must be in [1, 64], got {r}")
    recs = [torch.empty_like(p) if reconstruct else None for p in planes]
    arr, n = _planes(planes, recs)
    sse = torch.empty((n, len(planes)), dtype=torch.int64, device=planes[0].device)
    _lib.call("adct_compress_retain_planes", arr, len(planes), n, int(r), _ptr(sse), _stream())
    return recs, sse


@_device_guard
def sweep_retain_sse(images: torch.Tensor, r_min: int = 1, r_max: int = 45) -> torch.Tensor:
    """K7: SSE[N, r_max-r_min+1] for every r, one read of each image (cli.py:101-113)."""
    if not (1 <= r_min <= r_max <= 64):
        raise InvalidRetention(f"retention range must satisfy 1 <= r_min <= r_max <= 64, got {r_min}..{r_max}")
    images = _as_batch(images)
    n, h, w = images.shape
    sse = torch.empty((n, r_max - r_min + 1), dtype=torch.int64, device=images.device)
    _lib.call("adct_sweep_retain_sse", _ptr(images), n, h, w, _img_stride(images), r_min, r_max, _ptr(sse), None,
              _stream())
    return sse


@_device_guard
def sse_u8(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """Per-image integer SSE of two uint8 CUDA batches (N, ...) -> int64[N]."""
    if a.shape != b.shape:
        raise DimensionMismatch(f"shape mismatch: {tuple(a.shape)} vs {tuple(b.shape)}")
    a = a.contiguous()
    b = b.contiguous()
    n = a.shape[0] if a.dim() > 0 else 1
    numel = a.numel() // max(n, 1) if n else 0
    sse = torch.empty(n, dtype=torch.int64, device=a.device)
    _lib.call("adct_sse_u8", _ptr(a), _ptr(b), n, numel, numel, numel, _ptr(sse), _stream())
    return sse


@_device_guard
def forward_f64(images: torch.Tensor) -> torch.Tensor:
    """C X C^T per block in float64 (forward_2d / coefficient_blocks, codec.py:68-71, 120-131)."""
    if images.dim() == 2:
        images = images.unsqueeze(0)
    if images.dim() != 3:
        raise BadDimensions(f"expected (N, H, W), got {tuple(images.shape)}")
    n, h, w = images.shape
    if h % 8 or w % 8:
        raise BadDimensions(f"image dimensions must be divisible by 8, got {(h, w)}")
    u8 = images.dtype == torch.uint8  # read as bytes by the kernel, no float64 copy
    x = images.contiguous() if u8 else images.to(dtype=torch.float64).contiguous()
    coef = torch.empty((n, (h // 8) * (w // 8), 8, 8), dtype=torch.float64, device=x.device)
    _lib.call("adct_forward_f64_u8" if u8 else "adct_forward_f64", _ptr(x), n, h, w, _ptr(coef), _stream())
    return coef


@_device_guard
def inverse_f64(coef: torch.Tensor, h: int, w: int, *, r: int = 64, clamp: bool = False) -> torch.Tensor:
    """untile(C^T mask_r(Y) C), optionally clamped (inverse_2d / reconstruct_image)."""
    if not 1 <= int(r) <= 64:
        raise InvalidRetention(f"retention count must be in [1, 64], got {r}")
    if h % 8 or w % 8:
        raise BadDimensions(f"image dimensions must be divisible by 8, got {(h, w)}")
    nb = (h // 8) * (w // 8)
    c = coef.to(dtype=torch.float64).contiguous()
    if c.numel() % (64 * max(nb, 1)) or (nb and c.numel() // 64 % nb):
        raise BadDimensions(f"coefficients {tuple(coef.shape)} do not tile a {h}x{w} image")
    n = c.numel() // (64 * nb) if nb else 0
    out = torch.empty((n, h, w), dtype=torch.float64, device=c.device)
    _lib.call("adct_inverse_f64", _ptr(c), n, h, w, int(r), int(clamp), _ptr(out), _stream())
    return out


def psnr_from_sse(sse, n_pixels: int, *, scale: float = 1.0) -> np.ndarray:
    """10 log10(255^2 / (sse / (scale * n_pixels))), inf at 0 (metrics.py:59-65)."""
    s = np.asarray(sse.cpu() if isinstance(sse, torch.Tensor) else sse, dtype=np.float64)
    mse = s / (scale * float(n_pixels))
    with np.errstate(divide="ignore"):
        return np.where(mse == 0, np.inf, 10.0 * np.log10(255.0**2 / np.where(mse == 0, 1.0, mse)))


# --- dense float64 transforms for any 8x8 matrix (exact DCT, registry kernels) ---

def _cmat(C) -> "ctypes.Array":
    a = np.ascontiguousarray(np.asarray(C, dtype=np.float64).reshape(64))
    if a.size != 64:
        raise BadDimensions("transform matrix must be 8x8")
    return (ctypes.c_double * 64)(*a.tolist())


def _f64_or_u8(images: torch.Tensor):
    if images.dim() == 2:
        images = images.unsqueeze(0)
    if images.dim() != 3:
        raise BadDimensions(f"expected (N, H, W), got {tuple(images.shape)}")
    n, h, w = images.shape
    if h % 8 or w % 8:
        raise BadDimensions(f"image dimensions must be divisible by 8, got {(h, w)}")
    if images.dtype == torch.uint8:
        return images.contiguous(), 0
    return images.to(torch.float64).contiguous(), 1


@_device_guard
def forward_dense(images: torch.Tensor, C) -> torch.Tensor:
    """Y = C X C^T per block for any 8x8 C, float64 (coefficient_blocks, codec.py:120-131)."""
    x, f64 = _f64_or_u8(images)
    n, h, w = x.shape
    coef = torch.empty((n, (h // 8) * (w // 8), 8, 8), dtype=torch.float64, device=x.device)
    _lib.call("adct_forward_dense", _ptr(x), f64, n, h, w, _cmat(C), _ptr(coef), _stream())
    return coef


@_device_guard
def inverse_dense(coef: torch.Tensor, h: int, w: int, C, *, r: int = 64, clamp: bool = False) -> torch.Tensor:
    """untile(C^T mask_r(Y) C), optionally clamped (reconstruct_image, codec.py:134-141)."""
    if not 1 <= int(r) <= 64:
        raise InvalidRetention(f"retention count must be in [1, 64], got {r}")
    if h % 8 or w % 8:
        raise BadDimensions(f"image dimensions must be divisible by 8, got {(h, w)}")
    nb = (h // 8) * (w // 8)
    c = coef.to(torch.float64).contiguous()
    n = c.numel() // (64 * nb) if nb else 0
    out = torch.empty((n, h, w), dtype=torch.float64, device=c.device)
    _lib.call("adct_inverse_dense", _ptr(c), n, h, w, _cmat(C), int(r), int(clamp), _ptr(out), _stream())
    return out


@_device_guard
def sweep_dense_sse(images: torch.Tensor, C, r_min: int, r_max: int) -> torch.Tensor:
    """float64 SSE[N, r] of the reference's unrounded, clamped reconstructions for any C."""
    if not (1 <= r_min <= r_max <= 64):
        raise InvalidRetention(f"retention range must satisfy 1 <= r_min <= r_max <= 64, got {r_min}..{r_max}")
    x, f64 = _f64_or_u8(images)
    n, h, w = x.shape
    sse = torch.empty((n, r_max - r_min + 1), dtype=torch.float64, device=x.device)
    _lib.call("adct_sweep_dense", _ptr(x), f64, n, h, w, _cmat(C), r_min, r_max, _ptr(sse), _stream())
    return sse


@_device_guard
def sweep_retain_sse_unrounded(images: torch.Tensor, r_min: int = 1, r_max: int = 45, *, rounded: bool = True):
    """(rounded SSE, 4096 x unrounded SSE), both int64[N, r] — exact.
    rounded=False skips the rounded SSE (returned as None), which is all the
    reference's own convention (run_sweep) needs."""
    if not (1 <= r_min <= r_max <= 64):
        raise InvalidRetention(f"retention range must satisfy 1 <= r_min <= r_max <= 64, got {r_min}..{r_max}")
    images = _as_batch(images)
    n, h, w = images.shape
    ssef = torch.empty((n, r_max - r_min + 1), dtype=torch.int64, device=images.device)
    sse = torch.empty_like(ssef) if rounded else None
    _lib.call("adct_sweep_retain_sse", _ptr(images), n, h, w, _img_stride(images), r_min, r_max, _ptr(sse),
              _ptr(ssef), _stream())
    return sse, ssef
