"""Drop-in mirror of the reference codec API (adct/codec.py:24-155).

Same names, argument meaning, return types and contract errors.  Arrays are
numpy (as in the reference) or torch tensors; numpy inputs are copied to the
GPU, computed there by libadct_cuda.so and copied back.  There is no CPU
compute path: a missing library or GPU raises.

Routing:
* `forward_2d_unscaled` on 8-bit-range integers -> K1 exact integer kernel;
  any other real input -> the dense float64 kernel with K (exact for
  integers).  Device tensors choose by dtype (uint8), never by scanning
  values, so no call synchronises the host with the GPU.
* `forward_2d`, `inverse_2d`, `coefficient_blocks`, `reconstruct_image`,
  `compress_image` keep the reference's float64 semantics (unrounded,
  clamped) -> float64 flow-graph kernels (agree with the reference's dense
  float64 matmuls to ~1e-13).
* The batched, rounded uint8 hot path is `batch.compress_retain` /
  `batch.compress_quant` (exact integer pipeline).
Any other `Transform` (the exact DCT, the reference registry's comparison
kernels — anything with an 8x8 `.matrix`) runs on the dense float64 8x8
kernels (adct_*_dense).
"""

from __future__ import annotations

import warnings
from functools import lru_cache

import numpy as np
import torch

from . import batch
from .errors import BadDimensions, InvalidRetention
from .quant import fold_scaling_into_quantization  # noqa: F401  (re-export, codec.py:90)
from .transforms import is_proposed

_ZZ_CACHE: tuple[int, ...] | None = None


def _zigzag() -> tuple[int, ...]:
    """JPEG zigzag scan as flat row-major indices: anti-diagonals u+v = s,
    odd s with increasing row, even s with decreasing row."""
    order = []
    for s in range(15):
        rows = list(range(max(0, s - 7), min(s, 7) + 1))
        if s % 2 == 0:
            rows.reverse()
        order += [u * 8 + (s - u) for u in rows]
    return tuple(order)


#: Standard JPEG zigzag scan (codec.py:24-33), generated, not typed.
ZIGZAG_INDICES: tuple[int, ...] = _zigzag()


def zigzag_positions() -> tuple[tuple[int, int], ...]:
    return tuple((i // 8, i % 8) for i in ZIGZAG_INDICES)


@lru_cache(maxsize=None)
def retention_mask(r: int) -> np.ndarray:
    """Boolean 8x8 mask of the first r zigzag positions (codec.py:41-50)."""
    if not 1 <= r <= 64:
        raise InvalidRetention(f"retention count must be in [1, 64], got {r}")
    mask = np.zeros(64, dtype=bool)
    mask[list(ZIGZAG_INDICES[:r])] = True
    mask = mask.reshape(8, 8)
    mask.setflags(write=False)
    return mask


def retain_coefficients(block, r: int) -> np.ndarray:
    """Zero all but the first r zigzag coefficients (codec.py:53-58)."""
    block = np.asarray(block, dtype=np.float64)
    if block.shape != (8, 8):
        raise BadDimensions(f"expected an 8x8 block, got {block.shape}")
    return np.where(retention_mask(r), block, 0.0)


def compression_ratio(r: int) -> float:
    """100 (64 - r) / 64 (codec.py:61-65)."""
    if not 1 <= r <= 64:
        raise InvalidRetention(f"retention count must be in [1, 64], got {r}")
    return 100.0 * (64 - r) / 64


# --- device plumbing ----------------------------------------------------------

def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1702_00817_b200 computes on CUDA only; no GPU is visible")
    return torch.device("cuda", torch.cuda.current_device())


def _image_dtype(a) -> torch.dtype:
    """uint8 images travel and are read as bytes (1/8 of the float64 copy the
    reference makes, codec.py:127); anything else as float64."""
    if isinstance(a, torch.Tensor):
        return torch.uint8 if a.dtype == torch.uint8 else torch.float64
    return torch.uint8 if np.asarray(a).dtype == np.uint8 else torch.float64


def _to_dev(a, dtype=None) -> tuple[torch.Tensor, bool]:
    """(tensor on device, was_numpy)."""
    if isinstance(a, torch.Tensor):
        t = a if a.is_cuda else a.to(_device())
        return (t if dtype is None else t.to(dtype)), False
    t = _host_tensor(a).to(_device())
    return (t if dtype is None else t.to(dtype)), True


def _host_tensor(a) -> torch.Tensor:
    """A CPU tensor viewing numpy data.  Read-only arrays (the reference
    freezes its image samples) are viewed as they are: the view is only read
    (copied to the device), so torch's non-writable warning does not apply."""
    arr = np.ascontiguousarray(np.asarray(a))
    if arr.flags.writeable:
        return torch.from_numpy(arr)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)
        return torch.from_numpy(arr)


def _back(t: torch.Tensor, to_numpy: bool):
    if to_numpy:
        torch.cuda.current_stream().synchronize()
        return t.cpu().numpy()
    return t


def _matrix(t) -> np.ndarray:
    m = np.asarray(getattr(t, "matrix"), dtype=np.float64)
    if m.shape != (8, 8):
        raise BadDimensions(f"transform matrix must be 8x8, got {m.shape}")
    return m


def _is_u8_range_integral(a) -> bool:
    """Whether `a` can take the exact 8-bit integer kernel.  Device tensors
    decide by dtype alone (a value scan would be a device-wide reduction and a
    host sync on every call); other device dtypes take the dense float64
    kernel, exact for integer values.  Host arrays are scanned on the host."""
    if isinstance(a, torch.Tensor):
        return a.dtype == torch.uint8
    a = np.asarray(a)
    if a.dtype == np.uint8:
        return True
    if a.dtype.kind == "f":
        return bool(np.all((a == np.round(a)) & (a >= 0) & (a <= 255)))
    if a.dtype.kind in "iub":
        return bool(np.all((a >= 0) & (a <= 255)))
    return False


def _blocks_as_images(block) -> tuple[object, tuple]:
    shape = tuple(block.shape)
    if len(shape) < 2 or shape[-2:] != (8, 8):
        raise BadDimensions(f"expected (..., 8, 8) blocks, got {shape}")
    lead = shape[:-2]
    n = int(np.prod(lead)) if lead else 1
    return block.reshape(n, 8, 8), lead


# --- reference API ------------------------------------------------------------

def forward_2d(t, block):
    """C B C^T (codec.py:68-71), float64, over (..., 8, 8)."""
    x, was_np = _to_dev(block, _image_dtype(block))
    xs, lead = _blocks_as_images(x)
    y = batch.forward_f64(xs) if is_proposed(t) else batch.forward_dense(xs, _matrix(t))
    return _back(y.reshape(*lead, 8, 8) if lead else y.reshape(8, 8), was_np)


def forward_2d_unscaled(t, block):
    """K B K^T without the diagonal scaling (codec.py:74-81); integer-exact.
    8-bit integer blocks of the proposed kernel take K1 (exact integer
    flow graph); anything else the dense float64 kernel with K itself (exact
    for integer values, the reference's own product otherwise)."""
    integral_in = (block.dtype.kind in "iub") if not isinstance(block, torch.Tensor) else not block.dtype.is_floating_point
    if is_proposed(t) and _is_u8_range_integral(block):
        x, was_np = _to_dev(block, torch.uint8)
        xs, lead = _blocks_as_images(x)
        z = batch.forward_int(xs).reshape(*lead, 8, 8) if lead else batch.forward_int(xs).reshape(8, 8)
        z = z.to(torch.int64) if integral_in else z.to(torch.float64)
        return _back(z, was_np)
    k = np.asarray(t.kernel.entries, dtype=np.float64)
    x, was_np = _to_dev(block, torch.float64)
    xs, lead = _blocks_as_images(x)
    z = batch.forward_dense(xs, k)
    z = z.reshape(*lead, 8, 8) if lead else z.reshape(8, 8)
    return _back(torch.round(z).to(torch.int64) if integral_in else z, was_np)


def inverse_2d(t, coeffs):
    """C^T Y C (codec.py:84-87), float64, over (..., 8, 8)."""
    y, was_np = _to_dev(coeffs, torch.float64)
    ys, lead = _blocks_as_images(y)
    if is_proposed(t):
        x = batch.inverse_f64(ys.reshape(-1, 1, 8, 8), 8, 8, r=64, clamp=False)
    else:
        x = batch.inverse_dense(ys.reshape(-1, 1, 8, 8), 8, 8, _matrix(t), r=64, clamp=False)
    x = x.reshape(*lead, 8, 8) if lead else x.reshape(8, 8)
    return _back(x, was_np)


def coefficient_blocks(t, image):
    """Forward-transform every 8x8 tile; (n_blocks, 8, 8) float64 in raster block order (codec.py:120-131)."""
    shape = tuple(image.shape)
    if len(shape) != 2 or shape[0] % 8 or shape[1] % 8:
        raise BadDimensions(f"image dimensions must be divisible by 8, got {shape}")
    x, was_np = _to_dev(image, _image_dtype(image))
    c = batch.forward_f64(x.unsqueeze(0)) if is_proposed(t) else batch.forward_dense(x.unsqueeze(0), _matrix(t))
    return _back(c[0], was_np)


def reconstruct_image(t, coeffs, r: int, height: int, width: int):
    """Inverse of the first r zigzag coefficients, untiled and clamped to [0,255] (codec.py:134-141)."""
    if not 1 <= r <= 64:
        raise InvalidRetention(f"retention count must be in [1, 64], got {r}")
    c, was_np = _to_dev(coeffs, torch.float64)
    c = c.reshape(1, -1, 8, 8)
    if is_proposed(t):
        out = batch.inverse_f64(c, int(height), int(width), r=int(r), clamp=True)[0]
    else:
        out = batch.inverse_dense(c, int(height), int(width), _matrix(t), r=int(r), clamp=True)[0]
    return _back(out, was_np)


def compress_image(t, image, r: int):
    """Forward, keep r zigzag coefficients, inverse, clamp (codec.py:144-155); float64, unrounded."""
    if not 1 <= r <= 64:
        raise InvalidRetention(f"retention count must be in [1, 64], got {r}")
    shape = tuple(image.shape)
    if len(shape) != 2 or shape[0] % 8 or shape[1] % 8:
        raise BadDimensions(f"image dimensions must be divisible by 8, got {shape}")
    m = None if is_proposed(t) else _matrix(t)
    x, was_np = _to_dev(image, _image_dtype(image))
    if m is None:
        c = batch.forward_f64(x.unsqueeze(0))
        out = batch.inverse_f64(c, shape[0], shape[1], r=int(r), clamp=True)[0]
    else:
        c = batch.forward_dense(x.unsqueeze(0), m)
        out = batch.inverse_dense(c, shape[0], shape[1], m, r=int(r), clamp=True)[0]
    return _back(out, was_np)
