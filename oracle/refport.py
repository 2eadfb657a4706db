"""float64 restatement of the reference's own code path (TEST INFRASTRUCTURE /
CPU BASELINE ONLY — see oracle/__init__.py).

This is the algorithm of codec.py:120-155 and metrics.py:49-65 as the
reference runs it: dense float64 matrices C = D T (kernels.py:121-124), two
stacked matmuls per direction, np.where masking, clip.  bench.py times it as
the reference CPU arm ("port"): /root/reference cannot travel to the GPU box.
"""

from __future__ import annotations

import math

import numpy as np

from .exact import T, retention_mask, tile, untile

_S8, _S2 = 1 / math.sqrt(8), 1 / math.sqrt(2)
D = np.array([_S8, _S2, 0.5, _S2, _S8, _S2, 0.5, _S2])  # kernels.py:157
C = D[:, None] * T  # ApproximateTransform.matrix, kernels.py:121-124


def coefficient_blocks(image: np.ndarray) -> np.ndarray:
    """codec.py:120-131."""
    return C @ tile(np.asarray(image, dtype=np.float64)) @ C.T


def reconstruct_image(coeffs: np.ndarray, r: int, h: int, w: int) -> np.ndarray:
    """codec.py:134-141 (mask, C^T Y C, untile, clip; no rounding)."""
    kept = np.where(retention_mask(r).astype(bool), coeffs, 0.0)
    return np.clip(untile(C.T @ kept @ C, h, w), 0.0, 255.0)


def compress_image(image: np.ndarray, r: int) -> np.ndarray:
    """codec.py:144-155."""
    image = np.asarray(image, dtype=np.float64)
    return reconstruct_image(coefficient_blocks(image), r, *image.shape)


def mse(a, b) -> float:
    """metrics.py:49-56."""
    return float(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2))


def psnr(m: float) -> float:
    """metrics.py:59-65."""
    return math.inf if m == 0 else 10.0 * math.log10(255.0**2 / m)


def compress_rounded(image: np.ndarray, r: int) -> np.ndarray:
    """Reference float64 output snapped to the 1/64 grid, then rounded half away
    and clamped (BASELINE config 1 'round and clamp').  The snap makes ties
    deterministic: the float64 path lands within 2e-13 of k/64."""
    y = compress_image(image, r)
    k = np.round(y * 64.0)
    assert np.abs(y * 64.0 - k).max() < 1e-6
    return np.clip(np.floor((k + 32) / 64), 0, 255).astype(np.uint8)


def image_quality(image: np.ndarray, r: int) -> tuple[float, float]:
    """(mse, psnr) of one image under the reference's own convention."""
    rec = compress_image(image, r)
    m = mse(image, rec)
    return m, psnr(m)


def quant_float64(image: np.ndarray, Qp: np.ndarray) -> np.ndarray:
    """Quantised pipeline composed from the reference's float64 functions:
    forward_2d_unscaled (codec.py:74-81) of X-128, divide by Q', round half
    away, multiply, inverse_2d (codec.py:84-87) of the rescaled coefficients
    D Z' D, +128, round half away, clamp.  Used to show exact.compress_quant
    differs from the float composition only at exact .5 ties."""
    x = tile(np.asarray(image, dtype=np.float64)) - 128.0
    Z = T.astype(np.float64) @ x @ T.T.astype(np.float64)
    q = np.sign(Z) * np.floor(np.abs(Z) / Qp + 0.5)
    Y = np.outer(D, D) * (q * Qp)
    xr = C.T @ Y @ C + 128.0
    h, w = np.asarray(image).shape
    return untile(xr, h, w)
