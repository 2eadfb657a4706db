"""Mirror of the reference metrics API (adct/metrics.py:24-97).

`mse` runs on the GPU (exact integer SSE for uint8 inputs via adct_sse_u8,
float64 reduction otherwise); `psnr`, `ape_vs_dct` and `summarize` are host
arithmetic on scalars, exactly as in the reference.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Iterable

import numpy as np
import torch

from . import batch
from .errors import DimensionMismatch, EmptyGroup

PEAK = 255.0


@dataclass(frozen=True)
class QualityRecord:
    image_id: str
    transform_name: str
    r: int
    mse: float
    psnr: float


@dataclass(frozen=True)
class CorpusSummary:
    transform_name: str
    r: int
    avg_mse: float
    avg_psnr: float
    n_images: int


def _device_pair(a, b):
    dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else None
    if dev is None:
        raise RuntimeError("paper_1702_00817_b200 computes on CUDA only; no GPU is visible")

    def conv(x):
        if isinstance(x, torch.Tensor):
            return x.to(dev)
        return torch.from_numpy(np.ascontiguousarray(np.asarray(x))).to(dev)

    return conv(a), conv(b)


def mse(original, reconstructed) -> float:
    """mean((o - r)^2) as float (metrics.py:49-56)."""
    oshape = tuple(np.shape(original)) if not isinstance(original, torch.Tensor) else tuple(original.shape)
    rshape = tuple(np.shape(reconstructed)) if not isinstance(reconstructed, torch.Tensor) else tuple(reconstructed.shape)
    if oshape != rshape:
        raise DimensionMismatch(f"shape mismatch: {oshape} vs {rshape}")
    a, b = _device_pair(original, reconstructed)
    n = a.numel()
    if n == 0:
        return float("nan")
    if a.dtype == torch.uint8 and b.dtype == torch.uint8:
        sse = batch.sse_u8(a.reshape(1, -1), b.reshape(1, -1))
        return float(sse.item()) / n
    d = a.to(torch.float64) - b.to(torch.float64)
    return float((d * d).mean().item())


def psnr(mse_value: float) -> float:
    """10 log10(255^2 / mse); inf at 0 (metrics.py:59-65)."""
    if mse_value < 0:
        raise ValueError("mse cannot be negative")
    if mse_value == 0:
        return math.inf
    return 10.0 * math.log10(PEAK**2 / mse_value)


def ape_vs_dct(avg_mse_approx: float, avg_mse_dct: float) -> float:
    if avg_mse_dct == 0:
        raise ZeroDivisionError("reference average MSE is zero")
    return 100.0 * abs(avg_mse_approx - avg_mse_dct) / avg_mse_dct


def summarize(records: Iterable[QualityRecord], *, psnr_from_avg_mse: bool = False) -> list[CorpusSummary]:
    """Per-(transform, r) averages; avg_psnr is the mean of per-image PSNRs by default (metrics.py:75-97)."""
    groups: dict[tuple[str, int], list[QualityRecord]] = {}
    for rec in records:
        groups.setdefault((rec.transform_name, rec.r), []).append(rec)
    if not groups:
        raise EmptyGroup("no records to summarize")
    out = []
    for name, r in sorted(groups):
        members = groups[(name, r)]
        avg_mse = float(np.mean([m.mse for m in members]))
        avg_psnr = psnr(avg_mse) if psnr_from_avg_mse else float(np.mean([m.psnr for m in members]))
        out.append(CorpusSummary(name, r, avg_mse, avg_psnr, len(members)))
    return out
