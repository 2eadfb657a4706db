"""Mirror of the reference metrics API (adct/metrics.py:24-97).

`mse` runs on the GPU (exact integer SSE for uint8 inputs via adct_sse_u8,
float64 reduction otherwise); `psnr`, `ape_vs_dct` and `summarize` are host
arithmetic on scalars with the reference's results; the CSV writers produce
the reference's report format.
"""

from __future__ import annotations

import csv
import math
from collections import defaultdict
from dataclasses import dataclass
from typing import Iterable, TextIO

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
        from .codec import _host_tensor

        return _host_tensor(x).to(dev)

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
    """One CorpusSummary per (transform, r), in key order (metrics.py:75-97).
    avg_psnr is the mean of the per-image PSNRs, or with psnr_from_avg_mse
    the PSNR of avg_mse; EmptyGroup when there is nothing to average."""
    by_key: dict[tuple[str, int], list[QualityRecord]] = defaultdict(list)
    for rec in records:
        by_key[rec.transform_name, rec.r].append(rec)
    if not by_key:
        raise EmptyGroup("no records to summarize")
    out = []
    for key in sorted(by_key):
        mses = np.array([m.mse for m in by_key[key]], dtype=np.float64)
        psnrs = np.array([m.psnr for m in by_key[key]], dtype=np.float64)
        avg_mse = float(mses.mean())
        out.append(CorpusSummary(key[0], key[1], avg_mse,
                                 psnr(avg_mse) if psnr_from_avg_mse else float(psnrs.mean()), len(mses)))
    return out


# --- CSV reports (metrics.py:100-122): same columns, order and number format ---

def format_float(x: float) -> str:
    """%.6g ('inf' for a lossless PSNR)."""
    return f"{x:.6g}"


_RECORD_COLUMNS = (("image_id", lambda m: m.image_id), ("transform", lambda m: m.transform_name),
                   ("r", lambda m: m.r), ("mse", lambda m: format_float(m.mse)),
                   ("psnr", lambda m: format_float(m.psnr)))
_SUMMARY_COLUMNS = (("transform", lambda s: s.transform_name), ("r", lambda s: s.r),
                    ("avg_mse", lambda s: format_float(s.avg_mse)), ("avg_psnr", lambda s: format_float(s.avg_psnr)),
                    ("n_images", lambda s: s.n_images))


def _write_table(fp: TextIO, columns, rows, key) -> None:
    w = csv.writer(fp, lineterminator="\n")
    w.writerow([name for name, _ in columns])
    w.writerows([[get(row) for _, get in columns] for row in sorted(rows, key=key)])


def write_quality_csv(fp: TextIO, records: Iterable[QualityRecord]) -> None:
    """Per-image records sorted by (transform, r, image_id)."""
    _write_table(fp, _RECORD_COLUMNS, records, key=lambda m: (m.transform_name, m.r, m.image_id))


def write_summary_csv(fp: TextIO, summaries: Iterable[CorpusSummary]) -> None:
    """Per-(transform, r) summaries sorted by (transform, r)."""
    _write_table(fp, _SUMMARY_COLUMNS, summaries, key=lambda s: (s.transform_name, s.r))
