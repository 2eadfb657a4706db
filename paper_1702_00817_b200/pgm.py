"""PGM ingestion straight into page-locked batch buffers.

The reference reads one PGM at a time into float64 samples
(corpus.read_pgm, corpus.py:65-111).  Here a whole corpus of P5 files is read
with `readinto` directly into one page-locked uint8 (N, H, W) buffer — no
float conversion, no intermediate copy — which the host pipeline then streams
through the GPU (H2D overlapped with compute and D2H).  Header parsing and
the contract errors follow the reference: P2/P5 magic, whitespace and '#'
comments, maxval in (0, 255], exactly one whitespace byte before a P5 raster,
TruncatedData on short rasters, samples above maxval rejected.
"""

from __future__ import annotations

import os
from pathlib import Path
from typing import Sequence

import numpy as np

from .errors import BadDimensions, IoFailure, MalformedHeader, TruncatedData, UnsupportedMaxval

_WS = b" \t\r\n"


def _tokens(data: bytes, start: int = 0):
    i, n = start, len(data)
    while i < n:
        c = data[i : i + 1]
        if c in _WS:
            i += 1
        elif c == b"#":
            while i < n and data[i : i + 1] not in b"\r\n":
                i += 1
        else:
            j = i
            while j < n and data[j : j + 1] not in _WS + b"#":
                j += 1
            yield data[i:j], j
            i = j


def parse_header(data: bytes) -> tuple[bytes, int, int, int, int]:
    """(magic, width, height, maxval, offset just past the header's last token)."""
    tok = _tokens(data)
    try:
        magic, _ = next(tok)
    except StopIteration:
        raise MalformedHeader("empty file") from None
    if magic not in (b"P2", b"P5"):
        raise MalformedHeader(f"not a PGM file (magic {magic!r})")
    vals, end = [], 0
    for _ in range(3):
        try:
            t, end = next(tok)
            vals.append(int(t))
        except StopIteration:
            raise MalformedHeader("header ended early") from None
        except ValueError:
            raise MalformedHeader(f"non-integer header token {t!r}") from None
    w, h, maxval = vals
    if w <= 0 or h <= 0:
        raise MalformedHeader(f"bad dimensions {w}x{h}")
    if not 0 < maxval <= 255:
        raise UnsupportedMaxval(f"maxval {maxval} outside (0, 255]")
    return magic, w, h, maxval, end


def read_pgm_u8(path: str | os.PathLike, out: np.ndarray | None = None) -> np.ndarray:
    """One PGM as uint8 (H, W); P5 rasters are read straight into `out`."""
    with open(path, "rb") as f:
        head = f.read(4096)
        magic, w, h, maxval, end = parse_header(head)
        if out is None:
            out = np.empty((h, w), dtype=np.uint8)
        elif out.shape != (h, w) or out.dtype != np.uint8:
            raise BadDimensions(f"{path}: {h}x{w} does not fit the batch slot {out.shape}")
        if magic == b"P5":
            f.seek(end + 1)  # exactly one whitespace byte before the raster
            got = f.readinto(memoryview(out).cast("B"))
            if got < w * h:
                raise TruncatedData(f"expected {w * h} bytes, found {got}")
        else:
            data = head + f.read()
            vals = []
            for t, _ in _tokens(data, end):
                try:
                    vals.append(int(t))
                except ValueError:
                    raise MalformedHeader(f"non-integer sample {t!r}") from None
                if len(vals) == w * h:
                    break
            if len(vals) < w * h:
                raise TruncatedData(f"expected {w * h} samples, found {len(vals)}")
            arr = np.asarray(vals, dtype=np.int64)
            if arr.max(initial=0) > 255:
                raise MalformedHeader("sample exceeds declared maxval")
            out[...] = arr.reshape(h, w)
    if maxval < 255 and int(out.max(initial=0)) > maxval:
        raise MalformedHeader("sample exceeds declared maxval")
    return out


def load_batch(paths: Sequence[str | os.PathLike], *, pinned: bool = True) -> np.ndarray:
    """All files (same size) into one (N, H, W) uint8 buffer; when `pinned`,
    the buffer is page-locked host memory (pipeline.pinned_empty, freed with
    the array) that the host pipeline streams at the PCIe limit."""
    if not paths:
        raise ValueError("no files")
    with open(paths[0], "rb") as f:
        _, w, h, _, _ = parse_header(f.read(4096))
    if pinned:
        from .pipeline import pinned_empty

        batch = pinned_empty((len(paths), h, w))
    else:
        batch = np.empty((len(paths), h, w), dtype=np.uint8)
    for k, p in enumerate(paths):
        read_pgm_u8(p, batch[k])
    return batch


def write_pgm_u8(image: np.ndarray, path: str | os.PathLike) -> None:
    """P5, maxval 255 (corpus.write_pgm, corpus.py:114-121, for uint8 samples)."""
    img = np.asarray(image)
    if img.dtype != np.uint8:
        img = np.floor(img.astype(np.float64) + 0.5).clip(0, 255).astype(np.uint8)
    h, w = img.shape
    try:
        with open(path, "wb") as f:
            f.write(f"P5\n{w} {h}\n255\n".encode("ascii"))
            f.write(np.ascontiguousarray(img).tobytes())
    except OSError as exc:
        raise IoFailure(f"cannot write {path}: {exc}") from exc


def compress_files(paths: Sequence[str | os.PathLike], r: int, out_dir: str | os.PathLike | None = None,
                   device: int = 0, chunk_bytes: int = 16 << 20):
    """End to end: PGM files -> pinned batch -> GPU retain-r -> per-file (mse, psnr)
    of the rounded reconstruction; optionally writes the reconstructions."""
    from .metrics import psnr
    from .pipeline import HostPipeline, pinned_empty

    imgs = load_batch(paths, pinned=True)
    rec = pinned_empty(imgs.shape)
    with HostPipeline(device, chunk_bytes=chunk_bytes) as p:
        _, sse = p.compress_retain(imgs, r, rec, register=False)
    n_px = imgs.shape[1] * imgs.shape[2]
    results = []
    for k, path in enumerate(paths):
        m = float(sse[k]) / n_px
        results.append((Path(path).stem, m, psnr(m)))
        if out_dir is not None:
            Path(out_dir).mkdir(parents=True, exist_ok=True)
            write_pgm_u8(rec[k], Path(out_dir) / (Path(path).stem + f"_r{r}.pgm"))
    return results


# --- reference-shaped API (corpus.py:26-121) ------------------------------------

class GrayImage:
    """8-bit-valued grayscale image with float64 samples (corpus.py:26-43)."""

    def __init__(self, width: int, height: int, samples) -> None:
        if width <= 0 or height <= 0:
            raise ValueError("image dimensions must be positive")
        s = np.array(samples, dtype=np.float64).reshape(height, width)
        if not np.isfinite(s).all():
            raise ValueError("samples must be finite")
        if s.min() < 0 or s.max() > 255:
            raise ValueError("samples must lie in [0, 255]")
        s.setflags(write=False)
        self.width, self.height, self.samples = width, height, s


def read_pgm(path) -> GrayImage:
    """P2/P5 PGM -> GrayImage (corpus.read_pgm contract)."""
    u8 = read_pgm_u8(path)
    return GrayImage(u8.shape[1], u8.shape[0], u8)


def write_pgm(image: GrayImage, path) -> None:
    """P5, maxval 255, samples rounded half away from zero (corpus.write_pgm)."""
    write_pgm_u8(np.floor(np.asarray(image.samples) + 0.5).astype(np.uint8), path)
