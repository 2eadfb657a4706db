"""PGM ingestion straight into page-locked batch buffers.

The reference reads one PGM at a time into float64 samples
(corpus.read_pgm, corpus.py:65-111).  Here a whole corpus of P5 files is read
with `readinto` directly into one page-locked uint8 (N, H, W) buffer — no
float conversion, no intermediate copy — which the host pipeline then streams
through the GPU (H2D overlapped with compute and D2H).  Header parsing and
the contract error classes follow the reference (P2/P5 magic, whitespace and
'#' comments, maxval in (0, 255], exactly one whitespace byte before a P5
raster, TruncatedData on short rasters, samples above maxval rejected).  The
reference's float64 GrayImage / read_pgm / write_pgm stay with the reference:
a drop-in caller keeps using them, and this module is the uint8 batch path.
"""

from __future__ import annotations

import os
import re
from pathlib import Path
from typing import Sequence

import numpy as np

from .errors import BadDimensions, IoFailure, MalformedHeader, TruncatedData, UnsupportedMaxval

# A header field is a run of bytes other than PGM whitespace (space, tab,
# CR, LF) and '#'; a '#' starts a comment that ends at the line break.  One
# regex alternates the two so comments are skipped in a single scan.
_FIELD_OR_COMMENT = re.compile(rb"#[^\r\n]*|[^ \t\r\n#]+")


def _fields(data: bytes, pos: int = 0):
    """(field, offset just past it) for every header field from `pos` on."""
    for m in _FIELD_OR_COMMENT.finditer(data, pos):
        if not m.group().startswith(b"#"):
            yield m.group(), m.end()


def parse_header(data: bytes) -> tuple[bytes, int, int, int, int]:
    """(magic, width, height, maxval, offset just past maxval) of a P2/P5
    header, raising the reference's contract errors (corpus.py:65-91):
    MalformedHeader for a bad magic, missing or non-integer fields and
    non-positive sizes; UnsupportedMaxval outside (0, 255]."""
    fields = _fields(data)
    first = next(fields, None)
    if first is None:
        raise MalformedHeader("no PGM header: the file is empty")
    if first[0] not in (b"P2", b"P5"):
        raise MalformedHeader(f"magic {first[0]!r} is neither P2 nor P5")
    nums = []
    end = first[1]
    for name in ("width", "height", "maxval"):
        f = next(fields, None)
        if f is None:
            raise MalformedHeader(f"PGM header stops before its {name}")
        try:
            nums.append(int(f[0]))
        except ValueError:
            raise MalformedHeader(f"PGM {name} {f[0]!r} is not an integer") from None
        end = f[1]
    w, h, maxval = nums
    if w <= 0 or h <= 0:
        raise MalformedHeader(f"PGM size {w}x{h} is not positive")
    if not 0 < maxval <= 255:
        raise UnsupportedMaxval(f"PGM maxval {maxval}: only 1..255 (8-bit samples) is supported")
    return first[0], w, h, maxval, end


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
                raise TruncatedData(f"P5 raster holds {got} of {w * h} bytes")
        else:
            # P2: decimal samples after the header, same field/comment rules
            toks = [t for t, _ in _fields(head + f.read(), end)][: w * h]
            if len(toks) < w * h:
                raise TruncatedData(f"P2 raster holds {len(toks)} of {w * h} samples")
            try:
                vals = np.array([int(t) for t in toks], dtype=np.int64)
            except ValueError:
                raise MalformedHeader("P2 raster has a sample that is not an integer") from None
            if vals.max(initial=0) > maxval or vals.min(initial=0) < 0:
                raise MalformedHeader(f"P2 sample outside 0..{maxval} (the declared maxval)")
            out[...] = vals.reshape(h, w)
    if maxval < 255 and int(out.max(initial=0)) > maxval:
        raise MalformedHeader(f"P5 sample above the declared maxval {maxval}")
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
