"""GPU-backed corpus sweep — the reference's caller of the hot path re-pointed
at the batch kernels (reference cli.py:53-152).

`run_sweep` keeps the reference's contract: for every (transform, image, r)
it records the MSE and PSNR of the *unrounded, clamped* reconstruction
(codec.reconstruct_image + metrics.mse, cli.py:105-113), then summarises per
(transform, r) and computes the APE of the average MSE against the exact DCT.
The loop over images and r is replaced by one launch per image batch:

* "proposed": `adct_sweep_retain_sse` — one read per image, exact integer
  SSE for every r (the unrounded SSE is 4096 x the reference's, exactly);
* any other transform ("dct", or a registry transform object with an 8x8
  `.matrix`): `adct_sweep_dense` — float64, incremental per r.

`write_sweep_outputs` writes records.csv, summary.csv and run_metadata.json in
the reference's format (cli.py:127-152, metrics.py:100-122).

`compare_transforms` is the GPU form of cli.cmd_lena (cli.py:187-204): one
image, one r, PSNR per transform and optionally the reconstructions as PGM.
"""

from __future__ import annotations

import json
from dataclasses import asdict, dataclass
from pathlib import Path
from typing import Sequence

import numpy as np
import torch

from . import batch, codec, metrics, transforms


@dataclass(frozen=True)
class ExperimentConfig:
    """Mirror of cli.ExperimentConfig (cli.py:53-73); `transforms` holds names
    ("dct", "proposed") or transform objects (e.g. registry kernels)."""

    transforms: tuple
    r_min: int = 2
    r_max: int = 45
    corpus_path: str | None = None
    seed: int = 2012
    n_images: int = 45
    psnr_from_avg_mse: bool = False

    def __post_init__(self) -> None:
        if not self.transforms:
            raise ValueError("at least one transform is required")
        if not (1 <= self.r_min <= self.r_max <= 64):
            raise ValueError(f"retention range [{self.r_min}, {self.r_max}] not within [1, 64]")

    @property
    def r_values(self) -> range:
        return range(self.r_min, self.r_max + 1)


def _reference_registry():
    """The installed reference package's kernel registry (kernels.py:312-327:
    default_registry() over its bundled data/kernels.txt), or None.  In a
    drop-in deployment the reference package is what calls into this one, so
    its registry and data file are the source of the comparison kernels; this
    package does not carry a second copy of either."""
    try:
        from adct import kernels as ref_kernels
    except ImportError:
        return None
    return ref_kernels.default_registry()


def resolve_transform(t):
    """Name -> transform (cli.py:40-50): "dct" and "proposed" are built in,
    any other name is looked up in the installed reference's registry
    (bas2008, bas2009, bas2011, cb2011, level1, ...); transform objects
    (ours, the reference's, or anything with an 8x8 `.matrix`) pass through."""
    if not isinstance(t, str):
        return t
    if t == "dct":
        return transforms.exact_dct_matrix()
    if t == "proposed":
        return transforms.proposed_transform()
    reg = _reference_registry()
    if reg is None:
        raise ValueError(f"unknown transform {t!r}: registry names need the reference package `adct` "
                         "importable (its data/kernels.txt); or pass the transform object")
    if t not in reg:
        raise ValueError(f"unknown transform {t!r}; available: dct, proposed, {', '.join(reg.names())}")
    return reg.get(t)


def load_corpus_images(config: ExperimentConfig):
    """(image_id, samples) pairs like cli.load_corpus_images (cli.py:76-84):
    every *.pgm of `config.corpus_path` in name order (read as uint8 straight
    into one batch by pgm.load_batch; MissingImage when there are none), else
    the reference's synthetic corpus (corpus.synthesize_corpus, needs the
    reference package)."""
    from pathlib import Path

    from . import pgm
    from .errors import MissingImage

    if config.corpus_path is not None:
        paths = sorted(Path(config.corpus_path).glob("*.pgm"))
        if not paths:
            raise MissingImage(f"no .pgm files in {config.corpus_path}")
        shapes = {pgm.parse_header(open(p, "rb").read(4096))[1:3] for p in paths}
        if len(shapes) == 1:
            stack = pgm.load_batch(paths, pinned=False)
            return [(p.stem, stack[k]) for k, p in enumerate(paths)]
        return [(p.stem, pgm.read_pgm_u8(p)) for p in paths]
    try:
        from adct import corpus as ref_corpus
    except ImportError:
        raise ValueError("no corpus_path and no reference package for the synthetic corpus; "
                         "pass images or a PGM directory") from None
    imgs = ref_corpus.synthesize_corpus(config.seed, config.n_images)
    return [(f"synth-{i:03d}", g.samples) for i, g in enumerate(imgs)]


def _name(t) -> str:
    return t if isinstance(t, str) else t.name


def _group_by_shape(images):
    groups: dict[tuple, list[int]] = {}
    for k, (_, s) in enumerate(images):
        groups.setdefault((tuple(np.shape(s)), np.asarray(s).dtype.kind), []).append(k)
    return groups


def _is_u8_exact(arr: np.ndarray) -> bool:
    return arr.dtype == np.uint8 or (
        arr.dtype.kind in "fiu" and bool(np.all((arr >= 0) & (arr <= 255) & (arr == np.round(arr))))
    )


def sweep_mse(t, stack: np.ndarray, r_min: int, r_max: int, device=None) -> np.ndarray:
    """MSE[N, r] of the unrounded clamped reconstructions of an (N, H, W) stack."""
    dev = device or torch.device("cuda", torch.cuda.current_device())
    n, h, w = stack.shape
    tr = resolve_transform(t)
    if transforms.is_proposed(tr) and _is_u8_exact(stack):
        u8 = stack if stack.dtype == np.uint8 else stack.astype(np.uint8)
        x = codec._host_tensor(u8).to(dev)
        _, ssef = batch.sweep_retain_sse_unrounded(x, r_min, r_max, rounded=False)
        torch.cuda.current_stream().synchronize()
        return ssef.cpu().numpy().astype(np.float64) / (4096.0 * h * w)
    x = codec._host_tensor(stack).to(dev)
    if x.dtype != torch.uint8:
        x = x.to(torch.float64)
    sse = batch.sweep_dense_sse(x, np.asarray(tr.matrix, dtype=np.float64), r_min, r_max)
    torch.cuda.current_stream().synchronize()
    return sse.cpu().numpy() / float(h * w)


def _batch_of(images, idx) -> np.ndarray:
    """(N, H, W) batch of images[idx]: a zero-copy view when they are
    consecutive C-contiguous planes of one allocation (a corpus loaded as one
    batch, pgm.load_batch, synth.images_np), else one stacked copy."""
    arrs = [np.asarray(images[k][1]) for k in idx]
    a0 = arrs[0]
    owner = a0.base
    if owner is not None and all(a.base is owner and a.flags.c_contiguous and a.dtype == a0.dtype
                                 and a.shape == a0.shape for a in arrs):
        plane = a0.nbytes
        p0 = a0.__array_interface__["data"][0]
        if all(a.__array_interface__["data"][0] == p0 + k * plane for k, a in enumerate(arrs)):
            # every plane lies inside `owner`, back to back: one strided view covers them
            return np.lib.stride_tricks.as_strided(a0, shape=(len(arrs),) + a0.shape,
                                                   strides=(plane,) + a0.strides, writeable=False)
    return np.stack(arrs)


def run_sweep(config: ExperimentConfig, images: Sequence[tuple[str, np.ndarray]] | None = None):
    """(records, summaries, ape) exactly as cli.run_sweep (cli.py:87-124) returns them.

    `images` are (image_id, samples) pairs; None loads them like the
    reference (load_corpus_images: config.corpus_path or the synthesizer).
    One batched sweep per (transform, image shape).  The summaries come
    straight from the MSE matrix, with the reference's own float64 averages
    (metrics.summarize, metrics.py:75-97: np.mean over the images in order).
    Transforms sharing a name merge their groups as the reference does, and
    then go through metrics.summarize itself."""
    if images is None:
        images = load_corpus_images(config)
    records: list[metrics.QualityRecord] = []
    groups = _group_by_shape(images)
    batches = {key: _batch_of(images, idx) for key, idx in groups.items()}
    r_values = list(config.r_values)
    names = [_name(t) for t in config.transforms]
    per_name: dict[str, tuple[np.ndarray, np.ndarray]] = {}
    for t, name in zip(config.transforms, names):
        m = np.empty((len(images), len(r_values)), dtype=np.float64)
        for key, idx in groups.items():
            m[idx] = sweep_mse(t, batches[key], config.r_min, config.r_max)
        p = np.empty_like(m)
        for k, (image_id, _) in enumerate(images):
            for j, r in enumerate(r_values):
                err = float(m[k, j])
                p[k, j] = metrics.psnr(err)  # math.log10, as the reference's per-record psnr
                records.append(metrics.QualityRecord(image_id, name, r, err, float(p[k, j])))
        per_name[name] = (m, p)
    if images and len(set(names)) == len(names):
        summaries = []
        for name in sorted(names):
            m, p = per_name[name]
            avg_m = np.ascontiguousarray(m.T).mean(axis=1)  # per r, over the images in order
            avg_p = np.ascontiguousarray(p.T).mean(axis=1)
            for j, r in enumerate(r_values):
                am = float(avg_m[j])
                ap = metrics.psnr(am) if config.psnr_from_avg_mse else float(avg_p[j])
                summaries.append(metrics.CorpusSummary(name, r, am, ap, len(images)))
    else:
        summaries = metrics.summarize(records, psnr_from_avg_mse=config.psnr_from_avg_mse)
    avg_mse = {(s.transform_name, s.r): s.avg_mse for s in summaries}
    ape = {}
    if "dct" in names:
        for s in summaries:
            ref = avg_mse[("dct", s.r)]
            ape[(s.transform_name, s.r)] = metrics.ape_vs_dct(s.avg_mse, ref) if ref > 0 else float("nan")
    return records, summaries, ape


_fmt = metrics.format_float


def write_sweep_outputs(out_dir, config: ExperimentConfig, records, summaries, ape) -> None:
    """records.csv, summary.csv, run_metadata.json (cli.py:127-152)."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    with open(out / "records.csv", "w", newline="") as fp:
        metrics.write_quality_csv(fp, records)
    with open(out / "summary.csv", "w") as fp:
        fp.write("transform,r,compression_ratio,avg_mse,avg_psnr,ape_vs_dct,n_images\n")
        for s in sorted(summaries, key=lambda m: (m.transform_name, m.r)):
            cells = [
                s.transform_name, str(s.r), _fmt(codec.compression_ratio(s.r)), _fmt(s.avg_mse),
                _fmt(s.avg_psnr), _fmt(ape[(s.transform_name, s.r)]) if ape else "", str(s.n_images),
            ]
            fp.write(",".join(cells) + "\n")
    meta = asdict(config)
    meta["transforms"] = [_name(t) for t in config.transforms]
    meta["psnr_convention"] = "psnr_of_avg_mse" if config.psnr_from_avg_mse else "mean_of_per_image_psnr"
    meta["ape_convention"] = "avg_mse"
    with open(out / "run_metadata.json", "w") as fp:
        json.dump(meta, fp, indent=2, sort_keys=True)
        fp.write("\n")


def compare_transforms(image, r: int, transforms_=("dct", "proposed"), *, out_dir=None, stem: str = "image"):
    """PSNR of every transform's retain-r reconstruction of one image, in the
    order given (cli.cmd_lena, cli.py:187-204: reference float semantics,
    unrounded clamped reconstruction, metrics.mse + metrics.psnr).  With
    `out_dir`, each reconstruction is written as `<stem>_<name>_r<r>.pgm`
    (samples rounded half away, corpus.write_pgm).  Registry transforms are
    passed as objects.  Returns [(name, psnr_db)]."""
    from . import pgm

    img = np.asarray(image)
    if out_dir is not None:
        out_dir = Path(out_dir)
        out_dir.mkdir(parents=True, exist_ok=True)
    rows = []
    for t in transforms_:
        tr = resolve_transform(t)
        recon = np.asarray(codec.compress_image(tr, img, r))
        value = metrics.psnr(metrics.mse(img, recon))
        rows.append((_name(t), value))
        if out_dir is not None:  # samples rounded half away (corpus.write_pgm, corpus.py:114-121)
            pgm.write_pgm_u8(recon, out_dir / f"{stem}_{_name(t)}_r{r}.pgm")
    return rows

