"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference package `adct` (pure Python/numpy) is imported read-only from
/root/reference; nothing is copied.  Outputs:

* images.npz   — the seeded input images the fixtures were computed on
                 (BASELINE generator, paper_1702_00817_b200.synth numpy path),
                 stored so the fixtures do not depend on regenerating them.
* golden.json  — reference results: SPEC.md known answers evaluated by the
                 reference, config-0 coefficients (sha256 + sample blocks) and
                 float64 round-trip error, config-1 retain-r PSNR/SSE for
                 r = 1..45, quantised-pipeline results composed from the
                 reference's own functions for q in {10, 50, 75, 90}.

Rounded results (SSE of rounded reconstructions) are obtained from the
reference's float64 output snapped to the exact 1/64 grid (|64 x - k| < 1e-6
is asserted) and rounded half away from zero, so ties are resolved
deterministically.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import adct  # noqa: E402  (the reference)
from adct import codec, fast, kernels, metrics  # noqa: E402

from paper_1702_00817_b200 import synth  # noqa: E402  (generator only)
from paper_1702_00817_b200.quant import q50_luma  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def snap_round(y: np.ndarray) -> np.ndarray:
    k = np.round(y * 64.0)
    assert np.abs(y * 64.0 - k).max() < 1e-6, "reference output not on the 1/64 grid"
    return np.clip(np.floor((k + 32) / 64), 0, 255).astype(np.uint8), k


def make_images() -> dict[str, np.ndarray]:
    imgs = {
        "c0_seed0_512": synth.images_np([0], 512, 512, 16, 8.0, 64.0)[0],
        "c1_seed1_128": synth.images_np([1], 128, 128, 16, 8.0, 64.0)[0],
        "c1_seed2_128": synth.images_np([2], 128, 128, 16, 8.0, 64.0)[0],
        "c2_seed3_128": synth.images_np([3], 128, 128, 32, 16.0, 128.0)[0],
        "ragged_40x24": synth.images_np([4], 40, 24, 16, 8.0, 64.0)[0],
    }
    rng = np.random.default_rng(7)
    imgs["noise_64"] = rng.integers(0, 256, (64, 64), dtype=np.uint8)
    sat = rng.integers(0, 256, (32, 48), dtype=np.uint8)
    sat[:, :24] = np.where(sat[:, :24] > 127, 255, 0)
    imgs["saturated_32x48"] = sat
    return imgs


def kats() -> dict:
    t = kernels.proposed_transform()
    out = {}
    out["T"] = kernels.proposed_kernel().entries.tolist()
    out["gram"] = kernels.proposed_kernel().gram().tolist()
    out["stages"] = [m.tolist() for m in fast.stage_matrices()]
    oc = fast.count_operations()
    out["op_count"] = [oc.additions, oc.multiplications, oc.shifts]
    out["fast_forward_1to8"] = fast.fast_forward(list(range(1, 9)))[0].tolist()
    out["fast_forward_ones"] = fast.fast_forward([1] * 8)[0].tolist()
    out["scaling_diag"] = t.scaling.diag.tolist()
    out["zigzag"] = list(codec.ZIGZAG_INDICES)
    out["compression_ratio"] = {str(r): codec.compression_ratio(r) for r in (1, 2, 25, 45, 64)}
    ones = np.ones((8, 8))
    f = codec.fold_scaling_into_quantization(t, ones)
    out["fold_ones_00"] = float(f[0, 0])
    out["fold_ones_11"] = float(f[1, 1])
    out["psnr"] = {"1": metrics.psnr(1.0), "65025": metrics.psnr(255.0**2), "0": str(metrics.psnr(0.0))}
    out["mse_2x2"] = metrics.mse(np.array([[0, 1], [2, 3]]), np.array([[1, 2], [3, 4]]))
    const = np.full((8, 8), 128.0)
    out["forward_const128_dc"] = float(codec.forward_2d(t, const)[0, 0])
    dc = np.zeros((8, 8))
    dc[0, 0] = 1024.0
    out["inverse_dc1024"] = codec.inverse_2d(t, dc).tolist()
    return out


def config0(img: np.ndarray) -> dict:
    t = kernels.proposed_transform()
    tiles = codec._tile(img.astype(np.int64))
    coef = np.stack([codec.forward_2d_unscaled(t, b) for b in tiles]).astype(np.int64)
    fl = img.astype(np.float64)
    rt = codec._tile(fl)
    err = max(float(np.abs(codec.inverse_2d(t, codec.forward_2d(t, b)) - b).max()) for b in rt)
    return {
        "coef_sha256_int64": sha(coef),
        "coef_sum": int(coef.sum()),
        "coef_abs_max": int(np.abs(coef).max()),
        "coef_blocks_0_3": coef[:4].tolist(),
        "coef_block_last": coef[-1].tolist(),
        "roundtrip_max_err": err,
    }


def config1(img: np.ndarray, rs) -> dict:
    t = kernels.proposed_transform()
    fl = img.astype(np.float64)
    res = {}
    for r in rs:
        y = codec.compress_image(t, fl, r)
        m = metrics.mse(fl, y)
        rec, k = snap_round(y)
        d = img.astype(np.int64) - rec.astype(np.int64)
        ties = int(np.count_nonzero((k.astype(np.int64) % 64) == 32))
        res[str(r)] = {
            "mse_ref": m,
            "psnr_ref": metrics.psnr(m),
            "sse_rounded": int((d * d).sum()),
            "rec_sha256": sha(rec),
            "ties": ties,
        }
    return res


def quant_ref(img: np.ndarray, q: int) -> dict:
    """Quantised pipeline composed from the reference's functions (float64):
    fold_scaling_into_quantization (then rounded half away), forward_2d_unscaled
    of X-128, quantise, dequantise, inverse_2d of D Z' D, +128, snap, round."""
    t = kernels.proposed_transform()
    s = (5000.0 / q if q < 50 else 200.0 - 2.0 * q) / 100.0
    qpu = codec.fold_scaling_into_quantization(t, q50_luma().astype(np.float64) * s)
    Qp = np.maximum(1, np.floor(qpu + 0.5))
    d = t.scaling.diag
    tiles = codec._tile(img.astype(np.int64) - 128)
    outs = []
    for b in tiles:
        Z = codec.forward_2d_unscaled(t, b).astype(np.float64)
        qq = np.sign(Z) * np.floor(np.abs(Z) / Qp + 0.5)
        Y = np.outer(d, d) * (qq * Qp)
        outs.append(codec.inverse_2d(t, Y) + 128.0)
    h, w = img.shape
    y = codec._untile(np.stack(outs), h, w)
    rec, k = snap_round(y)
    dd = img.astype(np.int64) - rec.astype(np.int64)
    return {"qprime": Qp.astype(int).tolist(), "sse": int((dd * dd).sum()), "rec_sha256": sha(rec),
            "ties": int(np.count_nonzero((k.astype(np.int64) % 64) == 32))}


def main() -> None:
    imgs = make_images()
    np.savez_compressed(os.path.join(HERE, "images.npz"), **imgs)
    g = {"reference": f"adct {adct.__version__} (/root/reference/pkg/src)", "kat": kats()}
    g["config0"] = config0(imgs["c0_seed0_512"])
    g["config1"] = {}
    for name in ("c0_seed0_512", "c1_seed1_128", "c1_seed2_128", "ragged_40x24", "noise_64", "saturated_32x48"):
        rs = range(1, 46) if name != "c0_seed0_512" else (1, 2, 3, 6, 10, 15, 25, 36, 45)
        g["config1"][name] = config1(imgs[name], rs)
    g["quant"] = {}
    for name in ("c2_seed3_128", "noise_64", "saturated_32x48", "ragged_40x24"):
        g["quant"][name] = {str(q): quant_ref(imgs[name], q) for q in (10, 50, 75, 90)}
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(g, f, indent=1, default=lambda o: float(o))
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
