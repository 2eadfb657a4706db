"""GPU: dense 8x8 kernels for the exact DCT / arbitrary matrices, and the
GPU-backed run_sweep against a float64 restatement of cli.run_sweep."""

import json
import os

import numpy as np
import pytest
import torch

from oracle import exact, refport
from paper_1702_00817_b200 import batch, codec, metrics, sweep, transforms

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
IMAGES = dict(np.load(os.path.join(HERE, "golden", "images.npz")))
DCT = transforms.exact_dct_matrix()
GOLDEN = json.load(open(os.path.join(HERE, "golden", "golden.json")))


def ref_sweep_mse(C, img, rs):
    """cli.run_sweep's per-image inner loop in float64 (codec.py:120-141, metrics.py:49-56)."""
    tiles = exact.tile(img.astype(np.float64))
    coef = C @ tiles @ C.T
    h, w = img.shape
    out = []
    for r in rs:
        kept = np.where(exact.retention_mask(r).astype(bool), coef, 0.0)
        rec = np.clip(exact.untile(C.T @ kept @ C, h, w), 0, 255)
        out.append(np.mean((img.astype(np.float64) - rec) ** 2))
    return np.array(out)


def test_dense_forward_inverse_dct(cuda):
    img = IMAGES["c1_seed1_128"]
    C = DCT.matrix
    y = codec.coefficient_blocks(DCT, img.astype(np.float64))
    assert np.abs(y - C @ exact.tile(img.astype(np.float64)) @ C.T).max() < 1e-9
    for r in (1, 10, 64):
        rec = codec.reconstruct_image(DCT, y, r, 128, 128)
        kept = np.where(exact.retention_mask(r).astype(bool), y, 0.0)
        want = np.clip(exact.untile(C.T @ kept @ C, 128, 128), 0, 255)
        assert np.abs(rec - want).max() < 1e-9
    assert np.abs(codec.compress_image(DCT, img, 64) - img).max() < 1e-9


def test_dense_matches_flow_graph_for_proposed_matrix(cuda):
    """The dense kernel fed the proposed C = D T agrees with the flow-graph kernels."""
    t = transforms.proposed_transform()
    x = torch.from_numpy(IMAGES["c1_seed2_128"]).to(cuda)
    a = batch.forward_dense(x, t.matrix)
    b = batch.forward_f64(x)
    assert (a - b).abs().max().item() < 1e-9


def test_dense_sweep_equals_reference_loop(cuda):
    img = IMAGES["c1_seed1_128"]
    x = torch.from_numpy(img).to(cuda)
    got = batch.sweep_dense_sse(x, DCT.matrix, 1, 45)[0].cpu().numpy() / img.size
    want = ref_sweep_mse(DCT.matrix, img, range(1, 46))
    assert np.allclose(got, want, rtol=1e-10, atol=1e-10)
    got_f = batch.sweep_dense_sse(x.to(torch.float64) + 0.25, DCT.matrix, 3, 7)[0].cpu().numpy() / img.size
    assert np.allclose(got_f, ref_sweep_mse(DCT.matrix, img + 0.25, range(3, 8)), rtol=1e-10, atol=1e-10)


def test_exact_sweep_unrounded_matches_golden(cuda):
    name = "c1_seed2_128"
    x = torch.from_numpy(IMAGES[name]).to(cuda)
    sse, ssef = batch.sweep_retain_sse_unrounded(x, 1, 45)
    for r in range(1, 46):
        g = GOLDEN["config1"][name][str(r)]
        assert int(sse[0, r - 1]) == g["sse_rounded"]
        assert ssef[0, r - 1].item() / (4096.0 * IMAGES[name].size) == pytest.approx(g["mse_ref"], rel=1e-9)
    none, only = batch.sweep_retain_sse_unrounded(x, 1, 45, rounded=False)  # the run_sweep form
    assert none is None and torch.equal(only, ssef)
    odd = torch.from_numpy(IMAGES["noise_64"][:, :56]).to(cuda)  # unpaired units
    _, f1 = batch.sweep_retain_sse_unrounded(odd, 2, 9)
    _, f2 = batch.sweep_retain_sse_unrounded(odd, 2, 9, rounded=False)
    assert torch.equal(f1, f2)


def test_run_sweep_matches_reference_semantics(cuda, tmp_path):
    imgs = [("a", IMAGES["c1_seed1_128"]), ("b", IMAGES["c1_seed2_128"]), ("c", IMAGES["noise_64"].astype(np.float64))]
    cfg = sweep.ExperimentConfig(transforms=("dct", "proposed"), r_min=2, r_max=12)
    records, summaries, ape = sweep.run_sweep(cfg, imgs)
    assert len(records) == 2 * 3 * 11
    prop = transforms.proposed_transform()
    for rec in records:
        img = dict(imgs)[rec.image_id]
        C = DCT.matrix if rec.transform_name == "dct" else prop.matrix
        want = ref_sweep_mse(C, np.asarray(img), [rec.r])[0]
        assert rec.mse == pytest.approx(want, rel=1e-9, abs=1e-12)
        assert rec.psnr == pytest.approx(metrics.psnr(want), abs=1e-8)
    s = {(x.transform_name, x.r): x for x in summaries}
    assert ape[("dct", 5)] == 0.0 and ape[("proposed", 5)] > 0
    assert s[("proposed", 2)].n_images == 3
    sweep.write_sweep_outputs(tmp_path, cfg, records, summaries, ape)
    head = open(tmp_path / "summary.csv").read().splitlines()
    assert head[0] == "transform,r,compression_ratio,avg_mse,avg_psnr,ape_vs_dct,n_images"
    assert json.load(open(tmp_path / "run_metadata.json"))["psnr_convention"] == "mean_of_per_image_psnr"


def test_compare_transforms_is_cmd_lena(cuda, tmp_path):
    """sweep.compare_transforms = cli.cmd_lena: PSNR per transform at one r
    (reference float semantics) and the reconstructions as P5 files."""
    from paper_1702_00817_b200 import pgm

    img = IMAGES["c1_seed1_128"]
    reg = transforms.ApproximateTransform(transforms.TransformMatrix("flipped", -exact.T),
                                          transforms.proposed_scaling())
    rows = sweep.compare_transforms(img, 25, ("dct", "proposed", reg), out_dir=tmp_path, stem="c1")
    assert [n for n, _ in rows] == ["dct", "proposed", "flipped"]
    prop = transforms.proposed_transform()
    for (name, value), C in zip(rows, (DCT.matrix, prop.matrix, reg.matrix)):
        want = ref_sweep_mse(C, np.asarray(img, dtype=np.float64), [25])[0]
        assert value == pytest.approx(metrics.psnr(want), abs=1e-8)
        f = tmp_path / f"c1_{name}_r25.pgm"
        g = pgm.read_pgm_u8(f)
        recon = np.asarray(codec.compress_image(sweep.resolve_transform(
            {"dct": "dct", "proposed": "proposed"}.get(name, reg)), img, 25))
        assert np.array_equal(g, np.floor(recon + 0.5))
    assert rows[1][1] == pytest.approx(rows[2][1], abs=1e-9)  # -T gives the same reconstruction


def test_registry_style_transform_object(cuda):
    """Any object with an 8x8 .matrix works (e.g. a reference registry kernel)."""
    k = exact.T.astype(np.float64)
    m = np.diag(1 / np.sqrt((k * k).sum(1))) @ k  # row-normalised proposed kernel
    class T:
        name = "custom"
        matrix = m
    img = IMAGES["c1_seed2_128"]
    assert np.abs(codec.compress_image(T, img, 10) - refport.compress_image(img, 10)).max() < 1e-9
