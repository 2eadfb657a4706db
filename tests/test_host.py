"""Host-side logic on CPU: transform definitions, reference-mirror API
validation (errors raised before any device work), sharding arithmetic, the
numpy mirror of the synthetic generator."""

import numpy as np
import pytest

from oracle import exact
from paper_1702_00817_b200 import codec, errors, metrics, shard, synth, transforms


def test_transform_from_stages_equals_reference_matrix():
    t = transforms.proposed_transform()
    assert np.array_equal(t.kernel.entries, exact.T)
    assert np.abs(t.matrix @ t.matrix.T - np.eye(8)).max() < 1e-12
    a1, a2, a3, p = transforms.stage_matrices()
    assert np.array_equal(p @ a3 @ a2 @ a1, exact.T)
    assert transforms.is_proposed(t)
    assert not transforms.is_proposed(transforms.exact_dct_matrix())


def test_transform_validation_errors():
    with pytest.raises(errors.ZeroRow):
        transforms.TransformMatrix("z", np.zeros((8, 8), dtype=int))
    with pytest.raises(ValueError):
        transforms.TransformMatrix("b", np.full((8, 8), 3))
    bad = transforms.TransformMatrix("b", np.ones((8, 8), dtype=int))
    with pytest.raises(errors.NonOrthogonalKernel):
        transforms.ApproximateTransform(bad, transforms.proposed_scaling())


def test_dct_is_orthonormal():
    c = transforms.exact_dct_matrix().matrix
    assert np.abs(c @ c.T - np.eye(8)).max() < 1e-12
    assert c[1, 0] == pytest.approx(0.490393, abs=1e-6)


def test_zigzag_and_masks():
    assert codec.ZIGZAG_INDICES == exact.zigzag_indices()
    assert codec.zigzag_positions()[:3] == ((0, 0), (0, 1), (1, 0))
    m = codec.retention_mask(10)
    assert m.sum() == 10 and not m.flags.writeable
    assert m[:4, :4].sum() == 10  # N8: r = 10 keeps only u, v <= 3
    b = np.arange(64, dtype=float).reshape(8, 8)
    assert np.array_equal(codec.retain_coefficients(b, 64), b)
    assert codec.retain_coefficients(b, 1).sum() == 0.0 and codec.retain_coefficients(b, 1)[0, 0] == 0.0
    r3 = codec.retain_coefficients(b + 1, 3)
    assert np.count_nonzero(r3) == 3
    assert np.array_equal(codec.retain_coefficients(r3, 3), r3)  # idempotent
    assert codec.compression_ratio(2) == 96.875 and codec.compression_ratio(25) == 60.9375


@pytest.mark.parametrize("r", [0, 65, -3])
def test_invalid_retention_raised_before_compute(r):
    t = transforms.proposed_transform()
    img = np.zeros((16, 16), np.uint8)
    with pytest.raises(errors.InvalidRetention):
        codec.compress_image(t, img, r)
    with pytest.raises(errors.InvalidRetention):
        codec.retention_mask(r)
    with pytest.raises(errors.InvalidRetention):
        codec.compression_ratio(r)


def test_bad_dimensions_raised_before_compute():
    t = transforms.proposed_transform()
    with pytest.raises(errors.BadDimensions):
        codec.compress_image(t, np.zeros((12, 16)), 10)
    with pytest.raises(errors.BadDimensions):
        codec.coefficient_blocks(t, np.zeros((16, 20)))
    with pytest.raises(errors.BadDimensions):
        codec.coefficient_blocks(t, np.zeros((2, 16, 16)))
    with pytest.raises(errors.BadDimensions):
        codec.retain_coefficients(np.zeros((4, 4)), 3)


def test_non_8x8_transform_matrix_rejected_before_compute():
    class Bad:
        name = "bad"
        matrix = np.eye(4)

    with pytest.raises(errors.BadDimensions):
        codec.compress_image(Bad, np.zeros((8, 8)), 3)


def test_metrics_host_functions():
    assert metrics.psnr(1.0) == pytest.approx(48.13080360867909)
    assert metrics.psnr(0.0) == float("inf")
    with pytest.raises(ValueError):
        metrics.psnr(-1.0)
    with pytest.raises(errors.DimensionMismatch):
        metrics.mse(np.zeros((2, 2)), np.zeros((2, 3)))
    recs = [metrics.QualityRecord("a", "proposed", 10, 4.0, 42.0), metrics.QualityRecord("b", "proposed", 10, 2.0, 44.0)]
    (s,) = metrics.summarize(recs)
    assert s.avg_mse == 3.0 and s.avg_psnr == 43.0 and s.n_images == 2
    (s2,) = metrics.summarize(recs, psnr_from_avg_mse=True)
    assert s2.avg_psnr == pytest.approx(metrics.psnr(3.0))
    with pytest.raises(errors.EmptyGroup):
        metrics.summarize([])
    assert metrics.ape_vs_dct(1.1, 1.0) == pytest.approx(10.0)


@pytest.mark.parametrize("n,world", [(10, 4), (4096, 8), (3, 8), (0, 2), (7, 1)])
def test_shard_ranges_partition(n, world):
    parts = [shard.shard_range(n, r, world) for r in range(world)]
    assert parts[0].start == 0 and parts[-1].stop == n
    assert all(a.stop == b.start for a, b in zip(parts, parts[1:]))
    sizes = [p.count for p in parts]
    assert max(sizes) - min(sizes) <= 1 and sum(sizes) == n


def test_synth_numpy_generator_properties():
    p = synth.blob_params(5, 512, 512, 16, 8.0, 64.0)
    assert p.shape == (16, 4)
    assert np.all((p[:, 2] >= 8) & (p[:, 2] <= 64)) and np.all(np.abs(p[:, 3]) <= 80)
    a = synth.images_np([0, 1], 128, 128, 16, 8.0, 64.0)
    b = synth.images_np([0, 1], 128, 128, 16, 8.0, 64.0)
    assert a.dtype == np.uint8 and np.array_equal(a, b) and not np.array_equal(a[0], a[1])
    z = synth.hash_normal(3, np.arange(200000, dtype=np.uint64))
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1) < 0.01
    v = synth.video_blob_params(0, 5, 64, 64, 16, 8.0, 64.0)
    assert np.array_equal(v[0], synth.video_blob_params(0, 1, 64, 64, 16, 8.0, 64.0)[0])
    assert np.all(v[1:, :, 2:] == v[:1, :, 2:])  # only centres drift


def test_golden_images_reproduce_from_generator():
    import os

    imgs = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", "images.npz")))
    again = synth.images_np([1], 128, 128, 16, 8.0, 64.0)[0]
    assert np.mean(again != imgs["c1_seed1_128"]) < 1e-3


def test_lane_range_bound_for_every_r():
    """16-bit output fields are unambiguous for every retain mask."""
    import importlib.util
    import os

    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools", "range_bounds.py")
    spec = importlib.util.spec_from_file_location("range_bounds", path)
    rb = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(rb)
    worst = max(rb.worst(r) for r in range(1, 65))
    assert worst == 27136 and worst + 32 <= 32767


def test_flowgraph_api_kats():
    from paper_1702_00817_b200 import flowgraph

    y, cost = flowgraph.fast_forward([1, 2, 3, 4, 5, 6, 7, 8])
    assert y.tolist() == [36, -7, 0, 3, 0, 5, 0, 1] and (cost.additions, cost.multiplications, cost.shifts) == (14, 0, 0)
    assert flowgraph.fast_forward([1] * 8)[0].tolist() == [8, 0, 0, 0, 0, 0, 0, 0]
    rng = np.random.default_rng(0)
    for _ in range(200):
        x = rng.integers(-1024, 1025, 8)
        assert np.array_equal(flowgraph.fast_forward(x)[0], exact.T @ x)
    assert max(abs(v) for st in flowgraph.flow_intermediates([255, 0, 255, 0, 0, 255, 0, 255]) for v in st) <= 2040


def test_op_count_is_tallied_from_the_stages():
    from paper_1702_00817_b200 import flowgraph

    assert flowgraph.stage_costs() == (("A1", 8), ("A2", 4), ("A3", 2), ("P", 0))
    c = transforms.proposed_transform().declared_costs
    assert (c.additions, c.multiplications, c.shifts) == (14, 0, 0)  # kernels.py:160-163


def test_proposed_types_match_reference_objects(reference):
    """Our transform objects carry the reference's attribute values, and the
    reference's own objects are recognised as the paper's transform."""
    ours, ref = transforms.proposed_transform(), reference.proposed_transform()
    assert np.array_equal(ours.kernel.entries, ref.kernel.entries)
    assert np.array_equal(ours.scaling.diag, ref.scaling.diag)
    assert np.array_equal(ours.matrix, ref.matrix) and ours.name == ref.name
    assert ref.declared_costs.additions == ours.declared_costs.additions == 14
    assert transforms.is_proposed(ref) and not transforms.is_proposed(reference.exact_dct_matrix())
    assert np.abs(transforms.exact_dct_matrix().matrix - reference.exact_dct_matrix().matrix).max() < 1e-15


def test_type_contract_errors():
    from paper_1702_00817_b200 import errors as E

    z = exact.T.copy()
    z[3] = 0
    with pytest.raises(E.ZeroRow):
        transforms.TransformMatrix("z", z)
    with pytest.raises(ValueError):
        transforms.TransformMatrix("big", exact.T * 3)
    sgn = np.sign(transforms.exact_dct_matrix().matrix).astype(int)
    k = transforms.TransformMatrix("sdct", sgn)
    with pytest.raises(E.NonOrthogonalKernel):
        transforms.ApproximateTransform(k, transforms.DiagonalScaling(1 / np.sqrt(np.diag(k.gram()))))
    t = transforms.ApproximateTransform(k, transforms.DiagonalScaling(1 / np.sqrt(np.diag(k.gram()))), orthogonal=False)
    assert t.name == "sdct" and t.orthogonal is False and t.matrix.shape == (8, 8)
    with pytest.raises(ValueError):
        transforms.DiagonalScaling(np.r_[np.ones(7), 0.0])


def test_registry_names_resolve_through_the_reference(reference):
    """Names other than dct/proposed come from the installed reference's own
    registry (its data/kernels.txt), as cli.resolve_transform does."""
    from paper_1702_00817_b200 import sweep

    reg = reference.default_registry()
    assert len(reg.names()) >= 5
    for name in reg.names():
        t = sweep.resolve_transform(name)
        assert t is reg.get(name)
    assert transforms.is_proposed(sweep.resolve_transform("proposed"))
    with pytest.raises(ValueError):
        sweep.resolve_transform("no-such-kernel")


def test_load_corpus_images_from_pgm_dir(tmp_path):
    from paper_1702_00817_b200 import errors as E, pgm, sweep

    cfg = sweep.ExperimentConfig(("proposed",), corpus_path=str(tmp_path))
    with pytest.raises(E.MissingImage):
        sweep.load_corpus_images(cfg)
    rng = np.random.default_rng(4)
    imgs = {f"im{k}": rng.integers(0, 256, (16, 24), dtype=np.uint8) for k in (2, 0, 1)}
    for name, im in imgs.items():
        pgm.write_pgm_u8(im, tmp_path / f"{name}.pgm")
    got = sweep.load_corpus_images(cfg)
    assert [n for n, _ in got] == ["im0", "im1", "im2"]
    assert all(np.array_equal(a, imgs[n]) for n, a in got)
    pgm.write_pgm_u8(rng.integers(0, 256, (8, 8), dtype=np.uint8), tmp_path / "odd.pgm")  # mixed sizes
    assert [a.shape for _, a in sweep.load_corpus_images(cfg)][-1] == (8, 8)


def test_csv_writers_match_reference(reference):
    import io

    from paper_1702_00817_b200 import metrics

    recs = [metrics.QualityRecord(f"im{i}", t, r, 10.0 / (r + i), metrics.psnr(10.0 / (r + i)))
            for i in range(3) for t in ("proposed", "dct") for r in (2, 10)]
    recs.append(metrics.QualityRecord("zero", "dct", 64, 0.0, metrics.psnr(0.0)))
    ref_recs = [reference.metrics.QualityRecord(*vars(m).values()) for m in recs]
    a, b = io.StringIO(), io.StringIO()
    metrics.write_quality_csv(a, recs)
    reference.metrics.write_quality_csv(b, ref_recs)
    assert a.getvalue() == b.getvalue()
    for conv in (False, True):
        ours = metrics.summarize(recs, psnr_from_avg_mse=conv)
        ref = reference.metrics.summarize(ref_recs, psnr_from_avg_mse=conv)
        assert [tuple(vars(s).values()) for s in ours] == [tuple(vars(s).values()) for s in ref]
        a, b = io.StringIO(), io.StringIO()
        metrics.write_summary_csv(a, ours)
        reference.metrics.write_summary_csv(b, ref)
        assert a.getvalue() == b.getvalue()
    assert metrics.format_float(float("inf")) == reference.metrics.format_float(float("inf")) == "inf"


def test_missing_native_library_fails_loudly(tmp_path):
    """No CPU fallback: without libadct_cuda.so every compute entry point
    raises NativeLibraryError (child process: the path is read at import)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r'''
import numpy as np, torch
from paper_1702_00817_b200 import _lib, batch, codec, quant, transforms
for call in (lambda: _lib.lib(),
             lambda: quant.quant_table(50),
             lambda: batch.compress_retain(torch.zeros((1, 8, 8), dtype=torch.uint8), 10),
             lambda: codec.compress_image(transforms.proposed_transform(), np.zeros((8, 8)), 10)):
    try:
        call()
    except (_lib.NativeLibraryError, RuntimeError, ValueError) as exc:
        msg = str(exc)
        assert "not found" in msg or "CUDA" in msg or "GPU" in msg or "no CPU path" in msg, exc
    else:
        raise SystemExit("a call succeeded without the native library")
print("LOUD_OK")
'''
    env = dict(os.environ, PYTHONPATH=root, ADCT_LIB_PATH=str(tmp_path / "absent.so"))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, env=env)
    assert "LOUD_OK" in r.stdout, r.stderr[-2000:]
