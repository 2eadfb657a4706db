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


def test_registry_parse_and_scaling(tmp_path):
    from paper_1702_00817_b200 import errors as E
    from paper_1702_00817_b200.transforms import derive_scaling, load_registry

    t = exact.T
    txt = "# test file\nprop\n" + "\n".join(" ".join(str(v) for v in row) for row in t) + "\n14 0 0\n"
    sgn = np.sign(transforms.exact_dct_matrix().matrix).astype(int)
    txt += "sdct non-orthogonal\n" + "\n".join(" ".join(str(v) for v in row) for row in sgn) + "\n24 0 0\n"
    (tmp_path / "k.txt").write_text(txt)
    reg = load_registry(tmp_path / "k.txt")
    assert reg.names() == ("prop", "sdct") and len(reg) == 2
    assert np.allclose(reg.get("prop").scaling.diag, transforms.proposed_scaling().diag)
    assert reg.get("sdct").orthogonal is False
    with pytest.raises(E.NonOrthogonalKernel):
        derive_scaling(sgn)
    with pytest.raises(E.DuplicateName):
        reg.register(transforms.TransformMatrix("prop", t))


def test_registry_matches_live_reference(reference):
    """The reference's own data file parses identically here."""
    import importlib.resources as ir

    from paper_1702_00817_b200.transforms import load_registry

    path = ir.files("adct").joinpath("data/kernels.txt")
    ours = load_registry(path)
    ref = reference.default_registry()
    assert ours.names() == ref.names()
    for name in ref.names():
        assert np.array_equal(ours.get(name).kernel.entries, ref.get(name).kernel.entries)
        assert np.allclose(ours.get(name).scaling.diag, ref.get(name).scaling.diag, rtol=0, atol=1e-15)
        assert ours.get(name).orthogonal == ref.get(name).orthogonal


def test_apply_forward_inverse_kats():
    t = transforms.proposed_transform()
    x = np.arange(1, 9, dtype=np.float64)
    y = transforms.apply_forward(t, x)
    assert np.allclose(y / t.scaling.diag, [36, -7, 0, 3, 0, 5, 0, 1])
    assert np.abs(transforms.apply_inverse(t, y) - x).max() < 1e-9
    assert np.allclose(transforms.apply_inverse(t, np.r_[np.sqrt(8), np.zeros(7)]), np.ones(8))
