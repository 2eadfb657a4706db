"""The drop-in, proven on the reference's own call sites: the dispatch module
of INTEGRATION.md §3 rebinds adct.codec / adct.metrics hot functions to this
package's GPU wrappers, and the UNMODIFIED reference drivers (cli.run_sweep,
cli.py:87-124, and the `lena` command, cli.py:187-204) run on the GPU.  Their
records must equal the unpatched reference's: MSE to 1e-9 relative, PSNR to
1e-3 dB (BASELINE's float tolerance; the float64 kernels agree far closer)."""

import os
import re
import sys

import numpy as np
import pytest

from paper_1702_00817_b200 import pgm, synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def adct_pkg():
    for d in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(d, "adct")):
            if d not in sys.path:
                sys.path.insert(0, d)
            import adct
            import adct.cli  # noqa: F401

            return adct
    pytest.skip("reference package not installed (baseline/_ref)")


@pytest.fixture()
def dispatch(adct_pkg):
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    code = re.findall(r"```python\n(# adct/_gpu_dispatch.py.*?)```", text, re.S)[0]
    ns = {"__name__": "adct._gpu_dispatch"}
    exec(compile(code, "INTEGRATION.md:adct/_gpu_dispatch.py", "exec"), ns)
    yield ns
    ns["disable"]()


def _records(adct, cfg, images=None):
    recs, summ, ape = adct.cli.run_sweep(cfg, images)
    return ({(r.image_id, r.transform_name, r.r): (r.mse, r.psnr) for r in recs},
            {(s.transform_name, s.r): (s.avg_mse, s.avg_psnr, s.n_images) for s in summ}, ape)


def _assert_close(a, b):
    assert a.keys() == b.keys()
    for k in a:
        (ma, pa), (mb, pb) = a[k][:2], b[k][:2]
        assert ma == pytest.approx(mb, rel=1e-9, abs=1e-12), k
        # a lossless reconstruction (r = 64, exact DCT) leaves only float64
        # round-off (MSE ~1e-26, PSNR > 250 dB) whose digits carry no meaning
        assert (pa == pb == np.inf) or abs(pa - pb) < 1e-3 or min(pa, pb) > 250.0, k


def test_reference_run_sweep_on_the_gpu(adct_pkg, dispatch):
    """Synthetic float corpus (the reference's own generator), every transform
    the reference can resolve: the built-ins and its registry kernels."""
    adct = adct_pkg
    names = ("dct", "proposed") + tuple(adct.kernels.default_registry().names())
    cfg = adct.cli.ExperimentConfig(transforms=names, r_min=2, r_max=45, n_images=3, seed=7)
    ref_recs, ref_summ, ref_ape = _records(adct, cfg)
    calls = {"n": 0}
    dispatch["enable"]()
    orig = adct.codec.reconstruct_image

    def counting(*a, **k):
        calls["n"] += 1
        return orig(*a, **k)

    adct.codec.reconstruct_image = counting
    gpu_recs, gpu_summ, gpu_ape = _records(adct, cfg)
    assert calls["n"] == 3 * len(names) * 44  # the reference loop really called the GPU wrapper
    _assert_close(gpu_recs, ref_recs)
    _assert_close(gpu_summ, ref_summ)
    assert gpu_ape.keys() == ref_ape.keys()
    for k in ref_ape:
        assert gpu_ape[k] == pytest.approx(ref_ape[k], rel=1e-7, abs=1e-9) or np.isnan(ref_ape[k])


def test_reference_run_sweep_pgm_corpus(adct_pkg, dispatch, tmp_path):
    """uint8 PGM corpus through the reference's loader (corpus_path)."""
    adct = adct_pkg
    imgs = synth.images_np(range(3), 128, 192, 16, 8.0, 64.0)
    for k, im in enumerate(imgs):
        pgm.write_pgm_u8(im, tmp_path / f"img{k}.pgm")
    cfg = adct.cli.ExperimentConfig(transforms=("dct", "proposed"), r_min=1, r_max=64, corpus_path=str(tmp_path))
    ref = _records(adct, cfg)
    dispatch["enable"]()
    gpu = _records(adct, cfg)
    _assert_close(gpu[0], ref[0])
    _assert_close(gpu[1], ref[1])


def test_reference_lena_command_on_the_gpu(adct_pkg, dispatch, tmp_path, capsys):
    adct = adct_pkg
    img = synth.images_np([11], 256, 256, 16, 8.0, 64.0)[0]
    pgm.write_pgm_u8(img, tmp_path / "lena.pgm")
    assert adct.cli.main(["lena", str(tmp_path / "lena.pgm"), "--r", "25", "--out", str(tmp_path / "ref")]) == 0
    ref_out = capsys.readouterr().out
    dispatch["enable"]()
    assert adct.cli.main(["lena", str(tmp_path / "lena.pgm"), "--r", "25", "--out", str(tmp_path / "gpu")]) == 0
    gpu_out = capsys.readouterr().out
    parse = lambda out: {ln.split()[0]: float(ln.split()[1]) for ln in out.splitlines()[2:] if ln.strip()}  # noqa: E731
    ref_psnr, gpu_psnr = parse(ref_out), parse(gpu_out)
    assert ref_psnr.keys() == gpu_psnr.keys() and len(ref_psnr) >= 7
    assert all(abs(ref_psnr[k] - gpu_psnr[k]) <= 0.01 for k in ref_psnr)  # printed with 2 decimals
    for f in sorted((tmp_path / "ref").glob("*.pgm")):
        a, b = pgm.read_pgm_u8(f), pgm.read_pgm_u8(tmp_path / "gpu" / f.name)
        # identical except where float64 lands either side of an exact .5
        assert np.abs(a.astype(int) - b.astype(int)).max() <= 1
        assert np.mean(a != b) < 0.05


def test_reference_errors_and_functions_through_dispatch(adct_pkg, dispatch):
    adct = adct_pkg
    t = adct.kernels.proposed_transform()
    rng = np.random.default_rng(3)
    blocks = rng.integers(0, 256, (5, 8, 8))
    want = {n: getattr(adct.codec, n) for n in ("forward_2d", "forward_2d_unscaled", "inverse_2d")}
    dispatch["enable"]()
    z = adct.codec.forward_2d_unscaled(t, blocks)
    assert z.dtype.kind == "i" and np.array_equal(z, want["forward_2d_unscaled"](t, blocks))
    y = adct.codec.forward_2d(t, blocks)
    assert np.abs(y - want["forward_2d"](t, blocks)).max() < 1e-9
    assert np.abs(adct.codec.inverse_2d(t, y) - blocks).max() < 1e-9
    with pytest.raises(adct.errors.InvalidRetention):
        adct.codec.compress_image(t, np.zeros((16, 16)), 65)
    with pytest.raises(adct.errors.BadDimensions):
        adct.codec.coefficient_blocks(t, np.zeros((12, 16)))
    with pytest.raises(adct.errors.DimensionMismatch):
        adct.metrics.mse(np.zeros((8, 8)), np.zeros((8, 16)))


def _read_csv(path):
    import csv

    with open(path) as fp:
        return list(csv.reader(fp))


def _assert_csv_close(a, b):
    """Same rows and text cells; numeric cells (printed to 6 significant
    digits by the reference) equal to that precision."""
    assert len(a) == len(b) and a[0] == b[0]
    for ra, rb in zip(a[1:], b[1:]):
        assert len(ra) == len(rb)
        for x, y in zip(ra, rb):
            try:
                fx, fy = float(x), float(y)
            except ValueError:
                assert x == y
                continue
            assert fx == pytest.approx(fy, rel=2e-6, abs=1e-12) or (np.isnan(fx) and np.isnan(fy)), (ra, rb)


@pytest.mark.parametrize("corpus", ["synthetic", "pgm"])
def test_reference_sweep_command_with_driver_dispatch(adct_pkg, dispatch, tmp_path, corpus):
    """enable(drivers=True): the unmodified `adct sweep` command (cli.main ->
    cmd_sweep -> run_sweep -> _write_sweep_outputs) runs the batched GPU sweep
    and writes the reference's own records.csv / summary.csv / metadata."""
    adct = adct_pkg
    names = ["dct", "proposed", sorted(adct.kernels.default_registry().names())[0]]
    args = ["sweep", "--transforms", ",".join(names), "--r-min", "1", "--r-max", "45"]
    if corpus == "pgm":  # uint8 images: the exact integer sweep for "proposed"
        d = tmp_path / "corpus"
        d.mkdir()
        for k, im in enumerate(synth.images_np(range(3), 64, 96, 16, 8.0, 64.0)):
            pgm.write_pgm_u8(im, d / f"im{k}.pgm")
        args += ["--corpus", str(d)]
    else:  # the reference's float synthesizer: dense float64 sweeps
        args += ["--n-images", "3", "--seed", "5"]
    orig = adct.cli.run_sweep
    assert adct.cli.main(args + ["--out", str(tmp_path / "ref")]) == 0
    dispatch["enable"](drivers=True)
    assert adct.cli.run_sweep is not orig
    assert adct.cli.main(args + ["--out", str(tmp_path / "gpu")]) == 0
    for f in ("records.csv", "summary.csv"):
        _assert_csv_close(_read_csv(tmp_path / "gpu" / f), _read_csv(tmp_path / "ref" / f))
    assert (tmp_path / "gpu" / "run_metadata.json").read_text() == (tmp_path / "ref" / "run_metadata.json").read_text()
    dispatch["disable"]()
    assert adct.cli.run_sweep is orig
