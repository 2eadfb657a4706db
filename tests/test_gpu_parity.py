"""GPU parity: CUDA path (through the C ABI) vs the CPU oracle, bit-exact."""

import numpy as np
import pytest
import torch

from oracle import exact
from paper_1702_00817_b200 import batch, quant, synth

pytestmark = pytest.mark.gpu


def _imgs(cuda, seeds, h=512, w=512, cfg=0):
    nb, smin, smax = synth.CONFIG_BLOBS[cfg]
    return synth.images_device(seeds, h, w, nb, smin, smax, device=cuda)


def test_forward_int32_config0(cuda):
    x = _imgs(cuda, [0])
    z = batch.forward_int(x)
    torch.cuda.synchronize()
    want = exact.forward_unscaled(x.cpu().numpy())
    assert z.shape == (1, 4096, 8, 8)
    assert np.array_equal(z.cpu().numpy().astype(np.int64), want)


@pytest.mark.parametrize("level_shift", [False, True])
@pytest.mark.parametrize("shape", [(2, 64, 64), (3, 40, 24), (1, 8, 8), (2, 16, 48)])
def test_forward_int_shapes(cuda, shape, level_shift):
    g = torch.Generator(device="cpu").manual_seed(sum(shape))
    x = torch.randint(0, 256, shape, dtype=torch.uint8, generator=g).to(cuda)
    for dt in (torch.int32, torch.int16):
        z = batch.forward_int(x, level_shift=level_shift, dtype=dt)
        torch.cuda.synchronize()
        want = exact.forward_unscaled(x.cpu().numpy(), level_shift=level_shift)
        assert np.array_equal(z.cpu().numpy().astype(np.int64), want)


@pytest.mark.parametrize("shape", [(5, 136, 272), (3, 72, 200), (70, 24, 48), (2, 8, 4096)])
def test_forward_int_ragged_warp_runs(cuda, shape):
    """Units per frame not a multiple of the 32-unit warp run (pair and
    single-block layouts), many frames, and a frame-strided batch."""
    n, h, w = shape
    g = torch.Generator(device="cpu").manual_seed(n * h + w)
    big = torch.randint(0, 256, (n, h * w + 48), dtype=torch.uint8, generator=g).to(cuda)
    x = big.as_strided((n, h, w), (h * w + 48, w, 1))
    want = exact.forward_unscaled(x.cpu().numpy(), level_shift=True)
    for dt in (torch.int32, torch.int16):
        out = torch.full((n, h * w // 64, 8, 8), 7, dtype=dt, device=cuda)
        z = batch.forward_int(x, level_shift=True, out=out)
        torch.cuda.synchronize()
        assert z.data_ptr() == out.data_ptr()
        assert np.array_equal(z.cpu().numpy().astype(np.int64), want)


@pytest.mark.parametrize("r", [1, 2, 3, 6, 10, 15, 25, 36, 45, 55, 63, 64])
def test_retain_matches_oracle(cuda, r):
    x = _imgs(cuda, [3, 4])
    rec, sse, ssef = batch.compress_retain(x, r, unrounded_sse=True)
    rec2, sse2, _ = batch.compress_retain(x, r)
    torch.cuda.synchronize()
    want_rec, want_sse, want_ssef = exact.compress_retain(x.cpu().numpy(), r)
    assert np.array_equal(rec.cpu().numpy(), want_rec)
    assert np.array_equal(rec2.cpu().numpy(), want_rec)  # pruned kernel == runtime-r kernel
    assert np.array_equal(sse.cpu().numpy(), want_sse)
    assert np.array_equal(sse2.cpu().numpy(), want_sse)
    assert np.array_equal(ssef.cpu().numpy(), want_ssef)


@pytest.mark.parametrize("r", list(range(1, 65)))
def test_retain_every_r_random_noise(cuda, r):
    """Full-range random pixels stress the 16-bit-lane bounds for every r."""
    g = torch.Generator().manual_seed(r)
    x = torch.randint(0, 256, (2, 64, 128), dtype=torch.uint8, generator=g)
    x[0, :32] = 255 * (x[0, :32] > 127)  # saturated edges
    xd = x.to(cuda)
    rec, sse, _ = batch.compress_retain(xd, r)
    torch.cuda.synchronize()
    want_rec, want_sse, _ = exact.compress_retain(x.numpy(), r)
    assert np.array_equal(rec.cpu().numpy(), want_rec)
    assert np.array_equal(sse.cpu().numpy(), want_sse)


@pytest.mark.parametrize("q", [1, 5, 10, 25, 50, 75, 90, 100])
def test_quant_matches_oracle(cuda, q):
    x = _imgs(cuda, [7, 8], 256, 256, cfg=2)
    g = torch.Generator().manual_seed(q)
    noise = torch.randint(0, 256, (1, 256, 256), dtype=torch.uint8, generator=g).to(cuda)
    x = torch.cat([x, noise])
    qt = quant.quant_table(q)
    rec, sse = batch.compress_quant(x, qt)
    torch.cuda.synchronize()
    want_rec, want_sse = exact.compress_quant(x.cpu().numpy(), exact.qprime(quant.q50_luma(), q))
    assert np.array_equal(rec.cpu().numpy(), want_rec)
    assert np.array_equal(sse.cpu().numpy(), want_sse)


@pytest.mark.parametrize("kind", ["huge", "mixed"])
def test_quant_custom_tables(cuda, kind):
    """Tables outside the JPEG-quality family: Q' up to 2^20 (the scalar
    quantiser's post-shift variant) and an odd/even/1 mix in the packed range."""
    rng = np.random.default_rng(11 if kind == "huge" else 12)
    if kind == "huge":
        qpu = rng.choice([1.0, 7.0, 40000.0, 65536.0, 300001.0, 1048576.0], size=(8, 8))
    else:
        qpu = rng.choice([1.0, 2.0, 3.0, 4.0, 6.0, 8.0, 12.0, 16.49, 16.5, 255.0], size=(8, 8))
    qt = quant.quant_table(qprime_unrounded=qpu)
    assert qt.wide == (1 if kind == "huge" else 0)
    x = _imgs(cuda, [21, 22], 128, 256, cfg=2)
    noise = torch.randint(0, 256, (1, 128, 256), dtype=torch.uint8,
                          generator=torch.Generator().manual_seed(5)).to(cuda)
    x = torch.cat([x, noise])
    rec, sse = batch.compress_quant(x, qt)
    torch.cuda.synchronize()
    want_rec, want_sse = exact.compress_quant(x.cpu().numpy(), quant.qtab_qprime(qt))
    assert np.array_equal(rec.cpu().numpy(), want_rec)
    assert np.array_equal(sse.cpu().numpy(), want_sse)


def test_ragged_width_retain_and_quant(cuda):
    g = torch.Generator().manual_seed(11)
    x = torch.randint(0, 256, (3, 24, 40), dtype=torch.uint8, generator=g)  # W % 16 == 8
    xd = x.to(cuda)
    rec, sse, _ = batch.compress_retain(xd, 10)
    qt = quant.quant_table(50)
    recq, sseq = batch.compress_quant(xd, qt)
    torch.cuda.synchronize()
    wr, ws, _ = exact.compress_retain(x.numpy(), 10)
    wq, wqs = exact.compress_quant(x.numpy(), exact.qprime(quant.q50_luma(), 50))
    assert np.array_equal(rec.cpu().numpy(), wr) and np.array_equal(sse.cpu().numpy(), ws)
    assert np.array_equal(recq.cpu().numpy(), wq) and np.array_equal(sseq.cpu().numpy(), wqs)


@pytest.mark.parametrize("q", [10, 75])
def test_planes_quant_one_launch(cuda, q):
    """Y + Cb + Cr in one launch: q = 75 on the packed kernel, q = 10 on the
    float-pair-inverse kernel (tiles of 128 units; the planes' unit counts are
    not multiples of the tile)."""
    g = torch.Generator().manual_seed(5)
    y = torch.randint(0, 256, (2, 64, 96), dtype=torch.uint8, generator=g)
    cb = torch.randint(0, 256, (2, 32, 48), dtype=torch.uint8, generator=g)
    cr = torch.randint(0, 256, (2, 32, 48), dtype=torch.uint8, generator=g)
    qt = quant.quant_table(q)
    recs, sse = batch.compress_quant_planes([y.to(cuda), cb.to(cuda), cr.to(cuda)], qt)
    torch.cuda.synchronize()
    qp = exact.qprime(quant.q50_luma(), q)
    for k, p in enumerate((y, cb, cr)):
        wr, ws = exact.compress_quant(p.numpy(), qp)
        assert np.array_equal(recs[k].cpu().numpy(), wr)
        assert np.array_equal(sse[:, k].cpu().numpy(), ws)


@pytest.mark.parametrize("r", [1, 10, 64])
def test_planes_retain_one_launch(cuda, r):
    """adct_compress_retain_planes: Y + Cb + Cr in one launch with per-frame,
    per-plane SSE; then planes whose 24-px width cannot pair blocks."""
    g = torch.Generator().manual_seed(6 + r)
    y = torch.randint(0, 256, (3, 72, 128), dtype=torch.uint8, generator=g)
    cb = torch.randint(0, 256, (3, 40, 64), dtype=torch.uint8, generator=g)
    cr = torch.randint(0, 256, (3, 40, 64), dtype=torch.uint8, generator=g)
    recs, sse = batch.compress_retain_planes([y.to(cuda), cb.to(cuda), cr.to(cuda)], r)
    torch.cuda.synchronize()
    for k, p in enumerate((y, cb, cr)):
        wr, ws, _ = exact.compress_retain(p.numpy(), r)
        assert np.array_equal(recs[k].cpu().numpy(), wr)
        assert np.array_equal(sse[:, k].cpu().numpy(), ws)
    y2 = torch.randint(0, 256, (2, 16, 24), dtype=torch.uint8, generator=g)  # 24 px: single-block units
    c2 = torch.randint(0, 256, (2, 8, 16), dtype=torch.uint8, generator=g)
    recs2, sse2 = batch.compress_retain_planes([y2.to(cuda), c2.to(cuda)], r)
    torch.cuda.synchronize()
    for k, p in enumerate((y2, c2)):
        wr, ws, _ = exact.compress_retain(p.numpy(), r)
        assert np.array_equal(recs2[k].cpu().numpy(), wr)
        assert np.array_equal(sse2[:, k].cpu().numpy(), ws)


@pytest.mark.parametrize("shape,r_min,r_max", [((3, 40, 24), 1, 64), ((2, 72, 144), 7, 30),
                                               ((5, 16, 2048), 64, 64), ((1, 8, 8), 2, 2)])
@pytest.mark.parametrize("kernel", ["inc", "full"])
def test_sweep_shapes_and_ranges(cuda, shape, r_min, r_max, kernel):
    """Both sweep kernels (incremental basis updates / full masked inverse,
    selected by ADCT_SWEEP_KERNEL in a child process) over unpaired widths,
    partial CTAs, r ranges not starting at 1, and a single r."""
    import os
    import subprocess
    import sys

    g = torch.Generator().manual_seed(sum(shape) + r_min)
    x = torch.randint(0, 256, shape, dtype=torch.uint8, generator=g)
    want = exact.sweep_sse(x.numpy(), r_min, r_max)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys, numpy as np, torch\n"
        "from paper_1702_00817_b200 import batch\n"
        "x = torch.from_numpy(np.load(sys.argv[1])).cuda()\n"
        f"s = batch.sweep_retain_sse(x, {r_min}, {r_max})\n"
        f"s2, sf = batch.sweep_retain_sse_unrounded(x, {r_min}, {r_max})\n"
        "assert torch.equal(s, s2)\n"
        "np.save(sys.argv[2], np.stack([s.cpu().numpy(), sf.cpu().numpy()]))\n"
    )
    import tempfile

    with tempfile.TemporaryDirectory() as td:
        np.save(os.path.join(td, "x.npy"), x.numpy())
        env = dict(os.environ, ADCT_SWEEP_KERNEL=kernel, PYTHONPATH=root)
        r = subprocess.run([sys.executable, "-c", code, os.path.join(td, "x.npy"), os.path.join(td, "s.npy")],
                           env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-3000:]
        got = np.load(os.path.join(td, "s.npy"))
    assert np.array_equal(got[0], want)
    want_f = np.stack([exact.compress_retain(x.numpy(), r)[2] for r in range(r_min, r_max + 1)], axis=1)
    assert np.array_equal(got[1], want_f)


def test_sweep_matches_oracle(cuda):
    x = _imgs(cuda, [0, 1, 2], 128, 128)
    s = batch.sweep_retain_sse(x, 1, 45)
    torch.cuda.synchronize()
    assert np.array_equal(s.cpu().numpy(), exact.sweep_sse(x.cpu().numpy(), 1, 45))


def test_empty_batch(cuda):
    x = torch.empty((0, 64, 64), dtype=torch.uint8, device=cuda)
    rec, sse, _ = batch.compress_retain(x, 10)
    assert rec.shape == (0, 64, 64) and sse.shape == (0,)


@pytest.mark.parametrize("env", [{"ADCT_QUANT_KERNEL": "grid"}, {"ADCT_WIDE_KERNEL": "scalar"},
                                 {"ADCT_PIPELINE_DEPTH": "2"}, {"ADCT_QUANT_FLOAT": "0"},
                                 {"ADCT_QUANT_FLOAT": "0", "ADCT_WIDE_KERNEL": "scalar"},
                                 {"ADCT_PIPELINE_THREADS": "1"}, {"ADCT_QUANT_JIT_AFTER": "1"},
                                 {"ADCT_FI_KERNEL": "all"}, {"ADCT_FI_KERNEL": "all", "ADCT_QUANT_JIT_AFTER": "1"},
                                 {"ADCT_FI_KERNEL": "all", "ADCT_FI_THREADS": "256"},
                                 {"ADCT_FI_KERNEL": "off"}])
def test_alternate_kernel_paths(cuda, env):
    """The A/B switches keep their kernels exact: one-tile-per-CTA quant
    kernel, scalar coarse-table kernel, the float-pair-inverse kernel for every
    table (generic and table-specialised, both tile sizes) or for none (the
    32-bit hybrid), a 2-deep host pipeline (child process: the switches are
    read once per process)."""
    import os
    import subprocess
    import sys
    import tempfile

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r'''
import sys, numpy as np, torch
from oracle import exact
from paper_1702_00817_b200 import batch, quant
from paper_1702_00817_b200.pipeline import HostPipeline
g = torch.Generator().manual_seed(3)
for shape in ((3, 64, 256), (2, 40, 24)):
    x = torch.randint(0, 256, shape, dtype=torch.uint8, generator=g)
    for q in (2, 10, 30, 75, 95):
        qt = quant.quant_table(q)
        rec, sse = batch.compress_quant(x.cuda(), qt)
        wr, ws = exact.compress_quant(x.numpy(), quant.qtab_qprime(qt))
        assert np.array_equal(rec.cpu().numpy(), wr) and np.array_equal(sse.cpu().numpy(), ws), (shape, q)
    with HostPipeline(0, chunk_bytes=1 << 15) as p:
        out = np.empty(shape, np.uint8)
        _, s2 = p.compress_retain(x.numpy(), 10, out)
        wr, ws, _ = exact.compress_retain(x.numpy(), 10)
        assert np.array_equal(out, wr) and np.array_equal(s2, ws)
print("ALT_OK")
'''
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, PYTHONPATH=root, **env),
                       capture_output=True, text=True, timeout=300)
    assert "ALT_OK" in r.stdout, r.stderr[-3000:]


def test_float_inverse_at_its_acceptance_limit(cuda):
    """Custom tables whose sum(Q'E) sits just under k_quant_fi's exactness
    bound (capi.cu fi_exact; the same tables tests/test_fi_model.py checks in
    a float32 model): the kernel on adversarial blocks equals the oracle."""
    rng = np.random.default_rng(99)
    budget = 2 * (2.0**24 - 64 * 8192 - 8224) - 1
    checker = ((np.indices((8, 8)).sum(axis=0) % 2) * 255).astype(np.uint8)
    for _ in range(4):
        w = rng.random((8, 8))
        qp = np.maximum(1, np.floor(budget * w / w.sum() / exact.E)).astype(np.int64)
        qt = quant.quant_table(qprime_unrounded=qp.astype(np.float64))
        assert np.array_equal(quant.qtab_qprime(qt), qp)
        x = np.concatenate([np.tile(checker, (2, 4)), (rng.integers(0, 2, (16, 32)) * 255).astype(np.uint8),
                            rng.integers(0, 256, (16, 32)).astype(np.uint8)])[None]
        rec, sse = batch.compress_quant(torch.from_numpy(x).to(cuda), qt)
        wr, ws = exact.compress_quant(x, qp)
        assert np.array_equal(rec.cpu().numpy(), wr) and np.array_equal(sse.cpu().numpy(), ws)
