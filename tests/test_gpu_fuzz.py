"""Seeded randomized parity: random batch shapes (multiples of 8, paired and
unpaired widths), frame-strided inputs, random r / quality / custom Q' tables,
with and without reconstructions — every fused entry point against the
oracle, bit-exact."""

import numpy as np
import pytest
import torch

from oracle import exact
from paper_1702_00817_b200 import batch, quant

pytestmark = pytest.mark.gpu

CASES = 24


def _batch(rng, cuda):
    n = int(rng.integers(1, 5))
    h = 8 * int(rng.integers(1, 12))
    w = 8 * int(rng.integers(1, 40))
    pad = 16 * int(rng.integers(0, 3))
    kind = rng.integers(0, 3)
    if kind == 0:  # uniform noise
        x = rng.integers(0, 256, (n, h * w + pad), dtype=np.uint8)
    elif kind == 1:  # saturated extremes (clamp paths)
        x = (rng.integers(0, 2, (n, h * w + pad)) * 255).astype(np.uint8)
    else:  # smooth ramp + noise
        base = (np.arange(h * w + pad) * 7 % 256).astype(np.int64)
        x = np.clip(base[None, :] + rng.integers(-20, 21, (n, h * w + pad)), 0, 255).astype(np.uint8)
    t = torch.from_numpy(x).to(cuda)
    view = t.as_strided((n, h, w), (h * w + pad, w, 1))
    host = np.stack([x[k, : h * w].reshape(h, w) for k in range(n)])
    return view, host


@pytest.mark.parametrize("case", range(CASES))
def test_random_retain(cuda, case):
    rng = np.random.default_rng(1000 + case)
    x, host = _batch(rng, cuda)
    r = int(rng.integers(1, 65))
    want_rec, want_sse, want_ssef = exact.compress_retain(host, r)
    rec, sse, ssef = batch.compress_retain(x, r, unrounded_sse=bool(case % 2))
    torch.cuda.synchronize()
    assert np.array_equal(rec.cpu().numpy(), want_rec)
    assert np.array_equal(sse.cpu().numpy(), want_sse)
    if ssef is not None:
        assert np.array_equal(ssef.cpu().numpy(), want_ssef)
    _, sse_only, _ = batch.compress_retain(x, r, reconstruct=False)
    torch.cuda.synchronize()
    assert np.array_equal(sse_only.cpu().numpy(), want_sse)


@pytest.mark.parametrize("case", range(CASES))
def test_random_quant(cuda, case):
    rng = np.random.default_rng(2000 + case)
    x, host = _batch(rng, cuda)
    if case % 3 == 2:  # custom unrounded table, mixed magnitudes
        qpu = rng.choice([1.0, 2.0, 2.5, 3.0, 7.49, 7.5, 16.0, 33.3, 100.0, 999.0, 8191.0, 9000.0], size=(8, 8))
        qt = quant.quant_table(qprime_unrounded=qpu)
    else:
        qt = quant.quant_table(int(rng.integers(1, 101)))
    qp = quant.qtab_qprime(qt)
    want_rec, want_sse = exact.compress_quant(host, qp)
    rec, sse = batch.compress_quant(x, qt)
    torch.cuda.synchronize()
    assert np.array_equal(rec.cpu().numpy(), want_rec), (qt.wide, qt.aligned)
    assert np.array_equal(sse.cpu().numpy(), want_sse)


@pytest.mark.parametrize("case", range(8))
def test_random_sweep_and_forward(cuda, case):
    rng = np.random.default_rng(3000 + case)
    x, host = _batch(rng, cuda)
    r0 = int(rng.integers(1, 65))
    r1 = int(rng.integers(r0, 65))
    s = batch.sweep_retain_sse(x, r0, r1)
    z = batch.forward_int(x, level_shift=bool(case % 2))
    torch.cuda.synchronize()
    assert np.array_equal(s.cpu().numpy(), exact.sweep_sse(host, r0, r1))
    assert np.array_equal(z.cpu().numpy().astype(np.int64), exact.forward_unscaled(host, level_shift=bool(case % 2)))


def test_random_quant_all_tables_on_float_inverse(cuda):
    """The float-pair-inverse kernel (k_quant_fi) for every table, not only
    the coarse ones it runs by default (ADCT_FI_KERNEL=all; child process:
    the switch is read once per process): the random quant cases again."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r'''
import numpy as np, torch, test_gpu_fuzz as F
from oracle import exact
from paper_1702_00817_b200 import batch, quant
cuda = torch.device("cuda", 0)
for case in range(F.CASES):
    rng = np.random.default_rng(5000 + case)
    x, host = F._batch(rng, cuda)
    if case % 3 == 2:
        qpu = rng.choice([1.0, 2.0, 2.5, 3.0, 7.49, 7.5, 16.0, 33.3, 100.0, 999.0, 8191.0, 9000.0], size=(8, 8))
        qt = quant.quant_table(qprime_unrounded=qpu)
    else:
        qt = quant.quant_table(int(rng.integers(1, 101)))
    want_rec, want_sse = exact.compress_quant(host, quant.qtab_qprime(qt))
    rec, sse = batch.compress_quant(x, qt)
    assert np.array_equal(rec.cpu().numpy(), want_rec) and np.array_equal(sse.cpu().numpy(), want_sse), case
print("FI_ALL_OK")
'''
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, PYTHONPATH=os.pathsep.join([root, os.path.join(root, "tests")]),
                                                        ADCT_FI_KERNEL="all"),
                       capture_output=True, text=True, timeout=300, cwd=root)
    assert "FI_ALL_OK" in r.stdout, r.stderr[-3000:]
