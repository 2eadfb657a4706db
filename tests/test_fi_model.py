"""CPU model of k_quant_fi's float arithmetic (csrc/adct_kernels.cuh, K3f).

The kernel's exactness claim is that, for every table the host accepts
(capi.cu fi_exact: 64*8192 + 8224 + sum(Q'E)/2 < 2^24), no FP32 operation of
the dequantise-and-inverse part ever rounds.  This test re-executes that part
in numpy with one float32 rounding after every operation, in the kernel's
order (inv8_dq: FFMA chains with +-k = Q'E/64, DC offset 128.5; inv8: FADD
rows; floor; clamp), on adversarial blocks (saturated checkerboards, stripes,
noise), and requires the result to equal the exact integer oracle.  The
quantised integers q come from the oracle: the device quantiser is verified
exhaustively by adct_qtab_build on its own."""

import numpy as np
import pytest

from oracle import exact
from paper_1702_00817_b200 import quant


def f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def fma(a, b, c):  # one rounding, like FFMA (the float64 product and sum are exact here)
    return f32(np.asarray(a, np.float64) * np.asarray(b, np.float64) + np.asarray(c, np.float64))


def inv8_dq(q, k, dc):
    """q, k: (..., 8) along u; returns x (..., 8) along i (kernel inv8_dq)."""
    X0 = fma(q[..., 0], k[..., 0], dc)
    b0, b1 = fma(q[..., 4], k[..., 4], X0), fma(q[..., 4], -k[..., 4], X0)
    a0, a3 = fma(q[..., 2], k[..., 2], b0), fma(q[..., 2], -k[..., 2], b0)
    a1, a2 = fma(q[..., 6], -k[..., 6], b1), fma(q[..., 6], k[..., 6], b1)
    x = [fma(q[..., 1], k[..., 1], a0), fma(q[..., 5], -k[..., 5], a1), fma(q[..., 3], -k[..., 3], a2),
         fma(q[..., 7], -k[..., 7], a3), fma(q[..., 7], k[..., 7], a3), fma(q[..., 3], k[..., 3], a2),
         fma(q[..., 5], k[..., 5], a1), fma(q[..., 1], -k[..., 1], a0)]
    return np.stack(x, axis=-1)


def inv8(X):
    """Plain inv8 with a float32 rounding after every add (kernel FADD2 rows)."""
    b0, b1 = f32(X[..., 0] + X[..., 4]), f32(X[..., 0] - X[..., 4])
    a0, a3 = f32(b0 + X[..., 2]), f32(b0 - X[..., 2])
    a1, a2 = f32(b1 - X[..., 6]), f32(b1 + X[..., 6])
    x = [f32(a0 + X[..., 1]), f32(a1 - X[..., 5]), f32(a2 - X[..., 3]), f32(a3 - X[..., 7]),
         f32(a3 + X[..., 7]), f32(a2 + X[..., 3]), f32(a1 + X[..., 5]), f32(a0 - X[..., 1])]
    return np.stack(x, axis=-1)


def fi_model(blocks: np.ndarray, qp: np.ndarray, qe: np.ndarray) -> np.ndarray:
    """(N, 8, 8) uint8 blocks -> reconstructed uint8 blocks, the kernel's way."""
    Z = np.einsum("ui,nij,vj->nuv", exact.T, blocks.astype(np.int64) - 128, exact.T)
    q = exact.quantize(Z, qp).astype(np.float64)
    k = f32(qe.astype(np.float64) / 64.0)
    # column pass: for each column v, inverse along u (dc only on column 0)
    cols = []
    for v in range(8):
        dc = np.full(blocks.shape[0], 128.5 if v == 0 else 0.0)
        if v == 0:
            cv = inv8_dq(q[:, :, v], k[:, v], dc)
        else:  # FMUL for the DC term of the other columns: the same as an FFMA with 0
            cv = inv8_dq(q[:, :, v], k[:, v], 0.0)
        cols.append(cv)  # (N, 8) over i
    c = np.stack(cols, axis=-1)  # (N, i, v)
    y = inv8(c)  # rows: (N, i, j)
    return np.clip(np.floor(y), 0, 255).astype(np.uint8)


def _adversarial_blocks(rng, n):
    checker = ((np.indices((8, 8)).sum(axis=0) % 2) * 255).astype(np.uint8)
    stripes_v = np.tile((np.arange(8) % 2 * 255).astype(np.uint8), (8, 1))
    stripes_h = stripes_v.T.copy()
    halves = np.zeros((8, 8), np.uint8)
    halves[:, 4:] = 255
    fixed = np.stack([checker, 255 - checker, stripes_v, stripes_h, halves, 255 - halves,
                      np.zeros((8, 8), np.uint8), np.full((8, 8), 255, np.uint8)])
    sat = (rng.integers(0, 2, (n, 8, 8)) * 255).astype(np.uint8)
    noise = rng.integers(0, 256, (n, 8, 8)).astype(np.uint8)
    return np.concatenate([fixed, sat, noise])


def _fi_accepts(qe: np.ndarray) -> bool:  # capi.cu fi_exact
    return 64 * 8192 + 8224 + qe.astype(np.float64).sum() / 2 < 2.0**24


@pytest.mark.parametrize("q", [1, 2, 5, 10, 15, 19, 25, 50, 75, 90, 100])
def test_fi_float_model_is_exact_for_quality_tables(q):
    rng = np.random.default_rng(q)
    qt = quant.quant_table(q)
    qp = quant.qtab_qprime(qt)
    qe = np.asarray(qt.qe, dtype=np.int64).reshape(8, 8)
    assert np.array_equal(qe, qp * exact.E)
    assert _fi_accepts(qe)
    blocks = _adversarial_blocks(rng, 400)
    want = exact.compress_quant(blocks.reshape(-1, 8, 8), qp)[0]
    assert np.array_equal(fi_model(blocks, qp, qe), want)


def test_fi_float_model_is_exact_at_the_acceptance_limit():
    """Custom tables with sum(Q'E) just under the fi_exact bound: the largest
    magnitudes the kernel may see still never round."""
    rng = np.random.default_rng(99)
    budget = 2 * (2.0**24 - 64 * 8192 - 8224) - 1
    for _ in range(6):
        w = rng.random((8, 8))
        qe_f = budget * w / w.sum()
        qp = np.maximum(1, np.floor(qe_f / exact.E)).astype(np.int64)
        qe = qp * exact.E
        assert _fi_accepts(qe)
        blocks = _adversarial_blocks(rng, 200)
        want = exact.compress_quant(blocks, qp)[0]
        assert np.array_equal(fi_model(blocks, qp, qe), want)
