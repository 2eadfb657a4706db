"""Out-of-bounds write detection without compute-sanitizer (closed on this
GPU pool): every entry point that writes device memory runs on an interior
view of a sentinel-filled buffer; the guard bands and the frame-stride gaps
must come back untouched, and the interior must be exact."""

import numpy as np
import pytest
import torch

from oracle import exact
from paper_1702_00817_b200 import batch, quant

pytestmark = pytest.mark.gpu
GUARD = 4096
SENT8 = 0xA5


def _guarded_u8(cuda, n, h, w, gap):
    """(view (n, h, w) with frame stride h*w + gap, whole buffer, guard slices)."""
    total = GUARD + n * (h * w + gap) + GUARD
    buf = torch.full((total,), SENT8, dtype=torch.uint8, device=cuda)
    view = buf[GUARD:].as_strided((n, h, w), (h * w + gap, w, 1))
    return view, buf


def _outside_untouched(buf, n, h, w, gap):
    b = buf.cpu().numpy()
    inside = np.zeros(b.size, dtype=bool)
    for k in range(n):
        s = GUARD + k * (h * w + gap)
        inside[s:s + h * w] = True
    return bool((b[~inside] == SENT8).all())


SHAPES = [(3, 40, 24, 16), (2, 64, 144, 48), (1, 8, 8, 0), (4, 16, 2048, 32)]


@pytest.mark.parametrize("n,h,w,gap", SHAPES)
def test_retain_and_quant_write_only_their_frames(cuda, n, h, w, gap):
    g = torch.Generator().manual_seed(n * w + gap)
    x = torch.randint(0, 256, (n, h, w), dtype=torch.uint8, generator=g)
    src, _ = _guarded_u8(cuda, n, h, w, gap)
    src.copy_(x.to(cuda))
    for run in ("retain", "quant10", "quant75"):
        out, obuf = _guarded_u8(cuda, n, h, w, gap)
        sse_buf = torch.full((n + 64,), -7, dtype=torch.int64, device=cuda)
        sse = sse_buf[32:32 + n]
        if run == "retain":
            batch.compress_retain(src, 10, out=out, sse_out=sse)
            want_rec, want_sse, _ = exact.compress_retain(x.numpy(), 10)
        else:
            qt = quant.quant_table(int(run[5:]))
            batch.compress_quant(src, qt, out=out, sse_out=sse)
            want_rec, want_sse = exact.compress_quant(x.numpy(), quant.qtab_qprime(qt))
        torch.cuda.synchronize()
        assert _outside_untouched(obuf, n, h, w, gap), run
        assert np.array_equal(out.cpu().numpy(), want_rec), run
        assert np.array_equal(sse.cpu().numpy(), want_sse), run
        s = sse_buf.cpu().numpy()
        assert (s[:32] == -7).all() and (s[32 + n:] == -7).all(), run


@pytest.mark.parametrize("n,h,w,gap", SHAPES)
def test_forward_and_sweep_write_only_their_outputs(cuda, n, h, w, gap):
    g = torch.Generator().manual_seed(7 + n * w + gap)
    x = torch.randint(0, 256, (n, h, w), dtype=torch.uint8, generator=g)
    src, _ = _guarded_u8(cuda, n, h, w, gap)
    src.copy_(x.to(cuda))
    nb = h * w // 64
    for dt in (torch.int32, torch.int16):
        cbuf = torch.full((GUARD + n * nb * 64 + GUARD,), -3, dtype=dt, device=cuda)
        coef = cbuf[GUARD:GUARD + n * nb * 64].view(n, nb, 8, 8)
        batch.forward_int(src, out=coef)
        torch.cuda.synchronize()
        c = cbuf.cpu().numpy()
        assert (c[:GUARD] == -3).all() and (c[GUARD + n * nb * 64:] == -3).all()
        assert np.array_equal(coef.cpu().numpy().astype(np.int64), exact.forward_unscaled(x.numpy()))
    s = batch.sweep_retain_sse(src, 3, 9)
    torch.cuda.synchronize()
    assert s.shape == (n, 7)
    assert np.array_equal(s.cpu().numpy(), exact.sweep_sse(x.numpy(), 3, 9))


@pytest.mark.parametrize("h,w", [(8, 65536), (65536, 16), (8, 8), (16384, 16384)])
def test_extreme_geometries(cuda, h, w):
    """Row-index arithmetic at the extremes: one block row of 4096 units,
    one unit per block row (upr == 1), a single block, and a 256 MiB image.
    Full oracle comparison where it is cheap, sampled otherwise."""
    g = torch.Generator().manual_seed(h + w)
    x = torch.randint(0, 256, (1, h, w), dtype=torch.uint8, generator=g).to(cuda)
    rec, sse, _ = batch.compress_retain(x, 10)
    qt = quant.quant_table(50)
    recq, sseq = batch.compress_quant(x, qt)
    torch.cuda.synchronize()
    if h * w <= (1 << 20):
        host = x.cpu().numpy()
        wr, ws, _ = exact.compress_retain(host, 10)
        assert np.array_equal(rec.cpu().numpy(), wr) and np.array_equal(sse.cpu().numpy(), ws)
        wq, wqs = exact.compress_quant(host, quant.qtab_qprime(qt))
        assert np.array_equal(recq.cpu().numpy(), wq) and np.array_equal(sseq.cpu().numpy(), wqs)
    else:  # 8-row bands at the start, middle and end: blocks are independent
        for r0 in (0, h // 2, h - 64):
            band = x[:, r0:r0 + 64].contiguous().cpu().numpy()
            wr, _, _ = exact.compress_retain(band, 10)
            assert np.array_equal(rec[:, r0:r0 + 64].cpu().numpy(), wr), r0
            wq, _ = exact.compress_quant(band, quant.qtab_qprime(qt))
            assert np.array_equal(recq[:, r0:r0 + 64].cpu().numpy(), wq), r0
        d = rec.to(torch.int64) - x.to(torch.int64)
        assert int(sse[0]) == int((d * d).sum())
        dq = recq.to(torch.int64) - x.to(torch.int64)
        assert int(sseq[0]) == int((dq * dq).sum())


@pytest.mark.parametrize("h,w", [(8, 65536), (65536, 16), (8, 16), (16384, 16384)])
def test_extreme_geometries_float_inverse(cuda, h, w):
    """The same extremes through k_quant_fi (q = 10: 128-unit tiles, the
    park in shared memory): exact where cheap, sampled bands otherwise."""
    g = torch.Generator().manual_seed(3 * h + w)
    x = torch.randint(0, 256, (1, h, w), dtype=torch.uint8, generator=g).to(cuda)
    qt = quant.quant_table(10)
    recq, sseq = batch.compress_quant(x, qt)
    torch.cuda.synchronize()
    if h * w <= (1 << 20):
        wq, wqs = exact.compress_quant(x.cpu().numpy(), quant.qtab_qprime(qt))
        assert np.array_equal(recq.cpu().numpy(), wq) and np.array_equal(sseq.cpu().numpy(), wqs)
    else:
        for r0 in (0, h // 2, h - 64):
            band = x[:, r0:r0 + 64].contiguous().cpu().numpy()
            wq, _ = exact.compress_quant(band, quant.qtab_qprime(qt))
            assert np.array_equal(recq[:, r0:r0 + 64].cpu().numpy(), wq), r0
        dq = recq.to(torch.int64) - x.to(torch.int64)
        assert int(sseq[0]) == int((dq * dq).sum())


def test_more_frames_than_one_grid_row(cuda):
    """More than 65,535 frames: the launches are chunked along grid.y
    (frame_base), the persistent quant kernel walks them in one grid.  Every
    kernel family, exact against the oracle on every frame."""
    n = 65_535 + 70
    g = torch.Generator().manual_seed(65)
    x = torch.randint(0, 256, (n, 8, 16), dtype=torch.uint8, generator=g)
    xd, xh = x.to(cuda), x.numpy()
    rec, sse, _ = batch.compress_retain(xd, 10)
    wr, ws, _ = exact.compress_retain(xh, 10)
    assert np.array_equal(rec.cpu().numpy(), wr) and np.array_equal(sse.cpu().numpy(), ws)
    for q in (75, 10):  # k_quant_p (persistent), k_quant_fi (chunked)
        qt = quant.quant_table(q)
        recq, sseq = batch.compress_quant(xd, qt)
        wq, wqs = exact.compress_quant(xh, quant.qtab_qprime(qt))
        assert np.array_equal(recq.cpu().numpy(), wq), q
        assert np.array_equal(sseq.cpu().numpy(), wqs), q
    z = batch.forward_int(xd)
    assert np.array_equal(z.cpu().numpy().astype(np.int64), exact.forward_unscaled(xh))
    s = batch.sweep_retain_sse(xd, 1, 12)
    assert np.array_equal(s.cpu().numpy(), exact.sweep_sse(xh, 1, 12))
    c = batch.forward_f64(xd)
    back = batch.inverse_f64(c, 8, 16, r=64)
    assert float((back - xd.to(torch.float64)).abs().max()) < 1e-9
