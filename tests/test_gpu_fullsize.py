"""GPU parity at BASELINE.json's stated sizes (every config, every image).

Each test runs the entry point bench.py times for that config on the full
seeded workload and compares every output with the plain-C exact oracle
(oracle/fast.py -> oracle/exact_c.c, pinned to oracle/exact.py and to the
reference-made golden vectors by tests/test_oracle.py):

* C1  45 x 512^2, seeds 0..44, SSE for every r = 1..45 (adct_sweep_retain_sse):
      rounded SSE and the reference's unrounded SSE bit-exact, per-image and
      mean PSNR, and the reference's own float64 algorithm (oracle/refport.py)
      within BASELINE's 1e-5 relative MSE / 1e-3 dB.
* C2  256 x 1024^2, q = 10, 50, 90 (batch.compress_quant): every image's SSE and
      every reconstructed byte, for the generic and the table-specialised kernel.
* C3  4096 x 2048^2, r = 10 (batch.compress_retain): the whole 16 GiB batch,
      every SSE and every reconstructed byte (compared in 1 GiB chunks).
* C4  512 frames of 3840x2160 4:2:0, q = 75 (adct_compress_quant_planes):
      every frame's per-plane SSE and every reconstructed byte.
"""

import numpy as np
import pytest
import torch

from oracle import exact, fast, refport
from paper_1702_00817_b200 import batch, quant, synth

pytestmark = pytest.mark.gpu


def _jit_launches():
    import ctypes

    from paper_1702_00817_b200 import _lib

    c, l, f = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _lib.lib().adct_quant_jit_stats(ctypes.byref(c), ctypes.byref(l), ctypes.byref(f))
    return l.value


def test_config1_full_sweep(cuda):
    imgs = synth.config_images_device(1, range(45), device=cuda)
    sse, ssef = batch.sweep_retain_sse_unrounded(imgs, 1, 45)
    # the bench's launch (rounded SSE only) gives the same rounded SSE
    sse_bench = batch.sweep_retain_sse(imgs, 1, 45)
    host = imgs.cpu().numpy()
    want, wantf = fast.sweep_sse(host, 1, 45)
    assert np.array_equal(sse.cpu().numpy(), want)
    assert np.array_equal(sse_bench.cpu().numpy(), want)
    assert np.array_equal(ssef.cpu().numpy(), wantf)
    npx = 512 * 512
    # per-image and corpus-mean PSNR (metrics.summarize default: mean of per-image PSNR)
    p_gpu = batch.psnr_from_sse(sse, npx)
    p_want = exact.psnr(want, npx)
    assert np.array_equal(p_gpu, p_want)
    assert np.array_equal(p_gpu.mean(axis=0), p_want.mean(axis=0))
    # BASELINE config 1: "checked against the float64 reference" — the
    # reference's own algorithm (float64 matmuls, unrounded clamped output)
    # against our exact unrounded SSE, every image and r
    for i in range(45):
        y = refport.coefficient_blocks(host[i])
        for k, r in enumerate(range(1, 46)):
            m_ref = refport.mse(host[i], refport.reconstruct_image(y, r, 512, 512))
            m_ours = float(ssef[i, k]) / (4096.0 * npx)
            assert m_ours == pytest.approx(m_ref, rel=1e-5)
            assert abs(refport.psnr(m_ours) - refport.psnr(m_ref)) < 1e-3


@pytest.mark.parametrize("q", [10, 50, 90])
def test_config2_full_quant(cuda, q):
    imgs = synth.config_images_device(2, range(256), device=cuda)
    qt = quant.quant_table(q)
    host = imgs.cpu().numpy()
    want_rec, want_sse = fast.compress_quant(host, quant.qtab_qprime(qt))
    before = _jit_launches()
    for it in range(4):  # generic kernel first, table-specialised from the 3rd use
        rec, sse = batch.compress_quant(imgs, qt)
        assert np.array_equal(sse.cpu().numpy(), want_sse), (q, it)
        assert torch.equal(rec, torch.from_numpy(want_rec).to(cuda)), (q, it)
    if not qt.wide:  # k_quant_p: the specialised kernel ran and was checked too
        assert _jit_launches() > before
    else:  # coarse table: k_quant_fi, which is never specialised
        assert _jit_launches() == before


def test_config3_full_batch(cuda):
    n, h, w = 4096, 2048, 2048
    imgs = synth.config_images_device(3, range(n), device=cuda)
    rec, sse, _ = batch.compress_retain(imgs, 10)
    sse = sse.cpu().numpy()
    chunk = 256  # 1 GiB of images per comparison
    for i0 in range(0, n, chunk):
        host = imgs[i0:i0 + chunk].cpu().numpy()
        want_rec, want_sse, _ = fast.compress_retain(host, 10)
        assert np.array_equal(sse[i0:i0 + chunk], want_sse), i0
        assert torch.equal(rec[i0:i0 + chunk], torch.from_numpy(want_rec).to(cuda)), i0
        del host, want_rec
    del imgs, rec
    torch.cuda.empty_cache()


def test_config4_all_frames(cuda):
    import ctypes

    from paper_1702_00817_b200 import _lib

    frames = 512
    planes = synth.video_planes_device(frames, device=cuda)
    qt = quant.quant_table(75)
    qp = quant.qtab_qprime(qt)
    runs = []
    for it in range(4):  # bench's launch; generic first, table-specialised from the 3rd use
        recs = [torch.empty_like(p) for p in planes]
        arr, _ = batch._planes(planes, recs)
        sse = torch.empty((frames, 3), dtype=torch.int64, device=cuda)
        _lib.call("adct_compress_quant_planes", arr, 3, frames, ctypes.byref(qt), sse.data_ptr(),
                  torch.cuda.current_stream().cuda_stream)
        if it in (0, 3):
            runs.append((recs, sse.cpu().numpy()))
    torch.cuda.synchronize()
    chunk = 64
    for f0 in range(0, frames, chunk):
        for k in range(3):
            host = planes[k][f0:f0 + chunk].cpu().numpy()
            want_rec, want_sse = fast.compress_quant(host, qp)
            want_rec = torch.from_numpy(want_rec).to(cuda)
            for it, (recs, got) in enumerate(runs):
                assert np.array_equal(got[f0:f0 + chunk, k], want_sse), (it, f0, k)
                assert torch.equal(recs[k][f0:f0 + chunk], want_rec), (it, f0, k)
    # the last frames of the drift are real content (not a degenerate frame)
    assert runs[0][1][-1, 0] > 0 and not torch.equal(planes[0][-1], planes[0][0])
