"""GPU: golden fixtures through the CUDA path, the reference-signature
wrappers, the host-buffer pipeline, the device generator, and full-size
configurations checked through size-independent properties."""

import hashlib
import json
import os

import numpy as np
import pytest
import torch

from oracle import exact, refport
from paper_1702_00817_b200 import batch, codec, metrics, quant, synth, transforms
from paper_1702_00817_b200.pipeline import HostPipeline

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = json.load(open(os.path.join(HERE, "golden", "golden.json")))
IMAGES = dict(np.load(os.path.join(HERE, "golden", "images.npz")))
T = transforms.proposed_transform()


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# --- golden vectors (reference results) straight through the CUDA path ---------

def test_config0_golden_int32(cuda):
    x = torch.from_numpy(IMAGES["c0_seed0_512"]).to(cuda)
    z = batch.forward_int(x)[0].cpu().numpy().astype(np.int64)
    g = GOLDEN["config0"]
    assert sha(z) == g["coef_sha256_int64"] and z[:4].tolist() == g["coef_blocks_0_3"]


def test_config0_float_roundtrip(cuda):
    img = IMAGES["c0_seed0_512"]
    y = codec.coefficient_blocks(T, img.astype(np.float64))
    ref = refport.coefficient_blocks(img)
    assert np.abs(y - ref).max() < 1e-9
    back = codec.reconstruct_image(T, y, 64, 512, 512)
    assert np.abs(back - img).max() < 1e-9


@pytest.mark.parametrize("name", ["c0_seed0_512", "c1_seed1_128", "c1_seed2_128", "ragged_40x24", "noise_64", "saturated_32x48"])
def test_config1_golden(cuda, name):
    img = IMAGES[name]
    x = torch.from_numpy(img).to(cuda)
    for r_s, g in GOLDEN["config1"][name].items():
        rec, sse, ssef = batch.compress_retain(x, int(r_s), unrounded_sse=True)
        assert int(sse.item()) == g["sse_rounded"]
        assert sha(rec[0].cpu().numpy()) == g["rec_sha256"]
        mse_ref_conv = ssef.item() / (4096.0 * img.size)
        assert mse_ref_conv == pytest.approx(g["mse_ref"], rel=1e-9, abs=1e-12)
        assert metrics.psnr(mse_ref_conv) == pytest.approx(g["psnr_ref"], abs=1e-9)


@pytest.mark.parametrize("name", ["c2_seed3_128", "noise_64", "saturated_32x48", "ragged_40x24"])
def test_quant_golden(cuda, name):
    x = torch.from_numpy(IMAGES[name]).to(cuda)
    for q_s, g in GOLDEN["quant"][name].items():
        rec, sse = batch.compress_quant(x, quant.quant_table(int(q_s)))
        assert int(sse.item()) == g["sse"] and sha(rec[0].cpu().numpy()) == g["rec_sha256"]


def test_sweep_golden(cuda):
    name = "c1_seed1_128"
    x = torch.from_numpy(IMAGES[name]).to(cuda)
    s = batch.sweep_retain_sse(x, 1, 45)[0].cpu().numpy()
    assert [int(v) for v in s] == [GOLDEN["config1"][name][str(r)]["sse_rounded"] for r in range(1, 46)]


# --- reference-signature wrappers ------------------------------------------------

def test_codec_wrappers_match_reference_float_semantics(cuda):
    img = IMAGES["c1_seed1_128"].astype(np.float64)
    for r in (1, 10, 25, 45, 64):
        ours = codec.compress_image(T, img, r)
        ref = refport.compress_image(img, r)
        assert isinstance(ours, np.ndarray) and ours.dtype == np.float64
        assert np.abs(ours - ref).max() < 1e-9
    blocks = np.random.default_rng(0).normal(100, 40, (5, 8, 8))
    y = codec.forward_2d(T, blocks)
    assert np.abs(y - refport.C @ blocks @ refport.C.T).max() < 1e-9
    assert np.abs(codec.inverse_2d(T, y) - blocks).max() < 1e-9
    single = codec.forward_2d(T, blocks[0])
    assert single.shape == (8, 8)
    ib = np.random.default_rng(1).integers(-1024, 1025, (20, 8, 8))
    assert np.array_equal(codec.forward_2d_unscaled(T, ib), exact.T @ ib @ exact.T.T)
    u8 = IMAGES["noise_64"][:8, :8]
    z = codec.forward_2d_unscaled(T, u8)
    assert z.dtype == np.int64 and np.array_equal(z, exact.T @ u8.astype(np.int64) @ exact.T.T)


def test_codec_non_integral_image(cuda):
    img = np.random.default_rng(3).uniform(0, 255, (32, 40))
    assert np.abs(codec.compress_image(T, img, 10) - refport.compress_image(img, 10)).max() < 1e-9


def test_metrics_mse_on_device(cuda):
    a = IMAGES["noise_64"]
    b = np.roll(a, 1)
    assert metrics.mse(a, b) == refport.mse(a, b)
    ta, tb = torch.from_numpy(a).to(cuda), torch.from_numpy(b).to(cuda)
    assert metrics.mse(ta, tb) == refport.mse(a, b)
    f = a.astype(np.float64) + 0.25
    assert metrics.mse(f, a) == pytest.approx(refport.mse(f, a), rel=1e-12)


def test_wrappers_accept_torch_and_return_torch(cuda):
    x = torch.from_numpy(IMAGES["c1_seed2_128"]).to(cuda).to(torch.float64)
    y = codec.compress_image(T, x, 10)
    assert isinstance(y, torch.Tensor) and y.is_cuda
    assert np.abs(y.cpu().numpy() - refport.compress_image(IMAGES["c1_seed2_128"], 10)).max() < 1e-9


# --- host pipeline (end-to-end API) --------------------------------------------------

@pytest.mark.parametrize("chunk_mb", [1, 8])
def test_host_pipeline_retain_and_quant(cuda, chunk_mb):
    imgs = synth.images_np(range(20, 27), 256, 256, 16, 8.0, 64.0)
    rec = np.empty_like(imgs)
    with HostPipeline(0, chunk_bytes=chunk_mb << 20) as p:
        _, sse = p.compress_retain(imgs, 10, rec)
        wr, ws, _ = exact.compress_retain(imgs, 10)
        assert np.array_equal(rec, wr) and np.array_equal(sse, ws)
        qt = quant.quant_table(75)
        _, sseq = p.compress_quant(imgs, qt, rec)
        wq, wqs = exact.compress_quant(imgs, exact.qprime(quant.q50_luma(), 75))
        assert np.array_equal(rec, wq) and np.array_equal(sseq, wqs)
        _, sse_only = p.compress_retain(imgs, 3)  # SSE only, no reconstruction copy
        assert np.array_equal(sse_only, exact.compress_retain(imgs, 3)[1])
    with HostPipeline(0, chunk_bytes=4096) as p:  # smaller than one image: staging grows
        _, sse_small = p.compress_retain(imgs, 10, rec)
        assert np.array_equal(sse_small, exact.compress_retain(imgs, 10)[1])


@pytest.mark.parametrize("chunk", [1 << 14, 1 << 22])
def test_host_pipeline_planes(cuda, chunk):
    """adct_pipeline_compress_quant_planes: host Y/Cb/Cr frames, chunked by
    frames (small chunk: one frame per chunk, staging grows), with and without
    reconstructions, against the per-plane oracle."""
    rng = np.random.default_rng(9)
    y = rng.integers(0, 256, (5, 48, 64), dtype=np.uint8)
    cb = rng.integers(0, 256, (5, 24, 32), dtype=np.uint8)
    cr = rng.integers(0, 256, (5, 24, 32), dtype=np.uint8)
    for q in (10, 75):
        qt = quant.quant_table(q)
        outs = [np.empty_like(p) for p in (y, cb, cr)]
        with HostPipeline(0, chunk_bytes=chunk) as p:
            got, sse = p.compress_quant_planes([y, cb, cr], qt, outs)
            _, sse_only = p.compress_quant_planes([y, cb, cr], qt)
        qp = quant.qtab_qprime(qt)
        for k, plane in enumerate((y, cb, cr)):
            wr, ws = exact.compress_quant(plane, qp)
            assert np.array_equal(got[k], wr) and np.array_equal(sse[:, k], ws), (q, k)
            assert np.array_equal(sse_only[:, k], ws)


def test_host_pipeline_empty_and_degenerate(cuda):
    """Zero images / frames and zero-size planes are no-ops with well-formed results."""
    from paper_1702_00817_b200 import errors

    with HostPipeline(0) as p:
        e = np.empty((0, 64, 64), np.uint8)
        _, sse = p.compress_retain(e, 10, np.empty_like(e))
        assert sse.shape == (0,)
        _, sseq = p.compress_quant(e, quant.quant_table(50))
        assert sseq.shape == (0,)
        outs, ssep = p.compress_quant_planes([e, np.empty((0, 32, 32), np.uint8)], quant.quant_table(50))
        assert ssep.shape == (0, 2)
        z = np.empty((3, 0, 8), np.uint8)  # zero-height images: exact zero SSE, nothing transferred
        _, sz = p.compress_retain(z, 10)
        assert np.array_equal(sz, np.zeros(3, np.int64))
        with pytest.raises(errors.BadDimensions):
            p.compress_retain(np.zeros((1, 12, 16), np.uint8), 10)
        with pytest.raises(errors.InvalidRetention):
            p.compress_retain(np.zeros((1, 8, 16), np.uint8), 65)


@pytest.mark.parametrize("mode", ["pageable", "register", "pinned_in", "pinned_out"])
def test_host_pipeline_staging_modes(cuda, mode):
    """Pageable numpy arrays go through the library's page-locked ring (many
    chunks per call, so every ring slot is reused several times); registered
    or pinned arrays are copied directly; mixed calls stage.  All exact."""
    from paper_1702_00817_b200.pipeline import pinned_empty

    imgs = synth.images_np(range(50, 63), 64, 128, 16, 8.0, 64.0)  # 13 images, 8 KiB each
    src, dst = imgs, np.empty_like(imgs)
    if mode == "pinned_in":
        src = pinned_empty(imgs.shape)
        src[...] = imgs
    if mode == "pinned_out":
        dst = pinned_empty(imgs.shape)
    wr, ws, _ = exact.compress_retain(imgs, 10)
    qt = quant.quant_table(50)
    wq, wqs = exact.compress_quant(imgs, quant.qtab_qprime(qt))
    with HostPipeline(0, chunk_bytes=2 * 8192) as p:  # 2 images per chunk: 7 chunks, 3 slots
        for rep in range(2):
            dst[...] = 0
            _, sse = p.compress_retain(src, 10, dst, register=(mode == "register"))
            assert np.array_equal(dst, wr) and np.array_equal(sse, ws), (mode, rep)
            _, sseq = p.compress_quant(src, qt, dst, register=(mode == "register"))
            assert np.array_equal(dst, wq) and np.array_equal(sseq, wqs), (mode, rep)
            _, sse_only = p.compress_quant(src, qt)
            assert np.array_equal(sse_only, wqs)


def test_host_pipeline_rejects_bad_rec(cuda):
    imgs = np.zeros((3, 16, 16), np.uint8)
    with HostPipeline(0) as p:
        for bad in (np.zeros((2, 16, 16), np.uint8), np.zeros((3, 16, 16), np.int16),
                    np.zeros((3, 16, 32), np.uint8)[:, :, ::2]):
            with pytest.raises(ValueError):
                p.compress_retain(imgs, 10, bad)
            with pytest.raises(ValueError):
                p.compress_quant(imgs, quant.quant_table(50), bad)


def test_batch_rejects_bad_out_and_sse(cuda):
    x = torch.zeros((3, 16, 16), dtype=torch.uint8, device=cuda)
    with pytest.raises(ValueError):
        batch.compress_retain(x, 10, out=torch.zeros((2, 16, 16), dtype=torch.uint8, device=cuda))
    with pytest.raises(ValueError):
        batch.compress_retain(x, 10, sse_out=torch.zeros(4, dtype=torch.int64, device=cuda))
    with pytest.raises(ValueError):
        batch.compress_quant(x, quant.quant_table(50), sse_out=torch.zeros((3, 2), dtype=torch.int64, device=cuda)[:, 0])
    with pytest.raises(ValueError):
        batch.compress_quant(x, quant.quant_table(50), out=torch.zeros((3, 16, 16), dtype=torch.int32, device=cuda))


def test_pinned_empty_buffers_through_pipeline(cuda):
    import gc

    from paper_1702_00817_b200.pipeline import pinned_empty

    imgs = synth.images_np(range(30, 35), 128, 192, 16, 8.0, 64.0)
    host_in = pinned_empty(imgs.shape)
    host_out = pinned_empty(imgs.shape)
    assert host_in.shape == imgs.shape and host_in.dtype == np.uint8 and host_in.flags.c_contiguous
    host_in[...] = imgs
    with HostPipeline(0, chunk_bytes=1 << 16) as p:
        _, sse = p.compress_retain(host_in, 10, host_out, register=False)
    wr, ws, _ = exact.compress_retain(imgs, 10)
    assert np.array_equal(host_out, wr) and np.array_equal(sse, ws)
    view = host_out[1:3]  # a view keeps the allocation alive
    del host_out
    gc.collect()
    assert np.array_equal(view, wr[1:3])
    assert pinned_empty((0, 8, 8)).size == 0
    f = pinned_empty(16, dtype=np.float64)
    f[:] = 1.5
    assert f.sum() == 24.0


# --- generator -------------------------------------------------------------------------

def test_device_generator_matches_numpy_mirror(cuda):
    seeds = [0, 1, 2]
    d = synth.images_device(seeds, 512, 512, 16, 8.0, 64.0, device=cuda).cpu().numpy()
    h = synth.images_np(seeds, 512, 512, 16, 8.0, 64.0)
    diff = np.abs(d.astype(int) - h.astype(int))
    assert diff.max() <= 1 and np.mean(diff != 0) < 1e-3


def test_video_planes_shapes_and_drift(cuda):
    y, cb, cr = synth.video_planes_device(3, device=cuda)
    assert y.shape == (3, 2160, 3840) and cb.shape == (3, 1080, 1920) and cr.shape == (3, 1080, 1920)
    assert not torch.equal(y[0], y[1])
    y2, _, _ = synth.video_planes_device(2, frame0=1, device=cuda)
    assert torch.equal(y2[0], y[1])  # frame i identical whatever the shard start


# --- full sizes: size-independent properties -------------------------------------------

def test_config3_full_size_sampled_parity(cuda):
    """A 64-image slice of config 3 (2048x2048, r = 10): every reconstruction and
    SSE of 4 sampled images equal the oracle; r = 64 is lossless over the
    whole slice; sum of SSE equals the SSE of the reconstructions."""
    nb, smin, smax = synth.CONFIG_BLOBS[3]
    x = synth.images_device(range(64), 2048, 2048, nb, smin, smax, device=cuda)
    rec, sse, _ = batch.compress_retain(x, 10)
    for i in (0, 17, 40, 63):
        wr, ws, _ = exact.compress_retain(x[i].cpu().numpy(), 10)
        assert np.array_equal(rec[i].cpu().numpy(), wr) and int(sse[i]) == ws
    assert torch.equal(batch.sse_u8(x, rec), sse)
    rec64, sse64, _ = batch.compress_retain(x, 64)
    assert int(sse64.sum()) == 0 and torch.equal(rec64, x)


def test_config4_frame_parity(cuda):
    y, cb, cr = synth.video_planes_device(2, device=cuda)
    qt = quant.quant_table(75)
    recs, sse = batch.compress_quant_planes([y, cb, cr], qt)
    qp = exact.qprime(quant.q50_luma(), 75)
    for k, p in enumerate((y, cb, cr)):
        wr, ws = exact.compress_quant(p.cpu().numpy(), qp)
        assert np.array_equal(recs[k].cpu().numpy(), wr) and np.array_equal(sse[:, k].cpu().numpy(), ws)


def test_forward_int16_config0(cuda):
    x = torch.from_numpy(IMAGES["c0_seed0_512"]).to(cuda)
    assert torch.equal(batch.forward_int(x, dtype=torch.int16).to(torch.int32), batch.forward_int(x))


def test_many_images_grid_y_chunking(cuda):
    """> 65535 images exercises the frame-chunked launch loop."""
    x = torch.randint(0, 256, (70000, 8, 16), dtype=torch.uint8, device=cuda)
    rec, sse, _ = batch.compress_retain(x, 5)
    idx = [0, 65534, 65535, 65536, 69999]
    wr, ws, _ = exact.compress_retain(x[idx].cpu().numpy(), 5)
    assert np.array_equal(rec[idx].cpu().numpy(), wr) and np.array_equal(sse[idx].cpu().numpy(), ws)


def test_config3_full_batch_properties(cuda):
    """Full config 3 (4096 x 2048^2, 16 GiB): one launch == 8 chunked launches
    bit for bit, deterministic across runs, SSE == independent device SSE of
    (input, reconstruction), and sampled images == the oracle."""
    nb, smin, smax = synth.CONFIG_BLOBS[3]
    x = synth.images_device(range(4096), 2048, 2048, nb, smin, smax, device=cuda)
    rec = torch.empty_like(x)
    _, sse, _ = batch.compress_retain(x, 10, out=rec)
    sse_chunks = torch.cat([batch.compress_retain(x[k * 512:(k + 1) * 512], 10, reconstruct=False)[1] for k in range(8)])
    assert torch.equal(sse, sse_chunks)
    h1 = torch.sum(rec.view(4096, -1)[:, ::4097].to(torch.int64), dim=1)
    rec2 = torch.empty_like(x)
    _, sse2, _ = batch.compress_retain(x, 10, out=rec2)
    assert torch.equal(sse, sse2) and torch.equal(rec, rec2)
    del rec2
    assert torch.equal(batch.sse_u8(x, rec), sse)
    for i in (0, 1234, 4095):
        wr, ws, _ = exact.compress_retain(x[i].cpu().numpy(), 10)
        assert int(sse[i]) == ws and np.array_equal(rec[i].cpu().numpy(), wr)
    assert int(h1.sum()) > 0


def test_forward_unscaled_device_tensors(cuda):
    """Device tensors route by dtype (no value scan, no host sync): uint8 takes
    the exact integer kernel, other dtypes the dense float64 kernel with K,
    exact for integer values and returned in the input's kind."""
    rng = np.random.default_rng(7)
    ib = rng.integers(-1024, 1025, (6, 8, 8))
    want = exact.T @ ib @ exact.T.T
    for dt in (torch.int32, torch.int64, torch.float32, torch.float64):
        z = codec.forward_2d_unscaled(T, torch.as_tensor(ib, dtype=dt, device=cuda))
        assert z.is_cuda and np.array_equal(z.cpu().numpy(), want), dt
        assert (z.dtype == torch.int64) == (not dt.is_floating_point)
    u8 = rng.integers(0, 256, (3, 8, 8)).astype(np.uint8)
    z = codec.forward_2d_unscaled(T, torch.as_tensor(u8, device=cuda))
    assert z.dtype == torch.int64 and np.array_equal(z.cpu().numpy(), exact.T @ u8.astype(np.int64) @ exact.T.T)
    fb = rng.normal(0, 50, (4, 8, 8))
    zf = codec.forward_2d_unscaled(T, torch.as_tensor(fb, device=cuda))
    assert np.abs(zf.cpu().numpy() - exact.T @ fb @ exact.T.T).max() < 1e-9


def test_host_pipeline_shared_by_threads(cuda):
    """Several Python threads on ONE HostPipeline (ctypes releases the GIL):
    the library serialises the calls, every result is exact."""
    import threading

    imgs = synth.images_np(range(60, 66), 128, 256, 16, 8.0, 64.0)
    want_rec, want_sse, _ = exact.compress_retain(imgs, 7)
    qt = quant.quant_table(30)
    wq, wqs = exact.compress_quant(imgs, quant.qtab_qprime(qt))
    errors = []
    with HostPipeline(0, chunk_bytes=1 << 16) as p:
        def work(k):
            try:
                for _ in range(3):
                    rec = np.empty_like(imgs)
                    if k % 2:
                        _, s = p.compress_retain(imgs, 7, rec)
                        ok = np.array_equal(rec, want_rec) and np.array_equal(s, want_sse)
                    else:
                        _, s = p.compress_quant(imgs, qt, rec)
                        ok = np.array_equal(rec, wq) and np.array_equal(s, wqs)
                    if not ok:
                        errors.append(k)
            except Exception as exc:  # noqa: BLE001
                errors.append(repr(exc))
        threads = [threading.Thread(target=work, args=(k,)) for k in range(4)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
    assert not errors, errors
