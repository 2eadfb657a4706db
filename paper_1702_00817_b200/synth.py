"""Seeded synthetic images of BASELINE.json (Gaussian blobs + N(0, 4^2) noise).

pixel = clip(rint(128 + sum_k a_k exp(-((y-cy_k)^2 + (x-cx_k)^2) / (2 s_k^2)) + 4 n(y,x)), 0, 255)

Draw order (fixed here; BASELINE does not specify one): for image seed s,
``rng = np.random.default_rng(s)``, ``u = rng.random((n_blobs, 4))`` and
cy = u0*H, cx = u1*W, s = smin + u2*(smax-smin), a = -80 + 160*u3.  The noise
n(y,x) is a counter-based Box-Muller normal of (noise_seed, y*W+x), so image i
is the same on any number of GPUs.  Video frames (config 4) move every blob
centre by an N(0, 2^2) step per frame (``rng.normal(0, 2, (frames, n_blobs, 2))``
cumulated, drawn after ``u``) and use noise_seed = (plane_seed << 20) + frame.

The device rasteriser (adct_synth_blobs) evaluates this in float32; the numpy
mirror below evaluates it in float64 for tests.  They agree except for rare
pixels whose value lands within float32 rounding of a .5 boundary (tested).
Generation is never inside a timed region.
"""

from __future__ import annotations


import numpy as np

from . import _lib

#: (n_blobs, sigma_min, sigma_max) per BASELINE config.
CONFIG_BLOBS = {0: (16, 8.0, 64.0), 1: (16, 8.0, 64.0), 2: (32, 16.0, 128.0), 3: (64, 16.0, 256.0), 4: (16, 8.0, 64.0)}

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_GOLD = np.uint64(0x9E3779B97F4A7C15)


def blob_params(seed: int, h: int, w: int, n_blobs: int, smin: float, smax: float) -> np.ndarray:
    """(n_blobs, 4) float64 rows (cy, cx, sigma, amp) for one image seed."""
    rng = np.random.default_rng(int(seed))
    u = rng.random((n_blobs, 4))
    return np.stack([u[:, 0] * h, u[:, 1] * w, smin + u[:, 2] * (smax - smin), -80.0 + 160.0 * u[:, 3]], axis=1)


def video_blob_params(plane_seed: int, frames: int, h: int, w: int, n_blobs: int, smin: float, smax: float) -> np.ndarray:
    """(frames, n_blobs, 4): config-4 blobs with an N(0, 2^2) random-walk drift of the centres."""
    rng = np.random.default_rng(int(plane_seed))
    u = rng.random((n_blobs, 4))
    base = np.stack([u[:, 0] * h, u[:, 1] * w, smin + u[:, 2] * (smax - smin), -80.0 + 160.0 * u[:, 3]], axis=1)
    steps = rng.normal(0.0, 2.0, (frames, n_blobs, 2))
    steps[0] = 0.0
    drift = np.cumsum(steps, axis=0)
    out = np.broadcast_to(base, (frames, n_blobs, 4)).copy()
    out[:, :, 0:2] += drift
    return out


def _mix64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def hash_normal(seed: int, idx: np.ndarray) -> np.ndarray:
    """numpy mirror of the device hash_normal (csrc/adct_kernels.cuh)."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed) * _GOLD + idx.astype(np.uint64) + np.uint64(1)
    h = _mix64(z)
    u1 = ((h >> np.uint64(40)).astype(np.float64) + 0.5) / 16777216.0
    u2 = (((h >> np.uint64(8)) & np.uint64(0xFFFFFF)).astype(np.float64) + 0.5) / 16777216.0
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def render_np(params: np.ndarray, h: int, w: int, noise_seed: int) -> np.ndarray:
    """float64 host rendering of one image (test mirror of the device kernel)."""
    y = np.arange(h, dtype=np.float64)[:, None]
    x = np.arange(w, dtype=np.float64)[None, :]
    cy, cx, s, a = (params[:, k][:, None] for k in range(4))
    gy = np.exp(-((y.T - cy) ** 2) / (2 * s * s))  # (n_blobs, h)
    gx = a * np.exp(-((x - cx) ** 2) / (2 * s * s))  # (n_blobs, w)
    acc = gy.T @ gx  # separable Gaussian sum, same factorisation as the device kernel
    idx = (np.arange(h, dtype=np.uint64)[:, None] * np.uint64(w) + np.arange(w, dtype=np.uint64)[None, :])
    v = 128.0 + acc + 4.0 * hash_normal(noise_seed, idx)
    return np.clip(np.rint(v), 0, 255).astype(np.uint8)


def images_np(seeds, h: int, w: int, n_blobs: int, smin: float, smax: float) -> np.ndarray:
    return np.stack([render_np(blob_params(s, h, w, n_blobs, smin, smax), h, w, s) for s in seeds])


def render_device(params: np.ndarray, noise_seeds, h: int, w: int, device="cuda"):
    """Rasterise (N, n_blobs, 4) parameters on the GPU into a (N, H, W) uint8 tensor."""
    import torch

    params = np.asarray(params, dtype=np.float32)
    n, nb, _ = params.shape
    pad = next(k for k in (16, 32, 64) if k >= nb) if nb <= 64 else None
    if pad is None:
        raise ValueError("at most 64 blobs")
    if pad != nb:  # zero-amplitude padding blobs
        extra = np.zeros((n, pad - nb, 4), np.float32)
        extra[:, :, 2] = 1.0
        params = np.concatenate([params, extra], axis=1)
    d_params = torch.from_numpy(np.ascontiguousarray(params)).to(device)
    d_seeds = torch.from_numpy(np.asarray(noise_seeds, dtype=np.uint64).view(np.int64)).to(device)
    out = torch.empty((n, h, w), dtype=torch.uint8, device=device)
    _lib.call(
        "adct_synth_blobs",
        out.data_ptr(), n, h, w, h * w, d_params.data_ptr(), pad, d_seeds.data_ptr(),
        torch.cuda.current_stream().cuda_stream,
    )
    return out


def images_device(seeds, h: int, w: int, n_blobs: int, smin: float, smax: float, device="cuda", chunk: int = 1024):
    """(len(seeds), H, W) uint8 CUDA batch; image i uses seed seeds[i] for blobs and noise."""
    import torch

    seeds = list(seeds)
    out = torch.empty((len(seeds), h, w), dtype=torch.uint8, device=device)
    for i0 in range(0, len(seeds), chunk):
        sl = seeds[i0 : i0 + chunk]
        params = np.stack([blob_params(s, h, w, n_blobs, smin, smax) for s in sl])
        out[i0 : i0 + len(sl)] = render_device(params, sl, h, w, device)
    return out


def config_images_device(config: int, seeds, device="cuda"):
    h, w = {0: (512, 512), 1: (512, 512), 2: (1024, 1024), 3: (2048, 2048)}[config]
    nb, smin, smax = CONFIG_BLOBS[config]
    return images_device(seeds, h, w, nb, smin, smax, device)


def video_planes_device(frames: int, frame0: int = 0, base_seed: int = 0, device="cuda"):
    """Config 4: Y (3840x2160) and Cb, Cr (1920x1080) planes of `frames` frames
    starting at frame0; plane seeds 3*base_seed + {0,1,2}."""
    import torch

    nb, smin, smax = CONFIG_BLOBS[4]
    dims = [(2160, 3840), (1080, 1920), (1080, 1920)]
    planes = []
    for k, (h, w) in enumerate(dims):
        ps = 3 * base_seed + k
        params = video_blob_params(ps, frame0 + frames, h, w, nb, smin, smax)[frame0:]
        noise = [(ps << 20) + f for f in range(frame0, frame0 + frames)]
        planes.append(render_device(params, noise, h, w, device))
    return planes
