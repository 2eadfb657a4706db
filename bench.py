#!/usr/bin/env python
"""Benchmark of the fused 8x8 approximate-DCT compress path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

A step = one fused compress launch over every image resident on the rank
(config 3: 4096 seeded 2048x2048 uint8 images per GPU, retain r=10; weak
scaling) + the NCCL all-reduce of the per-image SSE when N > 1 (or, with
--exchange fused, the exchange done by the kernel epilogue through torch
symmetric memory).  Inputs are generated on the GPU before timing (16 GiB per
GPU >> 126 MB L2, so no L2 flush is needed between steps).  `e2e` times the
same work through the C-ABI host pipeline from page-locked host buffers
(reconstructions returned; `e2e.metric_only`: only the SSE/PSNR vector).
Rank 0 prints one JSON line.

--impl reference times the reference's own CPU algorithm (the float64
restatement oracle/refport.py of codec.compress_image + metrics.mse/psnr;
/root/reference cannot travel to the GPU box) on the host cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gpixel/s for fused 8x8 approx-DCT fwd+quant+inv+PSNR; % of HBM roofline"
UNIT = "Gpixel/s"
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback, used only without MEASURED_PEAKS.json

CONFIGS = {
    3: dict(kind="retain", h=2048, w=2048, n=4096, r=10, blobs=(64, 16.0, 256.0),
            workload="config3: 4096 seeded 2048x2048 u8 images per GPU, fused fwd+retain(r=10)+inv+round+clamp+SSE/PSNR"),
    2: dict(kind="quant", h=1024, w=1024, n=256, q=(10, 50, 90), blobs=(32, 16.0, 128.0),
            workload="config2: 256 seeded 1024x1024 u8 images per GPU, fused level-shift+fwd+quant(q=10,50,90)+dequant+inv+SSE"),
    4: dict(kind="planes", frames=512, q=75,
            workload="config4: 512 seeded 3840x2160 YCbCr 4:2:0 frames per GPU, fused quant(q=75) of Y+Cb+Cr in one launch"),
    1: dict(kind="sweep", h=512, w=512, n=45, r=(1, 45), blobs=(16, 8.0, 64.0),
            workload="config1: 45 seeded 512x512 u8 images, SSE/PSNR for every r=1..45 from one read (k_sweep_inc); "
                     "11.8 MB, L2-resident and launch bound: value counts image pixels, not pixel-reconstructions"),
    0: dict(kind="forward", h=512, w=512, n=1, blobs=(16, 8.0, 64.0),
            workload="config0: 1 seeded 512x512 u8 image, exact int32 T X T^T coefficients (launch bound)"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_hbm_peak() -> tuple[float, str]:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy read+write, measured)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback 6650 GB/s (B200_PROFILING.md), MEASURED_PEAKS.json absent"


def ncu_traffic(config: int):
    """Per-launch DRAM bytes of the top kernel from the committed ncu summary, or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(f"config{config}")
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True,
            )
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": smax, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU side: reference algorithm (oracle/refport.py), all host cores
# ---------------------------------------------------------------------------

def _ref_task(args):
    img, r = args
    from oracle import refport

    rec = refport.compress_image(img, r)
    m = refport.mse(img, rec)
    return refport.psnr(m)


def _ref_sweep_task(args):
    """Reference experiment for one image (the paper's Fig. 2 sweep): the
    coefficients once, then reconstruct + mse + psnr for every r in range."""
    img, (r0, r1) = args
    from oracle import refport

    y = refport.coefficient_blocks(img)
    return [refport.psnr(refport.mse(img, refport.reconstruct_image(y, r, *img.shape))) for r in range(r0, r1 + 1)]


def _ref_forward_task(args):
    """Reference forward: codec.coefficient_blocks of one image (float64)."""
    img, _ = args
    from oracle import refport

    return float(refport.coefficient_blocks(img)[0, 0, 0])


def quant_jit_stats():
    """Counters of the run-time table specialisation of the quant kernels
    (adct_quant_jit_stats): kernels compiled and specialised launches so far."""
    import ctypes

    from paper_1702_00817_b200 import _lib

    c, l, f = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _lib.lib().adct_quant_jit_stats(ctypes.byref(c), ctypes.byref(l), ctypes.byref(f))
    return {"compiled": c.value, "specialised_launches": l.value, "failures": f.value,
            "after_uses": int(os.environ.get("ADCT_QUANT_JIT_AFTER", "3"))}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference_rate(images, r, budget_s: float, cores: int, task=None):
    """Gpixel/s of the reference algorithm over full `images`, one task per
    worker, for about `budget_s` seconds (task: _ref_task or _ref_quant_task)."""
    task = task or _ref_task
    import numpy as np
    from concurrent.futures import ProcessPoolExecutor

    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    h, w = images[0].shape
    with ProcessPoolExecutor(max_workers=cores) as ex:
        # calibrate on one full image per worker
        t0 = time.perf_counter()
        list(ex.map(task, [(images[k % len(images)], r) for k in range(cores)]))
        t_full = time.perf_counter() - t0
        rounds = max(1, int(budget_s / max(t_full, 1e-3)))
        tasks = [(images[k % len(images)], r) for k in range(cores * rounds)]
        t0 = time.perf_counter()
        list(ex.map(task, tasks))
        dt = time.perf_counter() - t0
    px = len(tasks) * h * w
    return px / dt / 1e9, dict(images=len(tasks), seconds=dt, image_shape=[h, w])


def _ref_quant_task(args):
    """Quantised pipeline composed of the reference's own float64 functions
    (oracle/refport.quant_float64: forward_2d_unscaled, folded Q', inverse_2d)
    + round + clamp + mse + psnr; the reference has no quantised driver."""
    img, qp = args
    import numpy as np

    from oracle import refport

    rec = np.clip(np.floor(refport.quant_float64(img, qp) + 0.5), 0, 255)
    return refport.psnr(refport.mse(img, rec))


def reference_arm(args) -> None:
    """--impl reference: the reference's CPU algorithm on the host cores."""
    import numpy as np

    from paper_1702_00817_b200 import synth

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    cores = len(os.sched_getaffinity(0))
    if cfg["kind"] in ("retain", "sweep", "forward"):
        h, w = cfg["h"], cfg["w"]
        nb, smin, smax = cfg["blobs"]
        r, task, what = {
            "retain": (cfg.get("r"), _ref_task, "oracle/refport.py float64 path (codec.compress_image + metrics.mse/psnr)"),
            "sweep": (cfg.get("r"), _ref_sweep_task, "oracle/refport.py float64 sweep (coefficients once, reconstruct+mse+psnr per r)"),
            "forward": (None, _ref_forward_task, "oracle/refport.coefficient_blocks (codec.py:120-131, float64)"),
        }[cfg["kind"]]
    else:
        from oracle import exact
        from paper_1702_00817_b200.quant import q50_luma

        if cfg["kind"] == "quant":
            h, w = cfg["h"], cfg["w"]
            nb, smin, smax = cfg["blobs"]
            q = cfg["q"][1]
        else:  # config 4: the Y plane of the video frames carries 2/3 of the pixels
            h, w, q = 2160, 3840, cfg["q"]
            nb, smin, smax = synth.CONFIG_BLOBS[4]
        r = exact.qprime(q50_luma(), q)
        task = _ref_quant_task
        what = f"oracle/refport.quant_float64 (reference float64 functions composed, q={q})"
    n_img = min(cores, 16)
    images = [synth.render_np(synth.blob_params(s, h, w, nb, smin, smax), h, w, s) for s in range(n_img)]
    # per-step sample: `rows` rows of one image per worker, sized so the whole run fits ~3 minutes
    budget_step = min(30.0, 180.0 / max(1, args.steps + args.warmup))
    from concurrent.futures import ProcessPoolExecutor

    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    with ProcessPoolExecutor(max_workers=cores) as ex:
        t0 = time.perf_counter()
        list(ex.map(task, [(images[k % n_img], r) for k in range(cores)]))
        t_full = time.perf_counter() - t0
        rows = int(h * min(1.0, budget_step / max(t_full, 1e-3)))
        rows = max(8, rows - rows % 8)
        strips = [(images[k % n_img][:rows], r) for k in range(cores)]
        for _ in range(args.warmup):
            list(ex.map(task, strips))
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            list(ex.map(task, strips))
            times.append(time.perf_counter() - t0)
    px_step = cores * rows * w
    total = sum(times)
    value = px_step * len(times) / total / 1e9
    sample = f"{cores} x ({rows}x{w}) strips of config-{args.config} images per step (one per core), {what}"
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Gaussian blobs + N(0,4^2) noise, BASELINE.json generator)",
        "config": {"workload": cfg["workload"]},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                         "cpu": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def gpu_arm(args) -> None:
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1702_00817_b200 import batch, quant, shard, synth
    from paper_1702_00817_b200.pipeline import HostPipeline, pinned_empty

    rank, world, local = shard.init_from_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = CONFIGS[args.config]
    if world != args.gpus:
        log(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}; using {world}")

    # ---- workload resident in HBM -------------------------------------------
    t_gen = time.perf_counter()
    if cfg["kind"] in ("sweep", "forward"):
        per = cfg["n"] if args.scaling == "weak" else shard.shard_range(cfg["n"], rank, world).count
        first = rank * cfg["n"] if args.scaling == "weak" else shard.shard_range(cfg["n"], rank, world).start
        nb, smin, smax = cfg["blobs"]
        imgs = synth.images_device(range(first, first + per), cfg["h"], cfg["w"], nb, smin, smax, device=dev)
        px_rank = per * cfg["h"] * cfg["w"]
        n_total = per * world if args.scaling == "weak" else cfg["n"]
        if cfg["kind"] == "sweep":
            r0, r1 = cfg["r"]
            sse = torch.empty((per, r1 - r0 + 1), dtype=torch.int64, device=dev)
            import ctypes
            from paper_1702_00817_b200 import _lib
            def step_kernel():
                _lib.call("adct_sweep_retain_sse", imgs.data_ptr(), per, cfg["h"], cfg["w"], cfg["h"] * cfg["w"],
                          r0, r1, sse.data_ptr(), None, torch.cuda.current_stream().cuda_stream)
        else:
            coef = torch.empty((per, cfg["h"] * cfg["w"] // 64, 8, 8), dtype=torch.int32, device=dev)
            sse = torch.zeros((per, 1), dtype=torch.int64, device=dev)
            import ctypes
            from paper_1702_00817_b200 import _lib
            def step_kernel():
                _lib.call("adct_forward_int32", imgs.data_ptr(), per, cfg["h"], cfg["w"], cfg["h"] * cfg["w"], 0,
                          coef.data_ptr(), torch.cuda.current_stream().cuda_stream)
        launches_per_step = 1
    elif cfg["kind"] in ("retain", "quant"):
        per = cfg["n"] if args.scaling == "weak" else shard.shard_range(cfg["n"], rank, world).count
        first = rank * cfg["n"] if args.scaling == "weak" else shard.shard_range(cfg["n"], rank, world).start
        nb, smin, smax = cfg["blobs"]
        imgs = synth.images_device(range(first, first + per), cfg["h"], cfg["w"], nb, smin, smax, device=dev)
        rec = torch.empty_like(imgs)
        sse = torch.empty(per, dtype=torch.int64, device=dev)
        px_rank = per * cfg["h"] * cfg["w"]
        n_total = per * world if args.scaling == "weak" else cfg["n"]
        if cfg["kind"] == "retain" and args.exchange == "fused":
            # SSE exchange fused into the kernel epilogue:
            # P2P stores into every rank's symmetric-memory vector + one
            # stream-ordered barrier instead of the NCCL all-reduce
            if not dist.is_initialized():
                os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
                os.environ.setdefault("MASTER_PORT", "29561")
                dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
            base = rank * per if args.scaling == "weak" else shard.shard_range(n_total, rank, world).start
            exchange = shard.SseExchange(n_total, dev)
            def step_kernel():
                exchange.compress_retain(imgs, cfg["r"], base, out=rec, sse_out=sse)
            launches_per_step = 1
        elif cfg["kind"] == "retain":
            def step_kernel():
                batch.compress_retain(imgs, cfg["r"], out=rec, sse_out=sse)
            launches_per_step = 1
        else:
            qtabs = [quant.quant_table(q) for q in cfg["q"]]
            sse_q = torch.empty((len(qtabs), per), dtype=torch.int64, device=dev)  # one row per quality
            sse = sse_q.t()  # (per, n_q) view: what the all-reduce exchanges
            def step_kernel():
                for k, qt in enumerate(qtabs):
                    batch.compress_quant(imgs, qt, out=rec, sse_out=sse_q[k])
            launches_per_step = len(qtabs)
            px_rank *= len(qtabs)
    else:  # config 4 planes
        frames = cfg["frames"] if args.scaling == "weak" else shard.shard_range(cfg["frames"], rank, world).count
        f0 = rank * cfg["frames"] if args.scaling == "weak" else shard.shard_range(cfg["frames"], rank, world).start
        planes = synth.video_planes_device(frames, frame0=f0, device=dev)
        qt = quant.quant_table(cfg["q"])
        import ctypes
        from paper_1702_00817_b200 import _lib
        recs = [torch.empty_like(p) for p in planes]
        arr, _ = batch._planes(planes, recs)
        sse = torch.empty((frames, 3), dtype=torch.int64, device=dev)
        n_total = frames * world if args.scaling == "weak" else cfg["frames"]
        if args.exchange == "fused":  # exchange of the (frame, plane) SSE in the kernel epilogue
            if not dist.is_initialized():
                os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
                os.environ.setdefault("MASTER_PORT", "29562")
                dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
            exchange = shard.SseExchange(n_total * 3, dev)
            def step_kernel():
                exchange.compress_quant_planes(planes, qt, f0, out=recs)
        else:
            def step_kernel():
                _lib.call("adct_compress_quant_planes", arr, 3, frames, ctypes.byref(qt), sse.data_ptr(),
                          torch.cuda.current_stream().cuda_stream)
        launches_per_step = 1
        px_rank = frames * sum(p.shape[1] * p.shape[2] for p in planes)
        per = frames
    torch.cuda.synchronize()
    log(f"[rank {rank}] workload ready in {time.perf_counter() - t_gen:.1f}s: {px_rank / 1e9:.2f} Gpx per step")

    fused_exchange = cfg["kind"] in ("retain", "planes") and args.exchange == "fused"

    def step():
        step_kernel()
        if world > 1 and not fused_exchange:
            full = torch.zeros((n_total,) + tuple(sse.shape[1:]), dtype=torch.int64, device=dev)
            base = rank * per if args.scaling == "weak" else shard.shard_range(n_total, rank, world).start
            full[base : base + per] = sse
            dist.all_reduce(full)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    graphed = False
    if cfg["kind"] in ("sweep", "forward", "quant") and not args.no_graph:
        # short launches (configs 0/1: one small launch; config 2: three
        # ~0.16 ms launches per step): replay the step's C-ABI launches from a
        # CUDA graph so host-side call overhead does not leave the GPU idle
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step_kernel()
        graph.replay()
        torch.cuda.synchronize()
        step_kernel = graph.replay
        graphed = True

    # ---- timed region ----------------------------------------------------------
    stream = torch.cuda.current_stream()
    k_start = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    k_end = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_start.record(stream)
    for i in range(args.steps):
        k_start[i].record(stream)
        step_kernel()
        k_end[i].record(stream)
        if world > 1 and not fused_exchange:
            full = torch.zeros((n_total,) + tuple(sse.shape[1:]), dtype=torch.int64, device=dev)
            base = rank * per if args.scaling == "weak" else shard.shard_range(n_total, rank, world).start
            full[base : base + per] = sse
            dist.all_reduce(full)
    t_end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    elapsed_ms = t_start.elapsed_time(t_end)
    kern_ms = sum(a.elapsed_time(b) for a, b in zip(k_start, k_end)) / args.steps / launches_per_step
    if world > 1:
        t = torch.tensor([elapsed_ms, kern_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms, kern_ms = t.tolist()

    total_px = px_rank * world * args.steps
    value = total_px / (elapsed_ms * 1e-3) / 1e9
    px_launch = px_rank / launches_per_step
    bytes_per_px = {"sweep": 1, "forward": 5}.get(cfg["kind"], 2)  # u8 in (+ u8 out | + int32 coefficients)
    alg_bytes = bytes_per_px * px_launch + 8 * per * (sse.shape[1] if sse.dim() > 1 else 1)
    achieved = alg_bytes / (kern_ms * 1e-3) / 1e9
    peak, peak_src = measured_hbm_peak()

    # ---- end to end: host buffers through the C-ABI pipeline (every rank) -------
    def timed_e2e(call, outs):
        """Mean wall time of 3 host-pipeline calls after one warm call; max over ranks."""
        call(outs)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(3):
            call(outs)
        dt = (time.perf_counter() - t0) / 3
        if world > 1:
            t = torch.tensor([dt], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = t.item()
        return dt

    e2e = None
    if not args.no_e2e and cfg["kind"] in ("retain", "quant", "planes"):
        # page-locked host buffers from adct_host_alloc (cudaHostAlloc), filled
        # from the device copies before the timed region
        if cfg["kind"] == "planes":  # frames of Y/Cb/Cr host planes
            m = min(per, max(1, args.e2e_images // 4))
            host_in = [pinned_empty((m,) + tuple(p.shape[1:])) for p in planes]
            for a, p in zip(host_in, planes):
                a[...] = p[:m].cpu().numpy()
            host_out = [pinned_empty(a.shape) for a in host_in]
            n_sse = 3 * m
            qt4 = quant.quant_table(cfg["q"])
            chunk = max(args.e2e_chunk_mb << 20, 5 * sum(a[0].nbytes for a in host_in))  # ~5 frames: measured best
            api = "adct_pipeline_compress_quant_planes (C ABI) via paper_1702_00817_b200.pipeline"
            units = {"frames_per_step": world * m}
        else:
            m = min(per, args.e2e_images)
            host_in = [pinned_empty(tuple(imgs[:m].shape))]
            host_in[0][...] = imgs[:m].cpu().numpy()
            host_out = [pinned_empty(host_in[0].shape)]
            n_sse = m
            qt0 = quant.quant_table(cfg["q"][0]) if cfg["kind"] == "quant" else None
            chunk = args.e2e_chunk_mb << 20
            api = "adct_pipeline_compress_* (C ABI) via paper_1702_00817_b200.pipeline"
            units = {"images_per_step": world * m}
        try:
            with HostPipeline(local, chunk_bytes=chunk) as pipe:
                if cfg["kind"] == "planes":
                    call = lambda outs: pipe.compress_quant_planes(host_in, qt4, outs, register=False)
                elif cfg["kind"] == "retain":
                    call = lambda outs: pipe.compress_retain(host_in[0], cfg["r"], outs and outs[0], register=False)
                else:
                    call = lambda outs: pipe.compress_quant(host_in[0], qt0, outs and outs[0], register=False)
                dt = timed_e2e(call, host_out)  # reconstructions come back to the host every step
                dt_metric = timed_e2e(call, None)  # inputs in, per-image SSE (-> PSNR) back
            px = world * sum(a.size for a in host_in)
            nbytes = sum(a.nbytes for a in host_in)
            e2e = {"value": px / dt / 1e9, "unit": UNIT,
                   "h2d_bytes_per_step": int(world * nbytes),
                   "d2h_bytes_per_step": int(world * (nbytes + 8 * n_sse)),
                   **units,
                   "api": api + ", every rank, max time over ranks",
                   "metric_only": {"value": px / dt_metric / 1e9, "unit": UNIT,
                                   "h2d_bytes_per_step": int(world * nbytes),
                                   "d2h_bytes_per_step": int(world * 8 * n_sse),
                                   "note": "reconstructions kept on the device; only the SSE/PSNR vector is read back"}}
        finally:
            del host_in, host_out

    # ---- CPU baseline (rank 0, N=1) ---------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = len(os.sched_getaffinity(0))
        if cfg["kind"] in ("retain", "sweep", "forward"):
            sample_imgs = [imgs[k].cpu().numpy() for k in range(min(per, 8))]
            task = {"retain": _ref_task, "sweep": _ref_sweep_task, "forward": _ref_forward_task}[cfg["kind"]]
            v, info = cpu_reference_rate(sample_imgs, cfg.get("r"), args.cpu_seconds, cores, task=task)
            algo = f"oracle/refport.py = reference float64 algorithm ({task.__doc__.split(chr(10))[0] if task.__doc__ else 'codec.compress_image + metrics.mse/psnr'})"
        else:
            from oracle import exact

            q = cfg["q"][1] if cfg["kind"] == "quant" else cfg["q"]
            src = imgs if cfg["kind"] == "quant" else planes[0]
            sample_imgs = [src[k].cpu().numpy() for k in range(min(per, 4))]
            v, info = cpu_reference_rate(sample_imgs, exact.qprime(quant.q50_luma(), q), args.cpu_seconds, cores,
                                         task=_ref_quant_task)
            algo = f"oracle/refport.quant_float64 = reference float64 functions composed (q={q})"
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "cpu": cpu_model(),
               "sample": f"{info['images']} full {info['image_shape'][0]}x{info['image_shape'][1]} config-{args.config} images, "
                         f"one per task on {cores} processes, {info['seconds']:.1f}s; {algo}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (seeded Gaussian blobs + N(0,4^2) noise, BASELINE.json generator, rendered on GPU)",
            "config": {"workload": cfg["workload"], "units_per_gpu": per, "pixels_per_step": px_rank * world,
                       "parallelism": f"dp{world} (images sharded, SSE "
                                      + ("exchange fused into the kernel epilogue)" if fused_exchange else "all-reduce)"),
                       "l2": "inputs >> 126 MB L2 (no flush needed)" if px_rank > (256 << 20)
                             else "inputs L2-resident (launch/ALU bound config; no roofline claim)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic(args.config),
                         "kernel_ms": kern_ms, "algorithmic_bytes_per_launch": alg_bytes, "peak_source": peak_src},
            "clocks": clk,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "cuda_graph": graphed,
            "quant_jit": quant_jit_stats(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=3, choices=sorted(CONFIGS),
                    help="3 (default, large-batch headline), 4, 2, 1 (sweep), 0 (forward)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="configs 0/1/2: launch through the C ABI every step")
    ap.add_argument("--exchange", default="allreduce", choices=["allreduce", "fused"],
                    help="configs 3 and 4: SSE exchange by NCCL all-reduce (default) or fused into the kernel "
                         "epilogue through torch symmetric memory")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--e2e-images", type=int, default=256)
    ap.add_argument("--e2e-chunk-mb", type=int, default=32)
    args = ap.parse_args()
    if args.warmup < 3:
        log("warmup raised to 3 (timing rules)")
        args.warmup = 3
    if args.impl == "reference":
        reference_arm(args)
    else:
        gpu_arm(args)


if __name__ == "__main__":
    main()
