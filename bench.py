#!/usr/bin/env python
"""Benchmark of the fused 8x8 approximate-DCT compress path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

A step = one fused compress launch over every image resident on the rank +
the exchange of the per-image SSE when N > 1 (NCCL all-gather into a
preallocated vector, or with --exchange fused the kernel epilogue's P2P
stores through torch symmetric memory).  Default scaling is strong, as
BASELINE.json words it: config 3 is 4096 images *in total* sharded by image
over the N GPUs (config 4: 512 frames in total, sharded by frame);
--scaling weak gives every rank the full config instead.  Inputs are generated
on the GPU before timing (config 3: 16 GiB >> 126 MB L2, so no L2 flush is
needed between steps).  `e2e` times the same work through the C-ABI host
pipeline from page-locked host buffers (reconstructions returned;
`e2e.metric_only`: only the SSE/PSNR vector).  The default config-3 run also
measures configs 4 and 2 (the quantised kernels) in the same process and
reports them under `secondary`.  Rank 0 prints one JSON line.

--impl reference times the reference package itself (`adct`, installed
unmodified into baseline/_ref: codec.compress_image + metrics.mse/psnr, and
the reference's own functions composed for the quantised configs) on all
host cores; oracle/refport.py stands in only when baseline/_ref is absent.

--plan prints the workload split (no GPU work) — used by the CPU tests to
check the multi-rank accounting under torchrun + gloo.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
REF_DIR = os.path.join(ROOT, "baseline", "_ref")

METRIC = "Gpixel/s for fused 8x8 approx-DCT fwd+quant+inv+PSNR; % of HBM roofline"
UNIT = "Gpixel/s"
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback, used only without MEASURED_PEAKS.json

CONFIGS = {
    3: dict(kind="retain", h=2048, w=2048, n=4096, r=10, blobs=(64, 16.0, 256.0),
            workload="config3: 4096 seeded 2048x2048 u8 images, fused fwd+retain(r=10)+inv+round+clamp+SSE/PSNR"),
    2: dict(kind="quant", h=1024, w=1024, n=256, q=(10, 50, 90), blobs=(32, 16.0, 128.0),
            workload="config2: 256 seeded 1024x1024 u8 images, fused level-shift+fwd+quant(q=10,50,90)+dequant+inv+SSE"),
    4: dict(kind="planes", n=512, q=75,
            workload="config4: 512 seeded 3840x2160 YCbCr 4:2:0 frames, fused quant(q=75) of Y+Cb+Cr in one launch"),
    1: dict(kind="sweep", h=512, w=512, n=45, r=(1, 45), blobs=(16, 8.0, 64.0),
            workload="config1: 45 seeded 512x512 u8 images, SSE/PSNR for every r=1..45 from one read (k_sweep_inc); "
                     "11.8 MB, L2-resident and launch bound: value counts image pixels, not pixel-reconstructions"),
    0: dict(kind="forward", h=512, w=512, n=1, blobs=(16, 8.0, 64.0),
            workload="config0: 1 seeded 512x512 u8 image, exact int32 T X T^T coefficients (launch bound)"),
}
PLANE_DIMS = ((2160, 3840), (1080, 1920), (1080, 1920))  # config 4: Y, Cb, Cr


def log(*a):
    print(*a, file=sys.stderr, flush=True)


_OUT = None  # the real stdout (main() points fd 1 at stderr)


def emit(line: dict) -> None:
    out = _OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


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


# ---------------------------------------------------------------------------
# Workload split (shared by the GPU arm and --plan)
# ---------------------------------------------------------------------------

def px_per_unit(cfg) -> int:
    if cfg["kind"] == "planes":
        return sum(h * w for h, w in PLANE_DIMS)
    return cfg["h"] * cfg["w"]


def plan(config: int, rank: int, world: int, scaling: str) -> dict:
    """Units (images or frames) of this rank: strong scaling splits the
    config's units contiguously ([rank*n/N, (rank+1)*n/N), shard.shard_range);
    weak scaling gives every rank the whole config (units rank*n ...)."""
    from paper_1702_00817_b200 import shard

    cfg = CONFIGS[config]
    n = cfg["n"]
    if scaling == "weak":
        per, first, n_total = n, rank * n, n * world
        pad = n
    else:
        sh = shard.shard_range(n, rank, world)
        per, first, n_total = sh.count, sh.start, n
        pad = -(-n // world)  # ceil: every rank's exchange slot (all-gather needs equal sizes)
    launches = len(cfg["q"]) if cfg["kind"] == "quant" else 1
    px_rank = per * px_per_unit(cfg) * launches  # pixels processed by this rank per step
    return dict(per=per, first=first, n_total=n_total, pad=pad, launches=launches, px_rank=px_rank,
                pixels_per_step=(n_total * px_per_unit(cfg) * launches))


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
# CPU side: the reference package (baseline/_ref) on all host cores
# ---------------------------------------------------------------------------

def _reference_module():
    """(adct, kind): the unmodified reference from baseline/_ref, else None
    (the refport stand-in is used)."""
    if os.path.isdir(os.path.join(REF_DIR, "adct")):
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        try:
            import adct.codec  # noqa: F401
            import adct.kernels  # noqa: F401
            import adct.metrics  # noqa: F401

            return sys.modules["adct"]
        except Exception:
            return None
    return None


_REF_T = None


def _ref_task(args):
    """One reference task on one full image.  kind:
    retain  codec.compress_image + metrics.mse + metrics.psnr (codec.py:144-155, metrics.py:49-65)
    sweep   codec.coefficient_blocks once, then reconstruct_image + mse + psnr per r (cli.py:105-113)
    forward codec.coefficient_blocks (codec.py:120-131)
    quant   the reference's functions composed (the reference has no quantised driver):
            forward_2d_unscaled of the level-shifted tiles, Q' = fold_scaling_into_quantization
            rounded, round-half-away quantise/dequantise, inverse_2d of D Z' D, +128, round, clamp."""
    global _REF_T
    kind, img, param = args
    import numpy as np

    adct = _reference_module()
    if adct is None:  # stand-in: oracle/refport.py restates the same float64 path
        from oracle import refport

        if kind == "retain":
            return refport.psnr(refport.mse(img, refport.compress_image(img, param)))
        if kind == "sweep":
            y = refport.coefficient_blocks(img)
            return [refport.psnr(refport.mse(img, refport.reconstruct_image(y, r, *img.shape)))
                    for r in range(param[0], param[1] + 1)]
        if kind == "forward":
            return float(refport.coefficient_blocks(img)[0, 0, 0])
        rec = np.clip(np.floor(refport.quant_float64(img, param) + 0.5), 0, 255)
        return refport.psnr(refport.mse(img, rec))
    from adct import codec, kernels, metrics

    if _REF_T is None:
        _REF_T = kernels.proposed_transform()
    t = _REF_T
    x = np.asarray(img, dtype=np.float64)
    if kind == "retain":
        return metrics.psnr(metrics.mse(x, codec.compress_image(t, x, param)))
    if kind == "sweep":
        y = codec.coefficient_blocks(t, x)
        return [metrics.psnr(metrics.mse(x, codec.reconstruct_image(t, y, r, *x.shape)))
                for r in range(param[0], param[1] + 1)]
    if kind == "forward":
        return float(codec.coefficient_blocks(t, x)[0, 0, 0])
    # quant: param = the scaled base table Q50 * s(q) (8x8 float64)
    qpu = codec.fold_scaling_into_quantization(t, param)
    qp = np.maximum(1.0, np.floor(qpu + 0.5))
    h, w = x.shape
    tiles = (x - 128.0).reshape(h // 8, 8, w // 8, 8).swapaxes(1, 2).reshape(-1, 8, 8)
    z = codec.forward_2d_unscaled(t, tiles)
    zq = np.sign(z) * np.floor(np.abs(z) / qp + 0.5) * qp
    d = t.scaling.diag
    xr = codec.inverse_2d(t, zq * np.outer(d, d)) + 128.0
    rec = np.clip(np.floor(xr + 0.5), 0, 255).reshape(h // 8, w // 8, 8, 8).swapaxes(1, 2).reshape(h, w)
    return metrics.psnr(metrics.mse(x, rec))


def _ref_kind_param(config: int):
    import numpy as np

    cfg = CONFIGS[config]
    if cfg["kind"] in ("retain", "sweep", "forward"):
        return cfg["kind"], cfg.get("r")
    from paper_1702_00817_b200.quant import q50_luma, quality_scale

    q = cfg["q"][1] if cfg["kind"] == "quant" else cfg["q"]
    return "quant", np.asarray(q50_luma(), dtype=np.float64) * quality_scale(q)


def _ref_images(config: int, count: int):
    """`count` seeded images of the config (host mirror of the generator)."""
    from paper_1702_00817_b200 import synth

    cfg = CONFIGS[config]
    if cfg["kind"] == "planes":  # config 4: the Y plane carries 2/3 of the pixels
        h, w = PLANE_DIMS[0]
        nb, smin, smax = synth.CONFIG_BLOBS[4]
    else:
        h, w = cfg["h"], cfg["w"]
        nb, smin, smax = cfg["blobs"]
    return [synth.render_np(synth.blob_params(s, h, w, nb, smin, smax), h, w, s) for s in range(count)]


def ref_describe(config: int) -> tuple[str, str]:
    """(kind for cpu_baseline, what was timed)."""
    adct = _reference_module()
    kind, _ = _ref_kind_param(config)
    if adct is None:
        return "port", f"oracle/refport.py ({kind}; baseline/_ref absent)"
    what = {"retain": "adct.codec.compress_image + adct.metrics.mse/psnr",
            "sweep": "adct.codec.coefficient_blocks + reconstruct_image/mse/psnr per r",
            "forward": "adct.codec.coefficient_blocks",
            "quant": "adct.codec.forward_2d_unscaled/fold_scaling_into_quantization/inverse_2d composed + metrics"}[kind]
    return "reference", f"unmodified reference package from baseline/_ref: {what}"


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _pool(cores):
    from concurrent.futures import ProcessPoolExecutor

    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    return ProcessPoolExecutor(max_workers=cores)


def cpu_reference_rate(config: int, budget_s: float, cores: int, images=None):
    """Gpixel/s of the reference on full images, streamed: one image per task,
    `cores` workers, tasks queued for about `budget_s` seconds."""
    kind, param = _ref_kind_param(config)
    images = images if images is not None else _ref_images(config, min(cores, 8))
    h, w = images[0].shape
    with _pool(cores) as ex:
        t0 = time.perf_counter()
        list(ex.map(_ref_task, [(kind, images[k % len(images)], param) for k in range(cores)]))
        t_full = time.perf_counter() - t0  # one round (also warms the workers)
        rounds = max(1, int(budget_s / max(t_full, 1e-3)))
        tasks = [(kind, images[k % len(images)], param) for k in range(cores * rounds)]
        t0 = time.perf_counter()
        list(ex.map(_ref_task, tasks, chunksize=1))
        dt = time.perf_counter() - t0
    return len(tasks) * h * w / dt / 1e9, dict(images=len(tasks), seconds=dt, image_shape=[h, w])


def reference_arm(args) -> None:
    """--impl reference: the reference package on the host cores.  A step is
    a bounded sample of the workload: `m` full images per core streamed
    through one process pool (one task per image, no barrier inside a step)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    cores = len(os.sched_getaffinity(0))
    kind, param = _ref_kind_param(args.config)
    images = _ref_images(args.config, min(cores, 8))
    h, w = images[0].shape
    ref_kind, what = ref_describe(args.config)
    budget_step = min(6.0, 150.0 / max(1, args.steps + args.warmup))
    with _pool(cores) as ex:
        t0 = time.perf_counter()
        list(ex.map(_ref_task, [(kind, images[k % len(images)], param) for k in range(cores)]))
        t_round = time.perf_counter() - t0
        m = max(1, int(budget_step / max(t_round, 1e-3)))
        tasks = [(kind, images[k % len(images)], param) for k in range(cores * m)]
        for _ in range(args.warmup):
            list(ex.map(_ref_task, tasks, chunksize=1))
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            list(ex.map(_ref_task, tasks, chunksize=1))
            times.append(time.perf_counter() - t0)
    px_step = len(tasks) * h * w
    total = sum(times)
    value = px_step * len(times) / total / 1e9
    sample = (f"{len(tasks)} full {h}x{w} config-{args.config} images per step ({m} per core, streamed, one task "
              f"per image); {what}")
    if cfg["kind"] == "quant":
        sample += f"; timed at q={cfg['q'][1]} (the middle of the config's qualities)"
    if cfg["kind"] == "planes":
        sample += "; Y planes (2/3 of each frame's pixels)"
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Gaussian blobs + N(0,4^2) noise, BASELINE.json generator)",
        "config": config_block(args.config, world, args.scaling, plan(args.config, 0, world, args.scaling)),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": ref_kind, "sample": sample,
                         "cpu": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


def config_block(config: int, world: int, scaling: str, p: dict, fused: bool = False) -> dict:
    cfg = CONFIGS[config]
    return {"workload": cfg["workload"], "units_per_gpu": p["per"], "pixels_per_step": p["pixels_per_step"],
            "parallelism": f"dp{world} ({'frames' if cfg['kind'] == 'planes' else 'images'} sharded, SSE "
                           + ("exchange fused into the kernel epilogue)" if fused else "all-gather)"),
            "scaling": scaling,
            "l2": "inputs >> 126 MB L2 (no flush needed)" if p["px_rank"] > (256 << 20)
                  else "inputs L2-resident (launch/ALU bound config; no roofline claim)"}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def quant_jit_stats():
    """Counters of the run-time table specialisation of the quant kernels."""
    import ctypes

    from paper_1702_00817_b200 import _lib

    c, l, f = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _lib.lib().adct_quant_jit_stats(ctypes.byref(c), ctypes.byref(l), ctypes.byref(f))
    return {"compiled": c.value, "specialised_launches": l.value, "failures": f.value,
            "after_uses": int(os.environ.get("ADCT_QUANT_JIT_AFTER", "3"))}


class Workload:
    """Resident inputs + the step's launches for one config on this rank."""

    def __init__(self, config: int, args, rank: int, world: int, dev):
        import ctypes

        import torch
        import torch.distributed as dist

        from paper_1702_00817_b200 import _lib, batch, quant, shard, synth

        self.cfg = cfg = CONFIGS[config]
        self.config = config
        self.p = p = plan(config, rank, world, args.scaling)
        self.world, self.rank, self.dev = world, rank, dev
        per, first = p["per"], p["first"]
        self.fused = cfg["kind"] in ("retain", "planes") and args.exchange == "fused"
        stream = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
        if cfg["kind"] == "planes":
            self.planes = synth.video_planes_device(per, frame0=first, device=dev)
            qt = quant.quant_table(cfg["q"])
            self.recs = [torch.empty_like(x) for x in self.planes]
            arr, _ = batch._planes(self.planes, self.recs)
            cols = 3
        else:
            nb, smin, smax = cfg["blobs"]
            self.imgs = synth.images_device(range(first, first + per), cfg["h"], cfg["w"], nb, smin, smax, device=dev)
            cols = {"quant": len(cfg.get("q", ())), "sweep": (cfg["r"][1] - cfg["r"][0] + 1) if cfg["kind"] == "sweep"
                    else 0}.get(cfg["kind"], 1)
        # this rank's SSE rows live in a padded slot so the exchange is one
        # all-gather into a preallocated vector (no per-step allocation or zeroing);
        # config 2 keeps one contiguous row per quality
        shape = (cols, p["pad"]) if cfg["kind"] == "quant" else (p["pad"], cols)
        self.sse_slot = torch.zeros(shape, dtype=torch.int64, device=dev)
        self.sse_all = (torch.zeros((world * shape[0], shape[1]), dtype=torch.int64, device=dev)
                        if world > 1 else None)
        sse = self.sse_slot[:, :per] if cfg["kind"] == "quant" else self.sse_slot[:per]
        if cfg["kind"] == "sweep":
            r0, r1 = cfg["r"]

            def step_kernel():
                _lib.call("adct_sweep_retain_sse", self.imgs.data_ptr(), per, cfg["h"], cfg["w"], cfg["h"] * cfg["w"],
                          r0, r1, sse.data_ptr(), None, stream())
        elif cfg["kind"] == "forward":
            coef = torch.empty((per, cfg["h"] * cfg["w"] // 64, 8, 8), dtype=torch.int32, device=dev)

            def step_kernel():
                _lib.call("adct_forward_int32", self.imgs.data_ptr(), per, cfg["h"], cfg["w"], cfg["h"] * cfg["w"], 0,
                          coef.data_ptr(), stream())
        elif cfg["kind"] == "retain":
            rec = torch.empty_like(self.imgs)
            if self.fused:
                # SSE exchange fused into the kernel epilogue: P2P
                # stores into every rank's symmetric-memory vector + one
                # stream-ordered barrier instead of the NCCL collective
                _ensure_pg(dev)
                exchange = shard.SseExchange(p["n_total"], dev)
                base = first if args.scaling == "strong" else rank * per

                def step_kernel():
                    exchange.compress_retain(self.imgs, cfg["r"], base, out=rec, sse_out=sse[:, 0])
            else:
                def step_kernel():
                    batch.compress_retain(self.imgs, cfg["r"], out=rec, sse_out=sse[:, 0])
        elif cfg["kind"] == "quant":
            qtabs = [quant.quant_table(q) for q in cfg["q"]]
            if args.quant_streams:
                # the qualities are independent compressions of the same batch
                # (own reconstruction buffers): one stream each, forked from and
                # joined back into the current stream, so each ~0.12 ms
                # persistent launch's ramp and tail overlap the next one's
                recs = [torch.empty_like(self.imgs) for _ in qtabs]
                side = [torch.cuda.Stream(dev) for _ in qtabs]

                def step_kernel():
                    main = torch.cuda.current_stream()
                    for k, qt in enumerate(qtabs):
                        side[k].wait_stream(main)
                        with torch.cuda.stream(side[k]):
                            batch.compress_quant(self.imgs, qt, out=recs[k], sse_out=sse[k])
                    for st in side:
                        main.wait_stream(st)
            else:
                rec = torch.empty_like(self.imgs)

                def step_kernel():
                    for k, qt in enumerate(qtabs):
                        batch.compress_quant(self.imgs, qt, out=rec, sse_out=sse[k])
        else:  # planes
            if self.fused:
                _ensure_pg(dev)
                exchange = shard.SseExchange(p["n_total"] * 3, dev)
                f0 = first if args.scaling == "strong" else rank * per

                def step_kernel():
                    exchange.compress_quant_planes(self.planes, qt, f0, out=self.recs)
            else:
                def step_kernel():
                    _lib.call("adct_compress_quant_planes", arr, 3, per, ctypes.byref(qt), sse.data_ptr(), stream())
        self.step_kernel = step_kernel
        self.dist = dist

    def exchange(self):
        if self.world > 1 and not self.fused:
            self.dist.all_gather_into_tensor(self.sse_all, self.sse_slot)


def _ensure_pg(dev):
    import torch.distributed as dist

    if not dist.is_initialized():  # one rank: a world-size-1 group for the symmetric-memory path
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29561")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)


def measure(config: int, args, rank: int, world: int, local: int, dev, steps: int, warmup: int,
            with_e2e: bool, with_cpu: bool) -> dict:
    """Time `steps` steps of one config (after `warmup`); returns the fields of a bench line."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1702_00817_b200 import quant
    from paper_1702_00817_b200.pipeline import HostPipeline, pinned_empty

    cfg = CONFIGS[config]
    t_gen = time.perf_counter()
    wl = Workload(config, args, rank, world, dev)
    p = wl.p
    torch.cuda.synchronize()
    log(f"[rank {rank}] config {config} ready in {time.perf_counter() - t_gen:.1f}s: "
        f"{p['px_rank'] / 1e9:.2f} Gpx per step on this rank")

    step_kernel = wl.step_kernel
    for _ in range(warmup):
        step_kernel()
        wl.exchange()
    torch.cuda.synchronize()
    graphed = False
    if cfg["kind"] in ("sweep", "forward", "quant") and not args.no_graph:
        # short launches (configs 0/1: one small launch; config 2: three
        # ~0.13 ms launches per step): replay the step's C-ABI launches from a
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
    k_start = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    k_end = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_start.record(stream)
    for i in range(steps):
        k_start[i].record(stream)
        step_kernel()
        k_end[i].record(stream)
        wl.exchange()
    t_end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    elapsed_ms = t_start.elapsed_time(t_end)
    kern_ms = sum(a.elapsed_time(b) for a, b in zip(k_start, k_end)) / steps / p["launches"]
    if world > 1:
        t = torch.tensor([elapsed_ms, kern_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms, kern_ms = t.tolist()

    value = p["pixels_per_step"] * steps / (elapsed_ms * 1e-3) / 1e9
    px_launch = p["px_rank"] / p["launches"]
    bytes_per_px = {"sweep": 1, "forward": 5}.get(cfg["kind"], 2)  # u8 in (+ u8 out | + int32 coefficients)
    cols = wl.sse_slot.shape[1] if cfg["kind"] != "quant" else 1
    alg_bytes = bytes_per_px * px_launch + 8 * p["per"] * cols
    achieved = alg_bytes / (kern_ms * 1e-3) / 1e9
    peak, peak_src = measured_hbm_peak()
    out = {"value": value, "elapsed_ms": elapsed_ms, "kern_ms": kern_ms, "alg_bytes": alg_bytes,
           "achieved": achieved, "peak": peak, "peak_src": peak_src, "clocks": clk, "graphed": graphed,
           "plan": p, "fused": wl.fused}

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

    if with_e2e and cfg["kind"] in ("retain", "quant", "planes"):
        per = p["per"]
        if cfg["kind"] == "planes":  # frames of Y/Cb/Cr host planes
            m = min(per, max(1, args.e2e_images // 4))
            host_in = [pinned_empty((m,) + tuple(x.shape[1:])) for x in wl.planes]
            for a, x in zip(host_in, wl.planes):
                a[...] = x[:m].cpu().numpy()
            host_out = [pinned_empty(a.shape) for a in host_in]
            n_sse = 3 * m
            qt4 = quant.quant_table(cfg["q"])
            chunk = max(args.e2e_chunk_mb << 20, 5 * sum(a[0].nbytes for a in host_in))  # ~5 frames: measured best
            api = "adct_pipeline_compress_quant_planes (C ABI) via paper_1702_00817_b200.pipeline"
            units = {"frames_per_step": world * m}
        else:
            m = min(per, args.e2e_images)
            host_in = [pinned_empty(tuple(wl.imgs[:m].shape))]
            host_in[0][...] = wl.imgs[:m].cpu().numpy()
            host_out = [pinned_empty(host_in[0].shape)]
            n_sse = m
            qt0 = quant.quant_table(cfg["q"][0]) if cfg["kind"] == "quant" else None
            chunk = args.e2e_chunk_mb << 20
            api = "adct_pipeline_compress_* (C ABI) via paper_1702_00817_b200.pipeline"
            units = {"images_per_step": world * m}
        try:
            with HostPipeline(local, chunk_bytes=chunk) as pipe:
                if cfg["kind"] == "planes":
                    call = lambda outs: pipe.compress_quant_planes(host_in, qt4, outs, register=False)  # noqa: E731
                elif cfg["kind"] == "retain":
                    call = lambda outs: pipe.compress_retain(host_in[0], cfg["r"], outs and outs[0], register=False)  # noqa: E731
                else:
                    call = lambda outs: pipe.compress_quant(host_in[0], qt0, outs and outs[0], register=False)  # noqa: E731
                dt = timed_e2e(call, host_out)  # reconstructions come back to the host every step
                dt_metric = timed_e2e(call, None)  # inputs in, per-image SSE (-> PSNR) back
                # what a drop-in caller hands over: ordinary (pageable) numpy
                # arrays, staged by the library through its own page-locked ring
                pg_in = [np.array(a) for a in host_in]
                pg_out = [np.empty_like(a) for a in host_in]
                host_in_pinned = host_in
                host_in = pg_in
                dt_pageable = timed_e2e(call, pg_out)
                host_in = host_in_pinned
                del pg_in, pg_out
            px = world * sum(a.size for a in host_in)
            nbytes = sum(a.nbytes for a in host_in)
            out["e2e"] = {"value": px / dt / 1e9, "unit": UNIT,
                          "h2d_bytes_per_step": int(world * nbytes),
                          "d2h_bytes_per_step": int(world * (nbytes + 8 * n_sse)),
                          **units,
                          "api": api + ", every rank, max time over ranks",
                          "pageable": {"value": px / dt_pageable / 1e9, "unit": UNIT,
                                       "h2d_bytes_per_step": int(world * nbytes),
                                       "d2h_bytes_per_step": int(world * (nbytes + 8 * n_sse)),
                                       "note": "plain pageable numpy arrays in and out (a drop-in caller's buffers); "
                                               "the library stages them through its own page-locked ring"},
                          "metric_only": {"value": px / dt_metric / 1e9, "unit": UNIT,
                                          "h2d_bytes_per_step": int(world * nbytes),
                                          "d2h_bytes_per_step": int(world * 8 * n_sse),
                                          "note": "reconstructions kept on the device; only the SSE/PSNR vector is read back"}}
        finally:
            del host_in, host_out

    # ---- CPU baseline (rank 0, N=1) ---------------------------------------------
    if with_cpu and rank == 0 and world == 1:
        cores = len(os.sched_getaffinity(0))
        if cfg["kind"] == "planes":
            sample_imgs = [wl.planes[0][k].cpu().numpy() for k in range(min(p["per"], 4))]
        else:
            sample_imgs = [wl.imgs[k].cpu().numpy() for k in range(min(p["per"], 8))]
        v, info = cpu_reference_rate(config, args.cpu_seconds, cores, images=sample_imgs)
        kind, what = ref_describe(config)
        out["cpu_baseline"] = {
            "value": v, "unit": UNIT, "cores": cores, "kind": kind, "cpu": cpu_model(),
            "sample": f"{info['images']} full {info['image_shape'][0]}x{info['image_shape'][1]} config-{config} "
                      f"images, one task per image streamed over {cores} processes, {info['seconds']:.1f}s; {what}"}
    del wl
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return out


def gpu_arm(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_1702_00817_b200 import shard

    rank, world, local = shard.init_from_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world != args.gpus:
        log(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}; using {world}")

    main = measure(args.config, args, rank, world, local, dev, args.steps, args.warmup,
                   with_e2e=not args.no_e2e, with_cpu=not args.no_cpu)
    secondary = {}
    if args.config == 3 and not args.no_secondary:
        # the quantised kernels measured in the same run (same box, same clock record)
        # (config 2's step is ~0.4 ms: 10x the steps keep the timed region long
        # enough for the 50 ms nvidia-smi clock sampler to see it)
        for c, steps in ((4, max(3, min(args.steps, 20))), (2, max(3, min(10 * args.steps, 1000)))):
            s = measure(c, args, rank, world, local, dev, steps, max(args.warmup, 4), with_e2e=False, with_cpu=False)
            secondary[f"config{c}"] = {
                "value": s["value"], "unit": UNIT, "steps": steps, "ms_per_step": s["elapsed_ms"] / steps,
                "config": config_block(c, world, args.scaling, s["plan"], s["fused"]),
                "roofline": {"bound": "hbm", "achieved": s["achieved"], "peak": s["peak"], "unit": "GB/s",
                             "frac": s["achieved"] / s["peak"], "traffic": ncu_traffic(c), "kernel_ms": s["kern_ms"],
                             "algorithmic_bytes_per_launch": s["alg_bytes"]},
                "clocks": s["clocks"], "cuda_graph": s["graphed"]}

    if rank == 0:
        p = main["plan"]
        line = {
            "metric": METRIC, "value": main["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": main["elapsed_ms"] / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (seeded Gaussian blobs + N(0,4^2) noise, BASELINE.json generator, rendered on GPU)",
            "config": config_block(args.config, world, args.scaling, p, main["fused"]),
            "roofline": {"bound": "hbm", "achieved": main["achieved"], "peak": main["peak"], "unit": "GB/s",
                         "frac": main["achieved"] / main["peak"], "traffic": ncu_traffic(args.config),
                         "kernel_ms": main["kern_ms"], "algorithmic_bytes_per_launch": main["alg_bytes"],
                         "peak_source": main["peak_src"]},
            "clocks": main["clocks"],
            "e2e": main.get("e2e"),
            "gpu_launches": p["launches"] * args.steps,
            "cuda_graph": main["graphed"],
            "quant_jit": quant_jit_stats(),
            "cpu_baseline": main.get("cpu_baseline"),
        }
        if secondary:
            line["secondary"] = secondary
        emit(line)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


def plan_arm(args) -> None:
    """--plan: the workload split as the GPU arm would use it (no GPU work)."""
    from paper_1702_00817_b200 import shard

    rank, world, _ = shard.init_from_env("gloo" if not os.environ.get("ADCT_DIST_BACKEND") else None)
    p = plan(args.config, rank, world, args.scaling)
    if world > 1:
        import torch
        import torch.distributed as dist

        got = [None] * world
        dist.all_gather_object(got, p)
        units = sum(g["per"] for g in got)
        firsts = [g["first"] for g in got]
        dist.barrier()
        dist.destroy_process_group()
    else:
        units, firsts = p["per"], [p["first"]]
    if rank == 0:
        emit({"plan": p, "units_all_ranks": units, "first_unit_per_rank": firsts,
              "config": config_block(args.config, world, args.scaling, p)})


def main() -> None:
    global _OUT
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=3, choices=sorted(CONFIGS),
                    help="3 (default, large-batch headline), 4, 2, 1 (sweep), 0 (forward)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong (default): the config's units split over the GPUs; weak: every GPU runs the whole config")
    ap.add_argument("--plan", action="store_true", help="print the per-rank workload split and exit (no GPU work)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="config 3: skip the config 4 / config 2 secondary lines")
    ap.add_argument("--no-graph", action="store_true", help="configs 0/1/2: launch through the C ABI every step")
    ap.add_argument("--exchange", default="allreduce", choices=["allreduce", "fused"],
                    help="configs 3 and 4: SSE exchange by NCCL collective (default) or fused into the kernel "
                         "epilogue through torch symmetric memory")
    ap.add_argument("--quant-streams", type=int, default=1,
                    help="config 2: run the three qualities on concurrent streams (1, default: +4%%) or back to back (0)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--e2e-images", type=int, default=256)
    ap.add_argument("--e2e-chunk-mb", type=int, default=32)
    args = ap.parse_args()
    # stdout carries exactly one JSON line: anything else the libraries print
    # to fd 1 (e.g. NCCL's "NCCL version ..." banner when symmetric memory
    # initialises it) is sent to stderr, and the JSON goes to a saved copy of fd 1
    _OUT = os.fdopen(os.dup(1), "w")
    sys.stdout.flush()
    os.dup2(2, 1)
    if args.warmup < 3:
        log("warmup raised to 3 (timing rules)")
        args.warmup = 3
    if args.plan:
        plan_arm(args)
    elif args.impl == "reference":
        reference_arm(args)
    else:
        gpu_arm(args)


if __name__ == "__main__":
    main()
