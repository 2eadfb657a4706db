"""e2e from pageable numpy through the host pipeline's staging ring, per
ADCT_PIPELINE_THREADS and chunk size (config-3 images), plus the box's raw
host memcpy bandwidth for reference.  Prints one line per setting."""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1702_00817_b200 import synth  # noqa: E402
from paper_1702_00817_b200.pipeline import HostPipeline  # noqa: E402

n = int(os.environ.get("E2E_IMAGES", "256"))
imgs_d = synth.config_images_device(3, range(n), device="cuda")
src = imgs_d.cpu().numpy()
dst = np.empty_like(src)
dst[...] = 1  # fault the pages in
nbytes = src.nbytes

for th in (1, 4, 8, 16):
    a = np.empty(64 << 20, np.uint8); a[:] = 1; b = np.empty_like(a); b[:] = 2
    pieces = np.array_split(np.arange(a.size), th)
    def cp(ix):
        b[ix[0]:ix[-1] + 1] = a[ix[0]:ix[-1] + 1]
    with ThreadPoolExecutor(th) as ex:
        list(ex.map(cp, pieces))
        t0 = time.perf_counter()
        for _ in range(10):
            list(ex.map(cp, pieces))
        dt = (time.perf_counter() - t0) / 10
    print(f"host memcpy {th:2d} threads: {a.nbytes / dt / 1e9:.1f} GB/s", flush=True)

for th in (2, 4, 8, 12, 16):
    for chunk_mb in (16, 32, 64):
        os.environ["ADCT_PIPELINE_THREADS"] = str(th)
        with HostPipeline(0, chunk_bytes=chunk_mb << 20) as p:
            p.compress_retain(src, 10, dst)
            t0 = time.perf_counter()
            for _ in range(3):
                p.compress_retain(src, 10, dst)
            dt = (time.perf_counter() - t0) / 3
        print(f"pageable e2e threads={th:2d} chunk={chunk_mb}MiB: {src.size / dt / 1e9:.2f} Gpixel/s", flush=True)
