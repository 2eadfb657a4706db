"""Raw host<->device copy bandwidth with pinned buffers (ceiling for e2e)."""
import time, json, sys
import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1702_00817_b200.pipeline import HostPipeline, pin, unpin


GB = 1 << 30
h = torch.empty(GB, dtype=torch.uint8).pin_memory()
h2 = torch.empty(GB, dtype=torch.uint8).pin_memory()
d = torch.empty(GB, dtype=torch.uint8, device="cuda")
d2 = torch.empty(GB, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
res = {}
for name, fn in [
    ("h2d", lambda: d.copy_(h, non_blocking=True)),
    ("d2h", lambda: h.copy_(d, non_blocking=True)),
]:
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5): fn()
    torch.cuda.synchronize()
    res[name] = 5 * GB / (time.perf_counter() - t) / 1e9
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
both(); torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5): both()
torch.cuda.synchronize()
res["bidir_each"] = 5 * GB / (time.perf_counter() - t) / 1e9
imgs = torch.randint(0, 256, (256, 2048, 2048), dtype=torch.uint8).numpy()
out = np.empty_like(imgs)
pin(imgs); pin(out)
import os
for depth in (2, 3, 4, 6):
    os.environ["ADCT_PIPELINE_DEPTH"] = str(depth)
    for mb in (16, 32, 64):
        with HostPipeline(0, chunk_bytes=mb << 20) as p:
            p.compress_retain(imgs, 10, out, register=False)
            t = time.perf_counter()
            for _ in range(3): p.compress_retain(imgs, 10, out, register=False)
            res[f"pipeline_d{depth}_chunk{mb}MB_gpix"] = 3 * imgs.size / (time.perf_counter() - t) / 1e9
unpin(imgs); unpin(out)
print(json.dumps(res))
