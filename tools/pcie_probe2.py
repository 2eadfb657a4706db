"""Pinned-memory kind vs PCIe rate: cudaHostAlloc (torch pin_memory) vs
cudaHostRegister'd numpy buffers, for raw bidirectional copies and for the
C-ABI pipeline."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1702_00817_b200.pipeline import HostPipeline, pin, unpin

GB = 1 << 30
res = {}
d = torch.empty(GB, dtype=torch.uint8, device="cuda")
d2 = torch.empty(GB, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def bidir(h_in, h_out):
    def both():
        with torch.cuda.stream(s1):
            d.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d2, non_blocking=True)
    both(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        both()
    torch.cuda.synchronize()
    return 5 * GB / (time.perf_counter() - t) / 1e9


a = torch.empty(GB, dtype=torch.uint8).pin_memory()
b = torch.empty(GB, dtype=torch.uint8).pin_memory()
res["bidir_hostalloc"] = bidir(a, b)
na = np.ones(GB, np.uint8); nb = np.ones(GB, np.uint8)
pin(na); pin(nb)
res["bidir_registered"] = bidir(torch.from_numpy(na), torch.from_numpy(nb))
unpin(na); unpin(nb)

n = 256
img_t = torch.randint(0, 256, (n, 2048, 2048), dtype=torch.uint8).pin_memory()
out_t = torch.empty_like(img_t).pin_memory()
imgs, out = img_t.numpy(), out_t.numpy()
for mb in (32, 64):
    with HostPipeline(0, chunk_bytes=mb << 20) as p:
        p.compress_retain(imgs, 10, out, register=False)
        t = time.perf_counter()
        for _ in range(3):
            p.compress_retain(imgs, 10, out, register=False)
        res[f"pipeline_hostalloc_chunk{mb}MB_gpix"] = 3 * imgs.size / (time.perf_counter() - t) / 1e9
print(json.dumps(res))
