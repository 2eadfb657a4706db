"""Every device entry point once on small inputs (for compute-sanitizer)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1702_00817_b200 import batch, quant, synth, transforms
from paper_1702_00817_b200.pipeline import HostPipeline

dev = torch.device("cuda", 0)
g = torch.Generator().manual_seed(0)
x = torch.randint(0, 256, (3, 64, 96), dtype=torch.uint8, generator=g).to(dev)
xr = torch.randint(0, 256, (2, 24, 40), dtype=torch.uint8, generator=g).to(dev)  # ragged width
for dt in (torch.int32, torch.int16):
    batch.forward_int(x, dtype=dt); batch.forward_int(xr, dtype=dt, level_shift=True)
for r in (1, 10, 45, 64):
    batch.compress_retain(x, r); batch.compress_retain(x, r, unrounded_sse=True); batch.compress_retain(xr, r)
for q in (10, 50, 75):
    qt = quant.quant_table(q)
    batch.compress_quant(x, qt); batch.compress_quant(xr, qt)
planes = [x, x[:, :32, :48].contiguous(), x[:, :32, :48].contiguous()]
batch.compress_quant_planes(planes, quant.quant_table(75)); batch.compress_retain_planes(planes, 10)
batch.sweep_retain_sse(x, 1, 45); batch.sweep_retain_sse_unrounded(xr, 3, 9)
C = transforms.exact_dct_matrix().matrix
c = batch.forward_dense(x, C); batch.inverse_dense(c, 64, 96, C, r=10, clamp=True); batch.sweep_dense_sse(xr, C, 1, 12)
f = batch.forward_f64(x); batch.inverse_f64(f, 64, 96, r=20, clamp=True)
batch.sse_u8(x, x.flip(2).contiguous())
synth.images_device([0, 1], 64, 96, 16, 8.0, 64.0, device=dev)
imgs = x.cpu().numpy(); rec = np.empty_like(imgs)
with HostPipeline(0, chunk_bytes=64 * 96 * 2) as p:
    p.compress_retain(imgs, 10, rec); p.compress_quant(imgs, quant.quant_table(50), rec)
    hp = [pl.cpu().numpy() for pl in planes]
    p.compress_quant_planes(hp, quant.quant_table(10), [np.empty_like(a) for a in hp])
from paper_1702_00817_b200.pipeline import pinned_empty
buf = pinned_empty((2, 64, 96)); buf[...] = 7
batch.compress_quant(x, quant.quant_table(2))  # Q' > 8191 somewhere: scalar coarse-table kernel
peers = [torch.zeros(8, dtype=torch.int64, device=dev) for _ in range(2)]
ptrs = torch.tensor([v.data_ptr() for v in peers], dtype=torch.int64, device=dev)
arr = torch.zeros(9, dtype=torch.int32, device=dev)
batch.compress_retain_exchange(x, 10, ptrs.data_ptr(), 2, 1, arr)
peers9 = [torch.zeros(12, dtype=torch.int64, device=dev) for _ in range(2)]
ptrs9 = torch.tensor([v.data_ptr() for v in peers9], dtype=torch.int64, device=dev)
batch.compress_quant_planes_exchange(planes, quant.quant_table(75), ptrs9.data_ptr(), 2, 1, arr)
torch.cuda.synchronize()
print("sanitize smoke done")
