"""Per-quality quant kernel timing on config 2 (256 x 1024^2)."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1702_00817_b200 import batch, quant, synth

dev = torch.device("cuda", 0)
x = synth.config_images_device(2, range(256), device=dev)
rec = torch.empty_like(x)
res = {}
for q in (10, 25, 50, 75, 90):
    qt = quant.quant_table(q)
    f = lambda: batch.compress_quant(x, qt, out=rec)
    for _ in range(4):  # past ADCT_QUANT_JIT_AFTER (3): the table-specialised kernel is built here
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): f()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    res[f"q{q}"] = {"ms": ms, "gpix_s": x.numel() / ms / 1e6, "wide": qt.wide, "aligned": qt.aligned}
print(json.dumps(res))
