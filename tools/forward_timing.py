"""Forward-transform kernel timing (K1): int32 and int16 coefficients for a
large batch (inputs and outputs >> L2) and for config 0 (one 512^2 image)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1702_00817_b200 import batch, synth

dev = torch.device("cuda", 0)
PEAK = 6552.3


def timeit(f, reps=20):
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


res = {}
for name, n, hw in (("large", 256, 1024), ("config0", 1, 512)):
    x = synth.images_device(range(n), hw, hw, 16, 8.0, 64.0, device=dev)
    for bits in (32, 16):
        dt = torch.int32 if bits == 32 else torch.int16
        out = torch.empty((n, hw * hw // 64, 8, 8), dtype=dt, device=dev)
        ms = timeit(lambda: batch.forward_int(x, out=out))
        gb = x.numel() * (1 + bits // 8) / 1e9
        res[f"{name}_int{bits}"] = {"ms": ms, "gpix_s": x.numel() / ms / 1e6, "GB_s": gb / ms * 1e3,
                                    "frac": gb / ms * 1e3 / PEAK}
print(json.dumps(res, indent=1))
