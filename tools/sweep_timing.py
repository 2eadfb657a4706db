"""Config 1 (45 seeded 512x512 images, SSE for r = 1..45) and config 0 timings."""
import json, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1702_00817_b200 import batch, synth

dev = torch.device("cuda", 0)
x = synth.config_images_device(1, range(45), device=dev)
res = {}
def timeit(fn, reps=20):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
res["config1_sweep_rounded_ms"] = timeit(lambda: batch.sweep_retain_sse(x, 1, 45))
res["config1_sweep_rounded_and_unrounded_ms"] = timeit(lambda: batch.sweep_retain_sse_unrounded(x, 1, 45))
res["config1_sweep_unrounded_only_ms"] = timeit(lambda: batch.sweep_retain_sse_unrounded(x, 1, 45, rounded=False))
res["config1_45_separate_retain_launches_ms"] = timeit(lambda: [batch.compress_retain(x, r, reconstruct=False) for r in range(1, 46)], 5)
x0 = synth.config_images_device(0, [0], device=dev)
res["config0_forward_int32_ms"] = timeit(lambda: batch.forward_int(x0))
res["config0_forward_int16_ms"] = timeit(lambda: batch.forward_int(x0, dtype=torch.int16))
print(json.dumps(res))
