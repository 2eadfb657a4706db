"""Per-rank share of config 3 (4096 x 2048^2, retain r=10) on one GPU: the
fused kernel over 4096/N images for N = 1, 2, 4, 8, CUDA events, inputs
resident.  The kernel time of the 1/N share, against the full batch's, is
what strong scaling over N GPUs can at best reach (plus one all-gather of a
32 KiB SSE vector per step, not measurable on one GPU).  A projection, not a
multi-GPU measurement."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1702_00817_b200 import batch, synth


def main():
    dev = torch.device("cuda", 0)
    x = synth.config_images_device(3, range(4096), device=dev)
    out = torch.empty_like(x)
    sse = torch.empty(4096, dtype=torch.int64, device=dev)
    res = {}
    for n_gpu in (1, 2, 4, 8):
        k = 4096 // n_gpu
        xs, os_, ss = x[:k], out[:k], sse[:k]
        for _ in range(3):
            batch.compress_retain(xs, 10, out=os_, sse_out=ss)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20 * n_gpu
        a.record()
        for _ in range(reps):
            batch.compress_retain(xs, 10, out=os_, sse_out=ss)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        res[f"share_1_of_{n_gpu}"] = {"images": k, "kernel_ms": round(ms, 4),
                                      "gpix_s_per_gpu": round(k * 2048 * 2048 / ms / 1e6, 1)}
    t1 = res["share_1_of_1"]["kernel_ms"]
    for n_gpu in (2, 4, 8):
        r = res[f"share_1_of_{n_gpu}"]
        r["kernel_speedup_vs_1"] = round(t1 / r["kernel_ms"], 2)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
