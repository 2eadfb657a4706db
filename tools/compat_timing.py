"""Timing of the compatibility kernels (float64 reference-API paths, SURVEY
§8 rows a7/a9/a13 and f1): forward_f64 / inverse_f64 (proposed transform,
flow graph), forward_dense / inverse_dense / sweep_dense_sse (any 8x8 matrix,
here the exact DCT), on config 1's corpus (45 x 512^2) and on a larger
batch (64 x 1024^2).  Prints one JSON object: per kernel ms, Gpixel/s and the
achieved rate of algorithmic bytes (input + output, 1 B per uint8 pixel,
8 B per float64 value)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1702_00817_b200 import batch, synth, transforms


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    dev = torch.device("cuda", 0)
    dct = np.asarray(transforms.exact_dct_matrix().matrix, dtype=np.float64)
    res = {}
    cases = {"config1_45x512": synth.config_images_device(1, range(45), device=dev),
             "64x1024": synth.config_images_device(2, range(64), device=dev)}
    for name, u8 in cases.items():
        n, h, w = u8.shape
        px = n * h * w
        f64 = u8.to(torch.float64)
        coef = batch.forward_f64(u8)
        rows = {
            "forward_f64(u8)": (lambda: batch.forward_f64(u8), 1 + 8),
            "forward_f64(f64)": (lambda: batch.forward_f64(f64), 8 + 8),
            "inverse_f64(r=10,clamp)": (lambda: batch.inverse_f64(coef, h, w, r=10, clamp=True), 8 + 8),
            "forward_dense(u8,DCT)": (lambda: batch.forward_dense(u8, dct), 1 + 8),
            "inverse_dense(r=10,clamp,DCT)": (lambda: batch.inverse_dense(coef, h, w, dct, r=10, clamp=True), 8 + 8),
            "sweep_dense_sse(u8,DCT,r=1..45)": (lambda: batch.sweep_dense_sse(u8, dct, 1, 45), 1),
        }
        for k, (fn, bpp) in rows.items():
            ms = timed(fn)
            res[f"{name}/{k}"] = {"ms": round(ms, 4), "gpix_s": round(px / ms / 1e6, 1),
                                  "algo_GBps": round(px * bpp / ms / 1e6, 1)}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
