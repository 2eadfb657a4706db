"""The drop-in measured at the reference's own call site: the UNMODIFIED
`adct.cli.run_sweep` (cli.py:87-124, installed in baseline/_ref) over config
1's corpus (45 seeded 512x512 uint8 images, r = 1..45), timed three ways:

* `reference`  - the reference package alone, on the host (one process, as
                 the reference runs it; a bounded image sample, scaled);
* `dispatched` - the same unmodified function after the INTEGRATION.md §3
                 dispatch module rebinds adct.codec / adct.metrics to this
                 package's GPU wrappers (every coefficient_blocks /
                 reconstruct_image / mse call crosses PCIe with float64
                 arrays, because the reference's loop asks for them);
* `native`     - the same call with the dispatch's drivers=True: cli.run_sweep
                 rebound to this package's sweep.run_sweep (same records),
                 which moves each image once as uint8 and computes every r
                 in one kernel.

Prints one JSON object (seconds for the whole sweep, and image-pixels/s)."""

import json
import os
import re
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import adct  # noqa: E402
import adct.cli  # noqa: E402
from paper_1702_00817_b200 import synth  # noqa: E402


def main():
    n_cpu = int(os.environ.get("DROPIN_CPU_IMAGES", "4"))
    imgs = synth.images_np(range(45), 512, 512, 16, 8.0, 64.0)
    corpus = [(f"img{i:02d}", imgs[i]) for i in range(45)]
    px = 45 * 512 * 512
    out = {"corpus": "config 1: 45 x 512x512 uint8, r = 1..45"}
    for names in (("proposed",), ("dct", "proposed")):
        key = "+".join(names)
        cfg = adct.cli.ExperimentConfig(transforms=names, r_min=1, r_max=45)
        t = time.perf_counter()
        adct.cli.run_sweep(cfg, corpus[:n_cpu])
        cpu_s = (time.perf_counter() - t) * 45 / n_cpu
        text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
        code = re.findall(r"```python\n(# adct/_gpu_dispatch.py.*?)```", text, re.S)[0]
        ns = {"__name__": "adct._gpu_dispatch"}
        exec(compile(code, "INTEGRATION.md:adct/_gpu_dispatch.py", "exec"), ns)
        ns["enable"]()
        try:
            adct.cli.run_sweep(cfg, corpus[:2])  # warm-up (library load, first launches)
            torch.cuda.synchronize()
            t = time.perf_counter()
            adct.cli.run_sweep(cfg, corpus)
            torch.cuda.synchronize()
            disp_s = time.perf_counter() - t
        finally:
            ns["disable"]()
        ns["enable"](drivers=True)  # the reference's run_sweep itself rebound to the batched sweep
        try:
            adct.cli.run_sweep(cfg, corpus[:2])
            torch.cuda.synchronize()
            t = time.perf_counter()
            adct.cli.run_sweep(cfg, corpus)
            torch.cuda.synchronize()
            nat_s = time.perf_counter() - t
        finally:
            ns["disable"]()
        out[key] = {
            "reference_s": round(cpu_s, 3), "reference_sample_images": n_cpu,
            "dispatched_s": round(disp_s, 4), "native_s": round(nat_s, 4),
            "reference_mpix_s": round(px / cpu_s / 1e6, 2), "dispatched_mpix_s": round(px / disp_s / 1e6, 1),
            "native_mpix_s": round(px / nat_s / 1e6, 1),
            "speedup_dispatched": round(cpu_s / disp_s, 1), "speedup_native": round(cpu_s / nat_s, 1),
        }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
