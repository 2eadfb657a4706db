"""e2e (pinned host -> GPU -> host) throughput of the C-ABI pipeline vs chunk
size, pipeline depth and images per call (config-3 images, retain r=10)."""
import json, os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

if len(sys.argv) > 1:  # child: one depth (ADCT_PIPELINE_DEPTH is read at create time)
    import torch
    from paper_1702_00817_b200 import synth
    from paper_1702_00817_b200.pipeline import HostPipeline, pin, unpin
    n_max = 1024
    dev = torch.device("cuda", 0)
    imgs = synth.config_images_device(3, range(64), device=dev).cpu().numpy()
    host_in = np.empty((n_max, 2048, 2048), np.uint8)
    for k in range(n_max):
        host_in[k] = imgs[k % 64]
    host_out = np.empty_like(host_in)
    pin(host_in); pin(host_out)
    res = {}
    for chunk_mb in (16, 32, 64, 128):
        with HostPipeline(0, chunk_bytes=chunk_mb << 20) as pipe:
            for n in (256, 1024):
                a, b = host_in[:n], host_out[:n]
                pipe.compress_retain(a, 10, b, register=False)
                t0 = time.perf_counter()
                for _ in range(3):
                    pipe.compress_retain(a, 10, b, register=False)
                dt = (time.perf_counter() - t0) / 3
                res[f"depth{os.environ.get('ADCT_PIPELINE_DEPTH', '3')}_chunk{chunk_mb}MB_n{n}"] = round(n * 2048 * 2048 / dt / 1e9, 2)
    unpin(host_in); unpin(host_out)
    print(json.dumps(res))
else:
    for d in (2, 3, 4):
        env = dict(os.environ, ADCT_PIPELINE_DEPTH=str(d))
        print(subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True).stdout.strip())
