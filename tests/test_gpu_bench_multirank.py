"""bench.py's multi-rank path on the one GPU a gpurun box has: two ranks
under torchrun with the test hooks ADCT_DIST_BACKEND=gloo (collectives on the
CPU, so no kernel waits on another rank's) and ADCT_DEVICE_MAP=0 (both ranks
on GPU 0).  Real kernels, the strong-scaling split of config 3, the secondary
configs, the e2e pipeline on every rank and max-over-ranks timing; rank 0
prints the one JSON line."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_on_one_gpu(cuda):
    env = dict(os.environ, ADCT_DIST_BACKEND="gloo", ADCT_DEVICE_MAP="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29571", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-cpu"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["config"]["units_per_gpu"] == 2048 and d["config"]["pixels_per_step"] == 4096 * 2048 * 2048
    assert d["e2e"]["value"] > 0 and set(d["secondary"]) == {"config4", "config2"}
    assert d["secondary"]["config4"]["config"]["units_per_gpu"] == 256
