"""Multi-rank path on CPU: two gloo ranks shard a batch, compute per-image SSE
on their slice (oracle as the stand-in compute), and all-reduce; the result
must equal the single-process answer bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import exact
from paper_1702_00817_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    r, w, _ = shard.init_from_env("gloo")
    assert (r, w) == (rank, world)
    rng = np.random.default_rng(123)
    imgs = rng.integers(0, 256, (n, 32, 48), dtype=np.uint8)

    def compute(sh):
        part = imgs[sh.start : sh.stop]
        if sh.count == 0:
            return torch.zeros(0, dtype=torch.int64)
        return torch.from_numpy(exact.compress_retain(part, 10)[1].astype(np.int64))

    full = shard.run_sharded(n, compute)
    planes = torch.zeros((n, 3), dtype=torch.int64)
    sh = shard.shard_range(n, rank, world)
    planes[sh.start : sh.stop] = rank + 1
    g = shard.global_sse(planes[sh.start : sh.stop], sh, n)
    if rank == 0:
        np.save(out_path, np.concatenate([full.numpy(), g.numpy()[:, 0]]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [7, 2])
def test_two_rank_sse_allreduce_matches_single_process(tmp_path, n):
    out = str(tmp_path / "r.npy")
    mp.spawn(_worker, args=(2, _free_port(), n, out), nprocs=2, join=True)
    got = np.load(out)
    rng = np.random.default_rng(123)
    imgs = rng.integers(0, 256, (n, 32, 48), dtype=np.uint8)
    want = exact.compress_retain(imgs, 10)[1]
    assert np.array_equal(got[:n], want)
    owner = np.array([1 + (i >= shard.shard_range(n, 0, 2).stop) for i in range(n)])
    assert np.array_equal(got[n:], owner)
