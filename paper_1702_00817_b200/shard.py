"""Batch sharding across the GPUs of one box (north-star subsystem 5).

Images (or video frames) are independent, so rank k of N owns the contiguous
range [k*n/N, (k+1)*n/N) and runs the fused kernel on it with no data-path
communication.  The only exchange is the per-image int64 SSE vector, after
which every rank holds the exact global SSE and PSNR — bit-identical for any
N because integer sums are order independent.  Two ways to exchange it:

* `global_sse` / `run_sharded`: one all-reduce(SUM) (each rank fills its
  slice, zeros elsewhere) — NCCL over NVLink.
* `SseExchange`: the retain kernel's epilogue stores each
  finished image's SSE straight into every rank's symmetric-memory vector
  (P2P over NVLink), then one stream-ordered symmetric-memory barrier; no
  collective launch.

torch.distributed is the plumbing: NCCL over NVLink/NVSwitch on the B200 box,
gloo on CPU for the multi-rank tests.
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Callable

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    start: int
    stop: int

    @property
    def count(self) -> int:
        return self.stop - self.start


def shard_range(n: int, rank: int, world: int) -> Shard:
    """Contiguous balanced split: sizes differ by at most one, earlier ranks larger."""
    if world < 1 or not 0 <= rank < world or n < 0:
        raise ValueError(f"bad shard request n={n} rank={rank} world={world}")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    stop = start + base + (1 if rank < extra else 0)
    return Shard(rank, world, start, stop)


def init_from_env(backend: str | None = None) -> tuple[int, int, int]:
    """(rank, world, local_rank) from torchrun's environment; initialises the
    default process group when WORLD_SIZE > 1 (NCCL if CUDA, else gloo)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    # Test hooks: ADCT_DIST_BACKEND=gloo runs the collectives on the CPU and
    # ADCT_DEVICE_MAP=0 puts every rank on GPU 0, so the multi-rank logic can
    # be exercised on a one-GPU box (no kernel ever waits on another rank).
    if os.environ.get("ADCT_DEVICE_MAP") is not None:
        local = int(os.environ["ADCT_DEVICE_MAP"])
    backend = backend or os.environ.get("ADCT_DIST_BACKEND")
    if world > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group(backend, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world, local


def global_sse(local_sse: torch.Tensor, shard: Shard, n_total: int, group=None) -> torch.Tensor:
    """Scatter this rank's per-unit SSE into a zero int64[n_total, ...] vector and
    all-reduce(SUM) it; returns the global vector (identical on every rank)."""
    full = torch.zeros((n_total,) + tuple(local_sse.shape[1:]), dtype=torch.int64, device=local_sse.device)
    full[shard.start : shard.stop] = local_sse
    if shard.world > 1:
        dist.all_reduce(full, op=dist.ReduceOp.SUM, group=group)
    return full


def run_sharded(
    n_total: int,
    compute: Callable[[Shard], torch.Tensor],
    *,
    rank: int | None = None,
    world: int | None = None,
    group=None,
) -> torch.Tensor:
    """Run `compute(shard)` (-> int64 SSE for the shard's units) on this rank's
    range and return the all-reduced global SSE."""
    if world is None:
        world = dist.get_world_size(group) if dist.is_initialized() else 1
    if rank is None:
        rank = dist.get_rank(group) if dist.is_initialized() else 0
    sh = shard_range(n_total, rank, world)
    local = compute(sh)
    if local.shape[0] != sh.count:
        raise ValueError(f"compute returned {local.shape[0]} rows for a shard of {sh.count}")
    return global_sse(local, sh, n_total, group)


class SseExchange:
    """Global SSE vector in torch symmetric memory, filled by the fused
    retain kernel's epilogue on every rank (adct_compress_retain_exchange).

        ex = SseExchange(n_total, device)
        rec, local = ex.compress_retain(images_of_this_rank, r, shard.start)
        ex.sse  # int64 [n_total], identical on every rank after the call

    Each call is bracketed by two stream-ordered symmetric-memory barriers:
    the one before the pushes keeps a rank from overwriting a peer's vector
    while the peer's reads of the previous call (enqueued before its own
    call) are pending; the one after makes every rank's pushes visible.
    """

    def __init__(self, n_total: int, device, group=None):
        import torch.distributed._symmetric_memory as symm_mem

        if not dist.is_initialized():
            raise RuntimeError("SseExchange needs an initialised process group (NCCL)")
        group = group or dist.group.WORLD
        self.n_total = int(n_total)
        self.sse = symm_mem.empty(self.n_total, dtype=torch.int64, device=device)
        self.sse.zero_()
        torch.cuda.synchronize(device)  # zeroed before any peer can store into it
        self._hdl = symm_mem.rendezvous(self.sse, group.group_name)
        self.n_peers = int(self._hdl.world_size)
        self._arrivals: torch.Tensor | None = None

    def compress_retain(self, images: torch.Tensor, r: int, offset: int, *, out=None, sse_out=None):
        from . import batch

        n = images.shape[0] if images.dim() == 3 else 1
        if offset < 0 or offset + n > self.n_total:
            raise ValueError(f"images [{offset}, {offset + n}) outside the exchange vector of {self.n_total}")
        if self._arrivals is None or self._arrivals.numel() < n:
            self._arrivals = torch.zeros(max(n, 1), dtype=torch.int32, device=images.device)
        # stream-ordered barrier BEFORE the pushes: no rank stores into a peer's
        # vector while that peer may still read the previous call's values
        # (its reads were enqueued before its own barrier)
        self._hdl.barrier(channel=1)
        rec, local = batch.compress_retain_exchange(
            images, r, self._hdl.buffer_ptrs_dev, self.n_peers, offset, self._arrivals, out=out, sse_out=sse_out
        )
        self._hdl.barrier(channel=0)  # stream-ordered: every rank's pushes are visible after this
        return rec, local

    def compress_quant_planes(self, planes, qtab, frame_offset: int, *, out=None):
        """Frames [frame_offset, frame_offset + N) of n_planes planes; the
        vector holds entry frame * n_planes + plane (n_total = frames * planes)."""
        from . import batch

        n, k = planes[0].shape[0], len(planes)
        off = int(frame_offset) * k
        if frame_offset < 0 or off + n * k > self.n_total:
            raise ValueError(f"frames [{frame_offset}, {frame_offset + n}) x {k} planes outside the exchange vector")
        if self._arrivals is None or self._arrivals.numel() < n * k:
            self._arrivals = torch.zeros(max(n * k, 1), dtype=torch.int32, device=planes[0].device)
        self._hdl.barrier(channel=1)  # see compress_retain: no store while a peer may still read
        recs, local = batch.compress_quant_planes_exchange(
            planes, qtab, self._hdl.buffer_ptrs_dev, self.n_peers, off, self._arrivals, out=out
        )
        self._hdl.barrier(channel=0)
        return recs, local

