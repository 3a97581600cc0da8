"""Multi-GPU volume reconstruction: one process per GPU, slices sharded, no
collective on the data path; NCCL only to gather results.

Slices of a volume are independent (each is its own linogram -> image), so rank r
of G owns the contiguous slice range ``shard(n_slices, G, r)`` and runs its own
``Plan`` on its own GPU.  ``gather_volume`` collects the per-rank images on rank 0 only
(``torch.distributed.gather``: NCCL over NVLink on GPUs, gloo on CPU tensors).
"""
from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist


def shard(n_slices: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced range (start, count) of slices owned by `rank`."""
    if world < 1 or not (0 <= rank < world) or n_slices < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(n_slices, world)
    start = rank * base + min(rank, extra)
    count = base + (1 if rank < extra else 0)
    return start, count


def reconstruct_shard(reconstruct: Callable[[torch.Tensor], torch.Tensor],
                      make_slices: Callable[[int, int], torch.Tensor],
                      n_slices: int, world: int, rank: int, chunk: int) -> torch.Tensor:
    """Reconstruct this rank's slices in chunks of `chunk` (plan max_batch).

    make_slices(start, count) -> [count, 4, N, 2N] linograms on this rank's device;
    reconstruct(lin) -> [count, N, N].  Returns [count_local, N, N].
    """
    start, count = shard(n_slices, world, rank)
    outs = []
    for s0 in range(start, start + count, chunk):
        k = min(chunk, start + count - s0)
        outs.append(reconstruct(make_slices(s0, k)))
    if not outs:
        return None
    return torch.cat(outs, dim=0)


def gather_volume(local: torch.Tensor | None, n_slices: int, N: int, world: int, rank: int,
                  device) -> torch.Tensor | None:
    """Gather every rank's [count_r, N, N] block to rank 0 as [n_slices, N, N].

    Blocks are padded to the largest shard so one fixed-size gather suffices.
    Returns the volume on rank 0, None elsewhere.
    """
    cmax = shard(n_slices, world, 0)[1]
    buf = torch.zeros((cmax, N, N), dtype=torch.float32, device=device)
    if local is not None and local.shape[0] > 0:
        buf[: local.shape[0]].copy_(local)
    if world == 1:
        return buf[:n_slices].clone()
    # gather to rank 0 only (NCCL: grouped point-to-point sends into rank 0 over
    # NVLink; gloo on CPU tensors); the other ranks receive nothing
    parts = [torch.empty_like(buf) for _ in range(world)] if rank == 0 else None
    dist.gather(buf, gather_list=parts, dst=0)
    if rank != 0:
        return None
    vol = torch.empty((n_slices, N, N), dtype=torch.float32, device=device)
    for r in range(world):
        s, c = shard(n_slices, world, r)
        if c:
            vol[s: s + c].copy_(parts[r][:c])
    return vol
