"""Multi-process host logic of the slice-sharded volume path, world_size 2 on CPU
with gloo (-m "not gpu").  The per-slice compute is replaced by a deterministic
stand-in: this tests sharding, chunking and the gather, not the kernels."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2007_06289_b200.dist import gather_volume, reconstruct_shard, shard


def test_shard_partitions_exactly():
    for n in (0, 1, 7, 64, 256):
        for w in (1, 2, 3, 4, 8):
            seen = []
            for r in range(w):
                s, c = shard(n, w, r)
                seen.extend(range(s, s + c))
            assert seen == list(range(n)), (n, w)
            counts = [shard(n, w, r)[1] for r in range(w)]
            assert max(counts) - min(counts) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def fake_slices(start, count, N=8):
    # slice i is filled with values derived from i: order mistakes are visible
    base = torch.arange(start, start + count, dtype=torch.float32).view(-1, 1, 1, 1)
    return base + torch.zeros((count, 4, N, 2 * N))


def fake_reconstruct(lin):
    return lin[:, 0, :, : lin.shape[2]] * 2.0 + 1.0


def _worker(rank, world, port, n_slices, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    N = 8
    local = reconstruct_shard(fake_reconstruct, lambda s, c: fake_slices(s, c, N), n_slices,
                              world, rank, chunk=3)
    vol = gather_volume(local, n_slices, N, world, rank, "cpu")
    if rank == 0:
        q.put(vol.clone())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_slices", [5, 8])
def test_gather_volume_gloo_world2(n_slices):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_slices, q)) for r in range(2)]
    for p in procs:
        p.start()
    vol = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref = fake_reconstruct(fake_slices(0, n_slices))
    assert torch.equal(vol, ref)
