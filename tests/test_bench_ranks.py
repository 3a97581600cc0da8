"""bench.py's multi-rank logic at world size 2 on CPU with gloo (-m "not gpu"):
distinct seeded slices per rank, barrier-bracketed timing of exactly K steps, the
max over ranks, the whole-job aggregate and the separately timed gather to rank 0.
The per-step compute is a stand-in (a rank-dependent sleep); the kernels are
covered by the -m gpu tests."""
import os
import socket
import time

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
from paper_2007_06289_b200.dist import gather_volume


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def cpu_timer():
    t = {}

    def start():
        t["0"] = time.perf_counter()

    def stop():
        return 1e3 * (time.perf_counter() - t["0"])
    return start, stop


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world),
                      RANK=str(rank), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w, r, lr = bench.rank_env()
    B, K, N = 3, 4, 8
    ids = bench.slice_ids(r, B)
    calls = []

    def step():
        calls.append(1)
        time.sleep(0.01 * (r + 1))          # rank 1 is the slow one

    ms = bench.time_steps(step, K, dist.barrier, lambda: None, cpu_timer)
    mx = bench.max_over_ranks([ms, float(r)], w)
    value = bench.aggregate(w, B, K, mx[0])
    # images of this rank's slices: value = slice id, gathered to rank 0 in slice order
    img = torch.tensor(ids, dtype=torch.float32).view(B, 1, 1) + torch.zeros((B, N, N))
    vol = gather_volume(img, w * B, N, w, r, "cpu")
    q.put(dict(rank=r, world=w, local=lr, ids=ids, ms=ms, max=mx, value=value, calls=len(calls),
               vol=None if vol is None else vol[:, 0, 0].tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_bench_rank_logic_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(2)], key=lambda d: d["rank"])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    r0, r1 = res
    assert r0["world"] == r1["world"] == 2 and (r0["local"], r1["local"]) == (0, 1)
    # disjoint, seeded slice ranges
    assert r0["ids"] == [0, 1, 2] and r1["ids"] == [3, 4, 5]
    # exactly K steps each
    assert r0["calls"] == r1["calls"] == 4
    # max over ranks: both ranks agree, and it is the slow rank's time
    assert r0["max"] == r1["max"]
    assert r0["max"][0] == pytest.approx(max(r0["ms"], r1["ms"]))
    assert r0["max"][1] == 1.0
    assert r1["ms"] >= 4 * 20.0 * 0.9
    # whole-job aggregate: all ranks' slices over the slowest rank's time
    assert r0["value"] == pytest.approx(2 * 3 * 4 / (r0["max"][0] / 1e3))
    # gather to rank 0 only, in global slice order
    assert r0["vol"] == [0.0, 1.0, 2.0, 3.0, 4.0, 5.0] and r1["vol"] is None


@pytest.mark.parametrize("per_worker_gb", [1.6, 1e6])
def test_pool_workers_bounded(per_worker_gb):
    usable, total, model = bench.host_cores()
    w = bench.pool_workers(per_worker_gb)
    assert 1 <= w <= usable <= (total or usable)
    if per_worker_gb > 1e5:
        assert w == 1


def test_alg_and_design_bytes():
    """36 N^2 B per slice; the design bytes of the two FHT passes exceed it
    (the intermediate R round trip)."""
    N = 2048
    assert bench.alg_bytes_per_slice(N) == 36 * N * N
    path = {"fast": True, "tile_width": 64, "lookahead_tiles": 3}
    a = bench.kernel_design_bytes("fht_pass_a", N, 32, 64, path)
    b = bench.kernel_design_bytes("fht_pass_b", N, 32, 64, path)
    assert a + b > bench.alg_bytes_per_slice(N)
