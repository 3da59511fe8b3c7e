"""Multi-process host logic of the batch driver on CPU (gloo, world_size 2): sharding
covers every mesh exactly once, the stats all_gather reassembles rows in mesh order,
and the time reduction is a MAX over ranks."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2403_14723_b200 import batch


def test_shard_covers_all():
    for world in (1, 2, 3, 4, 8):
        got = sorted(i for r in range(world) for i in batch.shard(64, r, world))
        assert got == list(range(64))
    assert batch.shard(5, 1, 2) == [1, 3]
    with pytest.raises(ValueError):
        batch.shard(4, 2, 2)


def test_config5_interleaves_kinds():
    m = batch.config5_meshes()
    assert len(m) == 64
    for world in (1, 2, 4, 8):
        for r in range(world):
            kinds = {m[i]["kind"] for i in batch.shard(64, r, world)}
            assert kinds == {"jittered", "regular"}


def test_checksum_order_sensitive():
    off = torch.tensor([0, 3, 7], dtype=torch.int32)
    a = torch.tensor([0, 1, 2, 2, 3, 4, 5], dtype=torch.int32)
    b = torch.tensor([1, 0, 2, 2, 3, 4, 5], dtype=torch.int32)
    assert batch.loop_checksum(off, a) != batch.loop_checksum(off, b)
    assert batch.loop_checksum(off, a) == batch.loop_checksum(off, a.clone())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 7
        mine = batch.shard(n, rank, world)
        rows = torch.tensor([[i, 100 + i, 10 * i, 0, 0, 0, i * i] for i in mine], dtype=torch.int64).reshape(-1, 7)
        full = batch.gather_stats(rows, n, world)
        t = batch.max_time(1.5 + rank, torch.device("cpu"), world)
        q.put((rank, full.tolist(), t))
    finally:
        dist.destroy_process_group()


def test_gather_and_max_over_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, full, t in res:
        assert [row[0] for row in full] == list(range(7))
        assert all(row[1] == 100 + row[0] and row[6] == row[0] ** 2 for row in full)
        assert t == 2.5
