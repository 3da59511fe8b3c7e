"""Batch driver: independent triangulations sharded over ranks (BASELINE config 5).

A single mesh is not split across GPUs (its twin gathers are random).
Independent meshes are: mesh i goes to rank i mod world, each rank converts its meshes
through the C ABI with no data movement between GPUs, and the only collectives are a
few KB after the compute: an all_gather of per-mesh counts (NCCL on GPUs, gloo in the
CPU tests) and an all_reduce(MAX) of the device time.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

STAT_FIELDS = ("mesh", "n_triangles", "n_polygons", "n_loop_entries", "n_tips", "n_border", "checksum")


def shard(n_items: int, rank: int, world: int) -> list[int]:
    """Round-robin assignment: item i -> rank i mod world (interleaves mesh kinds)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return list(range(rank, n_items, world))


def loop_checksum(offsets: torch.Tensor, loops: torch.Tensor) -> int:
    """Order-sensitive 61-bit checksum of a CSR polygon list (harness-side consistency
    check across ranks / runs; not part of the conversion)."""
    x = loops.to(torch.int64) + 1
    w = (torch.arange(x.numel(), dtype=torch.int64, device=x.device) * 2654435761) & 0x7FFFFFFF
    s = int((x * (w + 1)).sum().item())  # wraps mod 2^64: deterministic, order-sensitive
    o = offsets.to(torch.int64)
    wo = (torch.arange(o.numel(), dtype=torch.int64, device=o.device) * 40503) & 0xFFFFF
    return (s ^ int((o * (wo + 1)).sum().item())) & ((1 << 63) - 1)


def gather_stats(local: torch.Tensor, n_total: int, world: int) -> torch.Tensor:
    """all_gather of per-mesh stat rows [k_local, F] (k varies by rank) -> [n_total, F]
    ordered by mesh index (column 0)."""
    F = local.shape[1]
    kmax = (n_total + world - 1) // world
    pad = torch.full((kmax, F), -1, dtype=torch.int64, device=local.device)
    pad[: local.shape[0]] = local
    if world == 1:
        rows = pad
    else:
        bufs = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(bufs, pad)
        rows = torch.cat(bufs, 0)
    rows = rows[rows[:, 0] >= 0]
    order = torch.argsort(rows[:, 0])
    return rows[order]


def max_time(t_ms: float, device, world: int) -> float:
    t = torch.tensor([t_ms], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def config5_meshes(count: int = 64, s: int = 2000):
    """BASELINE config 5: `count` grids of s x s vertices, jittered (a = 0.2, seeds
    1000..) and regular (Alg. 13) in alternating blocks of 8, so that under the
    round-robin shard every rank of a 1/2/4/8-GPU run gets both kinds."""
    out = []
    nj = 0
    for i in range(count):
        if (i // 8) % 2 == 0:
            out.append(dict(index=i, s=s, a=0.2, seed=1000 + nj, kind="jittered"))
            nj += 1
        else:
            out.append(dict(index=i, s=s, a=0.0, seed=0, kind="regular"))
    return out
