"""Row sharding of a low-bit GeMM over ranks.

C[i, :] depends only on A[i, :] and B (gemm.cpp:35-51), so the M rows of A
partition across ranks with no reduction: rank r owns a contiguous block of
rows and regenerates / receives only those, B is replicated (weights,
prepared once), and no collective touches the data path.  `gather_rows`
assembles C on rank 0 where a test needs the whole matrix (int16 has no NCCL
type: the shard travels as bytes).

Process model: one process per GPU, launched by torchrun; torch.distributed
(nccl on GPUs, gloo for the CPU tests) is plumbing only.
"""
from __future__ import annotations

from typing import Optional, Tuple

import torch
import torch.distributed as dist


def row_range(m: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous, balanced row block [r0, r1) of rank `rank` out of `world`."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    return m * rank // world, m * (rank + 1) // world


def max_shard_rows(m: int, world: int) -> int:
    return max(row_range(m, r, world)[1] - row_range(m, r, world)[0] for r in range(world))


def gather_rows(c_shard: torch.Tensor, m: int, group=None, dst: int = 0) -> Optional[torch.Tensor]:
    """Gather each rank's int16 [rows_r, n] shard of C into the full [m, n] C
    on rank `dst` (None elsewhere).  Shards are padded to the largest shard
    and sent as raw bytes."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = c_shard.shape[1]
    rows_max = max_shard_rows(m, world)
    send = torch.zeros((rows_max, n), dtype=c_shard.dtype, device=c_shard.device)
    send[: c_shard.shape[0]] = c_shard
    send_b = send.view(torch.uint8).reshape(-1)
    if rank == dst:
        bufs = [torch.empty_like(send_b) for _ in range(world)]
        dist.gather(send_b, gather_list=bufs, dst=dst, group=group)
        parts = []
        for r in range(world):
            r0, r1 = row_range(m, r, world)
            parts.append(bufs[r].view(c_shard.dtype).reshape(rows_max, n)[: r1 - r0])
        return torch.cat(parts, dim=0)
    dist.gather(send_b, dst=dst, group=group)
    return None
