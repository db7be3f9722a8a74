"""CPU, world_size 2 over gloo: the multi-GPU row-sharding logic (§8e).

Each rank regenerates only its A rows from the counter-based generator,
computes its C shard (here with the oracle, standing in for the GPU kernel,
which the 1-GPU tests cover), and rank 0 gathers the int16 shards as bytes and
compares with the single-process result.  Uneven shards are included."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2205_09120_b200.shard import gather_rows, row_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cases, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Port
    port_lib = Port()
    try:
        for ci, (mode, m, n, k, da, db, seed) in enumerate(cases):
            r0, r1 = row_range(m, rank, world)
            a = port_lib.generate(da, seed, 0, r1 - r0, k, row0=r0)  # only this rank's rows
            b = port_lib.generate(db, seed, 1, k, n)                 # B replicated
            c = torch.from_numpy(port_lib.gemm(mode, a, b)) if r1 > r0 else torch.zeros((0, n), dtype=torch.int16)
            full = gather_rows(c, m)
            if rank == 0:
                want = port_lib.gemm(mode, port_lib.generate(da, seed, 0, m, k), b)
                results[ci] = bool(np.array_equal(full.numpy(), want))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_row_sharded_gemm_gathers_to_rank0(world):
    cases = [(1, 301, 40, 200, 0, 0, 47), (0, 64, 33, 129, 1, 1, 45), (2, 5, 17, 77, 2, 1, 44), (1, 2, 8, 16, 0, 0, 1)]
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), cases, results), nprocs=world, join=True)
    assert len(results) == len(cases) and all(results.values()), dict(results)


def test_row_range_partition():
    for m in (1, 7, 1048576, 1000003):
        for world in (1, 2, 4, 8):
            spans = [row_range(m, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
