"""The row-sharded multi-GPU path through the CUDA kernels.

World 2 and 3, all ranks on cuda:0 (gpurun and the round-end tiers give one
GPU; NCCL refuses two ranks on one device, so the ranks talk over gloo with
the shards staged through host memory — the data path is identical to the
NCCL run's: no collective until the output gather).  Each rank regenerates
ONLY its rows of config 5's A from the counter-based generator (row0 = its
first row), encodes them, runs AUTO (the fp4 kernel K5 on reference planes)
and K5 on NIBBLES planes, and rank 0 gathers C with shard.gather_rows and
compares the whole 2 GiB result with the sha256 of the reference library's
own output (tests/golden/golden_configs.json).  Rows are independent
(/root/reference/proj/src/gemm.cpp:32-53), so the gathered C must be
bit-identical to the single-GPU one.
"""
import hashlib
import json
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, want, results):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2205_09120_b200 as lb
        from paper_2205_09120_b200.shard import gather_rows, row_range
        m, n, k = 1048576, 1024, 2048
        r0, r1 = row_range(m, rank, world)
        a = lb.generate(0, 47, 0, r1 - r0, k, row0=r0)  # only this rank's rows
        w = lb.prepare_weights(lb.pack_b(lb.encode_ternary(lb.generate(0, 47, 1, k, n))))  # B replicated
        ok = True
        for layout in (0, 2):
            ap = lb.encode_ternary(a, layout=layout)
            c = lb.gemm_lowbit(lb.TNN, ap, w, (r1 - r0, n, k))
            del ap
            full = gather_rows(c.cpu(), m)
            del c
            if rank == 0:
                h = hashlib.sha256(np.ascontiguousarray(full.numpy(), "<i2").tobytes()).hexdigest()
                ok = ok and h == want
            del full
        if rank == 0:
            results["ok"] = ok
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_row_sharded_config5_through_kernels(world):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    with open(os.path.join(ROOT, "tests", "golden", "golden_configs.json")) as f:
        want = json.load(f)["c5"]["sha256"]
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), want, results), nprocs=world, join=True)
    assert results.get("ok") is True


def test_bench_under_torchrun():
    # the launcher path the driver uses for N GPUs, at N = 1: torchrun -> NCCL process group ->
    # the timed loop with barriers and the max-over-ranks reduction -> the output gather
    import subprocess
    import sys
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--gpus", "1", "--steps", "3",
           "--warmup", "3", "--no-extra", "--no-cpu-baseline", "--no-e2e"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 1 and line["value"] > 1000 and line["gather"] is not None
