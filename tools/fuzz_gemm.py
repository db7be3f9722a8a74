"""Randomised gemm_lowbit shapes (every mode, AUTO and each kernel, reference / nibble layouts, gemm_i8) against the oracle.
SECONDS of fuzzing, seeded; prints the failing case if any."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2205_09120_b200 as lb
from oracle.oracle import Port, BNN, TNN, TBN
from tests.golden.make_golden import mode_dists

port = Port()
rng = np.random.default_rng(int(os.environ.get("SEED", "1")))
t_end = time.time() + float(os.environ.get("SECONDS", "180"))
n = 0
while time.time() < t_end:
    mode = int(rng.choice([BNN, TNN, TBN]))
    m = int(rng.choice([rng.integers(1, 200), rng.integers(1, 1500), rng.integers(1, 6000)]))
    nn = int(rng.choice([rng.integers(1, 64), rng.integers(1, 300), rng.integers(1, 1100)]))
    k = int(rng.choice([rng.integers(1, 300), rng.integers(1, 2500), rng.integers(1, 9000)]))
    if 2.0 * m * nn * k > 6e9:
        continue
    da, db = mode_dists(mode)
    a = port.generate(da, 2000 + n, 0, m, k)
    b = port.generate(db, 2000 + n, 1, k, nn)
    want = port.gemm(mode, a, b)
    at, bt = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    bp = lb.encode_ternary(bt) if mode == TNN else lb.encode_binary(bt)
    w = lb.prepare_weights(lb.pack_b(bp))
    case = dict(mode=mode, m=m, n=nn, k=k, seed=2000 + n)
    try:
        ap = lb.encode_binary(at) if mode == BNN else lb.encode_ternary(at)
        for kern in (lb.KERNEL_AUTO, lb.KERNEL_TENSOR, lb.KERNEL_TENSOR_I8, lb.KERNEL_TENSOR_1CTA, lb.KERNEL_BITSERIAL):
            got = lb.gemm_lowbit(mode, ap, w, (m, nn, k), kernel=kern).cpu().numpy()
            if not np.array_equal(got, want):
                print("MISMATCH", case, "kernel", kern, int((got != want).sum()))
                sys.exit(1)
        ap4 = lb.encode_binary(at, layout=2) if mode == BNN else lb.encode_ternary(at, layout=2)
        got = lb.gemm_lowbit(mode, ap4, w, (m, nn, k), kernel=lb.KERNEL_TENSOR).cpu().numpy()
        if not np.array_equal(got, want):
            print("MISMATCH", case, "nibbles")
            sys.exit(1)
        a16 = torch.zeros((m, (k + 15) // 16 * 16), dtype=torch.int8, device="cuda")
        a16[:, :k] = at
        got = lb.gemm_lowbit_i8(mode, a16[:, :k], w, (m, nn, k)).cpu().numpy()
        if not np.array_equal(got, want):
            print("MISMATCH", case, "gemm_i8")
            sys.exit(1)
    except Exception as ex:
        print("ERROR", case, repr(ex))
        sys.exit(1)
    n += 1
print(f"fuzz OK: {n} GeMM shapes x 7 paths")
