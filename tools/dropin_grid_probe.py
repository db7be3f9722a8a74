"""The reference's non-aligned gemm grid (test_gemm.cpp:50-61) through the
host-buffer entry (pageable numpy memory, what the C++ drop-in passes) and
through the device entry with every kernel; prints each mismatching case."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2205_09120_b200 as lb
from oracle.oracle import Port, a_mode_ternary, b_mode_ternary
from tests.golden.make_golden import mode_dists
port = Port()
bad = 0
i = 0
for mode in (lb.BNN, lb.TNN, lb.TBN):
    da, db = mode_dists(mode)
    for m in (1, 15, 17, 70):
        for n in (1, 7, 9, 25):
            for k in (1, 7, 9, 500):
                i += 1
                a = port.generate(da, 31, 2 * i, m, k)
                b = port.generate(db, 31, 2 * i + 1, k, n)
                want = port.gemm(mode, a, b)
                at, bt = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
                ap = lb.encode_ternary(at) if a_mode_ternary(mode) else lb.encode_binary(at)
                bp = lb.encode_ternary(bt) if b_mode_ternary(mode) else lb.encode_binary(bt)
                pb = lb.pack_b(bp)
                sb = (k + 7) // 8
                a0 = ap.plane0.cpu().numpy()[:, :sb].copy()
                a1 = ap.plane1.cpu().numpy()[:, :sb].copy() if ap.plane1 is not None else None
                panels = pb.panels.cpu().numpy().copy()
                for kern in (lb.KERNEL_AUTO, lb.KERNEL_TENSOR, lb.KERNEL_TENSOR_I8, lb.KERNEL_BITSERIAL):
                    got = lb.gemm_lowbit_host(mode, a0, a1, m, k, panels, b_mode_ternary(mode), n, k, (m, n, k),
                                              kernel=kern)
                    if not np.array_equal(got, want):
                        bad += 1
                        d = np.argwhere(got != want)
                        print("HOST", mode, (m, n, k), "kernel", kern, "ndiff", len(d), d[:4].tolist(),
                              got[tuple(d[0])], want[tuple(d[0])])
                    got = lb.gemm_lowbit(mode, ap, lb.prepare_weights(pb), (m, n, k), kernel=kern).cpu().numpy()
                    if not np.array_equal(got, want):
                        bad += 1
                        d = np.argwhere(got != want)
                        print("DEV", mode, (m, n, k), "kernel", kern, "ndiff", len(d), d[:4].tolist())
print("bad", bad)
