"""Quick standalone GPU check (one kernel at a time, for bring-up under a timeout)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2205_09120_b200 as lb
from oracle.oracle import Port
port = Port()
kernel = int(sys.argv[1]) if len(sys.argv) > 1 else 1
for mode, (m, n, k), (da, db) in [(lb.TNN, (360, 96, 256), (0, 0)), (lb.BNN, (200, 130, 300), (1, 1)),
                                  (lb.TBN, (129, 64, 512), (2, 1)), (lb.TNN, (1000, 600, 2048), (0, 0))]:
    a = port.generate(da, 43, 0, m, k); b = port.generate(db, 43, 1, k, n)
    want = port.gemm(mode, a, b)
    at, bt = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    ap = lb.encode_binary(at) if mode == lb.BNN else lb.encode_ternary(at)
    bp = lb.encode_ternary(bt) if mode == lb.TNN else lb.encode_binary(bt)
    w = lb.prepare_weights(lb.pack_b(bp))
    got = lb.gemm_lowbit(mode, ap, w, (m, n, k), kernel=kernel).cpu().numpy()
    bad = np.argwhere(got != want)
    print(mode, (m, n, k), "kernel", kernel, "mismatches", len(bad), bad[:5].tolist(),
          [ (int(got[tuple(x)]), int(want[tuple(x)])) for x in bad[:5]], flush=True)
