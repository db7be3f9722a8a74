"""Debug helper: one fp4 GeMM case vs the oracle, with mismatch geometry."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2205_09120_b200 as lb
from oracle.oracle import Port
from tests.golden.make_golden import mode_dists
port = Port()
def run(mode, m, n, k, seed=300):
    da, db = mode_dists(mode)
    a = port.generate(da, seed + k, 0, m, k); b = port.generate(db, seed + k, 1, k, n)
    at = torch.from_numpy(a).cuda(); bt = torch.from_numpy(b).cuda()
    ap = lb.encode_binary(at, layout=2) if mode == 0 else lb.encode_ternary(at, layout=2)
    bp = lb.encode_ternary(bt) if mode == 1 else lb.encode_binary(bt)
    got = lb.gemm_lowbit(mode, ap, lb.prepare_weights(lb.pack_b(bp)), (m, n, k), kernel=2).cpu().numpy()
    want = port.gemm(mode, a, b)
    bad = np.argwhere(got != want)
    print(f"mode={mode} m={m} n={n} k={k}: {len(bad)} bad of {m*n}", end="")
    if len(bad):
        rows = np.unique(bad[:, 0]); cols = np.unique(bad[:, 1])
        print(f"; rows {rows[:8]}..{rows[-3:]} ({len(rows)}), cols {cols[:8]}..{cols[-3:]} ({len(cols)}), "
              f"diff sample {(got - want)[bad[0][0], bad[0][1]]}")
    else:
        print()
for args in [(1, 19000, 300, 2300), (2, 19000, 300, 2300), (1, 19000, 300, 2048), (1, 19000, 300, 2304),
             (1, 19000, 208, 2300), (1, 4000, 300, 2300), (1, 19000, 300, 4096)]:
    run(*args)
