"""K7T bring-up: one small TNN conv through the halo path against the C oracle, with the
mismatch pattern (which output channels / positions differ)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2205_09120_b200 as lb
from oracle.oracle import Port
port = Port()
for (b, h, w, c, cout) in [(1, 4, 6, 128, 128), (2, 9, 9, 128, 64), (1, 12, 56, 128, 128), (2, 20, 30, 128, 40)]:
    fm = port.generate(0, 7, 0, b * h * w, c).reshape(b, h, w, c)
    wt = port.generate(0, 7, 1, 9 * c, cout)
    wc = lb.prepare_weights(lb.pack_b(lb.encode_ternary(torch.from_numpy(wt).cuda())))
    got = lb.conv2d_lowbit(lb.TNN, torch.from_numpy(fm).cuda(), False, wc, 3, 3, 1, 1).cpu().numpy().astype(np.int32)
    want = np.stack([port.conv2d_lowbit(lb.TNN, fm[i], False, wt, False, 3, 3, 1, 1) for i in range(b)])
    bad = got != want
    print((b, h, w, c, cout), "mismatches", int(bad.sum()), "of", bad.size)
    if bad.any():
        idx = np.argwhere(bad)
        print(" channels with errors:", sorted(set(idx[:, 3].tolist()))[:40])
        print(" (y,x) with errors:", sorted(set(map(tuple, idx[:, 1:3].tolist())))[:20])
        i = tuple(idx[0]); print(" first", i, "got", got[i], "want", want[i])
        # is got a permutation of want within each position?
        y, x = idx[0][1], idx[0][2]
        g, wv = got[0, y, x], want[0, y, x]
        print(" got[0,y,x][:16]", g[:16].tolist()); print(" want[0,y,x][:16]", wv[:16].tolist())
        # search for each got value's location in want (same image)
        for ch in range(4):
            loc = np.argwhere(want[0] == g[ch])[:3]
            print("  got ch", ch, "value", g[ch], "appears in want at", loc.tolist())
