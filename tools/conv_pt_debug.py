"""Small K6 tap-pair debug case: c = 128, 3x3, stride 1, pad 1; prints where
outputs differ from the oracle."""
import sys

import numpy as np
import torch

import paper_2205_09120_b200 as lb
from oracle.oracle import Port

p = Port()
b, h, w, c, cout = int(sys.argv[1]) if len(sys.argv) > 1 else 2, 6, 7, 128, 8
fm = p.generate(0, 5, 0, b * h * w, c).reshape(b, h, w, c)
wt = p.generate(0, 5, 1, 9 * c, cout)
bp = lb.encode_ternary(torch.from_numpy(wt).cuda())
wts = lb.prepare_weights(lb.pack_b(bp))
got = lb.conv2d_lowbit(1, torch.from_numpy(fm).cuda(), False, wts, 3, 3, 1, 1, kernel=2).cpu().numpy()
for img in range(b):
    want = p.direct_conv(fm[img], False, wt, 3, 3, 1, 1)
    bad = np.argwhere(got[img].astype(np.int32) != want)
    print("img", img, "bad", len(bad), "of", want.size)
    for y, x, o in bad[:12]:
        print(" ", y, x, o, "got", got[img, y, x, o], "want", want[y, x, o])
# which single-tap error explains the difference: tap (ky,kx) read at pixel offset dx
# instead of 0 (dx = None: tap missing)
want = p.direct_conv(fm[0], False, wt, 3, 3, 1, 1)
diff = got[0].astype(np.int32) - want
fpad = np.zeros((h + 2, w + 8, c), np.int32)
fpad[1:h + 1, 4:w + 4] = fm[0]


def cont(ky, kx, dx):
    sl = slice((ky * 3 + kx) * c, (ky * 3 + kx + 1) * c)
    out = np.zeros_like(want)
    for y in range(h):
        for x in range(w):
            out[y, x] = fpad[y + ky, x + kx + 3 + dx] @ wt[sl].astype(np.int32)
    return out


terms = {}
for ky in range(3):
    for kx in range(3):
        base = cont(ky, kx, 0)
        terms[(ky, kx, None)] = -base
        for dx in (-2, -1, 1, 2):
            terms[(ky, kx, dx)] = cont(ky, kx, dx) - base
print("diff nonzero", np.count_nonzero(diff))
for key, t in terms.items():
    if np.array_equal(diff, t):
        print("diff == single", key)
# per-row-of-filter: does the error come from group g0 or g1 of each ky?
for ky in range(3):
    for grp in ((0,), (1, 2)):
        s_ = sum(terms[(ky, kx, None)] for kx in grp)
        r = diff - s_
        print("ky", ky, "taps", grp, "missing -> residual nonzero", np.count_nonzero(r))
