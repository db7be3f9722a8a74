"""Per-CTA entry / work start / work end of K7T on c4 (TUNING build, LOWBIT_HALO_DEBUG=32)."""
import ctypes as C
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_09120_b200 as lb
fm = lb.generate(0, 46, 0, 64 * 56 * 56, 128).view(64, 56, 56, 128)
w = lb.prepare_weights(lb.pack_b(lb.encode_ternary(lb.generate(0, 46, 1, 9 * 128, 128))))
o = torch.empty((64, 56, 56, 128), dtype=torch.int16, device="cuda")
for _ in range(5):
    lb.conv2d_lowbit(1, fm, False, w, 3, 3, 1, 1, kernel=2, out=o)
torch.cuda.synchronize()
buf = (C.c_ulonglong * 640)()
assert lb._lib.lib.lowbit_debug_ts_ctas(buf) == 0
rows = [(buf[4 * i], buf[4 * i + 1], buf[4 * i + 2], buf[4 * i + 3]) for i in range(148)]
t0 = min(r[0] for r in rows)
ent = sorted(r[0] - t0 for r in rows); ws = sorted(r[1] - t0 for r in rows); we = sorted(r[2] - t0 for r in rows)
dur = sorted(r[2] - r[1] for r in rows)
q = lambda xs, p: xs[int(p * (len(xs) - 1))]
for name, xs in (("entry", ent), ("work start", ws), ("work end", we), ("work duration", dur)):
    print(f"{name:14s} ns: min {xs[0]} p25 {q(xs, .25)} median {q(xs, .5)} p75 {q(xs, .75)} max {xs[-1]}")
d13 = sorted(r[2] - r[1] for i, r in enumerate(rows) if i < 1792 - 12 * 148)
d12 = sorted(r[2] - r[1] for i, r in enumerate(rows) if i >= 1792 - 12 * 148)
print("13-tile CTAs work duration ns:", d13[0], q(d13, .5), d13[-1], "| 12-tile CTAs:", d12[0], q(d12, .5), d12[-1])
late = sorted(rows, key=lambda r: -r[2])[:8]
print("latest CTAs (block, sm, entry, end):", [(rows.index(r), r[3], r[0] - t0, r[2] - t0) for r in late])
sb = (C.c_ulonglong * 640)()
if hasattr(lb._lib.lib, "lowbit_debug_ts_setup") and lb._lib.lib.lowbit_debug_ts_setup(sb) == 0:
    a = sorted(sb[4 * i] - rows[i][0] for i in range(148)); b = sorted(sb[4 * i + 1] - rows[i][0] for i in range(148))
    c = sorted(sb[4 * i + 2] - rows[i][0] for i in range(148))
    print("setup, ns after the CTA's entry (median / max): barriers initialised %d / %d, TMEM allocated %d / %d, CTA barrier passed %d / %d"
          % (q(a, .5), a[-1], q(b, .5), b[-1], q(c, .5), c[-1]))
