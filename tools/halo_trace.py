"""Per-tile event timeline of K7's first leader CTA on c4 (LOWBIT_HALO_DEBUG must include 32).
Columns are clock64 cycles relative to the first producer event."""
import ctypes as C
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_09120_b200 as lb
fm = lb.generate(0, 46, 0, 64 * 56 * 56, 128).view(64, 56, 56, 128)
w = lb.prepare_weights(lb.pack_b(lb.encode_ternary(lb.generate(0, 46, 1, 9 * 128, 128))))
o = torch.empty((64, 56, 56, 128), dtype=torch.int16, device="cuda")
for _ in range(3):
    lb.conv2d_lowbit(1, fm, False, w, 3, 3, 1, 1, kernel=2, out=o)
torch.cuda.synchronize()
ph = (C.c_ulonglong * 4)()
lb._lib.lib.lowbit_debug_halo_phases(ph, 1)
lb.conv2d_lowbit(1, fm, False, w, 3, 3, 1, 1, kernel=2, out=o)
torch.cuda.synchronize()
assert lb._lib.lib.lowbit_debug_halo_phases(ph, 0) == 0
print("phases (us): first entry -> last setup end %.2f, -> last work end %.2f, -> last exit %.2f (total %.2f)" % (
    (ph[1] - ph[0]) / 1e3, (ph[2] - ph[1]) / 1e3, (ph[3] - ph[2]) / 1e3, (ph[3] - ph[0]) / 1e3))
buf = (C.c_ulonglong * 1024)()
assert lb._lib.lib.lowbit_debug_halo_trace(buf) == 0
ev = [[buf[e * 64 + i] for i in range(64)] for e in range(16)]
t0 = min(x for x in ev[0] if x)
names = ["prod:issue", "cv:raw_full", "cv:a_empty", "cv:done", "mma:acc", "mma:a_full", "mma:issued",
         "epi:full", "epi:tmem_ld", "epi:done"]
print("tile " + " ".join(f"{n:>12}" for n in names))
for i in range(14):
    print(f"{i:4d} " + " ".join(f"{(ev[e][i] - t0) if ev[e][i] else -1:12d}" for e in range(10)))
print("epilogue warp 0, cycles after epi:full: ld1 wait, cvt1, ld2 wait, cvt2, transpose, done")
for i in range(8):
    print(i, [ev[e][i] - ev[7][i] for e in (10, 11, 12, 13, 14, 9)])
print("converter warp 0: start -> first load landed, -> last load landed, -> converted + stored, -> fenced")
for i in range(13):
    print(i, [ev[10][i] - ev[2][i], ev[11][i] - ev[10][i], ev[15][i] - ev[11][i], ev[3][i] - ev[15][i]])
def avg(xs):
    xs = [x for x in xs if x > -10**12]
    return sum(xs) / max(len(xs), 1)
T = range(4, 12)
print("steady state (tiles 4-11): producer period %.0f, raw latency issue->converter %.0f, converter busy %.0f, "
      "MMA issue span %.0f, MMA period %.0f, epilogue span %.0f" % (
          avg([ev[0][i + 1] - ev[0][i] for i in T]), avg([ev[1][i] - ev[0][i] for i in T]),
          avg([ev[3][i] - ev[2][i] for i in T]), avg([ev[6][i] - ev[5][i] for i in T]),
          avg([ev[6][i + 1] - ev[6][i] for i in T]), avg([ev[9][i] - ev[7][i] for i in T])))
print("MMA waits per tile (tiles 4-11): tmem_empty->a_full %.0f, a_full->issued %.0f; converter done -> MMA a_full %.0f" % (
    avg([ev[5][i] - ev[4][i] for i in T]), avg([ev[6][i] - ev[5][i] for i in T]), avg([ev[5][i] - ev[3][i] for i in T])))
