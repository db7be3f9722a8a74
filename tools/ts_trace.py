"""Per-tile event timeline of K7T's CTA 0 on c4 (TUNING build, LOWBIT_HALO_DEBUG=32)."""
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
L = lb._lib.lib
ph = (C.c_ulonglong * 4)()
L.lowbit_debug_ts_phases(ph, 1)
lb.conv2d_lowbit(1, fm, False, w, 3, 3, 1, 1, kernel=2, out=o)
torch.cuda.synchronize()
L.lowbit_debug_ts_phases(ph, 0)
print("phases (us): first entry -> last setup end %.2f, -> last work end %.2f (total %.2f)" % (
    (ph[1] - ph[0]) / 1e3, (ph[2] - ph[1]) / 1e3, (ph[2] - ph[0]) / 1e3))
buf = (C.c_ulonglong * 1024)()
L.lowbit_debug_ts_trace(buf)
ev = [[buf[e * 64 + i] for i in range(64)] for e in range(16)]
t0 = min(x for x in ev[0] if x)
names = ["prod:issue", "wait:raw", "cv:start", "cv:done", "mma:acc", "mma:a_full", "mma:issued", "epi:full",
         "epi:release", "epi:done"]
print("tile " + " ".join(f"{n:>11}" for n in names))
for i in range(14):
    print(f"{i:4d} " + " ".join(f"{(ev[e][i] - t0) if ev[e][i] else -1:11d}" for e in range(10)))
def avg(xs):
    return sum(xs) / max(len(xs), 1)
T = range(3, 11)
print("steady (tiles 3-10): conv busy %.0f, conv period %.0f, MMA a_full->issued %.0f, MMA period %.0f, "
      "epi full->release %.0f, full->done %.0f, issued->epi full %.0f" % (
          avg([ev[3][i] - ev[2][i] for i in T]), avg([ev[2][i + 1] - ev[2][i] for i in T]),
          avg([ev[6][i] - ev[5][i] for i in T]), avg([ev[6][i + 1] - ev[6][i] for i in T]),
          avg([ev[8][i] - ev[7][i] for i in T]), avg([ev[9][i] - ev[7][i] for i in T]),
          avg([ev[7][i] - ev[6][i] for i in T])))
