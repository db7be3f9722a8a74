"""Per-tile event timeline of K6's first leader CTA (LOWBIT_CONV_DEBUG must include 32)."""
import ctypes as C
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_09120_b200 as lb
b = int(os.environ.get("PROBE_B", "64"))
fm = lb.generate(0, 46, 0, b * 56 * 56, 128).view(b, 56, 56, 128)
w = lb.prepare_weights(lb.pack_b(lb.encode_ternary(lb.generate(0, 46, 1, 9 * 128, 128))))
ws = torch.empty(int(lb._lib.lib.lowbit_conv2d_workspace_bytes(1, b, 56, 56, 128, 3, 3, 1, 1)), dtype=torch.uint8,
                 device="cuda")
o = torch.empty((b, 56, 56, 128), dtype=torch.int16, device="cuda")
for _ in range(3):
    lb.conv2d_lowbit(1, fm, False, w, 3, 3, 1, 1, kernel=2, out=o, workspace=ws)
torch.cuda.synchronize()
buf = (C.c_ulonglong * 1024)()
assert lb._lib.lib.lowbit_debug_conv_trace(buf) == 0
ev = [[buf[e * 64 + i] for i in range(64)] for e in range(16)]
t0 = min(x for x in ev[5] + ev[0] if x)
names = ["mma:acc_free", "mma:a_full", "mma:issued", "epi:full", "epi:drained", "prod:a_empty", "prod:issued",
         "mma:loop_end"]
print("tile " + " ".join(f"{n:>13}" for n in names))
for i in range(16):
    print(f"{i:4d} " + " ".join(f"{(ev[e][i] - t0) if ev[e][i] else -1:13d}" for e in range(8)))
print("epilogue warp 0 (from tmem_full): tmem_ld done, sts done, fence done, store issued")
for i in range(6):
    print(i, [ev[e][i] - ev[3][i] for e in (9, 10, 11, 12, 4)])
