"""K4 (fused im2col + encode) alone on c4: int8 NHWC in, two bit planes out; events after an L2 flush, median of 9."""
import ctypes as C
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_09120_b200 as lb
L = lb._lib
fm = lb.generate(0, 46, 0, 64 * 56 * 56, 128).view(64, 56, 56, 128)
pitch = lb.plane_pitch(1152)
p0 = torch.empty(200704 * pitch, dtype=torch.uint8, device="cuda")
p1 = torch.empty(200704 * pitch, dtype=torch.uint8, device="cuda")
fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
f = lambda: L.check(L.lib.lowbit_conv_encode(0, C.c_void_p(fm.data_ptr()), 64, 56, 56, 128, 3, 3, 1, 1, 0,
                                             C.c_void_p(p0.data_ptr()), C.c_void_p(p1.data_ptr()), pitch, None, st))
f(); torch.cuda.synchronize()
ts = []
for _ in range(9):
    fl.zero_(); fl.view(torch.int64).sum()  # flush L2, lines left clean (as bench.py)
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record(); f(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
t = sorted(ts)[4]
nb = 64 * 56 * 56 * 128 + 2 * 200704 * pitch
print(f"K4 c4: {t * 1e3:.1f} us, {nb / t / 1e6:.0f} GB/s")
