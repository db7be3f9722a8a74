"""Config-4-shaped BNN conv on a binary map padded with +1 (binary_pad_value): K7 (AUTO) vs the K4 encode +
GeMM path (KERNEL_BITSERIAL: K4 + K2, and K4 + the AUTO GeMM through a workspace-only call is what round 1 ran)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_09120_b200 as lb
fm = lb.generate(1, 48, 0, 64 * 56 * 56, 128).view(64, 56, 56, 128)
w = lb.prepare_weights(lb.pack_b(lb.encode_binary(lb.generate(1, 48, 1, 9 * 128, 128))))
o = torch.empty((64, 56, 56, 128), dtype=torch.int16, device="cuda")
fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ops = 2.0 * 200704 * 128 * 1152
import ctypes as C
L = lb._lib
ws = torch.empty(int(L.lib.lowbit_conv2d_workspace_bytes(0, 64, 56, 56, 128, 3, 3, 1, 1)), dtype=torch.uint8,
                 device="cuda")
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for name, kern in (("AUTO (K7)", 0), ("K4 + K2", 1)):
    # the C ABI call itself (lb.conv2d_lowbit also reads the zero flag back: a host sync)
    f = lambda: L.check(L.lib.lowbit_conv2d(0, C.c_void_p(fm.data_ptr()), 64, 56, 56, 128, 1, C.c_void_p(w.buf.data_ptr()),
                                            0, 128, 1152, 3, 3, 1, 1, 1, C.c_void_p(ws.data_ptr()),
                                            C.c_void_p(flag.data_ptr()), C.c_void_p(o.data_ptr()), kern, st), "conv")
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        fl.zero_(); fl.view(torch.int64).sum()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); f(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    t = sorted(ts)[5]
    print(f"BNN c4-shaped conv, pad value +1, {name}: {t * 1e3:.1f} us ({ops / t / 1e9:.0f} TOPS), zero flag "
          f"{int(flag.item())}")
