"""Timing of K3 (int8 pair: c5 from lanes planes, lowbit_gemm_i8), the int8 implicit conv (c4,
kernel TENSOR_I8) and K6 (fp4 implicit conv: c4's map with stride 2).  Events, L2 flushed."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_09120_b200 as lb
fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def t(f, reps=10):
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        fl.zero_(); fl.view(torch.int64).sum()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); f(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    return sorted(ts)[reps // 2] * 1e3
M, N, K = 1048576, 1024, 2048
a = lb.generate(0, 47, 0, M, K)
w = lb.prepare_weights(lb.pack_b(lb.encode_ternary(lb.generate(0, 47, 1, K, N))))
c = torch.empty((M, N), dtype=torch.int16, device="cuda")
ap = lb.encode_ternary(a, layout=1)
r = {}
r["k3_c5_lanes_us"] = t(lambda: lb.gemm_lowbit(1, ap, w, (M, N, K), kernel=lb.KERNEL_TENSOR, out=c))
r["gemm_i8_c5_us"] = t(lambda: lb.gemm_lowbit_i8(1, a, w, (M, N, K), out=c))
del ap, a, c
fm = lb.generate(0, 46, 0, 64 * 56 * 56, 128).view(64, 56, 56, 128)
wc = lb.prepare_weights(lb.pack_b(lb.encode_ternary(lb.generate(0, 46, 1, 9 * 128, 128))))
ws = torch.empty(int(lb._lib.lib.lowbit_conv2d_workspace_bytes(1, 64, 56, 56, 128, 3, 3, 2, 1)), dtype=torch.uint8,
                 device="cuda")
ws1 = torch.empty(int(lb._lib.lib.lowbit_conv2d_workspace_bytes(1, 64, 56, 56, 128, 3, 3, 1, 1)), dtype=torch.uint8,
                  device="cuda")
o2 = torch.empty((64, 28, 28, 128), dtype=torch.int16, device="cuda")
o1 = torch.empty((64, 56, 56, 128), dtype=torch.int16, device="cuda")
r["k6_c4_stride2_us"] = t(lambda: lb.conv2d_lowbit(1, fm, False, wc, 3, 3, 2, 1, kernel=lb.KERNEL_TENSOR, out=o2,
                                                   workspace=ws))
r["i8_conv_c4_us"] = t(lambda: lb.conv2d_lowbit(1, fm, False, wc, 3, 3, 1, 1, kernel=lb.KERNEL_TENSOR_I8, out=o1,
                                                workspace=ws1))
print(" ".join("%s=%.1f" % kv for kv in r.items()))
