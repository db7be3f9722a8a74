"""Role timing of the fp4 pair kernel on config 5 (profiling experiment):
LOWBIT_DEBUG_FP4=8 python tools/fp4_stats.py"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_09120_b200 as lb
L = lb._lib
M, N, K = int(os.environ.get("M", 1048576)), int(os.environ.get("N", 1024)), int(os.environ.get("K", 2048))
a = lb.generate(0, 47, 0, M, K); ap = lb.encode_ternary(a, layout=int(os.environ.get("LAYOUT", 2))); del a
w = lb.prepare_weights(lb.pack_b(lb.encode_ternary(lb.generate(0, 47, 1, K, N))))
c = torch.empty((M, N), dtype=torch.int16, device="cuda")
for _ in range(3):
    lb.gemm_lowbit(1, ap, w, (M, N, K), kernel=2, out=c)
torch.cuda.synchronize()
buf = (C.c_ulonglong * 16)()
L.lib.lowbit_debug_fp4_stats(buf)  # reset
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); lb.gemm_lowbit(1, ap, w, (M, N, K), kernel=2, out=c); e.record(); torch.cuda.synchronize()
L.lib.lowbit_debug_fp4_stats(buf)
v = list(buf)
ms = s.elapsed_time(e)
print(f"kernel {ms:.3f} ms  {2*M*N*K/ms/1e9:.0f} TOPS")
nl = 74
kb = max(v[12], 1)
print(f"MMA/leader: total {v[3]/nl:.0f} cyc, wait a_ready {v[0]/nl:.0f}, b_full {v[1]/nl:.0f}, "
      f"tmem_empty {v[2]/nl:.0f}, sf_ready {v[11]/nl:.0f}; k-blocks {kb/nl:.0f} -> {v[3]/kb:.0f} cyc/kblock")
nc = 148 * 8
print(f"converter warp: total {v[7]/nc:.0f}, wait raw {v[4]/nc:.0f}, wait slot {v[5]/nc:.0f}, work {v[6]/nc:.0f}; "
      f"work per k-block {v[6]/nc/(kb/nl/2):.0f} cyc")
ne = 148 * 4
print(f"epilogue warp: total {v[9]/ne:.0f}, wait tmem_full {v[8]/ne:.0f}, tail+scales {v[10]/ne:.0f}, "
      f"first group {v[14]/ne:.0f}, other groups {v[15]/ne:.0f}")
