"""Stage timeline of pair 0's leader CTA in the fp4 kernel (profiling experiment):
LOWBIT_DEBUG_FP4=32 python tools/fp4_timeline.py"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2205_09120_b200 as lb
L = lb._lib
M, N, K = 1048576, 1024, 2048
a = lb.generate(0, 47, 0, M, K); ap = lb.encode_ternary(a, layout=2); del a
w = lb.prepare_weights(lb.pack_b(lb.encode_ternary(lb.generate(0, 47, 1, K, N))))
c = torch.empty((M, N), dtype=torch.int16, device="cuda")
for _ in range(3):
    lb.gemm_lowbit(1, ap, w, (M, N, K), kernel=2, out=c)
torch.cuda.synchronize()
buf = (C.c_longlong * (8 * 1024))()
L.lib.lowbit_debug_fp4_timeline(buf)
t = np.array(buf, dtype=np.int64).reshape(8, 1024)
t0 = t[0, 0]
s = slice(200, 800)
d = lambda a, b: np.median((t[b] - t[a])[s])
print("median over stages 200..799 (cycles):")
print(f"  stage period (MMA start t -> t+1):   {np.median(np.diff(t[0])[s]):.0f}")
print(f"  MMA wait A (0->1):                   {d(0,1):.0f}")
print(f"  MMA wait B (1->2):                   {d(1,2):.0f}")
print(f"  MMA issue (2->3):                    {d(2,3):.0f}")
print(f"  converter chain slot->red (4->5):    {d(4,5):.0f}")
print(f"  red -> MMA sees A (5->1):            {d(5,1):.0f}")
sh = np.median((t[4][4:] - t[3][:-4])[200:800])
print(f"  MMA issued t -> slot free for t+4:   {sh:.0f}")
print(f"  B TMA issue -> watcher sees (6->7):  {d(6,7):.0f}")
print(f"  watcher sees B -> MMA start (7->0):  {d(7,0):.0f}")
