"""c5 end to end through lowbit_gemm_lowbit_host with PAGEABLE (numpy) host buffers: host clock per call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2205_09120_b200 as lb
M, N, K = int(os.environ.get("M", 1048576)), 1024, 2048
a = lb.generate(0, 47, 0, M, K)
ap = lb.encode_ternary(a); del a
sb = (K + 7) // 8
a0 = ap.plane0.cpu().numpy()[:, :sb].copy(); a1 = ap.plane1.cpu().numpy()[:, :sb].copy(); del ap
pb = lb.pack_b(lb.encode_ternary(lb.generate(0, 47, 1, K, N)))
pan = pb.panels.cpu().numpy().copy()
out = np.zeros((M, N), np.int16)
f = lambda: lb.gemm_lowbit_host(1, a0, a1, M, K, pan, True, N, K, (M, N, K), out=out)
f()
ts = []
for _ in range(4):
    t0 = time.perf_counter(); f(); ts.append(time.perf_counter() - t0)
t = float(np.median(ts))
print(f"pageable e2e c5: {t * 1e3:.1f} ms, {2.0 * M * N * K / t / 1e12:.1f} TOPS "
      f"(threads {os.environ.get('LOWBIT_COPY_THREADS', 'default')}, slot {os.environ.get('LOWBIT_STAGE_MB', 16)} MB)")
