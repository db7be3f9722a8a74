"""Config 2: the 64-shape TBN sweep as one grouped launch, device time per launch in a graph of
20 back-to-back launches (LOWBIT_LIB selects an alternative build)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_09120_b200 as lb
SWEEP = [(M, N, K) for M in (72, 120, 240, 360) for N in (24, 48, 72, 96) for K in (128, 256, 384, 512)]
aps, ws, cs = [], [], []
for s, (M, N, K) in enumerate(SWEEP):
    a = lb.generate(2, 44, 2 * s, M, K)
    b = lb.generate(1, 44, 2 * s + 1, K, N)
    aps.append(lb.encode_ternary(a))
    ws.append(lb.prepare_weights(lb.pack_b(lb.encode_binary(b))))
    cs.append(torch.empty((M, N), dtype=torch.int16, device="cuda"))
probs = [(aps[s], ws[s], cs[s]) for s in range(len(SWEEP))]
f = lambda: lb.gemm_grouped(2, probs)
f(); torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(20):
        f()
g.replay(); torch.cuda.synchronize()
ts = []
for _ in range(5):
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record(); g.replay(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e) / 20 * 1e3)
print("grouped c2: %.2f us per launch (min %.2f)" % (sorted(ts)[2], min(ts)))
