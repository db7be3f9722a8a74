"""Tuning sweep: K5 (fp4 pair kernel) TOPS vs n (tile width) at fixed m, k.
Set LOWBIT_DEBUG_FP4 for the role-isolation experiments (results invalid)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_09120_b200 as lb

m, k = int(os.environ.get("M", 524288)), int(os.environ.get("K", 2048))
a = lb.generate(0, 1, 0, m, k)
ap = lb.encode_ternary(a, layout=2)
del a
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for n in [int(x) for x in os.environ.get("NS", "768 832 896 1024 448 512").split()]:
    w = lb.prepare_weights(lb.pack_b(lb.encode_ternary(lb.generate(0, 1, 1, k, n))))
    c = torch.empty((m, n), dtype=torch.int16, device="cuda")
    for _ in range(3):
        lb.gemm_lowbit(1, ap, w, (m, n, k), kernel=2, out=c)
    ts = []
    for _ in range(20):
        flush.zero_()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); lb.gemm_lowbit(1, ap, w, (m, n, k), kernel=2, out=c); e.record()
        torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    ts.sort(); t = ts[len(ts) // 2]
    print(f"n={n} ms={t:.4f} TOPS={2*m*n*k/t/1e9:.0f}", flush=True)
