"""Config 1 (TNN 360 x 96 x 256) latency per path: CUDA-graph replays of one call (launch path off the host)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_09120_b200 as lb
m, n, k = 360, 96, 256
a = lb.generate(0, 43, 0, m, k); b = lb.generate(0, 43, 1, k, n)
ap = lb.encode_ternary(a); w = lb.prepare_weights(lb.pack_b(lb.encode_ternary(b)))
c = torch.empty((m, n), dtype=torch.int16, device="cuda")
ref = lb.gemm_lowbit(1, ap, w, (m, n, k), kernel=lb.KERNEL_BITSERIAL)


def graph_us(fn, reps=50):
    fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record(); g.replay(); e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


for name, kern in [("auto", lb.KERNEL_AUTO), ("tensor_i8", lb.KERNEL_TENSOR_I8), ("tensor", lb.KERNEL_TENSOR),
                   ("1cta", lb.KERNEL_TENSOR_1CTA), ("bitserial", lb.KERNEL_BITSERIAL)]:
    try:
        us = graph_us(lambda: lb.gemm_lowbit(1, ap, w, (m, n, k), kernel=kern, out=c))
        assert torch.equal(c, ref)
        print(f"{name}: {us:.2f} us")
    except Exception as ex:
        print(name, "failed", ex)
us = graph_us(lambda: lb.gemm_grouped(1, [(ap, w, c)]))
assert torch.equal(c, ref)
print(f"grouped (1 problem): {us:.2f} us")

# config 2 sweep (TBN): per-shape latency by kernel, 20 back-to-back graph replays each
import itertools
tot = {"tensor_i8": 0.0, "1cta": 0.0, "tensor": 0.0}
wins = {"tensor_i8": 0, "1cta": 0, "tensor": 0}
for M, N, K in itertools.product((72, 120, 240, 360), (24, 48, 72, 96), (128, 256, 384, 512)):
    a = lb.generate(2, 44, 0, M, K); b = lb.generate(1, 44, 1, K, N)
    ap = lb.encode_ternary(a); w = lb.prepare_weights(lb.pack_b(lb.encode_binary(b)))
    c = torch.empty((M, N), dtype=torch.int16, device="cuda")
    ref = lb.gemm_lowbit(lb.TBN, ap, w, (M, N, K), kernel=lb.KERNEL_BITSERIAL)
    best, bestk = 1e9, None
    row = {}
    for name, kern in [("tensor_i8", lb.KERNEL_TENSOR_I8), ("1cta", lb.KERNEL_TENSOR_1CTA), ("tensor", lb.KERNEL_TENSOR)]:
        us = graph_us(lambda: lb.gemm_lowbit(lb.TBN, ap, w, (M, N, K), kernel=kern, out=c), reps=20)
        assert torch.equal(c, ref), (M, N, K, name)
        tot[name] += us
        row[name] = us
        if us < best:
            best, bestk = us, name
    wins[bestk] += 1
    if os.environ.get("PER_SHAPE"):
        print(M, N, K, " ".join(f"{k}={v:.2f}" for k, v in row.items()), "best", bestk)
print("c2 sweep, sum of per-shape latencies (us):", {k: round(v, 1) for k, v in tot.items()}, "wins:", wins)
