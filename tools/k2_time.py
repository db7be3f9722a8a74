"""K2 (bit-serial) timing: TNN on a 262144-row slice of c5, BNN c3 and a TBN shape; events, median of 5."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_09120_b200 as lb
for name, mode, m, n, k, da, db, seed in [("c5 slice TNN", lb.TNN, 262144, 1024, 2048, 0, 0, 47),
                                          ("c3 BNN", lb.BNN, 8192, 8192, 4096, 1, 1, 45),
                                          ("TBN", lb.TBN, 65536, 1024, 2048, 2, 1, 44)]:
    a = lb.generate(da, seed, 0, m, k)
    b = lb.generate(db, seed, 1, k, n)
    ap = lb.encode_binary(a) if mode == lb.BNN else lb.encode_ternary(a)
    w = lb.prepare_weights(lb.pack_b(lb.encode_ternary(b) if mode == lb.TNN else lb.encode_binary(b)))
    out = torch.empty((m, n), dtype=torch.int16, device="cuda")
    f = lambda: lb.gemm_lowbit(mode, ap, w, (m, n, k), kernel=lb.KERNEL_BITSERIAL, out=out)
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); f(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    t = sorted(ts)[2]
    print(f"{name}: {t:.3f} ms, {2.0 * m * n * k / t / 1e9:.1f} TOPS")
