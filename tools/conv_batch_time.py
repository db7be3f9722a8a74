"""c4's conv (56x56x128 ternary, 3x3 -> 128, s1 p1) at other batch sizes: device time per conv in a graph of 10 back to back."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2205_09120_b200 as lb
for batch in [int(x) for x in os.environ.get("BATCHES", "16,64,256,1024").split(",")]:
    fm = lb.generate(0, 46, 0, batch * 56 * 56, 128).view(batch, 56, 56, 128)
    w = lb.prepare_weights(lb.pack_b(lb.encode_ternary(lb.generate(0, 46, 1, 9 * 128, 128))))
    o = torch.empty((batch, 56, 56, 128), dtype=torch.int16, device="cuda")
    f = lambda: lb.conv2d_lowbit(1, fm, False, w, 3, 3, 1, 1, kernel=lb.KERNEL_TENSOR, out=o)
    t = sorted(bench.graph_time(torch, f, reps=10, inner=10) * 1e3 for _ in range(3))[1]
    nbytes = batch * 56 * 56 * 128 * 3
    print(f"batch {batch}: {t:.2f} us, {2.0 * batch * 3136 * 128 * 1152 / t / 1e6:.0f} TOPS, frac_hbm {nbytes / (t * 1e-6) / 1e9 / 6542.7:.3f}")
