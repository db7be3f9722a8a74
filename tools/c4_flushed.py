"""Config 4 on K7 the way bench.py reports it: cold L2 (graph of 10 x (flush, conv) minus 10 x flush) and back to back."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2205_09120_b200 as lb
fm = lb.generate(0, 46, 0, 64 * 56 * 56, 128).view(64, 56, 56, 128)
w = lb.prepare_weights(lb.pack_b(lb.encode_ternary(lb.generate(0, 46, 1, 9 * 128, 128))))
o = torch.empty((64, 56, 56, 128), dtype=torch.int16, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
f = lambda: lb.conv2d_lowbit(1, fm, False, w, 3, 3, 1, 1, kernel=lb.KERNEL_TENSOR, out=o)
cold = [bench.graph_time_flushed_avg(torch, f, flush) * 1e3 for _ in range(5)]
b2b = [bench.graph_time(torch, f, reps=10, inner=10) * 1e3 for _ in range(3)]
print("cold L2 us:", " ".join(f"{x:.2f}" for x in cold), "| back to back us:", " ".join(f"{x:.2f}" for x in b2b),
      "| frac_hbm cold %.3f b2b %.3f" % (77070336 / (sorted(cold)[2] * 1e-6) / 1e9 / 6542.7, 77070336 / (sorted(b2b)[1] * 1e-6) / 1e9 / 6542.7))
