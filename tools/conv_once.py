"""Config 4 (64x56x56x128 ternary NHWC, 3x3x128 -> 128, s1 p1) through conv2d_lowbit, a few times."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_09120_b200 as lb
fm = lb.generate(0, 46, 0, 64 * 56 * 56, 128).view(64, 56, 56, 128)
w = lb.prepare_weights(lb.pack_b(lb.encode_ternary(lb.generate(0, 46, 1, 9 * 128, 128))))
out = torch.empty((64, 56, 56, 128), dtype=torch.int16, device="cuda")
for _ in range(3):
    lb.conv2d_lowbit(lb.TNN, fm, False, w, 3, 3, 1, 1, out=out)
torch.cuda.synchronize()
print("ok", int(out.sum()))
