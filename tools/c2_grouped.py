"""Config 2's 64-shape TBN sweep as one grouped launch (a few calls, for ncu's launch list)."""
import itertools, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_09120_b200 as lb
probs = []
for M, N, K in itertools.product((72, 120, 240, 360), (24, 48, 72, 96), (128, 256, 384, 512)):
    a = lb.generate(2, 44, 0, M, K); b = lb.generate(1, 44, 1, K, N)
    probs.append((lb.encode_ternary(a), lb.prepare_weights(lb.pack_b(lb.encode_binary(b))),
                  torch.empty((M, N), dtype=torch.int16, device="cuda")))
for _ in range(3):
    lb.gemm_grouped(lb.TBN, probs)
torch.cuda.synchronize()
print("ok")
