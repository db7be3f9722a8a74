"""K6 timing vs batch (is the cost per tile or fixed?): conv 56x56x128 -> 128, 3x3 pad 1."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_09120_b200 as lb
w = lb.prepare_weights(lb.pack_b(lb.encode_ternary(lb.generate(0, 46, 1, 9 * 128, 128))))
for b in [int(x) for x in os.environ.get("PROBE_B", "1,4,16,64").split(",")]:
    fm = lb.generate(0, 46, 0, b * 56 * 56, 128).view(b, 56, 56, 128)
    ws = torch.empty(int(lb._lib.lib.lowbit_conv2d_workspace_bytes(1, b, 56, 56, 128, 3, 3, 1, 1)), dtype=torch.uint8,
                     device="cuda")
    o = torch.empty((b, 56, 56, 128), dtype=torch.int16, device="cuda")
    f = lambda: lb.conv2d_lowbit(1, fm, False, w, 3, 3, 1, 1, kernel=2, out=o, workspace=ws)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(50):
        f()
    e.record(); torch.cuda.synchronize()
    print(f"batch {b}: {s.elapsed_time(e) / 50 * 1000:.1f} us per conv (pack + K6)")
