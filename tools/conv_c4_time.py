"""Config 4 conv timing per path (kernel 2: fp4 K6 incl. the fm pack pass; 4: int8 implicit GeMM; 1: K4 + K2)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_09120_b200 as lb
fm = lb.generate(0, 46, 0, 64 * 56 * 56, 128).view(64, 56, 56, 128)
w = lb.prepare_weights(lb.pack_b(lb.encode_ternary(lb.generate(0, 46, 1, 9 * 128, 128))))
ws = torch.empty(int(lb._lib.lib.lowbit_conv2d_workspace_bytes(1, 64, 56, 56, 128, 3, 3, 1, 1)), dtype=torch.uint8,
                 device="cuda")
o = torch.empty((64, 56, 56, 128), dtype=torch.int16, device="cuda")
fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ops = 2.0 * 200704 * 128 * 1152
for kern in [int(x) for x in os.environ.get("KERNELS", "2,4,1").split(",")]:
    f = lambda: lb.conv2d_lowbit(1, fm, False, w, 3, 3, 1, 1, kernel=kern, out=o, workspace=ws)
    for _ in range(3):
        f()
    ts = []
    for _ in range(20):
        fl.zero_(); fl.view(torch.int64).sum()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); f(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    ts.sort(); t = ts[10]
    # back to back (launch overhead amortised; fm stays in L2 between calls)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(50):
        f()
    e.record(); torch.cuda.synchronize()
    tb = s.elapsed_time(e) / 50
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    tg = []
    for _ in range(20):
        fl.zero_(); fl.view(torch.int64).sum()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); g.replay(); e.record(); torch.cuda.synchronize(); tg.append(s.elapsed_time(e))
    tg.sort()
    g10 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g10):
        for _ in range(10):
            f()
    g10.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record(); g10.replay(); e.record(); torch.cuda.synchronize()
    t10 = s.elapsed_time(e) / 10
    print(f"kernel {kern}: graph of 10 back-to-back {t10*1e3:.1f} us; eager {t*1e3:.1f} us, back-to-back {tb*1e3:.1f} us, graph+flush {tg[10]*1e3:.1f} us "
          f"({ops/tg[10]/1e9:.0f} TOPS)")
