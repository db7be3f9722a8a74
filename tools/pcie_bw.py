"""Pinned host <-> device copy bandwidth on this box (1 vs 2 vs 4 concurrent D2H streams)."""
import torch
n = 2 << 30
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
for nstreams in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    part = n // nstreams
    for rep in range(2):
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for i, st in enumerate(streams):
            st.wait_event(s)
            with torch.cuda.stream(st):
                h[i * part:(i + 1) * part].copy_(d[i * part:(i + 1) * part], non_blocking=True)
        for st in streams:
            e.wait(st) if False else torch.cuda.current_stream().wait_stream(st)
        e.record()
        torch.cuda.synchronize()
    print(f"D2H {nstreams} stream(s): {n / (s.elapsed_time(e) * 1e-3) / 1e9:.1f} GB/s")
torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record(); d.copy_(h, non_blocking=True); e.record(); torch.cuda.synchronize()
print(f"H2D 1 stream: {n / (s.elapsed_time(e) * 1e-3) / 1e9:.1f} GB/s")
