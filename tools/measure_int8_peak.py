"""Measure dense int8 tensor throughput on this GPU with cuBLASLt (torch._int_mm)
as a roofline denominator for the tcgen05 kind::i8 path."""
import json, sys, torch
torch.cuda.set_device(0)
res = {}
for n in (4096, 8192, 16384):
    a = torch.randint(-1, 2, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-1, 2, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()
    for _ in range(3):
        c = torch._int_mm(a, b)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    s.record()
    for _ in range(reps):
        c = torch._int_mm(a, b)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    res[n] = {"ms": ms, "TOPS": 2.0 * n ** 3 / (ms * 1e-3) / 1e12}
print(json.dumps({"cublaslt_int8_int_mm": res}))
