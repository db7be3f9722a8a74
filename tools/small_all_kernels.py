"""Small K5 / K7 / K3 / K2 calls checked against the oracle (a quick all-kernels probe)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2205_09120_b200 as lb
from oracle.oracle import Port
port = Port()
for mode, (m, n, k), (da, db) in [(lb.TNN, (600, 300, 1024), (0, 0)), (lb.BNN, (300, 200, 512), (1, 1))]:
    a = port.generate(da, 61, 0, m, k); b = port.generate(db, 61, 1, k, n)
    want = port.gemm(mode, a, b)
    at, bt = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    w = lb.prepare_weights(lb.pack_b(lb.encode_ternary(bt) if mode == lb.TNN else lb.encode_binary(bt)))
    for layout, kern in [(2, lb.KERNEL_TENSOR), (0, lb.KERNEL_TENSOR), (0, lb.KERNEL_TENSOR_I8), (0, lb.KERNEL_BITSERIAL)]:
        ap = lb.encode_binary(at, layout=layout) if mode == lb.BNN else lb.encode_ternary(at, layout=layout)
        got = lb.gemm_lowbit(mode, ap, w, (m, n, k), kernel=kern).cpu().numpy()
        assert np.array_equal(got, want), (mode, layout, kern)
fm = port.generate(0, 62, 0, 2 * 9 * 9, 128).reshape(2, 9, 9, 128)
wt = port.generate(0, 62, 1, 9 * 128, 64)
wts = lb.prepare_weights(lb.pack_b(lb.encode_ternary(torch.from_numpy(wt).cuda())))
got = lb.conv2d_lowbit(lb.TNN, torch.from_numpy(fm).cuda(), False, wts, 3, 3, 1, 1).cpu().numpy()
for img in range(2):
    assert (got[img].astype(np.int32) == port.direct_conv(fm[img], False, wt, 3, 3, 1, 1)).all()
torch.cuda.synchronize()
print("small all-kernels run OK")
