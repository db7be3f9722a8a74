"""GPU parity of K5, the fp4 (tcgen05 kind::mxf4) bit-plane GeMM, against the
oracle and the reference's golden hashes.  A arrives in the NIBBLES plane
layout (element j of each 32-bit word at bit 4*(j%8) + j//8); results must be
bit-identical to gemm_lowbit (gemm.cpp:79-112) for every mode and shape,
including the depth extremes where the f32 accumulator's exactness matters.
"""
import hashlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle.oracle import BNN, TNN, TBN, a_mode_ternary, b_mode_ternary  # noqa: E402
from tests.golden.make_golden import mode_dists  # noqa: E402

NIBBLES = 2


@pytest.fixture(scope="module")
def lb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2205_09120_b200 as lb
    return lb


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def host(t):
    return t.cpu().numpy()


def sha(c):
    return hashlib.sha256(np.ascontiguousarray(c, "<i2").tobytes()).hexdigest()


def to_nibbles(planes: np.ndarray) -> np.ndarray:
    """Reference-layout plane rows -> LOWBIT_LAYOUT_NIBBLES."""
    rows, sb = planes.shape
    padded = np.zeros((rows, (sb + 3) // 4 * 4), np.uint8)
    padded[:, :sb] = planes
    words = padded.view("<u4").astype(np.uint64)
    out = np.zeros_like(words)
    for j in range(32):
        out |= ((words >> j) & 1) << (4 * (j % 8) + j // 8)
    return out.astype("<u4").view(np.uint8)[:, :sb]


def encode_a(lb, mode, a):
    return (lb.encode_ternary(dev(a), layout=NIBBLES) if a_mode_ternary(mode)
            else lb.encode_binary(dev(a), layout=NIBBLES))


def weights(lb, mode, b):
    bp = lb.encode_ternary(dev(b)) if b_mode_ternary(mode) else lb.encode_binary(dev(b))
    return lb.prepare_weights(lb.pack_b(bp))


@pytest.mark.parametrize("shape", [(1, 8), (7, 13), (33, 129), (257, 1000), (5, 2048)])
def test_encode_nibbles_layout(lb, port, shape):
    rows, cols = shape
    for tern in (False, True):
        v = port.generate(0 if tern else 1, 31, int(tern), rows, cols)
        w0, w1 = port.encode(v, tern)
        got = (lb.encode_ternary(dev(v), layout=NIBBLES) if tern else lb.encode_binary(dev(v), layout=NIBBLES))
        sb = (cols + 7) // 8
        assert (host(got.plane0)[:, :sb] == to_nibbles(w0)).all()
        if tern:
            assert (host(got.plane1)[:, :sb] == to_nibbles(w1)).all()
    with pytest.raises(lb.ZeroInBinaryInput):
        lb.encode_binary(torch.zeros((2, 40), dtype=torch.int8, device="cuda"), layout=NIBBLES)


SHAPES = [(1, 1, 1), (17, 9, 500), (70, 25, 7), (360, 96, 256), (300, 520, 1000), (129, 257, 4100),
          (1000, 300, 2048), (513, 224, 255), (256, 225, 257), (777, 448, 768), (64, 16, 64), (2000, 1000, 1536)]


@pytest.mark.parametrize("mode", [BNN, TNN, TBN])
def test_gemm_fp4_matches_oracle(lb, port, mode):
    da, db = mode_dists(mode)
    for i, (m, n, k) in enumerate(SHAPES):
        a = port.generate(da, 188 + i, 0, m, k)
        b = port.generate(db, 188 + i, 1, k, n)
        got = host(lb.gemm_lowbit(mode, encode_a(lb, mode, a), weights(lb, mode, b), (m, n, k), kernel=2))
        assert (got == port.gemm(mode, a, b)).all(), (mode, m, n, k)


# m >= 74 pair tiles (19k rows): the m-major schedule; k-block counts that keep
# the raw planes resident (even, <= 8 ternary / 16 binary), odd ones, and
# depths past the ring (streamed).
@pytest.mark.parametrize("mode", [BNN, TNN, TBN])
@pytest.mark.parametrize("k", [1000, 700, 2300, 4096])
def test_gemm_fp4_m_major_schedule(lb, port, mode, k):
    m, n = 19000, 300
    da, db = mode_dists(mode)
    a = port.generate(da, 300 + k, 0, m, k)
    b = port.generate(db, 300 + k, 1, k, n)
    got = host(lb.gemm_lowbit(mode, encode_a(lb, mode, a), weights(lb, mode, b), (m, n, k), kernel=2))
    assert (got == port.gemm(mode, a, b)).all(), (mode, m, n, k)


@pytest.mark.parametrize("mode", [BNN, TNN, TBN])
def test_gemm_fp4_depth_extremes(lb, port, mode):
    """k = k_max = 32767: |C| reaches 32767, so the f32 accumulator must stay exact."""
    m, n, k = 300, 40, 32767
    a = np.ones((m, k), np.int8)
    a[1::2] = -1
    b = np.ones((k, n), np.int8)
    b[:, 1::3] = -1
    got = host(lb.gemm_lowbit(mode, encode_a(lb, mode, a), weights(lb, mode, b), (m, n, k), kernel=2))
    want = port.gemm(mode, a, b)
    assert np.abs(want).max() == 32767
    assert (got == want).all()
    da, db = mode_dists(mode)
    a = port.generate(da, 7, 0, m, k)
    b = port.generate(db, 7, 1, k, n)
    got = host(lb.gemm_lowbit(mode, encode_a(lb, mode, a), weights(lb, mode, b), (m, n, k), kernel=2))
    assert (got == port.gemm(mode, a, b)).all()


def test_gemm_fp4_strided_output(lb, port):
    """ldc not a multiple of 8 elements -> the direct-store epilogue."""
    m, n, k = 400, 100, 700
    a = port.generate(0, 5, 0, m, k)
    b = port.generate(0, 5, 1, k, n)
    c = torch.full((m, n + 3), 12345, dtype=torch.int16, device="cuda")
    lb.gemm_lowbit(TNN, encode_a(lb, TNN, a), weights(lb, TNN, b), (m, n, k), kernel=2, out=c[:, :n])
    got = host(c)
    assert (got[:, :n] == port.gemm(TNN, a, b)).all()
    assert (got[:, n:] == 12345).all()


def test_nibbles_rejected_by_other_kernels(lb, port):
    ap = lb.encode_ternary(dev(port.generate(0, 3, 0, 16, 64)), layout=NIBBLES)
    w = lb.prepare_weights(lb.pack_b(lb.encode_ternary(dev(port.generate(0, 3, 1, 64, 8)))))
    for kernel in (1, 3):
        with pytest.raises(lb.InvalidArgument):
            lb.gemm_lowbit(TNN, ap, w, (16, 8, 64), kernel=kernel)


def test_config5_fp4_hash(lb, golden_configs):
    m, n, k = 1048576, 1024, 2048
    a = lb.generate(0, 47, 0, m, k)
    ap = lb.encode_ternary(a, layout=NIBBLES)
    del a
    w = lb.prepare_weights(lb.pack_b(lb.encode_ternary(lb.generate(0, 47, 1, k, n))))
    c = lb.gemm_lowbit(TNN, ap, w, (m, n, k), kernel=2)
    assert sha(host(c)) == golden_configs["c5"]["sha256"]


def test_config3_fp4_hash(lb, golden_configs):
    m = n = 8192
    k = 4096
    ap = lb.encode_binary(lb.generate(1, 45, 0, m, k), layout=NIBBLES)
    w = lb.prepare_weights(lb.pack_b(lb.encode_binary(lb.generate(1, 45, 1, k, n))))
    c = lb.gemm_lowbit(BNN, ap, w, (m, n, k), kernel=2)
    assert sha(host(c)) == golden_configs["c3"]["sha256"]


def test_gemm_fp4_cluster4_multicast_experiment(lb):
    """The 4-CTA-cluster variant with multicast B (a tuning experiment behind
    LOWBIT_FP4_CL4=1, read once per process) stays bit-exact."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import numpy as np, torch, paper_2205_09120_b200 as lb\n"
        "from oracle.oracle import Port\n"
        "p = Port()\n"
        "for mode, (m, n, k) in [(1, (40000, 520, 2048)), (0, (19000, 300, 1024)), (2, (25000, 1024, 512))]:\n"
        "    da, db = {0: (1, 1), 1: (0, 0), 2: (2, 1)}[mode]\n"
        "    a = p.generate(da, 9, 0, m, k); b = p.generate(db, 9, 1, k, n)\n"
        "    at = torch.from_numpy(a).cuda()\n"
        "    ap = lb.encode_binary(at, layout=2) if mode == 0 else lb.encode_ternary(at, layout=2)\n"
        "    bp = lb.encode_ternary(torch.from_numpy(b).cuda()) if mode == 1 else lb.encode_binary(torch.from_numpy(b).cuda())\n"
        "    got = lb.gemm_lowbit(mode, ap, lb.prepare_weights(lb.pack_b(bp)), (m, n, k), kernel=2).cpu().numpy()\n"
        "    assert (got == p.gemm(mode, a, b)).all(), (mode, m, n, k)\n"
        "print('ok')\n")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=root,
                       env=dict(os.environ, LOWBIT_FP4_CL4="1"))
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]
