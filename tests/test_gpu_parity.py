"""GPU parity: the CUDA path (through the C ABI) against the oracle and the
reference's own golden outputs.  Bit-exact everywhere (integer work).

Small/medium shapes compare full outputs with the C oracle; BASELINE.json's
configs compare against sha256 hashes of the REFERENCE library's own output
(tests/golden/golden_configs.json) plus size-independent properties.
"""
import hashlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle.oracle import BNN, TNN, TBN, a_mode_ternary, b_mode_ternary  # noqa: E402
from tests.golden.make_golden import SMALL_GEMM, mode_dists, sweep_shapes  # noqa: E402

# LOWBIT_KERNEL_BITSERIAL, LOWBIT_KERNEL_TENSOR (reference planes -> fp4 K5), LOWBIT_KERNEL_TENSOR_1CTA,
# LOWBIT_KERNEL_TENSOR_I8 (int8 K3, CTA pairs when m > 128)
KERNELS = [1, 2, 3, 4]


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


def gpu_gemm(lb, mode, a, b, kernel, k_blk=4096):
    """int8 host matrices -> device encode -> pack_b -> prepare -> gemm."""
    m, k = a.shape
    n = b.shape[1]
    ap = lb.encode_ternary(dev(a)) if a_mode_ternary(mode) else lb.encode_binary(dev(a))
    bp = lb.encode_ternary(dev(b)) if b_mode_ternary(mode) else lb.encode_binary(dev(b))
    pb = lb.pack_b(bp)
    w = lb.prepare_weights(pb)
    return host(lb.gemm_lowbit(mode, ap, w, (m, n, k), k_blk=k_blk, kernel=kernel))


def sha(c):
    return hashlib.sha256(np.ascontiguousarray(c, "<i2").tobytes()).hexdigest()


# ------------------------------------------------------------------ K1 / K1b
@pytest.mark.parametrize("shape", [(1, 8), (7, 13), (9, 17), (3, 64), (5, 100), (16, 504), (33, 129), (257, 1000)])
def test_encode_matches_oracle(lb, port, shape):
    rows, cols = shape
    for tern in (False, True):
        v = port.generate(0 if tern else 1, 11, int(tern), rows, cols)
        want0, want1 = port.encode(v, tern)
        got = lb.encode_ternary(dev(v)) if tern else lb.encode_binary(dev(v))
        sb = (cols + 7) // 8
        g0 = host(got.plane0)
        assert (g0[:, :sb] == want0).all() and not g0[:, sb:].any()
        if tern:
            g1 = host(got.plane1)
            assert (g1[:, :sb] == want1).all() and not g1[:, sb:].any()


def test_encode_strided_input(lb, port):
    big = port.generate(0, 12, 0, 40, 300)
    t = dev(big)[:, 5:205]  # ld 300, unaligned start
    got = lb.encode_ternary(t)
    w0, w1 = port.encode(np.ascontiguousarray(big[:, 5:205]), True)
    assert (host(got.plane0)[:, :25] == w0).all() and (host(got.plane1)[:, :25] == w1).all()


def test_encode_binary_rejects_zero(lb):
    v = torch.ones((3, 40), dtype=torch.int8, device="cuda")
    v[2, 37] = 0
    with pytest.raises(lb.ZeroInBinaryInput):
        lb.encode_binary(v)


def test_generator_matches_oracle(lb, port):
    for dist in (0, 1, 2):
        g = host(lb.generate(dist, 47, 3, 33, 777, row0=1000))
        assert (g == port.generate(dist, 47, 3, 33, 777, row0=1000)).all()


@pytest.mark.parametrize("shape", [(1, 1), (16, 8), (17, 9), (504, 8), (100, 25), (2048, 1024), (333, 130)])
def test_pack_b_matches_oracle(lb, port, shape):
    k, n = shape
    for tern in (False, True):
        v = port.generate(0 if tern else 1, 13, int(tern), k, n)
        b0, b1 = port.encode(v, tern)
        want = port.pack_b(b0, b1, k, n)
        got = lb.pack_b(lb.encode_ternary(dev(v)) if tern else lb.encode_binary(dev(v)))
        assert (host(got.panels)[: len(want)] == want).all()


def test_pack_b_golden(lb, port, golden):
    for case, (rows, cols) in enumerate([(1, 8), (7, 13), (9, 17), (3, 64), (5, 100), (16, 504), (33, 129)]):
        for tern in (0, 1):
            v = port.generate(0 if tern else 1, 1000 + case, tern, rows, cols)
            got = lb.pack_b(lb.encode_ternary(dev(v)) if tern else lb.encode_binary(dev(v)))
            want = golden[f"packb_{case}_{tern}"]
            assert (host(got.panels)[: len(want)] == want).all()


# ------------------------------------------------------------------ K2 / K3
@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("mode", [BNN, TNN, TBN])
def test_gemm_golden_small(lb, port, golden, mode, kernel):
    da, db = mode_dists(mode)
    for case, (m, n, k) in enumerate(SMALL_GEMM):
        if k == 32767:
            if mode != BNN:
                continue
            a, b = np.ones((m, k), np.int8), np.ones((k, n), np.int8)
        else:
            a = port.generate(da, 2000 + 100 * mode + case, 0, m, k)
            b = port.generate(db, 2000 + 100 * mode + case, 1, k, n)
        for k_blk in ((4096, 64) if k < 32767 else (4096,)):
            got = gpu_gemm(lb, mode, a, b, kernel, k_blk)
            want = golden[f"gemm_{mode}_{case}_{k_blk}"]
            assert (got == want).all(), (mode, kernel, m, n, k)


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("mode", [BNN, TNN, TBN])
def test_gemm_nonaligned_grid(lb, port, mode, kernel):  # test_gemm.cpp:50-61
    da, db = mode_dists(mode)
    i = 0
    for m in (1, 15, 17, 70):
        for n in (1, 7, 9, 25):
            for k in (1, 7, 9, 500):
                a = port.generate(da, 31, 2 * i, m, k)
                b = port.generate(db, 31, 2 * i + 1, k, n)
                i += 1
                assert (gpu_gemm(lb, mode, a, b, kernel) == port.gemm(mode, a, b)).all(), (m, n, k)


@pytest.mark.parametrize("kernel", KERNELS)
def test_gemm_acceptance_grid(lb, port, kernel):  # acceptance.cpp:75-105 (criterion 3)
    rng = np.random.default_rng(1003)
    for mode in (BNN, TNN, TBN):
        da, db = mode_dists(mode)
        for s, (m, n, k) in enumerate(sweep_shapes()):
            a = port.generate(da, 1003 + mode, 2 * s, m, k)
            b = port.generate(db, 1003 + mode, 2 * s + 1, k, n)
            assert (gpu_gemm(lb, mode, a, b, kernel).astype(np.int32) == port.reference_gemm_int(a, b)).all()
    for rep in range(50):
        mode = rep % 3
        da, db = mode_dists(mode)
        m, n, k = int(rng.integers(1, 101)), int(rng.integers(1, 61)), int(rng.integers(1, 601))
        a = port.generate(da, 1103, 2 * rep, m, k)
        b = port.generate(db, 1103, 2 * rep + 1, k, n)
        assert (gpu_gemm(lb, mode, a, b, kernel).astype(np.int32) == port.reference_gemm_int(a, b)).all()


@pytest.mark.parametrize("kernel", KERNELS)
def test_gemm_multi_tile_shapes(lb, port, kernel):
    # several M/N tiles, ragged edges, deep K, persistent-loop wraparound
    for mode, (m, n, k) in [(TNN, (300, 520, 1000)), (BNN, (1000, 300, 2048)), (TBN, (129, 257, 4100)),
                            (TNN, (2000, 64, 256)), (BNN, (64, 1000, 96))]:
        da, db = mode_dists(mode)
        a = port.generate(da, 77, 0, m, k)
        b = port.generate(db, 77, 1, k, n)
        assert (gpu_gemm(lb, mode, a, b, kernel) == port.gemm(mode, a, b)).all(), (mode, m, n, k)


@pytest.mark.parametrize("kernel", KERNELS)
def test_depth_extremes(lb, kernel):  # test_gemm.cpp:88-100
    a = np.ones((16, 32767), np.int8)
    b = np.ones((32767, 8), np.int8)
    assert (gpu_gemm(lb, BNN, a, b, kernel) == 32767).all()
    a = -np.ones((20, 32767), np.int8)
    assert (gpu_gemm(lb, TBN, a, b, kernel) == -32767).all()
    with pytest.raises(lb.DepthOverflow) as e:
        gpu_gemm(lb, BNN, np.ones((16, 32768), np.int8), np.ones((32768, 8), np.int8), kernel)
    assert (e.value.k, e.value.k_max) == (32768, 32767)


def test_kblk_invariance_and_errors(lb, port):  # test_gemm.cpp:74-86, 102-110
    a = port.generate(0, 33, 0, 33, 700)
    b = port.generate(0, 33, 1, 700, 19)
    r = [gpu_gemm(lb, TNN, a, b, 0, kb) for kb in (64, 512, 4096)]
    assert (r[0] == r[1]).all() and (r[1] == r[2]).all()
    with pytest.raises(lb.Error):
        gpu_gemm(lb, TNN, a, b, 0, 12)
    ap = lb.encode_ternary(dev(port.generate(0, 34, 0, 16, 16)))
    bb = lb.pack_b(lb.encode_binary(dev(port.generate(1, 34, 1, 16, 8))))
    bt = lb.pack_b(lb.encode_ternary(dev(port.generate(0, 34, 2, 16, 8))))
    for mode, pb in [(TNN, bb), (TBN, bt), (BNN, bb)]:
        with pytest.raises(lb.ModeMismatch):
            lb.gemm_lowbit(mode, ap, pb, (16, 8, 16))
    with pytest.raises(lb.OutOfBounds):
        lb.gemm_lowbit(TNN, ap, bt, (16, 8, 15))


def test_host_dropin_entry(lb, port, ref):
    # one whole reference-API call with host buffers (what the C++ shim uses)
    for mode, (m, n, k) in [(TNN, (360, 96, 256)), (BNN, (100, 33, 77)), (TBN, (257, 130, 1000))]:
        da, db = mode_dists(mode)
        a = port.generate(da, 55, 0, m, k)
        b = port.generate(db, 55, 1, k, n)
        a0, a1 = port.encode(a, a_mode_ternary(mode))
        b0, b1 = port.encode(b, b_mode_ternary(mode))
        panels = port.pack_b(b0, b1, k, n)
        got = lb.gemm_lowbit_host(mode, a0, a1, m, k, panels, b1 is not None, n, k, (m, n, k))
        assert (got == ref.gemm(mode, a, b)).all()


def test_host_dropin_threads(lb, port, ref):
    # host-buffer calls from several host threads at once: each thread owns its
    # scratch, streams and events (thread_local per device in capi.cu)
    from concurrent.futures import ThreadPoolExecutor
    cases = []
    for i, (mode, (m, n, k)) in enumerate([(TNN, (300, 96, 512)), (TBN, (129, 64, 300)),
                                           (BNN, (64, 200, 1024)), (TNN, (1000, 32, 128))]):
        da, db = mode_dists(mode)
        a = port.generate(da, 90 + i, 0, m, k)
        b = port.generate(db, 90 + i, 1, k, n)
        a0, a1 = port.encode(a, a_mode_ternary(mode))
        b0, b1 = port.encode(b, b_mode_ternary(mode))
        cases.append((mode, m, n, k, a0, a1, port.pack_b(b0, b1, k, n), b1 is not None, ref.gemm(mode, a, b)))

    def run(case):
        mode, m, n, k, a0, a1, panels, bt, want = case
        for _ in range(5):
            got = lb.gemm_lowbit_host(mode, a0, a1, m, k, panels, bt, n, k, (m, n, k))
            if not (got == want).all():
                return False
        return True

    with ThreadPoolExecutor(len(cases)) as ex:
        assert all(ex.map(run, cases))


# ------------------------------------------------------------------ BASELINE configs
def _device_inputs(lb, mode, seed, m, n, k, dist_a, dist_b):
    a = lb.generate(dist_a, seed, 0, m, k)
    b = lb.generate(dist_b, seed, 1, k, n)
    ap = lb.encode_ternary(a) if a_mode_ternary(mode) else lb.encode_binary(a)
    bp = lb.encode_ternary(b) if b_mode_ternary(mode) else lb.encode_binary(b)
    return a, b, ap, lb.prepare_weights(lb.pack_b(bp))


@pytest.mark.parametrize("kernel", KERNELS)
def test_config1_golden(lb, golden, golden_configs, kernel):
    _, _, ap, w = _device_inputs(lb, TNN, 43, 360, 96, 256, 0, 0)
    c = host(lb.gemm_lowbit(TNN, ap, w, (360, 96, 256), kernel=kernel))
    assert (c == golden["config1"]).all() and sha(c) == golden_configs["c1"]["sha256"]


@pytest.mark.parametrize("kernel", KERNELS)
def test_config2_sweep_golden(lb, golden_configs, kernel):
    for s, (m, n, k) in enumerate(sweep_shapes()):
        a = lb.generate(2, 44, 2 * s, m, k)
        b = lb.generate(1, 44, 2 * s + 1, k, n)
        w = lb.prepare_weights(lb.pack_b(lb.encode_binary(b)))
        c = host(lb.gemm_lowbit(TBN, lb.encode_ternary(a), w, (m, n, k), kernel=kernel))
        assert sha(c) == golden_configs["c2"]["sha256"][s], (m, n, k)


def _row_col_sum_check(a, b, c):
    """Size-independent identities: C.1 = A.(B.1) and 1^T C = (1^T A).B (exact, int64)."""
    b_rows = b.to(torch.float64).sum(dim=1)                   # B.1   [k]
    a_cols = torch.zeros(a.shape[1], dtype=torch.float64, device=a.device)
    c_cols = torch.zeros(c.shape[1], dtype=torch.int64, device=c.device)
    step = 65536
    for r0 in range(0, a.shape[0], step):
        af = a[r0:r0 + step].to(torch.float64)
        a_cols += af.sum(dim=0)
        want_rows = (af @ b_rows).round().to(torch.int64)
        c64 = c[r0:r0 + step].to(torch.int64)
        assert torch.equal(c64.sum(dim=1), want_rows), r0
        c_cols += c64.sum(dim=0)
    want_cols = (a_cols @ b.to(torch.float64)).round().to(torch.int64)
    assert torch.equal(c_cols, want_cols)


@pytest.mark.parametrize("kernel", [2, 3, 4])
def test_config3_full(lb, port, golden_configs, kernel):
    m = n = 8192
    k = 4096
    a, b, ap, w = _device_inputs(lb, BNN, 45, m, n, k, 1, 1)
    c = lb.gemm_lowbit(BNN, ap, w, (m, n, k), kernel=kernel)
    torch.cuda.synchronize()
    _row_col_sum_check(a, b, c)
    rows = [0, 1, 4095, 8191]
    want = port.gemm(BNN, port.generate(1, 45, 0, 1, k, row0=0), port.generate(1, 45, 1, k, n))
    assert (host(c[0:1]) == want).all()
    if "c3" in golden_configs:
        assert sha(host(c)) == golden_configs["c3"]["sha256"]
    del rows


def test_config3_bitserial_sampled(lb, port):
    # the bit-serial kernel at full c3 size: compare sampled row blocks with the oracle
    m = n = 8192
    k = 4096
    _, _, ap, w = _device_inputs(lb, BNN, 45, m, n, k, 1, 1)
    c = lb.gemm_lowbit(BNN, ap, w, (m, n, k), kernel=1)
    b = port.generate(1, 45, 1, k, n)
    for r0 in (0, 4000, 8190):
        want = port.gemm(BNN, port.generate(1, 45, 0, 2, k, row0=r0), b)
        assert (host(c[r0:r0 + 2]) == want).all()


@pytest.mark.parametrize("kernel", [2, 4])
def test_config5_full(lb, port, golden_configs, kernel):
    m, n, k = 1048576, 1024, 2048
    a, b, ap, w = _device_inputs(lb, TNN, 47, m, n, k, 0, 0)
    c = lb.gemm_lowbit(TNN, ap, w, (m, n, k), kernel=kernel)
    torch.cuda.synchronize()
    _row_col_sum_check(a, b, c)
    bb = port.generate(0, 47, 1, k, n)
    for r0 in (0, 524287, m - 3):
        want = port.gemm(TNN, port.generate(0, 47, 0, 3, k, row0=r0), bb)
        assert (host(c[r0:r0 + 3]) == want).all()
    if "c5" in golden_configs:
        assert sha(host(c)) == golden_configs["c5"]["sha256"]


# ------------------------------------------------------------------ grouped launch (§8f-3)
def test_grouped_config2_sweep(lb, golden_configs):
    problems = []
    for s, (m, n, k) in enumerate(sweep_shapes()):
        a = lb.generate(2, 44, 2 * s, m, k)
        b = lb.generate(1, 44, 2 * s + 1, k, n)
        w = lb.prepare_weights(lb.pack_b(lb.encode_binary(b)))
        problems.append((lb.encode_ternary(a), w, torch.empty((m, n), dtype=torch.int16, device="cuda")))
    outs = lb.gemm_grouped(TBN, problems)
    for s, c in enumerate(outs):
        assert sha(host(c)) == golden_configs["c2"]["sha256"][s], s


@pytest.mark.parametrize("mode", [BNN, TNN, TBN])
def test_grouped_mixed_shapes(lb, port, mode):
    da, db = mode_dists(mode)
    rng = np.random.default_rng(7 + mode)
    problems, wants = [], []
    for i in range(150):  # > 128: exercises the split into several launches
        m, n, k = int(rng.integers(1, 200)), int(rng.integers(1, 100)), int(rng.integers(1, 700))
        a = port.generate(da, 600 + mode, 2 * i, m, k)
        b = port.generate(db, 600 + mode, 2 * i + 1, k, n)
        ap = lb.encode_ternary(dev(a)) if a_mode_ternary(mode) else lb.encode_binary(dev(a))
        bp = lb.encode_ternary(dev(b)) if b_mode_ternary(mode) else lb.encode_binary(dev(b))
        problems.append((ap, lb.prepare_weights(lb.pack_b(bp)), torch.empty((m, n), dtype=torch.int16,
                                                                            device="cuda")))
        wants.append(port.gemm(mode, a, b))
    outs = lb.gemm_grouped(mode, problems)
    for got, want in zip(outs, wants):
        assert (host(got) == want).all()


# ------------------------------------------------------------------ B200 lane-interleaved A layout
def to_lanes(planes: np.ndarray) -> np.ndarray:
    """Reference-layout plane rows -> LOWBIT_LAYOUT_LANES (element j of each
    32-bit word moves from bit j to bit 8*(j%4) + j//4)."""
    rows, sb = planes.shape
    padded = np.zeros((rows, (sb + 3) // 4 * 4), np.uint8)
    padded[:, :sb] = planes
    words = padded.view("<u4").astype(np.uint64)
    out = np.zeros_like(words)
    for j in range(32):
        out |= ((words >> j) & 1) << (8 * (j % 4) + j // 4)
    return out.astype("<u4").view(np.uint8)[:, :sb]


@pytest.mark.parametrize("shape", [(1, 8), (7, 13), (33, 129), (257, 1000), (5, 2048)])
def test_encode_lanes_layout(lb, port, shape):
    rows, cols = shape
    for tern in (False, True):
        v = port.generate(0 if tern else 1, 21, int(tern), rows, cols)
        w0, w1 = port.encode(v, tern)
        got = (lb.encode_ternary(dev(v), layout=1) if tern else lb.encode_binary(dev(v), layout=1))
        sb = (cols + 7) // 8
        assert (host(got.plane0)[:, :sb] == to_lanes(w0)).all()
        if tern:
            assert (host(got.plane1)[:, :sb] == to_lanes(w1)).all()
    with pytest.raises(lb.ZeroInBinaryInput):
        lb.encode_binary(torch.zeros((2, 40), dtype=torch.int8, device="cuda"), layout=1)


@pytest.mark.parametrize("kernel", [2, 3])
@pytest.mark.parametrize("mode", [BNN, TNN, TBN])
def test_gemm_lanes_layout(lb, port, mode, kernel):
    da, db = mode_dists(mode)
    for i, (m, n, k) in enumerate([(1, 1, 1), (17, 9, 500), (70, 25, 7), (360, 96, 256), (300, 520, 1000),
                                   (129, 257, 4100), (1000, 300, 2048)]):
        a = port.generate(da, 88 + i, 0, m, k)
        b = port.generate(db, 88 + i, 1, k, n)
        ap = lb.encode_ternary(dev(a), layout=1) if a_mode_ternary(mode) else lb.encode_binary(dev(a), layout=1)
        bp = lb.encode_ternary(dev(b)) if b_mode_ternary(mode) else lb.encode_binary(dev(b))
        got = host(lb.gemm_lowbit(mode, ap, lb.prepare_weights(lb.pack_b(bp)), (m, n, k), kernel=kernel))
        assert (got == port.gemm(mode, a, b)).all(), (mode, m, n, k)


def test_lanes_layout_rejected_by_bitserial(lb, port):
    ap = lb.encode_ternary(dev(port.generate(0, 3, 0, 16, 64)), layout=1)
    w = lb.prepare_weights(lb.pack_b(lb.encode_ternary(dev(port.generate(0, 3, 1, 64, 8)))))
    with pytest.raises(lb.InvalidArgument):
        lb.gemm_lowbit(TNN, ap, w, (16, 8, 64), kernel=1)


def test_config5_lanes_hash(lb, golden_configs):
    m, n, k = 1048576, 1024, 2048
    a = lb.generate(0, 47, 0, m, k)
    ap = lb.encode_ternary(a, layout=1)
    del a
    w = lb.prepare_weights(lb.pack_b(lb.encode_ternary(lb.generate(0, 47, 1, k, n))))
    c = lb.gemm_lowbit(TNN, ap, w, (m, n, k), kernel=2)
    assert sha(host(c)) == golden_configs["c5"]["sha256"]


def test_config3_lanes_hash(lb, golden_configs):
    m = n = 8192
    k = 4096
    ap = lb.encode_binary(lb.generate(1, 45, 0, m, k), layout=1)
    w = lb.prepare_weights(lb.pack_b(lb.encode_binary(lb.generate(1, 45, 1, k, n))))
    c = lb.gemm_lowbit(BNN, ap, w, (m, n, k), kernel=2)
    assert sha(host(c)) == golden_configs["c3"]["sha256"]
