"""CPU: pin the oracle (oracle/lowbit_oracle.c) before trusting it.

1. The known-answer vectors of the reference's own unit tests
   (proj/tests/test_core.cpp, test_pack.cpp, test_kernels.cpp, test_gemm.cpp,
   test_conv.cpp), restated.
2. Golden fixtures produced by the reference library itself
   (tests/golden/make_golden.py -> golden_small.npz).
3. When oracle/_ref is present: randomized port-vs-reference equivalence.
"""
import numpy as np
import pytest

from oracle.oracle import BNN, TNN, TBN, OracleError, a_mode_ternary, b_mode_ternary
from tests.golden.make_golden import SMALL_GEMM, mode_dists, sweep_shapes, sha


def row(vals):
    return np.array([vals], np.int8)


# ---------------------------------------------------------------- core KATs
def test_encode_binary_golden_byte(port):  # test_core.cpp:25-29
    p0, _ = port.encode(row([1, -1, 1, 1, -1, -1, -1, 1]), False)
    assert p0.shape == (1, 1) and p0[0, 0] == 0b01110010


def test_encode_binary_all_plus_zero_plane(port):  # test_core.cpp:31-36
    p0, _ = port.encode(np.ones((16, 16), np.int8), False)
    assert not p0.any()


def test_encode_binary_rejects_zero(port):  # test_core.cpp:38-40
    with pytest.raises(OracleError) as e:
        port.encode(row([1, 0, -1]), False)
    assert e.value.name == "ZeroInBinaryInput"


def test_decode_binary_goldens(port):  # test_core.cpp:42-55
    assert (port.decode(np.array([[0x00]], np.uint8), None, 1, 8) == 1).all()
    d = port.decode(np.array([[0x01]], np.uint8), None, 1, 8)
    assert d[0, 0] == -1 and (d[0, 1:] == 1).all()


def test_binary_roundtrip_and_padding(port):  # test_core.cpp:57-66
    v = port.generate(1, 7, 0, 7, 13)
    p0, _ = port.encode(v, False)
    assert (port.decode(p0, None, 7, 13) == v).all()
    assert not (p0[:, 1] & ~np.uint8(0x1F)).any()


def test_encode_ternary_goldens(port):  # test_core.cpp:68-77
    p, m = port.encode(row([1, 0, -1]), True)
    assert p[0, 0] == 0x01 and m[0, 0] == 0x04
    p, m = port.encode(np.zeros((4, 4), np.int8), True)
    assert not p.any() and not m.any()


def test_ternary_roundtrip_disjoint(port):  # test_core.cpp:79-86
    v = port.generate(0, 9, 0, 9, 17)
    p, m = port.encode(v, True)
    assert not (p & m).any()
    assert (port.decode(p, m, 9, 17) == v).all()


# ---------------------------------------------------------------- pack KATs
def test_pack_a_binary_goldens(port):  # test_pack.cpp:18-26
    p0, _ = port.encode(np.ones((16, 8), np.int8), False)
    buf, _ = port.pack_block(0, p0, None, 16, 8, 0, 0, 8)
    assert not buf.any()
    v = np.ones((16, 8), np.int8)
    v[3, :] = -1
    p0, _ = port.encode(v, False)
    buf, _ = port.pack_block(0, p0, None, 16, 8, 0, 0, 8)
    assert [int(x) for x in buf[:16]] == [0xFF if i == 3 else 0 for i in range(16)]


def test_pack_b_binary_golden(port):  # test_pack.cpp:28-35
    v = np.ones((16, 8), np.int8)
    v[:, 5] = -1
    p0, _ = port.encode(v, False)
    buf, _ = port.pack_block(1, p0, None, 16, 8, 0, 0, 16)
    assert len(buf) == 16
    for d in range(2):
        assert [int(x) for x in buf[d * 8:d * 8 + 8]] == [0xFF if j == 5 else 0 for j in range(8)]


def test_pack_a_ternary_golden(port):  # test_pack.cpp:37-43
    v = np.zeros((16, 8), np.int8)
    v[0, 0] = 1
    p, m = port.encode(v, True)
    buf, _ = port.pack_block(2, p, m, 16, 8, 0, 0, 8)
    assert buf[0] == 1 and not buf[1:].any()


def test_pack_b_ternary_golden(port):  # test_pack.cpp:45-52
    v = np.zeros((8, 8), np.int8)
    v[0, 2] = -1
    p, m = port.encode(v, True)
    buf, _ = port.pack_block(3, p, m, 8, 8, 0, 0, 8)
    assert buf[5] == 1 and buf.sum() == 1


@pytest.mark.parametrize("k_eff", [8, 16, 64, 128, 504])
def test_pack_buffer_lengths(port, k_eff):  # test_pack.cpp:54-68
    db = (k_eff + 7) // 8
    for mode, rows, cols, group, tern in [(0, 16, k_eff, 16, False), (1, k_eff, 8, 8, False),
                                          (2, 16, k_eff, 32, True), (3, k_eff, 8, 16, True)]:
        v = port.generate(0 if tern else 1, k_eff, mode, rows, cols)
        p, m = port.encode(v, tern)
        buf, _ = port.pack_block(mode, p, m, rows, cols, 0, 0, k_eff)
        assert len(buf) == group * db


def test_pack_bounds(port):  # test_pack.cpp:122-128
    p0, _ = port.encode(port.generate(1, 3, 0, 16, 32), False)
    for args in [(16, 0, 8), (0, 0, 33), (0, 4, 8)]:
        with pytest.raises(OracleError) as e:
            port.pack_block(0, p0, None, 16, 32, *args)
        assert e.value.name == "OutOfBounds"


def test_pack_matches_reference(port, ref):
    for case, (rows, cols) in enumerate([(16, 40), (10, 16), (33, 129), (8, 8)]):
        for mode in range(4):
            tern = mode >= 2
            v = port.generate(0 if tern else 1, 77 + case, mode, rows, cols)
            p, m = port.encode(v, tern)
            lim = cols if mode in (0, 2) else rows
            for depth_start, k_eff in [(0, lim), (0, min(lim, 24)), (8, min(lim - 8, 16))]:
                if k_eff < 1:
                    continue
                a, la = port.pack_block(mode, p, m, rows, cols, 0, depth_start, k_eff)
                b, lb = ref.pack_block(mode, p, m, rows, cols, 0, depth_start, k_eff)
                assert la == lb and (a == b).all()


# ---------------------------------------------------------------- kernel/gemm KATs
def test_tile_goldens(port):  # test_kernels.cpp:65-126 via 16x8 gemm
    assert (port.gemm(BNN, np.ones((16, 8), np.int8), np.ones((8, 8), np.int8)) == 8).all()
    a2 = np.ones((16, 16), np.int8)
    np.fill_diagonal(a2, -1)
    assert (port.gemm(BNN, a2, np.ones((16, 8), np.int8)) == 14).all()
    a1 = np.zeros((16, 16), np.int8)
    a1[2, 5] = 1
    b1 = np.zeros((16, 8), np.int8)
    b1[5, 3] = -1
    c = port.gemm(TNN, a1, b1)
    assert c[2, 3] == -1 and np.count_nonzero(c) == 1
    c = port.gemm(TBN, np.ones((16, 8), np.int8), -np.ones((8, 8), np.int8))
    assert (c == -8).all()
    assert (port.gemm(TBN, np.zeros((16, 8), np.int8), -np.ones((8, 8), np.int8)) == 0).all()


def test_dot_binary(port):  # test_kernels.cpp:46-63
    z = np.zeros(1, np.uint8)
    assert port.dot_binary(z, z, 8) == 8
    assert port.dot_binary(z, np.array([0xFF], np.uint8), 8) == -8
    with pytest.raises(OracleError):
        port.dot_binary(np.zeros(63, np.uint8), np.zeros(63, np.uint8), 32768)


def test_gemm_all_plus(port):  # test_gemm.cpp:33-38
    assert (port.gemm(BNN, np.ones((16, 128), np.int8), np.ones((128, 8), np.int8)) == 128).all()


def test_gemm_depth_contract(port):  # test_gemm.cpp:88-100
    a = np.ones((16, 32768), np.int8)
    b = np.ones((32768, 8), np.int8)
    with pytest.raises(OracleError) as e:
        port.gemm(BNN, a, b)
    assert e.value.name == "DepthOverflow"
    assert (port.gemm(BNN, a[:, :32767], b[:32767]) == 32767).all()


def test_gemm_mode_mismatch(port):  # test_gemm.cpp:102-110
    a0, a1 = port.encode(port.generate(0, 34, 0, 16, 16), True)
    b0, _ = port.encode(port.generate(1, 34, 1, 16, 8), False)
    t0, t1 = port.encode(port.generate(0, 34, 2, 16, 8), True)
    pbb = port.pack_b(b0, None, 16, 8)
    pbt = port.pack_b(t0, t1, 16, 8)
    for mode, pb, tern in [(TNN, pbb, False), (TBN, pbt, True), (BNN, pbb, False)]:
        with pytest.raises(OracleError) as e:
            port.gemm_lowbit(mode, a0, a1, 16, 16, pb, tern, 8, 16, 16, 8, 16)
        assert e.value.name == "ModeMismatch"


def test_gemm_bad_kblk(port):  # gemm.cpp:9-12
    a0, _ = port.encode(np.ones((16, 16), np.int8), False)
    b0, _ = port.encode(np.ones((16, 8), np.int8), False)
    pb = port.pack_b(b0, None, 16, 8)
    for kb in (0, 7, 12):
        with pytest.raises(OracleError) as e:
            port.gemm_lowbit(BNN, a0, None, 16, 16, pb, False, 8, 16, 16, 8, 16, kb)
        assert e.value.name == "Error"


def test_k_max_table(port):  # test_gemm.cpp:203-210
    L = port.lib
    assert L.orc_k_max(8, 32) == 66051 and L.orc_k_max(4, 16) == 291 and L.orc_k_max_sign(16) == 32767
    assert L.orc_c_in_max(32767, 3, 3) == 3640 and L.orc_c_in_max(291, 3, 3) == 32
    assert L.orc_c_in_max(32767, 1, 1) == 32767


def test_reference_gemm_int_kats(port):  # test_gemm.cpp:212-230
    assert port.reference_gemm_int(row([-1]), row([-1]))[0, 0] == 1
    ra = port.generate(0, 38, 0, 13, 29)
    rb = port.generate(0, 38, 1, 29, 11)
    want = ra.astype(np.int32) @ rb.astype(np.int32)
    assert (port.reference_gemm_int(ra, rb) == want).all()


# ---------------------------------------------------------------- vs reference goldens
def test_encode_pack_vs_golden(port, golden):
    for case, (rows, cols) in enumerate([(1, 8), (7, 13), (9, 17), (3, 64), (5, 100), (16, 504), (33, 129)]):
        for tern in (0, 1):
            v = port.generate(0 if tern else 1, 1000 + case, tern, rows, cols)
            p0, p1 = port.encode(v, bool(tern))
            assert (p0 == golden[f"enc_{case}_{tern}_p0"]).all()
            if tern:
                assert (p1 == golden[f"enc_{case}_{tern}_p1"]).all()
            assert (port.pack_b(p0, p1, rows, cols) == golden[f"packb_{case}_{tern}"]).all()


@pytest.mark.parametrize("mode", [BNN, TNN, TBN])
def test_gemm_vs_golden(port, golden, mode):
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
            assert (port.gemm(mode, a, b, k_blk) == golden[f"gemm_{mode}_{case}_{k_blk}"]).all()


def test_conv_vs_golden(port, golden):
    cases = [(5, 5, 2, 3, 3, 2, 1, 3), (8, 8, 5, 3, 3, 1, 1, 4), (9, 9, 32, 1, 1, 2, 0, 4),
             (3, 3, 2, 3, 3, 1, 1, 2), (6, 7, 3, 3, 3, 1, 0, 5)]
    for mode in (BNN, TNN, TBN):
        da, db = mode_dists(mode)
        for case, (h, w, ch, kh, kw, s, p, cout) in enumerate(cases):
            fm = port.generate(da, 3000 + 100 * mode + case, 0, h * w, ch).reshape(h, w, ch)
            wt = port.generate(db, 3000 + 100 * mode + case, 1, kh * kw * ch, cout)
            for pv in ((1, -1) if mode == BNN else (1,)):
                got = port.conv2d_lowbit(mode, fm, mode == BNN, wt, mode != TNN, kh, kw, s, p, pv)
                assert (got == golden[f"conv_{mode}_{case}_{pv}"]).all()
                assert (port.direct_conv(fm, mode == BNN, wt, kh, kw, s, p, pv) == got).all()


def test_config1_and_sweep_vs_golden(port, golden, golden_configs):
    a = port.generate(0, 43, 0, 360, 256)
    b = port.generate(0, 43, 1, 256, 96)
    c1 = port.gemm(TNN, a, b)
    assert (c1 == golden["config1"]).all() and sha(c1) == golden_configs["c1"]["sha256"]
    for s, (m, n, k) in enumerate(sweep_shapes()):
        a = port.generate(2, 44, 2 * s, m, k)
        b = port.generate(1, 44, 2 * s + 1, k, n)
        assert sha(port.gemm(TBN, a, b)) == golden_configs["c2"]["sha256"][s]


def test_port_vs_reference_random(port, ref):
    rng = np.random.default_rng(5)
    for rep in range(40):
        mode = rep % 3
        m, n, k = int(rng.integers(1, 100)), int(rng.integers(1, 60)), int(rng.integers(1, 600))
        da, db = mode_dists(mode)
        a = port.generate(da, 9000 + rep, 0, m, k)
        b = port.generate(db, 9000 + rep, 1, k, n)
        kb = int(rng.choice([64, 512, 4096]))
        assert (port.gemm(mode, a, b, kb) == ref.gemm(mode, a, b, kb)).all()


def test_generator_distributions(port):
    v = port.generate(0, 1, 0, 300, 1000)
    frac = [(v == x).mean() for x in (-1, 0, 1)]
    assert all(abs(f - 1 / 3) < 0.01 for f in frac)
    v = port.generate(1, 1, 0, 300, 1000)
    assert set(np.unique(v)) == {-1, 1} and abs((v == 1).mean() - 0.5) < 0.01
    v = port.generate(2, 1, 0, 300, 1000)
    assert abs((v == 0).mean() - 0.5) < 0.01 and abs((v == 1).mean() - 0.25) < 0.01
    # shards regenerate exactly
    assert (port.generate(0, 1, 0, 100, 1000, row0=200) == port.generate(0, 1, 0, 300, 1000)[200:]).all()
