"""int8 values outside {-1, 0, +1} take their SIGN on every int8-direct path.

The reference never multiplies raw int8 values: conv2d_lowbit runs im2col ->
encode_ternary / encode_binary -> gemm_lowbit (conv.cpp:33-59), and the
encoders set the plus bit for v > 0 and the minus bit for v < 0
(core.cpp:13-28, 40-58).  So a feature-map value of 2 or -127 acts as +1 or
-1.  The device paths that read int8 maps or matrices directly — K7 (fused
halo conv), K6 (packed-fp4 implicit GeMM), the int8 implicit GeMM, K4 (fused
im2col + encode) and lowbit_gemm_i8 — must do the same.  Each case below pins
the conv path it exercises with lowbit_conv_select, and compares with the C
oracle's conv2d_lowbit / gemm (and with oracle/_ref, the reference library
itself, when it was built).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle.oracle import BNN, TNN, TBN, a_mode_ternary, b_mode_ternary  # noqa: E402

WIDE_T = np.array([-128, -127, -5, -2, -1, 0, 0, 0, 1, 2, 3, 64, 127], np.int8)
WIDE_B = np.array([-128, -127, -5, -2, -1, 1, 2, 3, 64, 127], np.int8)


@pytest.fixture(scope="module")
def lb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2205_09120_b200 as lb
    return lb


def wide(rng, shape, binary):
    return rng.choice(WIDE_B if binary else WIDE_T, size=shape).astype(np.int8)


def weights_for(lb, wt, mode):
    t = torch.from_numpy(wt).cuda()
    bp = lb.encode_ternary(t) if b_mode_ternary(mode) else lb.encode_binary(t)
    return lb.prepare_weights(lb.pack_b(bp))


def _ref_conv(port, ref, mode, fm, fm_binary, wt, ksz, stride, pad):
    outs = []
    for img in range(fm.shape[0]):
        want = port.conv2d_lowbit(mode, fm[img], fm_binary, wt, not b_mode_ternary(mode), ksz, ksz, stride, pad)
        if ref is not None:
            r = ref.conv2d_lowbit(mode, fm[img], fm_binary, wt, not b_mode_ternary(mode), ksz, ksz, stride, pad)
            assert (r == want).all(), "oracle port and oracle/_ref disagree"
        outs.append(want)
    return np.stack(outs)


# (mode, fm_binary, batch, h, w, c, cout, k, stride, pad, kernel, expected path)
CASES = [
    (TNN, False, 2, 9, 9, 128, 64, 3, 1, 1, 0, "HALO_FP4"),
    (TBN, False, 1, 12, 20, 256, 40, 3, 1, 1, 0, "HALO_FP4"),
    (BNN, True, 2, 8, 8, 128, 32, 3, 1, 0, 0, "HALO_FP4"),
    (BNN, True, 2, 8, 8, 128, 32, 3, 1, 1, 0, "HALO_FP4"),   # padded with binary_pad_value = +1
    (TNN, False, 2, 9, 9, 128, 64, 3, 2, 1, 0, "IMPLICIT_FP4"),
    (BNN, True, 1, 9, 7, 128, 48, 3, 2, 0, 0, "IMPLICIT_FP4"),
    (TNN, False, 2, 9, 9, 128, 64, 3, 1, 1, 4, "IMPLICIT_I8"),
    (TBN, False, 1, 7, 11, 256, 24, 3, 2, 1, 4, "IMPLICIT_I8"),
    (TNN, False, 2, 9, 9, 128, 64, 3, 1, 1, 1, "ENCODE_GEMM"),
    (BNN, True, 1, 6, 6, 40, 16, 3, 1, 1, 0, "ENCODE_GEMM"),
    (TBN, False, 1, 6, 5, 72, 16, 3, 1, 1, 2, "ENCODE_GEMM"),
]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[-1]}-{i}" for i, c in enumerate(CASES)])
def test_conv_wide_values_by_sign(lb, port, request, case):
    seed = 600 + CASES.index(case)  # deterministic inputs (hash() of a tuple holding str varies per process)
    mode, fm_binary, batch, h, w, c, cout, ksz, stride, pad, kernel, path = case
    try:
        ref = request.getfixturevalue("ref")
    except pytest.skip.Exception:
        ref = None
    assert lb.conv_select(mode, fm_binary, batch, h, w, c, cout, ksz, ksz, stride, pad, kernel) == \
        getattr(lb, "CONV_PATH_" + path), case
    rng = np.random.default_rng(seed)
    fm = wide(rng, (batch, h, w, c), fm_binary)
    wt = wide(rng, (ksz * ksz * c, cout), not b_mode_ternary(mode))
    want = _ref_conv(port, ref, mode, fm, fm_binary, wt, ksz, stride, pad)
    got = lb.conv2d_lowbit(mode, torch.from_numpy(fm).cuda(), fm_binary, weights_for(lb, wt, mode), ksz, ksz, stride,
                           pad, kernel=kernel).cpu().numpy()
    assert (got.astype(np.int32) == want).all(), case
    # the same map with every value replaced by its sign gives the same result
    sgn = np.sign(fm).astype(np.int8)
    got2 = lb.conv2d_lowbit(mode, torch.from_numpy(sgn).cuda(), fm_binary, weights_for(lb, wt, mode), ksz, ksz,
                            stride, pad, kernel=kernel).cpu().numpy()
    assert (got2 == got).all()


@pytest.mark.parametrize("mode", [BNN, TNN, TBN])
def test_gemm_from_int8_wide_values_by_sign(lb, port, mode):
    rng = np.random.default_rng(500 + mode)
    for m, n, k in [(17, 9, 512), (300, 520, 1008), (129, 257, 4096), (1000, 96, 2048)]:
        a = wide(rng, (m, k), not a_mode_ternary(mode))
        b = wide(rng, (k, n), not b_mode_ternary(mode))
        want = port.gemm(mode, a, b)
        w = weights_for(lb, b, mode)
        at = torch.from_numpy(a).cuda()
        got = lb.gemm_lowbit_i8(mode, at, w, (m, n, k)).cpu().numpy()
        assert (got == want).all(), ("gemm_i8", mode, m, n, k)
        for layout in (0, 1, 2):  # K1 encode (by sign) on every plane layout, then the default kernel
            ap = lb.encode_ternary(at, layout=layout) if a_mode_ternary(mode) else lb.encode_binary(at, layout=layout)
            got = lb.gemm_lowbit(mode, ap, w, (m, n, k)).cpu().numpy()
            assert (got == want).all(), ("encode", layout, mode, m, n, k)
