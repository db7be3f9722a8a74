"""GPU parity for K4 (fused im2col + encode) + GeMM = conv2d_lowbit
(conv.cpp:33-59), against the oracle's 6-loop direct convolution
(test_conv.cpp:22-47 restated in oracle/lowbit_oracle.c) and the reference's
own output hash for BASELINE.json config 4."""
import hashlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.oracle import BNN, TNN, TBN  # noqa: E402
from tests.golden.make_golden import mode_dists  # noqa: E402


@pytest.fixture(scope="module")
def lb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2205_09120_b200 as lb
    return lb


def weights_for(lb, wt, mode):
    t = torch.from_numpy(np.ascontiguousarray(wt)).cuda()
    bp = lb.encode_ternary(t) if mode == TNN else lb.encode_binary(t)
    return lb.prepare_weights(lb.pack_b(bp))


@pytest.mark.parametrize("kernel", [1, 2])
@pytest.mark.parametrize("mode", [BNN, TNN, TBN])
def test_conv_shape_suite(lb, port, mode, kernel):  # test_conv.cpp:118-138
    da, db = mode_dists(mode)
    i = 0
    for spatial in (1, 3, 5, 8, 9):
        for ch in (1, 5, 32, 64):
            for ksz in (1, 3):
                for stride in (1, 2):
                    for pad in (0, 1):
                        if spatial + 2 * pad < ksz:
                            continue
                        i += 1
                        batch = 2
                        fm = port.generate(da, 56, 3 * i, batch * spatial * spatial, ch).reshape(batch, spatial,
                                                                                                 spatial, ch)
                        wt = port.generate(db, 56, 3 * i + 1, ksz * ksz * ch, 4)
                        w = weights_for(lb, wt, mode)
                        got = lb.conv2d_lowbit(mode, torch.from_numpy(fm).cuda(), mode == BNN, w, ksz, ksz, stride,
                                               pad, kernel=kernel).cpu().numpy()
                        for img in range(batch):
                            want = port.direct_conv(fm[img], mode == BNN, wt, ksz, ksz, stride, pad)
                            assert (got[img].astype(np.int32) == want).all(), (mode, spatial, ch, ksz, stride, pad)


def test_conv_binary_pad_values(lb, port):  # test_conv.cpp:140-149
    fm = port.generate(1, 57, 0, 9, 2).reshape(3, 3, 2)
    wt = port.generate(1, 57, 1, 18, 2)
    w = weights_for(lb, wt, BNN)
    for pv in (1, -1):
        got = lb.conv2d_lowbit(BNN, torch.from_numpy(fm).cuda(), True, w, 3, 3, 1, 1, binary_pad_value=pv)
        assert (got[0].cpu().numpy().astype(np.int32) == port.direct_conv(fm, True, wt, 3, 3, 1, 1, pv)).all()
    with pytest.raises(lb.ZeroInBinaryInput):  # a 0 pad is a 0 in encode_binary(cols)
        lb.conv2d_lowbit(BNN, torch.from_numpy(fm).cuda(), True, w, 3, 3, 1, 1, binary_pad_value=0)
    # TBN pads a binary map with the pad value too, but encodes it ternary: 0 is allowed
    wtb = port.generate(1, 57, 2, 18, 2)
    got = lb.conv2d_lowbit(TBN, torch.from_numpy(fm).cuda(), True, weights_for(lb, wtb, TBN), 3, 3, 1, 1,
                           binary_pad_value=0)
    assert (got[0].cpu().numpy().astype(np.int32) == port.direct_conv(fm, True, wtb, 3, 3, 1, 1, 0)).all()


def test_conv_errors(lb, port):  # test_conv.cpp:151-164, conv.cpp:35-45
    w = weights_for(lb, np.zeros((9 * 3641, 1), np.int8), TNN)
    with pytest.raises(lb.ChannelOverflow) as e:
        lb.conv2d_lowbit(TNN, torch.zeros((1, 1, 3641), dtype=torch.int8, device="cuda"), False, w, 3, 3, 1, 1)
    assert (e.value.c_in, e.value.c_in_max) == (3641, 3640)
    w_ok = weights_for(lb, np.zeros((9 * 3640, 1), np.int8), TNN)
    out = lb.conv2d_lowbit(TNN, torch.zeros((3, 3, 3640), dtype=torch.int8, device="cuda"), False, w_ok, 3, 3, 1, 0)
    assert out.shape[1:3] == (1, 1) and int(out[0, 0, 0, 0]) == 0
    with pytest.raises(lb.EmptyOutput):
        lb.conv2d_lowbit(TNN, torch.zeros((2, 2, 1), dtype=torch.int8, device="cuda"), False,
                         weights_for(lb, np.zeros((9, 1), np.int8), TNN), 3, 3, 1, 0)
    with pytest.raises(lb.ModeMismatch):
        lb.conv2d_lowbit(BNN, torch.ones((3, 3, 1), dtype=torch.int8, device="cuda"), False,
                         weights_for(lb, np.ones((9, 1), np.int8), BNN), 3, 3, 1, 0)


def test_config4_full(lb, golden_configs):
    # 64 x 56 x 56 x 128 NHWC ternary, 3x3x128 -> 128, stride 1, pad 1 (M=200704, K=1152, N=128)
    fm = lb.generate(0, 46, 0, 64 * 56 * 56, 128).view(64, 56, 56, 128)
    wt = lb.generate(0, 46, 1, 9 * 128, 128)
    w = lb.prepare_weights(lb.pack_b(lb.encode_ternary(wt)))
    for kernel in (2, 4, 1):  # fp4 implicit GeMM (K6), int8 implicit GeMM, K4 + bit-serial
        out = lb.conv2d_lowbit(TNN, fm, False, w, 3, 3, 1, 1, kernel=kernel)
        h = hashlib.sha256(out.cpu().numpy().astype("<i2").tobytes()).hexdigest()
        assert h == golden_configs["c4"]["sha256"], kernel


@pytest.mark.parametrize("mode", [TNN, TBN])
def test_conv_implicit_gemm_im2col(lb, port, mode):
    """c % 128 == 0 and zero padding: the TMA-im2col implicit GeMMs (0/2: fp4 K6
    over the packed feature map, 4: int8 over the int8 map)."""
    da, db = mode_dists(mode)
    i = 0
    for (batch, h, w, ch, ksz, stride, pad) in [(2, 9, 9, 128, 3, 1, 1), (3, 8, 7, 128, 3, 2, 1), (1, 5, 5, 256, 3, 1, 0),
                                                (2, 6, 6, 128, 1, 1, 0), (1, 16, 16, 128, 3, 2, 0),
                                                (4, 11, 13, 128, 3, 1, 1)]:
        i += 1
        fm = port.generate(0, 70 + i, 0, batch * h * w, ch).reshape(batch, h, w, ch)  # ternary map -> pad 0
        wt = port.generate(db, 70 + i, 1, ksz * ksz * ch, 96)
        wts = weights_for(lb, wt, mode)
        for kernel in (0, 2, 4):
            got = lb.conv2d_lowbit(mode, torch.from_numpy(fm).cuda(), False, wts, ksz, ksz, stride, pad,
                                   kernel=kernel).cpu().numpy()
            for img in range(batch):
                want = port.direct_conv(fm[img], False, wt, ksz, ksz, stride, pad)
                assert (got[img].astype(np.int32) == want).all(), (mode, batch, h, w, ch, ksz, stride, pad, img)


def test_conv_fp4_binary_and_wide(lb, port):
    """K6 on a binary map without padding (BNN, ZeroInBinaryInput still raised),
    several n tiles (cout 400 -> 2 tiles of 208, the filter reloaded per tile)
    and 256 channels (2 channel blocks per tap)."""
    fm = port.generate(1, 90, 0, 2 * 7 * 7, 128).reshape(2, 7, 7, 128)
    wt = port.generate(1, 90, 1, 9 * 128, 64)
    got = lb.conv2d_lowbit(BNN, torch.from_numpy(fm).cuda(), True, weights_for(lb, wt, BNN), 3, 3, 1, 0).cpu().numpy()
    for img in range(2):
        assert (got[img].astype(np.int32) == port.direct_conv(fm[img], True, wt, 3, 3, 1, 0)).all()
    fm0 = fm.copy()
    fm0[1, 3, 3, 5] = 0
    with pytest.raises(lb.ZeroInBinaryInput):
        lb.conv2d_lowbit(BNN, torch.from_numpy(fm0).cuda(), True, weights_for(lb, wt, BNN), 3, 3, 1, 0)
    fm = port.generate(0, 91, 0, 3 * 10 * 9, 256).reshape(3, 10, 9, 256)
    wt = port.generate(0, 91, 1, 9 * 256, 400)
    got = lb.conv2d_lowbit(TNN, torch.from_numpy(fm).cuda(), False, weights_for(lb, wt, TNN), 3, 3, 1, 1).cpu().numpy()
    for img in range(3):
        assert (got[img].astype(np.int32) == port.direct_conv(fm[img], False, wt, 3, 3, 1, 1)).all()


@pytest.mark.parametrize("mode", [BNN, TNN, TBN])
def test_conv_fp4_tap_pairs(lb, port, mode):
    """K6's tap-pair form (c = 128, 3x3, stride 1, padding 1): the zero pixel
    leading each fm4 row, the out-of-bounds zero half of the (dummy, kx = 0)
    filter pair, narrow and wide rows, several images and n tiles."""
    da, db = mode_dists(mode)
    for i, (b, h, w, cout) in enumerate([(1, 1, 1, 8), (2, 3, 2, 16), (3, 5, 7, 40), (1, 9, 33, 300),
                                         (2, 14, 14, 496), (1, 2, 130, 24)]):
        fm = port.generate(da, 120 + i, 0, b * h * w, 128).reshape(b, h, w, 128)
        wt = port.generate(db, 120 + i, 1, 9 * 128, cout)
        got = lb.conv2d_lowbit(mode, torch.from_numpy(fm).cuda(), mode == BNN, weights_for(lb, wt, mode), 3, 3, 1,
                               1).cpu().numpy()
        for img in range(b):
            want = port.direct_conv(fm[img], mode == BNN, wt, 3, 3, 1, 1)
            assert (got[img].astype(np.int32) == want).all(), (mode, b, h, w, cout)


@pytest.mark.parametrize("mode", [BNN, TNN, TBN])
def test_gemm_from_int8(lb, port, mode):
    da, db = mode_dists(mode)
    for i, (m, n, k) in enumerate([(1, 1, 16), (17, 9, 512), (300, 520, 1008), (360, 96, 256), (129, 257, 4096),
                                   (1000, 300, 2048)]):
        a = port.generate(da, 90 + i, 0, m, k)
        b = port.generate(db, 90 + i, 1, k, n)
        bp = lb.encode_ternary(torch.from_numpy(b).cuda()) if mode == TNN else lb.encode_binary(torch.from_numpy(b).cuda())
        got = lb.gemm_lowbit_i8(mode, torch.from_numpy(a).cuda(), lb.prepare_weights(lb.pack_b(bp)), (m, n, k))
        assert (got.cpu().numpy() == port.gemm(mode, a, b)).all(), (mode, m, n, k)


@pytest.mark.parametrize("mode", [BNN, TNN, TBN])
def test_conv_halo_geometries(lb, port, mode):
    """K7 (fused halo conv) across its geometry: position pitch 32 / 64 / 128
    (4, 2 or 1 output rows per CTA tile, output heights not a multiple of
    them), two channel blocks, several n tiles, 1x1 / 3x3 / 5x5 filters, an
    odd number of CTA tiles (the idle CTA of the last pair), padding 0 / 1 /
    2 — each checked to run on K7 (lowbit_conv_select), then against the
    oracle's direct convolution (test_conv.cpp:22-47)."""
    da, db = mode_dists(mode)
    cases = [(2, 7, 14, 128, 64, 3, 1), (1, 3, 100, 128, 96, 3, 1), (2, 9, 9, 256, 64, 3, 1),
             (2, 14, 14, 128, 496, 3, 1), (3, 11, 13, 128, 64, 5, 2), (1, 5, 40, 128, 32, 1, 0),
             (1, 1, 1, 128, 8, 3, 1)]
    for i, (b, h, w, ch, cout, ksz, pad) in enumerate(cases):
        if mode == BNN:
            pad = 0  # a binary map pads with +-1: K4's path (test_conv_binary_pad_values)
            if h < ksz or w < ksz:
                continue
        assert lb.conv_select(mode, mode == BNN, b, h, w, ch, cout, ksz, ksz, 1, pad) == lb.CONV_PATH_HALO_FP4, \
            (b, h, w, ch, cout, ksz, pad)
        fm = port.generate(da, 150 + i, 0, b * h * w, ch).reshape(b, h, w, ch)
        wt = port.generate(db, 150 + i, 1, ksz * ksz * ch, cout)
        got = lb.conv2d_lowbit(mode, torch.from_numpy(fm).cuda(), mode == BNN, weights_for(lb, wt, mode), ksz, ksz, 1,
                               pad).cpu().numpy()
        for img in range(b):
            want = port.direct_conv(fm[img], mode == BNN, wt, ksz, ksz, 1, pad)
            assert (got[img].astype(np.int32) == want).all(), (mode, b, h, w, ch, cout, ksz, pad, img)


@pytest.mark.parametrize("mode", [BNN, TNN, TBN])
def test_conv_halo_column_blocks(lb, port, mode):
    """K7 with rows cut into column blocks of 32 positions (4 output rows per tile, 32 - (kw - 1)
    valid outputs per block): chosen when it takes no more tiles than whole rows (config 4's
    56 x 56 map) and for rows wider than 128 pixels.  Widths that end inside a block, heights not
    a multiple of 4, two channel blocks, several n tiles, 3x3 / 5x5 / 1x1 filters, padding 0-2;
    binary maps with every pad value (the converters write the pad codes at each block's edges)
    and a 0 in a binary map's last block (ZeroInBinaryInput)."""
    da, db = mode_dists(mode)
    cases = [(2, 56, 56, 128, 128, 3, 1), (1, 8, 130, 128, 24, 3, 1), (2, 12, 70, 256, 40, 3, 1),
             (1, 6, 200, 128, 64, 5, 2), (3, 9, 45, 128, 64, 3, 0), (1, 4, 300, 128, 496, 1, 0),
             (5, 7, 61, 128, 32, 3, 1)]
    for i, (b, h, w, ch, cout, ksz, pad) in enumerate(cases):
        binary = mode == BNN
        assert lb.conv_select(mode, binary, b, h, w, ch, cout, ksz, ksz, 1, pad) == lb.CONV_PATH_HALO_FP4, \
            (b, h, w, ch, cout, ksz, pad)
        fm = port.generate(da, 230 + i, 0, b * h * w, ch).reshape(b, h, w, ch)
        wt = port.generate(db, 230 + i, 1, ksz * ksz * ch, cout)
        wts = weights_for(lb, wt, mode)
        for pv in ((1, -1) if binary and pad else (1,)):
            got = lb.conv2d_lowbit(mode, torch.from_numpy(fm).cuda(), binary, wts, ksz, ksz, 1, pad,
                                   binary_pad_value=pv).cpu().numpy()
            for img in range(b):
                want = port.direct_conv(fm[img], binary, wt, ksz, ksz, 1, pad, pv)
                assert (got[img].astype(np.int32) == want).all(), (mode, pv, b, h, w, ch, cout, ksz, pad, img)
    if mode == BNN:
        fm = port.generate(1, 239, 0, 2 * 8 * 70, 128).reshape(2, 8, 70, 128)
        wt = port.generate(1, 239, 1, 9 * 128, 64)
        fm[1, 7, 69, 100] = 0  # the last pixel of the last block
        with pytest.raises(lb.ZeroInBinaryInput):
            lb.conv2d_lowbit(BNN, torch.from_numpy(fm).cuda(), True, weights_for(lb, wt, BNN), 3, 3, 1, 1)


@pytest.mark.parametrize("mode", [TNN, TBN])
def test_conv_halo_filter_sizes(lb, port, mode):
    """The halo convs across filter depths: K7T keeps the filter in tensor memory (cout <= 128, up to 14
    k-blocks of 128 channels that also fit its bounce buffers) and loads it in three barrier groups; K7
    takes the rest.  1x1 and 2x2 filters over 1-4 channel blocks (1, 2, 3, 4, 8, 12, 16 k-blocks), cout
    from 8 to 136, each against the oracle's direct convolution."""
    da, db = mode_dists(mode)
    cases = [(2, 8, 20, 128, 128, 1), (2, 8, 20, 256, 40, 1), (1, 9, 30, 384, 8, 1), (3, 6, 12, 128, 96, 2),
             (2, 7, 16, 256, 128, 2), (1, 6, 10, 384, 64, 2), (1, 5, 9, 512, 136, 2), (2, 5, 40, 512, 24, 1)]
    for i, (b, h, w, ch, cout, ksz) in enumerate(cases):
        # (three or four channel blocks can outgrow the halo kernels' shared memory: K6 takes those)
        path = lb.conv_select(mode, False, b, h, w, ch, cout, ksz, ksz, 1, 0)
        assert path == lb.CONV_PATH_HALO_FP4 or (ch >= 384 and path == lb.CONV_PATH_IMPLICIT_FP4), path
        fm = port.generate(da, 250 + i, 0, b * h * w, ch).reshape(b, h, w, ch)
        wt = port.generate(db, 250 + i, 1, ksz * ksz * ch, cout)
        got = lb.conv2d_lowbit(mode, torch.from_numpy(fm).cuda(), False, weights_for(lb, wt, mode), ksz, ksz, 1,
                               0).cpu().numpy()
        for img in range(b):
            want = port.direct_conv(fm[img], False, wt, ksz, ksz, 1, 0)
            assert (got[img].astype(np.int32) == want).all(), (mode, b, h, w, ch, cout, ksz, img)


@pytest.mark.parametrize("ch", [32, 40])
def test_conv_binary_zero_only_where_sampled(lb, port, ch):
    """ZeroInBinaryInput follows im2col's view (conv.cpp:9-31, core.cpp:23): a 0 in a
    column no window reads (w = 8, 3x3, stride 2, no padding: column 7) is not an
    error; a 0 in a sampled pixel is.  K4's encode-once ring (c % 32 == 0) and its
    per-word kernel (other c)."""
    fm = port.generate(1, 58, 0, 9 * 8, ch).reshape(1, 9, 8, ch)
    wt = port.generate(1, 58, 1, 9 * ch, 8)
    w = weights_for(lb, wt, BNN)
    fm[0, 4, 7, 3] = 0
    got = lb.conv2d_lowbit(BNN, torch.from_numpy(fm).cuda(), True, w, 3, 3, 2, 0, kernel=1).cpu().numpy()
    assert (got[0].astype(np.int32) == port.conv2d_lowbit(BNN, fm[0], True, wt, True, 3, 3, 2, 0)).all()
    fm[0, 4, 6, 3] = 0
    with pytest.raises(lb.ZeroInBinaryInput):
        lb.conv2d_lowbit(BNN, torch.from_numpy(fm).cuda(), True, w, 3, 3, 2, 0, kernel=1)


@pytest.mark.parametrize("mode", [TNN, TBN])
def test_conv_halo_strips(lb, port, mode):
    """K7 walks each CTA's contiguous strip of CTA tiles with a sliding window of
    input rows (each row converted once per strip; a new image restarts the
    window).  Batches large enough that strips span several tiles and cross
    image boundaries at different steps in the two CTAs of a pair, for every
    position pitch, two channel blocks and two n tiles."""
    da, db = mode_dists(mode)
    cases = [(64, 9, 9, 128, 64, 3, 1), (40, 20, 20, 256, 48, 3, 1), (24, 30, 56, 128, 128, 3, 1),
             (12, 33, 100, 128, 40, 3, 1), (48, 12, 12, 128, 256, 3, 0), (20, 15, 28, 128, 32, 5, 2)]
    for i, (b, h, w, ch, cout, ksz, pad) in enumerate(cases):
        assert lb.conv_select(mode, False, b, h, w, ch, cout, ksz, ksz, 1, pad) == lb.CONV_PATH_HALO_FP4
        fm = port.generate(da, 170 + i, 0, b * h * w, ch).reshape(b, h, w, ch)
        wt = port.generate(db, 170 + i, 1, ksz * ksz * ch, cout)
        got = lb.conv2d_lowbit(mode, torch.from_numpy(fm).cuda(), False, weights_for(lb, wt, mode), ksz, ksz, 1,
                               pad).cpu().numpy()
        for img in range(b):
            want = port.direct_conv(fm[img], False, wt, ksz, ksz, 1, pad)
            assert (got[img].astype(np.int32) == want).all(), (mode, b, h, w, ch, cout, ksz, pad, img)


@pytest.mark.parametrize("mode", [BNN, TBN, TNN])
def test_conv_halo_binary_padding(lb, port, mode):
    """K7 on binary maps padded with binary_pad_value (conv.cpp:13): the TMA fills
    out-of-image pixels with 0 and the converters overwrite them with the pad
    value's codes.  +1 and -1 for every mode, 0 for TBN / TNN (encoded ternary:
    allowed); a BNN map padded with 0 still raises ZeroInBinaryInput (K4)."""
    da, db = mode_dists(mode)
    cases = [(2, 9, 9, 128, 64, 3, 1), (3, 14, 20, 128, 40, 3, 1), (1, 7, 30, 128, 32, 5, 2), (2, 9, 9, 256, 64, 3, 1),
             (4, 6, 50, 128, 48, 3, 1)]
    for i, (b, h, w, ch, cout, ksz, pad) in enumerate(cases):
        assert lb.conv_select(mode, True, b, h, w, ch, cout, ksz, ksz, 1, pad) == lb.CONV_PATH_HALO_FP4
        fm = port.generate(1, 190 + i, 0, b * h * w, ch).reshape(b, h, w, ch)  # binary map
        wt = port.generate(db, 190 + i, 1, ksz * ksz * ch, cout)
        wts = weights_for(lb, wt, mode)
        for pv in ((1, -1) if mode == BNN else (1, -1, 0)):
            got = lb.conv2d_lowbit(mode, torch.from_numpy(fm).cuda(), True, wts, ksz, ksz, 1, pad,
                                   binary_pad_value=pv).cpu().numpy()
            for img in range(b):
                want = port.direct_conv(fm[img], True, wt, ksz, ksz, 1, pad, pv)
                assert (got[img].astype(np.int32) == want).all(), (mode, pv, b, h, w, ch, cout, ksz, pad, img)
    if mode == BNN:
        fm = port.generate(1, 199, 0, 2 * 9 * 9, 128).reshape(2, 9, 9, 128)
        wt = port.generate(1, 199, 1, 9 * 128, 64)
        with pytest.raises(lb.ZeroInBinaryInput):
            lb.conv2d_lowbit(BNN, torch.from_numpy(fm).cuda(), True, weights_for(lb, wt, BNN), 3, 3, 1, 1,
                             binary_pad_value=0)


@pytest.mark.parametrize("mode", [TNN, TBN])
def test_conv_halo_large_sums(lb, port, mode):
    # K7's products are +-0.5 and its f32 sums half-integers: drive them far from 0 (all-ones
    # maps, filters of one sign with odd-step tails) at the deepest filters K7 takes for this
    # map (3x3 over 256 channels: k = 2304; 5x5 over 128: k = 3200)
    for (c, ksz, pad) in ((256, 3, 1), (128, 5, 2)):
        k = ksz * ksz * c
        assert lb.conv_select(mode, False, 2, 6, 10, c, 48, ksz, ksz, 1, pad) == lb.CONV_PATH_HALO_FP4
        fm = np.ones((2, 6, 10, c), np.int8)
        fm[1, ::2] = -1
        fm[1, 1::3, 2::4] = 0
        cols = [np.ones(k, np.int8), -np.ones(k, np.int8)]
        x = np.ones(k, np.int8)
        x[k // 2:] = -1
        x[k // 2::7] = 1
        cols.append(x)
        x = np.ones(k, np.int8)
        x[1::3] = 0 if mode == TNN else 1
        x[5::64] = -1
        cols.append(x)
        rng = np.random.default_rng(c)
        while len(cols) < 48:
            p1 = rng.uniform(0.6, 1.0)
            x = np.where(rng.random(k) < p1, 1, -1).astype(np.int8)
            if mode == TNN:
                x[rng.random(k) < 0.1] = 0
            cols.append(x)
        wt = np.ascontiguousarray(np.stack(cols, axis=1))
        got = lb.conv2d_lowbit(mode, torch.from_numpy(fm).cuda(), False, weights_for(lb, wt, mode), ksz, ksz, 1,
                               pad).cpu().numpy()
        for img in range(2):
            want = port.direct_conv(fm[img], False, wt, ksz, ksz, 1, pad)
            assert (got[img].astype(np.int32) == want).all(), (mode, c, ksz)
        assert np.abs(got).max() > 1500


def test_conv_fuzz_against_reference_semantics(lb):
    """tools/fuzz_conv.py for 20 s: seeded random stride-1 convs (every mode, binary maps with every pad
    value, int8 values mapped by sign, widths past 128, 1-3 channel blocks, cout up to 312) through
    conv2d_lowbit against the oracle's im2col -> encode -> GeMM (conv.cpp:33-59)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SECONDS="20", SEED="7")
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "fuzz_conv.py")], env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0 and "fuzz OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
