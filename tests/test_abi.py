"""CPU: the C-ABI library loads, exports every symbol include/lowbit_cuda.h
declares, and reports the reference's error contract in the reference's order
(validation runs before any device work, so it is checkable without a GPU)."""
import ctypes as C
import re

import pytest

import paper_2205_09120_b200 as lb
from paper_2205_09120_b200 import _lib as L


def declared_symbols():
    text = open(L.HEADER_PATH).read()
    return sorted(set(re.findall(r"\b(lowbit_[a-z0-9_]+)\s*\(", text)))


def test_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L.lib, s), s
        assert s in L.SIGNATURES, f"{s} missing from the ctypes signature table"


def test_abi_version_and_strings():
    assert L.lib.lowbit_abi_version() == 1
    names = [L.lib.lowbit_status_string(i).decode() for i in range(12)]
    assert names[:9] == ["OK", "Error", "ZeroInBinaryInput", "InvalidCode", "OutOfBounds", "DepthOverflow",
                         "ModeMismatch", "ChannelOverflow", "EmptyOutput"]


def test_layout_helpers():
    assert [L.lib.lowbit_plane_pitch(c) for c in (1, 8, 9, 128, 129, 256, 2048)] == [16, 16, 16, 16, 32, 32, 256]
    # PackedB bytes: ceil(n/8) panels x group x ceil(k/8) (pack.cpp:36-44, gemm.cpp:59-77)
    assert L.lib.lowbit_packed_b_bytes(0, 8192, 4096) == 1024 * 8 * 512
    assert L.lib.lowbit_packed_b_bytes(1, 96, 256) == 12 * 16 * 32
    assert L.lib.lowbit_packed_b_bytes(1, 9, 17) == 2 * 16 * 3
    assert L.lib.lowbit_weights_bytes(1, 96, 256) > 0


def gemm_status(mode, a_ternary, b_ternary, a_rows, a_cols, b_n, b_k, m, n, k, k_blk=4096):
    a1 = C.c_void_p(16) if a_ternary else None  # never dereferenced: validation fails first
    return L.lib.lowbit_gemm(mode, C.c_void_p(16), a1, 16, a_rows, a_cols, None, b_ternary, b_n, b_k, m, n, k,
                             k_blk, None, n, 0, None)


def test_validation_order_matches_reference():
    # check_cfg first (gemm.cpp:9-12), even with a mode mismatch present
    assert gemm_status(L.TNN, 0, 0, 4, 4, 4, 4, 4, 4, 4, k_blk=7) == L.ERROR
    assert gemm_status(L.BNN, 0, 0, 4, 4, 4, 4, 4, 4, 4, k_blk=0) == L.ERROR
    # mode before dims (gemm.cpp:81-84, 94-99)
    assert gemm_status(L.TNN, 0, 1, 4, 4, 4, 4, 0, 0, 0) == L.MODE_MISMATCH   # binary A needs bnn
    assert gemm_status(L.BNN, 0, 1, 4, 4, 4, 4, 4, 4, 4) == L.MODE_MISMATCH   # bnn needs binary B
    assert gemm_status(L.BNN, 1, 0, 4, 4, 4, 4, 4, 4, 4) == L.MODE_MISMATCH   # bnn needs binary A
    assert gemm_status(L.TNN, 1, 0, 4, 4, 4, 4, 4, 4, 4) == L.MODE_MISMATCH   # tnn needs ternary B
    assert gemm_status(L.TBN, 1, 1, 4, 4, 4, 4, 4, 4, 4) == L.MODE_MISMATCH   # tbn needs binary B
    # check_dims (gemm.cpp:14-19)
    assert gemm_status(L.TNN, 1, 1, 4, 4, 4, 4, 0, 4, 4) == L.OUT_OF_BOUNDS
    assert gemm_status(L.TNN, 1, 1, 5, 4, 4, 4, 4, 4, 4) == L.OUT_OF_BOUNDS
    assert gemm_status(L.TNN, 1, 1, 4, 4, 3, 4, 4, 4, 4) == L.OUT_OF_BOUNDS
    assert gemm_status(L.BNN, 0, 0, 16, 32768, 8, 32768, 16, 8, 32768) == L.DEPTH_OVERFLOW
    v0, v1 = C.c_longlong(), C.c_longlong()
    L.lib.lowbit_last_error_values(C.byref(v0), C.byref(v1))
    assert (v0.value, v1.value) == (32768, 32767)
    assert L.lib.lowbit_last_error().decode() == "depth 32768 exceeds k_max 32767"  # errors.hpp:24-27
    # passes validation -> stops at the NULL device pointers, not in a kernel
    assert gemm_status(L.BNN, 0, 0, 16, 32767, 8, 32767, 16, 8, 32767) == L.INVALID_ARGUMENT


def test_exceptions_map_to_reference_types():
    with pytest.raises(lb.DepthOverflow) as e:
        L.check(gemm_status(L.BNN, 0, 0, 16, 40000, 8, 40000, 16, 8, 40000))
    assert e.value.k == 40000 and e.value.k_max == 32767
    with pytest.raises(lb.ModeMismatch):
        L.check(gemm_status(L.TNN, 1, 0, 4, 4, 4, 4, 4, 4, 4))
    assert issubclass(lb.ZeroInBinaryInput, lb.Error) and issubclass(lb.NoDevice, lb.Error)


def test_select_kernel_table():
    assert L.lib.lowbit_select_kernel(L.TNN, 1048576, 1024, 2048) == L.KERNEL_TENSOR
    assert L.lib.lowbit_select_kernel(L.BNN, 8192, 8192, 4096) == L.KERNEL_TENSOR
    # launch-bound shapes take the int8 tensor kernel (c1, the c2 sweep)
    assert L.lib.lowbit_select_kernel(L.TBN, 72, 24, 128) == L.KERNEL_TENSOR_I8   # one k-block, narrow output
    assert L.lib.lowbit_select_kernel(L.TBN, 72, 24, 512) == L.KERNEL_TENSOR      # narrow output: the fp4 kernel
    assert L.lib.lowbit_select_kernel(L.TNN, 360, 96, 256) == L.KERNEL_TENSOR_1CTA
    assert L.lib.lowbit_select_kernel(L.TNN, 4096, 128, 256) == L.KERNEL_TENSOR_I8
    assert L.lib.lowbit_select_kernel(L.TNN, 4096, 64, 512) == L.KERNEL_TENSOR


def test_conv_select_paths():
    """lowbit_conv_select: which conv kernel conv2d_lowbit takes (conv.cu)."""
    sel = lb.conv_select
    # config 4: 64 x 56 x 56 x 128, 3x3 -> 128, stride 1, pad 1, ternary map -> K7 fused halo
    assert sel(L.TNN, False, 64, 56, 56, 128, 128, 3, 3, 1, 1) == lb.CONV_PATH_HALO_FP4
    assert sel(L.TBN, False, 64, 56, 56, 128, 128, 3, 3, 1, 1) == lb.CONV_PATH_HALO_FP4
    # several n tiles (cout 496 -> 3 x 176), two channel blocks, 128-pixel rows, a 5x5 filter
    assert sel(L.TNN, False, 2, 14, 14, 128, 496, 3, 3, 1, 1) == lb.CONV_PATH_HALO_FP4
    assert sel(L.TNN, False, 2, 9, 9, 256, 64, 3, 3, 1, 1) == lb.CONV_PATH_HALO_FP4
    assert sel(L.TNN, False, 1, 3, 100, 128, 96, 3, 3, 1, 1) == lb.CONV_PATH_HALO_FP4
    assert sel(L.TBN, False, 2, 11, 13, 128, 64, 5, 5, 1, 2) == lb.CONV_PATH_HALO_FP4
    # a filter too large for K7 / K6's shared memory: the int8 implicit GeMM
    assert sel(L.TNN, False, 3, 10, 9, 256, 400, 3, 3, 1, 1) == lb.CONV_PATH_IMPLICIT_I8
    # binary map without padding: K7 (the converters raise ZeroInBinaryInput)
    assert sel(L.BNN, True, 2, 7, 7, 128, 64, 3, 3, 1, 0) == lb.CONV_PATH_HALO_FP4
    # stride 2: the fp4 implicit GeMM with a workspace, else the int8 one
    assert sel(L.TNN, False, 3, 8, 7, 128, 96, 3, 3, 2, 1) == lb.CONV_PATH_IMPLICIT_FP4
    assert sel(L.TNN, False, 3, 8, 7, 128, 96, 3, 3, 2, 1, has_workspace=False) == lb.CONV_PATH_IMPLICIT_I8
    # padded row wider than 128 pixels: K7 cuts the rows into column blocks
    assert sel(L.TNN, False, 1, 2, 130, 128, 24, 3, 3, 1, 1) == lb.CONV_PATH_HALO_FP4
    # a binary map padded with +-1: K7 writes the pad codes (stride 2: K6 / int8 im2col cannot, K4 does);
    # c not a multiple of 128: K4 encode + GeMM
    assert sel(L.BNN, True, 64, 56, 56, 128, 128, 3, 3, 1, 1) == lb.CONV_PATH_HALO_FP4
    assert sel(L.BNN, True, 3, 8, 7, 128, 96, 3, 3, 2, 1) == lb.CONV_PATH_ENCODE_GEMM
    assert sel(L.TNN, False, 1, 9, 9, 64, 32, 3, 3, 1, 1) == lb.CONV_PATH_ENCODE_GEMM
    # the int8 kernel request skips the fp4 ones; the bit-serial request takes the bit path
    assert sel(L.TNN, False, 64, 56, 56, 128, 128, 3, 3, 1, 1, kernel=L.KERNEL_TENSOR_I8) == lb.CONV_PATH_IMPLICIT_I8
    assert sel(L.TNN, False, 64, 56, 56, 128, 128, 3, 3, 1, 1, kernel=L.KERNEL_BITSERIAL) == lb.CONV_PATH_ENCODE_GEMM
