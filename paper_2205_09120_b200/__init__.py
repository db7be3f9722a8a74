"""paper_2205_09120_b200 — B200-native (sm_100a) low-bit GeMM.

Ternary (TNN), ternary-binary (TBN) and binary (BNN) matrix multiplication of
"Fast matrix multiplication for binary and ternary CNNs on ARM CPU"
(arXiv 2205.09120), rebuilt for B200 behind the reference `lowbit` API:

  include/lowbit_cuda.h          the C ABI (drop-in boundary)
  paper_2205_09120_b200/csrc/    CUDA kernels (K1 encode, K1b pack_b, K2 bit-serial, K3 tcgen05)
  paper_2205_09120_b200/cpp/     C++ drop-in for the reference headers (namespace lowbit)
  paper_2205_09120_b200/api.py   Python mirror of the same API

The C ABI library is mandatory: importing this package fails if it is not built.
"""
from ._lib import (  # noqa: F401
    BNN, TNN, TBN, KERNEL_AUTO, KERNEL_BITSERIAL, KERNEL_TENSOR, KERNEL_TENSOR_1CTA, KERNEL_TENSOR_I8, K_MAX16,
    Error, ZeroInBinaryInput, InvalidCode, OutOfBounds, DepthOverflow, ModeMismatch, ChannelOverflow,
    EmptyOutput, InvalidPlan, CudaError, InvalidArgument, NoDevice, LIB_PATH,
)
from .api import (  # noqa: F401
    Planes, PackedB, Weights, encode_binary, encode_ternary, pack_b, prepare_weights, gemm_lowbit,
    gemm_lowbit_host, generate, plane_pitch, select_kernel, empty_planes, conv2d_lowbit, conv_out_dim, gemm_grouped, gemm_lowbit_i8,
    conv_select, CONV_PATH_ENCODE_GEMM, CONV_PATH_IMPLICIT_I8, CONV_PATH_IMPLICIT_FP4, CONV_PATH_HALO_FP4,
)
