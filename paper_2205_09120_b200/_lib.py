"""ctypes binding of the C ABI (include/lowbit_cuda.h) exported by
paper_2205_09120_b200/liblowbit_cuda.so.

The library is the product: there is no CPU fallback.  Importing this module
without the built .so raises immediately; calling a compute entry point on a
host without an sm_100 GPU raises NoDevice / CudaError.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# LOWBIT_LIB: alternative build of the same library (tuning experiments only)
LIB_PATH = os.environ.get("LOWBIT_LIB") or os.path.join(HERE, "liblowbit_cuda.so")
HEADER_PATH = os.path.join(os.path.dirname(HERE), "include", "lowbit_cuda.h")

# lowbit_status
OK, ERROR, ZERO_IN_BINARY, INVALID_CODE, OUT_OF_BOUNDS, DEPTH_OVERFLOW, MODE_MISMATCH = range(7)
CHANNEL_OVERFLOW, EMPTY_OUTPUT, CUDA_ERROR, INVALID_ARGUMENT, NO_DEVICE = range(7, 12)
# lowbit_gemm_mode (gemm.hpp:24)
BNN, TNN, TBN = 0, 1, 2
# lowbit_kernel
KERNEL_AUTO, KERNEL_BITSERIAL, KERNEL_TENSOR, KERNEL_TENSOR_1CTA, KERNEL_TENSOR_I8 = 0, 1, 2, 3, 4
K_MAX16 = 32767
# lowbit_layout
LAYOUT_REFERENCE, LAYOUT_LANES = 0, 1


# ---------------------------------------------------------------------------
# Exceptions: the reference hierarchy (errors.hpp:8-45) plus device errors.
# ---------------------------------------------------------------------------
class Error(RuntimeError):
    """lowbit::Error"""


class ZeroInBinaryInput(Error):
    pass


class InvalidCode(Error):
    pass


class OutOfBounds(Error):
    pass


class DepthOverflow(Error):
    def __init__(self, msg, k=0, k_max=0):
        super().__init__(msg)
        self.k, self.k_max = k, k_max


class ModeMismatch(Error):
    pass


class ChannelOverflow(Error):
    def __init__(self, msg, c_in=0, c_in_max=0):
        super().__init__(msg)
        self.c_in, self.c_in_max = c_in, c_in_max


class EmptyOutput(Error):
    pass


class InvalidPlan(Error):
    pass


class CudaError(Error):
    """A CUDA runtime/driver failure (no reference analogue)."""


class InvalidArgument(Error):
    """A device-layout precondition was violated (no reference analogue)."""


class NoDevice(CudaError):
    """No sm_100 GPU visible: the product has no CPU fallback."""


_EXC = {
    ERROR: Error, ZERO_IN_BINARY: ZeroInBinaryInput, INVALID_CODE: InvalidCode, OUT_OF_BOUNDS: OutOfBounds,
    MODE_MISMATCH: ModeMismatch, EMPTY_OUTPUT: EmptyOutput, CUDA_ERROR: CudaError, INVALID_ARGUMENT: InvalidArgument,
    NO_DEVICE: NoDevice,
}

_P = C.c_void_p
_I = C.c_int
_LL = C.c_longlong

# name -> (restype, argtypes); every symbol declared in include/lowbit_cuda.h
SIGNATURES = {
    "lowbit_abi_version": (_I, []),
    "lowbit_status_string": (C.c_char_p, [_I]),
    "lowbit_last_error": (C.c_char_p, []),
    "lowbit_last_error_values": (None, [C.POINTER(_LL), C.POINTER(_LL)]),
    "lowbit_device_check": (_I, []),
    "lowbit_plane_pitch": (_LL, [_I]),
    "lowbit_encode": (_I, [_I, _P, _I, _I, _LL, _P, _P, _LL, _P, _P]),
    "lowbit_packed_b_bytes": (C.c_size_t, [_I, _I, _I]),
    "lowbit_pack_b": (_I, [_I, _P, _P, _I, _I, _LL, _P, _P]),
    "lowbit_weights_bytes": (C.c_size_t, [_I, _I, _I]),
    "lowbit_prepare_weights": (_I, [_I, _P, _I, _I, _P, _P]),
    "lowbit_gemm": (_I, [_I, _P, _P, _LL, _I, _I, _P, _I, _I, _I, _I, _I, _I, _I, _P, _LL, _I, _P]),
    "lowbit_encode_ex": (_I, [_I, _I, _P, _I, _I, _LL, _P, _P, _LL, _P, _P]),
    "lowbit_gemm_ex": (_I, [_I, _I, _P, _P, _LL, _I, _I, _P, _I, _I, _I, _I, _I, _I, _I, _P, _LL, _I, _P]),
    "lowbit_debug_pair_stats": (_I, [C.POINTER(C.c_ulonglong)]),
    "lowbit_debug_fp4_stats": (_I, [C.POINTER(C.c_ulonglong)]),
    "lowbit_debug_conv_trace": (_I, [C.POINTER(C.c_ulonglong)]),
    "lowbit_debug_halo_trace": (_I, [C.POINTER(C.c_ulonglong)]),
    "lowbit_debug_halo_phases": (_I, [C.POINTER(C.c_ulonglong), _I]),
    "lowbit_conv_select": (_I, [_I, _I, _I, _I, _I, _I, _I, _I, _I, _I, _I, _I, _I]),
    "lowbit_gemm_i8": (_I, [_I, _P, _LL, _I, _I, _P, _I, _I, _I, _I, _I, _I, _I, _P, _LL, _P]),
    "lowbit_select_kernel": (_I, [_I, _I, _I, _I]),
    "lowbit_gemm_lowbit_host": (_I, [_I, _P, _P, _I, _I, _P, _I, _I, _I, _I, _I, _I, _I, _P, _I, _P]),
    "lowbit_conv_rows": (_LL, [_I, _I, _I, _I, _I, _I, _I]),
    "lowbit_conv_encode": (_I, [_I, _P, _I, _I, _I, _I, _I, _I, _I, _I, _I, _P, _P, _LL, _P, _P]),
    "lowbit_conv2d_workspace_bytes": (C.c_size_t, [_I, _I, _I, _I, _I, _I, _I, _I, _I]),
    "lowbit_conv2d": (_I, [_I, _P, _I, _I, _I, _I, _I, _P, _I, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _I, _P]),
    "lowbit_conv2d_host": (_I, [_I, _P, _I, _I, _I, _I, _I, _P, _I, _I, _I, _I, _I, _I, _I, _I, _P, _P]),
    "lowbit_encode_host": (_I, [_I, _P, _I, _I, _P, _P, _P]),
    "lowbit_pack_b_host": (_I, [_I, _P, _P, _I, _I, _P, _P]),
    "lowbit_release_thread_state": (None, []),
    "lowbit_generate": (_I, [_I, C.c_ulonglong, _I, _LL, _LL, _LL, _P, _P]),
}



class GemmProblem(C.Structure):
    """lowbit_gemm_problem (include/lowbit_cuda.h)."""
    _fields_ = [("a0", C.c_void_p), ("a1", C.c_void_p), ("a_pitch", C.c_longlong), ("weights", C.c_void_p),
                ("m", C.c_int), ("n", C.c_int), ("k", C.c_int), ("c", C.c_void_p), ("ldc", C.c_longlong)]


SIGNATURES["lowbit_gemm_grouped"] = (_I, [_I, _I, _I, C.POINTER(GemmProblem), _P])

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
        "(the low-bit GeMM has no CPU fallback)")

lib = C.CDLL(LIB_PATH)
for _name, (_res, _args) in SIGNATURES.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def check(status: int, where: str = "") -> None:
    """Raise the reference exception type matching a lowbit_status."""
    if status == OK:
        return
    msg = lib.lowbit_last_error().decode() or lib.lowbit_status_string(status).decode()
    if where:
        msg = f"{where}: {msg}"
    v0, v1 = _LL(0), _LL(0)
    lib.lowbit_last_error_values(C.byref(v0), C.byref(v1))
    if status == DEPTH_OVERFLOW:
        raise DepthOverflow(msg, v0.value, v1.value)
    if status == CHANNEL_OVERFLOW:
        raise ChannelOverflow(msg, v0.value, v1.value)
    raise _EXC.get(status, Error)(msg)
