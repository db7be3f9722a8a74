"""Python host mirror of the reference `lowbit` API over the C ABI.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/lowbit/{core,pack,gemm}.hpp); device buffers are
torch CUDA tensors (torch is plumbing here: memory, streams).  Every compute
call goes through liblowbit_cuda.so — there is no CPU path.

    encode_binary / encode_ternary   core.hpp:63,66   -> Planes (device bit planes)
    pack_b                           gemm.hpp:75-76   -> PackedB (reference panel bytes, device)
    prepare_weights                  (GPU operand of PackedB; once per weight matrix)
    gemm_lowbit                      gemm.hpp:78-81   -> int16 [m, n] (device)
    gemm_lowbit_host                 host-buffer drop-in of the whole call
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Union

import numpy as np
import torch

from . import _lib as L
from ._lib import BNN, TNN, TBN, KERNEL_AUTO, KERNEL_BITSERIAL, KERNEL_TENSOR  # noqa: F401

GemmMode = {"bnn": BNN, "tnn": TNN, "tbn": TBN}


def _stream() -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t: Optional[torch.Tensor]):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def plane_pitch(cols: int) -> int:
    return int(L.lib.lowbit_plane_pitch(cols))


@dataclass
class Planes:
    """Device bit planes (BinaryPackedMatrix / TernaryPackedMatrix, core.hpp:36-61).

    plane0 is the binary plane or the plus plane; plane1 the minus plane
    (None for binary).  Rows are `pitch` bytes (multiple of 16)."""
    rows: int
    cols: int
    plane0: torch.Tensor
    plane1: Optional[torch.Tensor]
    layout: int = 0  # lowbit_layout: 0 reference bit order, 1 B200 lane-interleaved

    @property
    def ternary(self) -> bool:
        return self.plane1 is not None

    @property
    def pitch(self) -> int:
        return int(self.plane0.stride(0))

    @property
    def stride_bits(self) -> int:  # core.hpp:38
        return (self.cols + 7) // 8 * 8


@dataclass
class PackedB:
    """Reference PackedB (gemm.hpp:67-73): ceil(n/8) panels concatenated, on device."""
    ternary: bool
    n: int
    k: int
    panels: torch.Tensor


@dataclass
class Weights:
    """PackedB prepared for the GPU kernels (csrc/layout.cuh)."""
    ternary: bool
    n: int
    k: int
    buf: torch.Tensor


def empty_planes(rows: int, cols: int, ternary: bool, device="cuda") -> Planes:
    pitch = plane_pitch(cols)
    p0 = torch.zeros((rows, pitch), dtype=torch.uint8, device=device)
    p1 = torch.zeros((rows, pitch), dtype=torch.uint8, device=device) if ternary else None
    return Planes(rows, cols, p0, p1)


def _encode(values: torch.Tensor, ternary: bool, check_zero: bool = True, layout: int = 0) -> Planes:
    if values.dtype != torch.int8 or not values.is_cuda or values.dim() != 2:
        raise L.InvalidArgument("encode: expected a 2-D int8 CUDA tensor")
    if values.stride(1) != 1:
        values = values.contiguous()
    rows, cols = values.shape
    out = empty_planes(rows, cols, ternary, values.device)
    out.layout = layout
    flag = torch.zeros(1, dtype=torch.int32, device=values.device)
    L.check(L.lib.lowbit_encode_ex(int(ternary), layout, _ptr(values), rows, cols, values.stride(0),
                                   _ptr(out.plane0), _ptr(out.plane1), out.pitch, _ptr(flag), _stream()), "encode")
    if not ternary and check_zero and rows and cols and int(flag.item()):
        raise L.ZeroInBinaryInput("binary matrix contains a zero element")
    return out


def encode_binary(values: torch.Tensor, check_zero: bool = True, layout: int = 0) -> Planes:
    """core.cpp:13-28 (+1 -> 0, -1 -> 1; a 0 raises ZeroInBinaryInput).
    layout=1 writes the B200 lane-interleaved planes (tensor-core kernels only)."""
    return _encode(values, False, check_zero, layout)


def encode_ternary(values: torch.Tensor, layout: int = 0) -> Planes:
    """core.cpp:40-58 (plus plane, minus plane)."""
    return _encode(values, True, True, layout)


def pack_b(b: Planes) -> PackedB:
    """gemm.cpp:59-77: K x N planes (packed along N) -> PackedB panels."""
    k, n = b.rows, b.cols
    nbytes = int(L.lib.lowbit_packed_b_bytes(int(b.ternary), n, k))
    panels = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=b.plane0.device)
    L.check(L.lib.lowbit_pack_b(int(b.ternary), _ptr(b.plane0), _ptr(b.plane1), k, n, b.pitch, _ptr(panels),
                                _stream()), "pack_b")
    return PackedB(b.ternary, n, k, panels)


def prepare_weights(pb: PackedB) -> Weights:
    nbytes = int(L.lib.lowbit_weights_bytes(int(pb.ternary), pb.n, pb.k))
    buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=pb.panels.device)
    L.check(L.lib.lowbit_prepare_weights(int(pb.ternary), _ptr(pb.panels), pb.n, pb.k, _ptr(buf), _stream()),
            "prepare_weights")
    return Weights(pb.ternary, pb.n, pb.k, buf)


def gemm_lowbit(mode: int, a: Planes, b: Union[PackedB, Weights], dims, k_blk: int = 4096,
                kernel: int = KERNEL_AUTO, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """gemm.cpp:79-112.  dims = (m, n, k) (GemmDims).  Returns int16 [m, n]."""
    m, n, k = dims
    w = b if isinstance(b, Weights) else None
    if out is None:
        out = torch.empty((max(m, 1), max(n, 1)), dtype=torch.int16, device=a.plane0.device)
    if w is None and isinstance(b, PackedB):
        # validate before preparing, so errors come out in the reference order
        st = L.lib.lowbit_gemm(mode, _ptr(a.plane0), _ptr(a.plane1), a.pitch, a.rows, a.cols, None,
                               int(b.ternary), b.n, b.k, m, n, k, k_blk, None, out.stride(0), kernel, _stream())
        if st not in (L.OK, L.INVALID_ARGUMENT):
            L.check(st, "gemm_lowbit")
        w = prepare_weights(b)
    L.check(L.lib.lowbit_gemm_ex(mode, a.layout, _ptr(a.plane0), _ptr(a.plane1), a.pitch, a.rows, a.cols,
                                 _ptr(w.buf), int(w.ternary), w.n, w.k, m, n, k, k_blk, _ptr(out), out.stride(0),
                                 kernel, _stream()), "gemm_lowbit")
    return out


def gemm_lowbit_host(mode: int, a0: np.ndarray, a1: Optional[np.ndarray], a_rows: int, a_cols: int,
                     panels: np.ndarray, b_ternary: bool, b_n: int, b_k: int, dims, k_blk: int = 4096,
                     kernel: int = KERNEL_AUTO, out: Optional[np.ndarray] = None) -> np.ndarray:
    """Host buffers in, host int16 C out: one whole reference gemm_lowbit call
    (upload, prepare B, run, download) through lowbit_gemm_lowbit_host."""
    m, n, k = dims
    if out is None:
        out = np.empty((max(m, 1), max(n, 1)), np.int16)

    def hp(x):
        return C.c_void_p(x.ctypes.data) if x is not None else None

    L.check(L.lib.lowbit_gemm_lowbit_host(mode, hp(a0), hp(a1), a_rows, a_cols, hp(panels), int(b_ternary), b_n,
                                          b_k, m, n, k, k_blk, hp(out), kernel, _stream()), "gemm_lowbit")
    return out


def generate(dist: int, seed: int, matrix_id: int, rows: int, cols: int, row0: int = 0,
             device="cuda") -> torch.Tensor:
    """Counter-based synthetic {-1,0,+1} data, identical to oracle.generate."""
    out = torch.empty((rows, cols), dtype=torch.int8, device=device)
    L.check(L.lib.lowbit_generate(dist, seed, matrix_id, row0, rows, cols, _ptr(out), _stream()), "generate")
    return out


def select_kernel(mode: int, m: int, n: int, k: int) -> int:
    return int(L.lib.lowbit_select_kernel(mode, m, n, k))


CONV_PATH_ENCODE_GEMM, CONV_PATH_IMPLICIT_I8, CONV_PATH_IMPLICIT_FP4, CONV_PATH_HALO_FP4 = 1, 3, 6, 7


def conv_select(mode: int, fm_binary: bool, batch: int, h: int, w: int, c: int, cout: int, kh: int, kw: int,
                stride: int = 1, padding: int = 0, kernel: int = KERNEL_AUTO, has_workspace: bool = True) -> int:
    """The kernel conv2d_lowbit takes for this conv (lowbit_conv_select; host logic, no GPU needed)."""
    return int(L.lib.lowbit_conv_select(mode, int(fm_binary), batch, h, w, c, cout, kh, kw, stride, padding, kernel,
                                        int(has_workspace)))


def conv_out_dim(i: int, k: int, s: int, p: int) -> int:
    """conv.cpp:5-7"""
    return (i + 2 * p - k) // s + 1


def conv2d_lowbit(mode: int, fm: torch.Tensor, fm_binary: bool, weights: Weights, kh: int, kw: int, stride: int = 1,
                  padding: int = 0, binary_pad_value: int = 1, kernel: int = KERNEL_AUTO,
                  out: Optional[torch.Tensor] = None, workspace: Optional[torch.Tensor] = None) -> torch.Tensor:
    """conv2d_lowbit (conv.cpp:33-59) over an NHWC int8 batch [B, H, W, C]:
    K4 fused im2col+encode, then the GeMM kernels.  weights: the prepared
    (kh*kw*C) x cout sign matrix.  Returns int16 [B, OH, OW, cout]."""
    if fm.dim() == 3:
        fm = fm.unsqueeze(0)
    fm = fm.contiguous()
    b, h, w, c = fm.shape
    oh, ow = conv_out_dim(h, kh, stride, padding), conv_out_dim(w, kw, stride, padding)
    cout = weights.n
    if out is None:
        out = torch.empty((b, max(oh, 1), max(ow, 1), cout), dtype=torch.int16, device=fm.device)
    if workspace is None:
        nbytes = int(L.lib.lowbit_conv2d_workspace_bytes(mode, b, h, w, c, kh, kw, stride, padding))
        workspace = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=fm.device)
    # only a BNN conv checks its map for zeros (core.cpp:23); the flag is optional in the C ABI, and
    # zeroing one per call would put a second kernel launch in front of every ternary conv
    flag = torch.zeros(1, dtype=torch.int32, device=fm.device) if mode == BNN else None
    L.check(L.lib.lowbit_conv2d(mode, _ptr(fm), b, h, w, c, int(fm_binary), _ptr(weights.buf), int(weights.ternary),
                                cout, weights.k, kh, kw, stride, padding, binary_pad_value, _ptr(workspace),
                                _ptr(flag) if flag is not None else None, _ptr(out), kernel, _stream()),
            "conv2d_lowbit")
    if flag is not None and int(flag.item()):
        raise L.ZeroInBinaryInput("binary matrix contains a zero element")
    return out


def gemm_grouped(mode: int, problems, b_ternary: Optional[bool] = None):
    """One launch for many small gemm_lowbit problems (bench grid / config 2).
    problems: list of (a: Planes, w: Weights, out: int16 tensor)."""
    if b_ternary is None:
        b_ternary = mode == TNN
    arr = (L.GemmProblem * len(problems))()
    for i, (a, w, out) in enumerate(problems):
        arr[i] = L.GemmProblem(a.plane0.data_ptr(), a.plane1.data_ptr() if a.plane1 is not None else None, a.pitch,
                               w.buf.data_ptr(), a.rows, w.n, a.cols, out.data_ptr(), out.stride(0))
    L.check(L.lib.lowbit_gemm_grouped(mode, int(b_ternary), len(problems), arr, _stream()), "gemm_grouped")
    return [p[2] for p in problems]


def gemm_lowbit_i8(mode: int, a: torch.Tensor, w: Weights, dims, k_blk: int = 4096,
                   out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """gemm_lowbit from dense int8 sign values (the "from int8 A" form):
    TMA feeds the tensor cores directly, no encode.  a: int8 [m, k] CUDA, rows
    16-byte aligned."""
    m, n, k = dims
    if a.dtype != torch.int8 or not a.is_cuda or a.dim() != 2 or a.stride(1) != 1:
        raise L.InvalidArgument("gemm_lowbit_i8: expected a row-major 2-D int8 CUDA tensor")
    if out is None:
        out = torch.empty((max(m, 1), max(n, 1)), dtype=torch.int16, device=a.device)
    L.check(L.lib.lowbit_gemm_i8(mode, _ptr(a), a.stride(0), a.shape[0], a.shape[1], _ptr(w.buf), int(w.ternary),
                                 w.n, w.k, m, n, k, k_blk, _ptr(out), out.stride(0), _stream()), "gemm_lowbit_i8")
    return out
