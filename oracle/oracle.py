"""ctypes front-end for the parity checkers (TEST INFRASTRUCTURE ONLY).

Two libraries sit behind the same numpy-level API:

* ``Port``  -> oracle/liblowbit_oracle.so, the C restatement in
  oracle/lowbit_oracle.c (always buildable with gcc);
* ``Ref``   -> oracle/_ref/liblowbit_ref.so, the unmodified reference library
  compiled from /root/reference/proj/src by oracle/Makefile (present when the
  reference was available at build time; the .so travels with the repo copy).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module.  The product (paper_2205_09120_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liblowbit_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "liblowbit_ref.so")
# the same reference sources built with -march=x86-64-v3 (BASELINE.md §2's second CPU line)
REF_NATIVE_SO = os.path.join(HERE, "_ref", "liblowbit_ref_native.so")

BNN, TNN, TBN = 0, 1, 2
STATUS_NAMES = {
    0: "OK", 1: "Error", 2: "ZeroInBinaryInput", 3: "InvalidCode", 4: "OutOfBounds",
    5: "DepthOverflow", 6: "ModeMismatch", 7: "ChannelOverflow", 8: "EmptyOutput",
}


class OracleError(RuntimeError):
    def __init__(self, status: int, where: str):
        super().__init__(f"{where}: {STATUS_NAMES.get(status, status)}")
        self.status = status
        self.name = STATUS_NAMES.get(status, str(status))


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def build():
    """Compile the checkers (gcc/g++ only; no reference build system)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def stride_bytes(cols: int) -> int:
    return (cols + 7) // 8


def a_mode_ternary(mode: int) -> bool:
    return mode != BNN


def b_mode_ternary(mode: int) -> bool:
    return mode == TNN


class _Common:
    lib: C.CDLL

    def _chk(self, st, where):
        if st != 0:
            raise OracleError(st, where)

    def encode(self, values: np.ndarray, ternary: bool):
        """encode_binary / encode_ternary -> (plane0, plane1|None), each rows x stride."""
        v = np.ascontiguousarray(values, dtype=np.int8)
        rows, cols = v.shape
        sb = stride_bytes(cols)
        p0 = np.zeros((rows, sb), np.uint8)
        p1 = np.zeros((rows, sb), np.uint8) if ternary else None
        st = self._encode(ternary, v, rows, cols, p0, p1)
        self._chk(st, "encode")
        return p0, p1

    def pack_b(self, b0, b1, k: int, n: int) -> np.ndarray:
        ternary = b1 is not None
        out = np.zeros(((n + 7) // 8) * (16 if ternary else 8) * ((k + 7) // 8), np.uint8)
        st = self.lib_pack_b(int(ternary), _p(b0), _p(b1), k, n, _p(out))
        self._chk(st, "pack_b")
        return out


class Port(_Common):
    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build()
        self.lib = lib = C.CDLL(path)
        lib.orc_splitmix64.restype = C.c_uint64
        lib.orc_splitmix64.argtypes = [C.c_uint64]
        lib.orc_generate.argtypes = [C.c_int, C.c_uint64, C.c_int, C.c_longlong, C.c_longlong, C.c_longlong, C.c_void_p]
        lib.orc_packed_b_bytes.restype = C.c_size_t
        lib.orc_k_max.restype = C.c_longlong
        lib.orc_k_max_sign.restype = C.c_longlong
        lib.orc_c_in_max.restype = C.c_longlong
        lib.orc_c_in_max.argtypes = [C.c_longlong, C.c_int, C.c_int]
        self.lib_pack_b = lib.orc_pack_b

    def _encode(self, ternary, v, rows, cols, p0, p1):
        if ternary:
            return self.lib.orc_encode_ternary(_p(v), rows, cols, _p(p0), _p(p1))
        return self.lib.orc_encode_binary(_p(v), rows, cols, _p(p0))

    def generate(self, dist: int, seed: int, matrix_id: int, rows: int, cols: int, row0: int = 0) -> np.ndarray:
        out = np.empty((rows, cols), np.int8)
        self.lib.orc_generate(dist, seed, matrix_id, row0, rows, cols, _p(out))
        return out

    def decode(self, p0, p1, rows, cols):
        out = np.empty((rows, cols), np.int8)
        if p1 is None:
            self.lib.orc_decode_binary(_p(p0), rows, cols, _p(out))
        else:
            self.lib.orc_decode_ternary(_p(p0), _p(p1), rows, cols, _p(out))
        return out

    def pack_block(self, block_mode, p0, p1, rows, cols, start, depth_start, k_eff):
        group = self.lib.orc_block_group_bytes(block_mode)
        out = np.zeros(group * max(1, (k_eff + 7) // 8), np.uint8)
        lanes = C.c_int(0)
        st = self.lib.orc_pack_block(block_mode, _p(p0), _p(p1), rows, cols, start, depth_start, k_eff, _p(out),
                                     C.byref(lanes))
        self._chk(st, "pack_block")
        return out, lanes.value

    def gemm_lowbit(self, mode, a0, a1, a_rows, a_cols, pb, pb_ternary, pb_n, pb_k, m, n, k, k_blk=4096):
        c = np.zeros((m, n), np.int16) if m > 0 and n > 0 else np.zeros((1, 1), np.int16)
        st = self.lib.orc_gemm_lowbit(mode, int(a1 is not None), _p(a0), _p(a1), a_rows, a_cols, int(pb_ternary),
                                      _p(pb), pb_n, pb_k, m, n, k, k_blk, _p(c))
        self._chk(st, "gemm_lowbit")
        return c

    def gemm(self, mode, a: np.ndarray, b: np.ndarray, k_blk=4096) -> np.ndarray:
        """int8 sign matrices -> encode + pack_b + gemm_lowbit (int16)."""
        m, k = a.shape
        _, n = b.shape
        a0, a1 = self.encode(a, a_mode_ternary(mode))
        b0, b1 = self.encode(b, b_mode_ternary(mode))
        pb = self.pack_b(b0, b1, k, n)
        return self.gemm_lowbit(mode, a0, a1, m, k, pb, b1 is not None, n, k, m, n, k, k_blk)

    def reference_gemm_int(self, a, b):
        a = np.ascontiguousarray(a, np.int8)
        b = np.ascontiguousarray(b, np.int8)
        m, k = a.shape
        n = b.shape[1]
        c = np.zeros((m, n), np.int32)
        self.lib.orc_reference_gemm_int(_p(a), _p(b), m, n, k, _p(c))
        return c

    def dot_binary(self, a, b, k):
        out = C.c_int16(0)
        st = self.lib.orc_dot_binary(_p(a), _p(b), min(len(a), len(b)), k, C.byref(out))
        self._chk(st, "dot_binary")
        return out.value

    def conv_out_dim(self, i, k, s, p):
        return self.lib.orc_conv_out_dim(i, k, s, p)

    def im2col(self, fm, fm_binary, kh, kw, stride, padding, binary_pad_value=1):
        h, w, ch = fm.shape
        oh, ow = self.conv_out_dim(h, kh, stride, padding), self.conv_out_dim(w, kw, stride, padding)
        out = np.zeros((max(oh * ow, 1), kh * kw * ch), np.int8)
        st = self.lib.orc_im2col(_p(np.ascontiguousarray(fm, np.int8)), h, w, ch, int(fm_binary), kh, kw, stride,
                                 padding, binary_pad_value, _p(out))
        self._chk(st, "im2col")
        return out

    def conv2d_lowbit(self, mode, fm, fm_binary, wts, w_binary, kh, kw, stride, padding, binary_pad_value=1):
        h, w, ch = fm.shape
        cout = wts.shape[1]
        oh, ow = self.conv_out_dim(h, kh, stride, padding), self.conv_out_dim(w, kw, stride, padding)
        out = np.zeros((max(oh, 1), max(ow, 1), cout), np.int32)
        st = self.lib.orc_conv2d_lowbit(mode, _p(np.ascontiguousarray(fm, np.int8)), h, w, ch, int(fm_binary),
                                        _p(np.ascontiguousarray(wts, np.int8)), wts.shape[0], wts.shape[1],
                                        int(w_binary), kh, kw, stride, padding, cout, binary_pad_value, _p(out))
        self._chk(st, "conv2d_lowbit")
        return out

    def direct_conv(self, fm, fm_binary, wts, kh, kw, stride, padding, binary_pad_value=1):
        h, w, ch = fm.shape
        cout = wts.shape[1]
        oh, ow = self.conv_out_dim(h, kh, stride, padding), self.conv_out_dim(w, kw, stride, padding)
        out = np.zeros((oh, ow, cout), np.int32)
        self.lib.orc_direct_conv(_p(np.ascontiguousarray(fm, np.int8)), h, w, ch, int(fm_binary),
                                 _p(np.ascontiguousarray(wts, np.int8)), kh, kw, stride, padding, cout,
                                 binary_pad_value, _p(out))
        return out


class Ref(_Common):
    """The reference library itself (oracle/_ref/liblowbit_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = lib = C.CDLL(path)
        lib.ref_bench_prepare.restype = C.c_void_p
        lib.ref_bench_prepare.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                          C.c_void_p, C.c_void_p, C.c_int, C.c_int]
        lib.ref_bench_prepare_i8.restype = C.c_void_p
        lib.ref_bench_prepare_i8.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                             C.c_int, C.c_int]
        lib.ref_bench_conv.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                       C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]
        lib.ref_bench_run.argtypes = [C.c_void_p, C.c_void_p]
        lib.ref_bench_free.argtypes = [C.c_void_p]
        lib.ref_k_max.restype = C.c_longlong
        lib.ref_c_in_max.restype = C.c_longlong
        lib.ref_c_in_max.argtypes = [C.c_longlong, C.c_int, C.c_int]
        self.lib_pack_b = lib.ref_pack_b

    @staticmethod
    def available(path: str = REF_SO) -> bool:
        return os.path.exists(path)

    def _encode(self, ternary, v, rows, cols, p0, p1):
        return self.lib.ref_encode(int(ternary), _p(v), rows, cols, _p(p0), _p(p1))

    def pack_block(self, block_mode, p0, p1, rows, cols, start, depth_start, k_eff):
        out = np.zeros(32 * max(1, (k_eff + 7) // 8) + 32, np.uint8)
        lanes, nbytes = C.c_int(0), C.c_int(0)
        st = self.lib.ref_pack_block(block_mode, _p(p0), _p(p1), rows, cols, start, depth_start, k_eff, _p(out),
                                     C.byref(lanes), C.byref(nbytes))
        self._chk(st, "pack_block")
        return out[: nbytes.value].copy(), lanes.value

    def gemm_planes(self, mode, a0, a1, a_rows, a_cols, b0, b1, b_rows, b_cols, m, n, k, k_blk=4096):
        c = np.zeros((max(m, 1), max(n, 1)), np.int16)
        st = self.lib.ref_gemm_lowbit(mode, int(a1 is not None), _p(a0), _p(a1), a_rows, a_cols, int(b1 is not None),
                                      _p(b0), _p(b1), b_rows, b_cols, m, n, k, k_blk, _p(c))
        self._chk(st, "gemm_lowbit")
        return c

    def gemm(self, mode, a, b, k_blk=4096):
        m, k = a.shape
        n = b.shape[1]
        a0, a1 = self.encode(a, a_mode_ternary(mode))
        b0, b1 = self.encode(b, b_mode_ternary(mode))
        return self.gemm_planes(mode, a0, a1, m, k, b0, b1, k, n, m, n, k, k_blk)

    def reference_gemm_int(self, a, b):
        a = np.ascontiguousarray(a, np.int8)
        b = np.ascontiguousarray(b, np.int8)
        m, k = a.shape
        n = b.shape[1]
        c = np.zeros((m, n), np.int32)
        self._chk(self.lib.ref_reference_gemm_int(_p(a), _p(b), m, n, k, _p(c)), "reference_gemm_int")
        return c

    def conv2d_lowbit(self, mode, fm, fm_binary, wts, w_binary, kh, kw, stride, padding, binary_pad_value=1):
        h, w, ch = fm.shape
        cout = wts.shape[1]
        oh = (h + 2 * padding - kh) // stride + 1
        ow = (w + 2 * padding - kw) // stride + 1
        out = np.zeros((max(oh, 1), max(ow, 1), cout), np.int32)
        oh_c, ow_c = C.c_int(0), C.c_int(0)
        st = self.lib.ref_conv2d_lowbit(mode, _p(np.ascontiguousarray(fm, np.int8)), h, w, ch, int(fm_binary),
                                        _p(np.ascontiguousarray(wts, np.int8)), wts.shape[0], wts.shape[1],
                                        int(w_binary), kh, kw, stride, padding, cout, binary_pad_value, _p(out),
                                        C.byref(oh_c), C.byref(ow_c))
        self._chk(st, "conv2d_lowbit")
        return out

    # --- timing harness (CPU baseline) -------------------------------------
    def bench_prepare(self, mode, a0, a1, m, k, b0, b1, n, threads):
        h = self.lib.ref_bench_prepare(mode, int(a1 is not None), _p(a0), _p(a1), m, k, int(b1 is not None),
                                       _p(b0), _p(b1), n, threads)
        return h

    def bench_prepare_i8(self, mode, a, m, k, b0, b1, n, threads):
        """"From int8 A": the timed run encodes each shard before its gemm_lowbit."""
        return self.lib.ref_bench_prepare_i8(mode, _p(np.ascontiguousarray(a, np.int8)), m, k, int(b1 is not None),
                                             _p(b0), _p(b1), n, threads)

    def bench_conv(self, mode, fm, fm_binary, wts, w_binary, kh, kw, stride, padding, threads):
        """`images` single-image conv2d_lowbit calls (fm: images x h x w x c) on `threads` threads."""
        images, h, w, ch = fm.shape
        self._chk(self.lib.ref_bench_conv(mode, _p(np.ascontiguousarray(fm, np.int8)), images, h, w, ch,
                                          int(fm_binary), _p(np.ascontiguousarray(wts, np.int8)), wts.shape[0],
                                          wts.shape[1], int(w_binary), kh, kw, stride, padding, threads),
                  "bench_conv")

    def bench_run(self, h, c=None):
        self._chk(self.lib.ref_bench_run(h, _p(c)), "bench_run")

    def bench_free(self, h):
        self.lib.ref_bench_free(h)
