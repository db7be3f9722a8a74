// conv.cu — K4: convolution as fused im2col + encode, feeding the GeMM kernels.
//
// Reference: conv2d_lowbit = im2col -> encode_* -> pack_b -> gemm_lowbit ->
// widen to int32 (conv.cpp:33-59), one image per call, (ky, kx, c) column
// order, pad value 0 for ternary / binary_pad_value for binary activations.
//
// Here one launch reads the NHWC int8 batch and writes the implicit-GeMM A
// operand directly as bit planes (the 9x-redundant int8 im2col matrix never
// exists), then lowbit_gemm runs on it with M = batch*OH*OW.  Each thread
// builds one 32-bit word (32 consecutive depth positions) of one output
// pixel; when C % 32 == 0 a word is 32 contiguous channels of one input
// pixel, read with two 16-byte loads (repeated taps hit L2).
//
// Algorithmic bytes per launch: batch*H*W*C int8 read + rows*pitch*planes written.
#include <cstdio>
#include <cstring>

#include "common.cuh"
#include "encode.cuh"
#include "layout.cuh"
#include "tmap.cuh"
#include "hostctx.cuh"

namespace lb {

#ifndef K4_BLOCKS_PER_SM
#define K4_BLOCKS_PER_SM 4
#endif

struct ConvGeom {
    int batch, h, w, c, kh, kw, stride, pad, oh, ow, k;
};

// a_binary: write one binary plane (BNN's A) instead of plus/minus planes.
__global__ void conv_encode_kernel(int a_binary, const int8_t* __restrict__ fm, ConvGeom g, int pad_value,
                                   uint8_t* __restrict__ plane0, uint8_t* __restrict__ plane1, long long pitch,
                                   int* zero_flag) {
    const long long words_per_row = pitch / 4;
    const long long rows = (long long)g.batch * g.oh * g.ow;
    const long long total = rows * words_per_row;
    const bool fast = (g.c % 32) == 0;
    bool saw_zero = false;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long r = idx / words_per_row;
        const int wd = (int)(idx - r * words_per_row);
        const int img = (int)(r / (g.oh * g.ow));
        const int rem = (int)(r - (long long)img * g.oh * g.ow);
        const int oy = rem / g.ow, ox = rem - oy * g.ow;
        const int k0 = wd * 32;
        uint32_t plus = 0, minus = 0;
        if (k0 < g.k) {
            const int nvals = g.k - k0 < 32 ? g.k - k0 : 32;
            if (fast) {
                const int tap = k0 / g.c, c0 = k0 - tap * g.c;
                const int ky = tap / g.kw, kx = tap - ky * g.kw;
                const int y = oy * g.stride + ky - g.pad, x = ox * g.stride + kx - g.pad;
                if (y >= 0 && y < g.h && x >= 0 && x < g.w) {
                    encode_word32(fm + (((long long)img * g.h + y) * g.w + x) * g.c + c0, 32, plus, minus);
                } else if (pad_value > 0) {
                    plus = 0xFFFFFFFFu;
                } else if (pad_value < 0) {
                    minus = 0xFFFFFFFFu;
                }
            } else {
                for (int j = 0; j < nvals; ++j) {
                    const int kk = k0 + j;
                    const int tap = kk / g.c, ch = kk - tap * g.c;
                    const int ky = tap / g.kw, kx = tap - ky * g.kw;
                    const int y = oy * g.stride + ky - g.pad, x = ox * g.stride + kx - g.pad;
                    const int v = (y >= 0 && y < g.h && x >= 0 && x < g.w)
                                      ? fm[(((long long)img * g.h + y) * g.w + x) * g.c + ch]
                                      : pad_value;
                    if (v > 0) plus |= 1u << j;
                    if (v < 0) minus |= 1u << j;
                }
            }
            if (a_binary && ((plus | minus) != valid_mask32(nvals))) saw_zero = true;
        }
        if (a_binary) {
            reinterpret_cast<uint32_t*>(plane0 + r * pitch)[wd] = minus;
        } else {
            reinterpret_cast<uint32_t*>(plane0 + r * pitch)[wd] = plus;
            reinterpret_cast<uint32_t*>(plane1 + r * pitch)[wd] = minus;
        }
    }
    if (saw_zero && zero_flag) atomicOr(zero_flag, 1);
}

// c % 32 == 0: every 32-value word of a row is 32 channels of one tap.  A block
// takes one output row (img, oy) at a time: its kh input rows (padding
// resolved: out-of-image pixels hold pad_value) are staged in shared memory
// once, then threads walk the row's (ox, word) pairs with an incremental index
// and build each word from shared memory.  Input bytes cross L2 -> SM kh
// times instead of kh*kw times (im2col), and no per-word divisions remain.
__global__ void conv_encode_rows_kernel(int a_binary, const int8_t* __restrict__ fm, ConvGeom g, int pad_value,
                                        uint8_t* __restrict__ plane0, uint8_t* __restrict__ plane1, long long pitch,
                                        int* zero_flag) {
    extern __shared__ __align__(16) uint8_t conv_smem[];
    const int wpr = (int)(pitch / 4), kwords = g.k / 32;
    uint32_t* tap_of_word = reinterpret_cast<uint32_t*>(conv_smem);  // (ky << 24) | (kx << 16) | c0 / 32
    int8_t* rows_s = reinterpret_cast<int8_t*>(conv_smem + ((wpr * 4 + 15) & ~15));  // [kh][w][c]
    for (int wd = threadIdx.x; wd < wpr; wd += blockDim.x) {
        uint32_t e = 0xFFFFFFFFu;  // past the depth: a zero word
        if (wd < kwords) {
            const int k0 = wd * 32, tap = k0 / g.c, c0 = k0 - tap * g.c;
            const int ky = tap / g.kw, kx = tap - ky * g.kw;
            e = ((uint32_t)ky << 24) | ((uint32_t)kx << 16) | (uint32_t)(c0 / 32);
        }
        tap_of_word[wd] = e;
    }
    const int per_row = g.ow * wpr;
    const int ox_first = threadIdx.x / wpr, wd_first = threadIdx.x - ox_first * wpr;
    const int dox = blockDim.x / wpr, dwd = blockDim.x - dox * wpr;
    const long long row_bytes = (long long)g.w * g.c;  // one input row
    const int row16 = (int)(row_bytes / 16);
    const uint32_t padw = pad_value > 0 ? 0x01010101u : (pad_value < 0 ? 0xFFFFFFFFu : 0u);
    bool saw_zero = false;
    for (long long orow = blockIdx.x; orow < (long long)g.batch * g.oh; orow += gridDim.x) {
        const int img = (int)(orow / g.oh), oy = (int)(orow - (long long)img * g.oh);
        __syncthreads();  // the previous row's words are built
        for (int ky = 0; ky < g.kh; ++ky) {  // stage input row y = oy*s + ky - pad (or padding)
            const int y = oy * g.stride + ky - g.pad;
            uint4* dst = reinterpret_cast<uint4*>(rows_s + (long long)ky * row_bytes);
            if (y >= 0 && y < g.h) {
                const uint4* src = reinterpret_cast<const uint4*>(fm + ((long long)img * g.h + y) * row_bytes);
                for (int i = threadIdx.x; i < row16; i += blockDim.x) dst[i] = __ldg(src + i);
            } else {
                for (int i = threadIdx.x; i < row16; i += blockDim.x) dst[i] = make_uint4(padw, padw, padw, padw);
            }
        }
        __syncthreads();
        const long long r0 = orow * g.ow;  // first output pixel (GeMM row) of this output row
        int ox = ox_first, wd = wd_first;
        for (int t = threadIdx.x; t < per_row; t += blockDim.x) {
            const uint32_t e = tap_of_word[wd];
            uint32_t plus = 0, minus = 0;
            if (e != 0xFFFFFFFFu) {
                const int ky = (int)(e >> 24), kx = (int)((e >> 16) & 0xFF), c0 = (int)(e & 0xFFFF) * 32;
                const int x = ox * g.stride + kx - g.pad;
                if (x >= 0 && x < g.w) {
                    const uint4* q = reinterpret_cast<const uint4*>(rows_s + (long long)ky * row_bytes +
                                                                    (long long)x * g.c + c0);
                    encode_word32_regs(q[0], q[1], plus, minus);
                } else if (pad_value > 0) {
                    plus = 0xFFFFFFFFu;
                } else if (pad_value < 0) {
                    minus = 0xFFFFFFFFu;
                }
                if (a_binary && (plus | minus) != 0xFFFFFFFFu) saw_zero = true;
            }
            const long long r = r0 + ox;
            if (a_binary) {
                reinterpret_cast<uint32_t*>(plane0 + r * pitch)[wd] = minus;
            } else {
                reinterpret_cast<uint32_t*>(plane0 + r * pitch)[wd] = plus;
                reinterpret_cast<uint32_t*>(plane1 + r * pitch)[wd] = minus;
            }
            ox += dox;
            wd += dwd;
            if (wd >= wpr) {
                wd -= wpr;
                ++ox;
            }
        }
    }
    if (saw_zero && zero_flag) atomicOr(zero_flag, 1);
}

// c % 32 == 0, the encode-once form: a block walks a contiguous range of output
// rows; every input row it needs is encoded ONCE into a shared-memory ring of
// kh rows of (plus, minus) words per (pixel, 32-channel group) — the encode
// ALU work is the input size, not the kh*kw-fold im2col size — and each output
// word is then a shared-memory lookup.  A per-block table gives, for every
// (output column ox, word), the tap row ky and the word's offset inside a ring
// row (pixel ox*s + kx - pad, group); pad and past-the-depth words point at two
// extra entries (the pad value's words, zeros) through two extra "tap rows".
// So an output word is ring[slot_of_ky[ky] + offset]: no branches, no
// divisions.  Output rows leave as 16-byte stores of 4 consecutive words
// (pitch % 16 == 0), a block's output pixels being consecutive GeMM rows; the
// next output row's new input row is loaded during the current row's stores.
__global__ void conv_encode_ring_kernel(int a_binary, const int8_t* __restrict__ fm, ConvGeom g, int pad_value,
                                        uint8_t* __restrict__ plane0, uint8_t* __restrict__ plane1, long long pitch,
                                        int* zero_flag) {
    extern __shared__ __align__(16) uint8_t conv_smem[];
    const int wpr = (int)(pitch / 4), kwords = g.k / 32, G = g.c / 32;
    const int row_groups = g.w * G, ring_words = g.kh * row_groups;
    const int PAD_IDX = ring_words, ZERO_IDX = ring_words + 1;
    uint32_t* table = reinterpret_cast<uint32_t*>(conv_smem);  // [ox][word]: (tap row << 24) | offset
    uint32_t* encP = table + g.ow * wpr;                       // ring rows, pad entry, zero entry
    uint32_t* encM = encP + ring_words + 2;
    __shared__ int slot_of_ky[258];  // ring-row base of tap row ky (kh: the pad entry, kh + 1: the zero entry)
    for (int t = threadIdx.x; t < g.ow * wpr; t += blockDim.x) {
        const int ox = t / wpr, wd = t - ox * wpr;
        uint32_t e = (uint32_t)(g.kh + 1) << 24;  // past the depth: a zero word
        if (wd < kwords) {
            const int k0 = wd * 32, tap = k0 / g.c, c0 = k0 - tap * g.c;
            const int ky = tap / g.kw, kx = tap - ky * g.kw;
            const int x = ox * g.stride + kx - g.pad;
            e = (x >= 0 && x < g.w) ? ((uint32_t)ky << 24) | (uint32_t)(x * G + c0 / 32) : (uint32_t)g.kh << 24;
        }
        table[t] = e;
    }
    const uint32_t pad_p = pad_value > 0 ? 0xFFFFFFFFu : 0u, pad_m = pad_value < 0 ? 0xFFFFFFFFu : 0u;
    if (threadIdx.x == 0) {
        encP[PAD_IDX] = pad_p;
        encM[PAD_IDX] = pad_m;
        encP[ZERO_IDX] = 0;
        encM[ZERO_IDX] = 0;
        slot_of_ky[g.kh] = PAD_IDX;
        slot_of_ky[g.kh + 1] = ZERO_IDX;
    }
    const uint32_t zero_tap = (uint32_t)(g.kh + 1);
    const long long orows = (long long)g.batch * g.oh;
    const long long r_begin = orows * blockIdx.x / gridDim.x, r_end = orows * (blockIdx.x + 1) / gridDim.x;
    const int wpr4 = wpr / 4, per_row = g.ow * wpr4;
    bool saw_zero = false;
    int have_img = -1, have_hi = -1;  // ring holds padded input rows (have_hi - kh, have_hi] of image have_img
    // next output row's one new input row (stride 1, same image), loaded during this row's stores
    constexpr int PF = 2;             // groups per thread held in registers (row_groups <= PF * blockDim)
    uint4 pf[PF][2];
    int pf_yp = -1;
    int img = (int)(r_begin / g.oh), oy = (int)(r_begin - (long long)img * g.oh);
    for (long long orow = r_begin; orow < r_end; ++orow) {
        const int lo = oy * g.stride, hi = lo + g.kh - 1;  // padded input rows needed (y + pad)
        int first = lo;
        if (img == have_img && have_hi >= lo) first = have_hi + 1;
        __syncthreads();  // the previous row's lookups are done before the ring changes
        for (int yp = first; yp <= hi; ++yp) {  // encode padded row yp into ring slot yp % kh
            const int y = yp - g.pad, slot = yp % g.kh;
            uint32_t* dp = encP + slot * row_groups;
            uint32_t* dm = encM + slot * row_groups;
            if (yp == pf_yp) {  // prefetched during the previous row's stores
#pragma unroll
                for (int q = 0; q < PF; ++q) {
                    const int i = threadIdx.x + q * blockDim.x;
                    if (i < row_groups) {
                        uint32_t p, m;
                        encode_word32_regs(pf[q][0], pf[q][1], p, m);
                        dp[i] = p;
                        dm[i] = m;
                    }
                }
            } else if (y >= 0 && y < g.h) {
                const int8_t* src = fm + ((long long)img * g.h + y) * g.w * g.c;
                for (int i = threadIdx.x; i < row_groups; i += blockDim.x) {
                    const uint4* q = reinterpret_cast<const uint4*>(src + (long long)i * 32);
                    uint32_t p, m;
                    encode_word32_regs(__ldg(q), __ldg(q + 1), p, m);
                    dp[i] = p;
                    dm[i] = m;
                }
            } else {
                for (int i = threadIdx.x; i < row_groups; i += blockDim.x) {
                    dp[i] = pad_p;
                    dm[i] = pad_m;
                }
            }
        }
        for (int ky = threadIdx.x; ky < g.kh; ky += blockDim.x) slot_of_ky[ky] = ((lo + ky) % g.kh) * row_groups;
        have_img = img;
        have_hi = hi;
        __syncthreads();
        // prefetch the next output row's single new input row (stride 1 within an image)
        pf_yp = -1;
        if (orow + 1 < r_end && g.stride == 1 && oy + 1 < g.oh && row_groups <= PF * (int)blockDim.x) {
            const int yn = hi + 1 - g.pad;
            if (yn >= 0 && yn < g.h) {
                pf_yp = hi + 1;
                const int8_t* src = fm + ((long long)img * g.h + yn) * g.w * g.c;
#pragma unroll
                for (int q = 0; q < PF; ++q) {
                    const int i = threadIdx.x + q * blockDim.x;
                    if (i < row_groups) {
                        const uint4* qq = reinterpret_cast<const uint4*>(src + (long long)i * 32);
                        pf[q][0] = __ldg(qq);
                        pf[q][1] = __ldg(qq + 1);
                    }
                }
            }
        }
        uint8_t* out0 = plane0 + orow * g.ow * pitch;
        uint8_t* out1 = a_binary ? nullptr : plane1 + orow * g.ow * pitch;
        for (int t = threadIdx.x; t < per_row; t += blockDim.x) {  // t = ox * wpr4 + w4: 4 words
            const uint4 e4 = *reinterpret_cast<const uint4*>(table + 4 * t);
            const uint32_t ev[4] = {e4.x, e4.y, e4.z, e4.w};
            uint32_t P[4], M[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t tap = ev[j] >> 24;
                const int idx = slot_of_ky[tap] + (int)(ev[j] & 0xFFFFFFu);
                P[j] = encP[idx];
                M[j] = encM[idx];
                // binary maps: a 0 among the values this word takes (im2col's view, core.cpp:23)
                if (a_binary) saw_zero |= tap != zero_tap && (P[j] | M[j]) != 0xFFFFFFFFu;
            }
            const long long off = (long long)t * 16;  // ox * pitch + w4 * 16 (pitch = 16 * wpr4)
            if (a_binary) {
                *reinterpret_cast<uint4*>(out0 + off) = make_uint4(M[0], M[1], M[2], M[3]);
            } else {
                *reinterpret_cast<uint4*>(out0 + off) = make_uint4(P[0], P[1], P[2], P[3]);
                *reinterpret_cast<uint4*>(out1 + off) = make_uint4(M[0], M[1], M[2], M[3]);
            }
        }
        if (++oy == g.oh) {
            oy = 0;
            ++img;
        }
    }
    if (saw_zero && zero_flag) atomicOr(zero_flag, 1);
}

__global__ void widen_kernel(const int16_t* __restrict__ in, int32_t* __restrict__ out, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        out[i] = in[i];
}

}  // namespace lb

namespace lb {
size_t conv_fp4_workspace_bytes(int batch, int h, int w, int c, int pad);
bool conv_fp4_applies(int mode, int fm_binary, int c, int cout, int kh, int kw, int padding, long long rows,
                      int stride);
lowbit_status launch_conv_fp4(const int8_t* fm, int batch, int h, int w, int cch, int kh, int kw, int stride,
                              int pad, int check_zero, const void* weights, int b_ternary, int cout, int16_t* out,
                              void* workspace, int* zero_flag, cudaStream_t stream);
bool conv_halo_applies(int fm_binary, int h, int w, int c, int cout, int kh, int kw, int stride, int pad,
                       long long batch);
lowbit_status launch_conv_halo(const int8_t* fm, int batch, int h, int w, int cch, int kh, int kw, int pad,
                               int check_zero, int pad_value, const void* weights, int b_ternary, int cout,
                               int16_t* out, int* zero_flag, cudaStream_t stream);
lowbit_status launch_conv_pair_im2col(const int8_t* fm, int batch, int h, int w, int cch, int kh, int kw, int stride,
                                      int pad, const void* weights, int b_ternary, int cout, int16_t* out,
                                      cudaStream_t stream);
}

using namespace lb;

static int conv_out(int in, int k, int s, int p) { return (in + 2 * p - k) / s + 1; }

// conv.cpp:35-45 checks, in order, then the EmptyOutput of im2col (conv.cpp:12).
static lowbit_status validate_conv(int mode, int batch, int h, int w, int c, int fm_binary, int b_ternary, int cout,
                                   int k, int kh, int kw, int stride, int padding) {
    const long long kk = (long long)kh * kw * c;
    if (kk > LOWBIT_K_MAX16) {
        char buf[128];
        const long long cmax = LOWBIT_K_MAX16 / ((long long)kh * kw);
        std::snprintf(buf, sizeof buf, "input channels %d exceed c_in_max %lld", c, cmax);
        return lbhost::set_error(LOWBIT_CHANNEL_OVERFLOW, buf, c, cmax);
    }
    if (k != kk || cout < 1) return lbhost::set_error(LOWBIT_OUT_OF_BOUNDS, "out of bounds: weight matrix shape");
    const bool a_binary = mode == LOWBIT_BNN, b_binary = mode != LOWBIT_TNN;
    if (mode < 0 || mode > 2) return lbhost::set_error(LOWBIT_INVALID_ARGUMENT, "unknown gemm mode");
    if (a_binary && !fm_binary) return lbhost::set_error(LOWBIT_MODE_MISMATCH, "mode mismatch: bnn requires binary activations");
    if (b_binary && b_ternary) return lbhost::set_error(LOWBIT_MODE_MISMATCH, "mode mismatch: weights must be binary");
    if (!b_binary && !b_ternary) return lbhost::set_error(LOWBIT_MODE_MISMATCH, "mode mismatch: weights must be ternary");
    if (stride < 1 || batch < 1 || h < 0 || w < 0 || c < 1)
        return lbhost::set_error(LOWBIT_INVALID_ARGUMENT, "conv: bad geometry");
    if (conv_out(h, kh, stride, padding) < 1 || conv_out(w, kw, stride, padding) < 1)
        return lbhost::set_error(LOWBIT_EMPTY_OUTPUT, "convolution produces empty output");
    return LOWBIT_OK;
}

extern "C" long long lowbit_conv_rows(int batch, int h, int w, int kh, int kw, int stride, int padding) {
    const int oh = conv_out(h, kh, stride, padding), ow = conv_out(w, kw, stride, padding);
    if (oh < 1 || ow < 1 || batch < 1) return 0;
    return (long long)batch * oh * ow;
}

extern "C" lowbit_status lowbit_conv_encode(int a_binary, const int8_t* fm, int batch, int h, int w, int c, int kh,
                                            int kw, int stride, int padding, int pad_value, uint8_t* plane0,
                                            uint8_t* plane1, long long pitch, int* zero_flag, lowbit_stream stream) {
    ConvGeom g{batch, h, w, c, kh, kw, stride, padding, conv_out(h, kh, stride, padding),
               conv_out(w, kw, stride, padding), kh * kw * c};
    if (g.oh < 1 || g.ow < 1) return lbhost::set_error(LOWBIT_EMPTY_OUTPUT, "convolution produces empty output");
    if (!fm || !plane0 || (!a_binary && !plane1)) return lbhost::set_error(LOWBIT_INVALID_ARGUMENT, "conv_encode: NULL");
    if ((pitch & 3) || pitch < (g.k + 7) / 8)
        return lbhost::set_error(LOWBIT_INVALID_ARGUMENT, "conv_encode: bad pitch");
    const long long work = (long long)batch * g.oh * g.ow * (pitch / 4);
    const int wpr = (int)(pitch / 4);
    const long long smem = ((wpr * 4LL + 15) & ~15LL) + (long long)kh * w * c;
    const long long ring_smem = (long long)g.ow * wpr * 4 + 2LL * (kh * w * (c / 32) + 2) * 4;
    const bool aligned = (reinterpret_cast<uintptr_t>(fm) & 15) == 0 && (reinterpret_cast<uintptr_t>(plane0) & 15) == 0 &&
                         (a_binary || (reinterpret_cast<uintptr_t>(plane1) & 15) == 0) && (pitch & 15) == 0;
    if (c % 32 == 0 && kh < 256 && kw < 256 && ring_smem <= 96 * 1024 && aligned && (long long)w * (c / 32) < (1 << 24)) {
        static SmemOptIn ring_attr;
        // (the 48 KB a kernel gets without the opt-in counts its static shared memory too — the
        // kernel's 1 KB tap-row table: tools/fuzz_conv.py found a 48,496-byte ring failing to launch)
        if (ring_smem > 44 * 1024) LB_CUDA_TRY(ring_attr.ensure(conv_encode_ring_kernel, 96 * 1024));
        const long long orows = (long long)batch * g.oh;
        // K4_BLOCKS_PER_SM co-resident blocks per SM, each a contiguous run of output rows (it
        // re-encodes kh - stride input rows at its start)
        const long long cap = (long long)num_sms() * K4_BLOCKS_PER_SM;
        const int blocks = (int)(orows < cap ? orows : cap);
        conv_encode_ring_kernel<<<blocks, 256, (size_t)ring_smem, (cudaStream_t)stream>>>(
            a_binary, fm, g, pad_value, plane0, plane1, pitch, zero_flag);
    } else if (c % 32 == 0 && kh < 256 && kw < 256 && smem <= 160 * 1024 && (reinterpret_cast<uintptr_t>(fm) & 15) == 0) {
        static SmemOptIn attr;
        if (smem > 44 * 1024) LB_CUDA_TRY(attr.ensure(conv_encode_rows_kernel, (int)smem));
        const long long orows = (long long)batch * g.oh;
        const int blocks = (int)(orows < 148LL * 8 ? orows : 148LL * 8);
        conv_encode_rows_kernel<<<blocks, 256, (size_t)smem, (cudaStream_t)stream>>>(a_binary, fm, g, pad_value,
                                                                                     plane0, plane1, pitch, zero_flag);
    } else {
        conv_encode_kernel<<<grid_for(work, 256), 256, 0, (cudaStream_t)stream>>>(a_binary, fm, g, pad_value, plane0,
                                                                                   plane1, pitch, zero_flag);
    }
    LB_CUDA_TRY(cudaGetLastError());
    return LOWBIT_OK;
}

extern "C" size_t lowbit_conv2d_workspace_bytes(int mode, int batch, int h, int w, int c, int kh, int kw, int stride,
                                                int padding) {
    const long long rows = lowbit_conv_rows(batch, h, w, kh, kw, stride, padding);
    const size_t planes = (size_t)rows * lowbit_plane_pitch(kh * kw * c) * (mode == LOWBIT_BNN ? 1 : 2) + 256;
    const size_t fm4 = lb::conv_fp4_workspace_bytes(batch, h, w, c, padding);  // K6's packed fp4 feature map
    return planes > fm4 ? planes : fm4;
}

// Which conv kernel lowbit_conv2d runs (pointers assumed aligned; host logic only):
//   K7 fused halo conv — stride 1, any width (column blocks past 128 padded pixels), c % 128 == 0, the filter + two
//      halo stages fit in shared memory; any padding (binary maps padded with +-1 get the pad
//      codes written by the converters; a BNN map padded with 0 must raise ZeroInBinaryInput and
//      takes K4, decided in lowbit_conv2d where the pad value is known);
//   K6 fp4 implicit GeMM over a packed fp4 copy of the map — padding that reads as 0 (ternary map
//      or no padding), any stride (needs the workspace);
//   int8 implicit GeMM (TMA im2col over the int8 map) — TNN/TBN, c % 128 == 0, padding reads 0;
//   else K4 (fused im2col + encode) + lowbit_gemm.
// TMA's out-of-bounds fill is 0, so the im2col paths (K6, int8) keep binary maps padded with
// +-1 on K4 (conv.cpp:13).
extern "C" int lowbit_conv_select(int mode, int fm_binary, int batch, int h, int w, int c, int cout, int kh, int kw,
                                  int stride, int padding, int kernel, int has_workspace) {
    const long long rows = lowbit_conv_rows(batch, h, w, kh, kw, stride, padding);
    const bool tensor = kernel == LOWBIT_KERNEL_AUTO || kernel == LOWBIT_KERNEL_TENSOR;
    static const bool no_halo = lb::tuning_env("LOWBIT_CONV_NO_HALO") != nullptr;  // tuning experiment knob
    if (rows <= 0) return LOWBIT_CONV_PATH_ENCODE_GEMM;
    if (tensor && !no_halo && lb::conv_halo_applies(fm_binary, h, w, c, cout, kh, kw, stride, padding, batch))
        return LOWBIT_CONV_PATH_HALO_FP4;
    if (tensor && has_workspace && lb::conv_fp4_applies(mode, fm_binary, c, cout, kh, kw, padding, rows, stride))
        return LOWBIT_CONV_PATH_IMPLICIT_FP4;
    const bool pad_is_zero = padding == 0 || !fm_binary;
    if (mode != LOWBIT_BNN && pad_is_zero && c % 128 == 0 && rows <= 0x7FFFFFFFLL &&
        (tensor || kernel == LOWBIT_KERNEL_TENSOR_I8))
        return LOWBIT_CONV_PATH_IMPLICIT_I8;
    return LOWBIT_CONV_PATH_ENCODE_GEMM;
}

extern "C" lowbit_status lowbit_conv2d(int mode, const int8_t* fm, int batch, int h, int w, int c, int fm_binary,
                                       const void* weights, int b_ternary, int cout, int k, int kh, int kw, int stride,
                                       int padding, int binary_pad_value, void* workspace, int* zero_flag,
                                       int16_t* out, int kernel, lowbit_stream stream) {
    lowbit_status st = validate_conv(mode, batch, h, w, c, fm_binary, b_ternary, cout, k, kh, kw, stride, padding);
    if (st) return st;
    if (!weights || !out) return lbhost::set_error(LOWBIT_INVALID_ARGUMENT, "conv2d: NULL pointer");
    const long long rows = lowbit_conv_rows(batch, h, w, kh, kw, stride, padding);
    // Implicit GeMM straight from the int8 feature map (TMA im2col -> UMMA, no
    // bit planes, no workspace) whenever padding reads as 0 — ternary
    // activations, or no padding — and the channel count tiles into 128-byte
    // k-blocks.  BNN keeps the bit path: its padding is +-1 and a 0 activation
    // must raise ZeroInBinaryInput (conv.cpp:13, core.cpp:23).
    const bool aligned = (reinterpret_cast<uintptr_t>(fm) & 15) == 0 &&
                         (reinterpret_cast<uintptr_t>(weights) & 255) == 0 &&
                         (reinterpret_cast<uintptr_t>(out) & 15) == 0;
    int path = aligned ? lowbit_conv_select(mode, fm_binary, batch, h, w, c, cout, kh, kw, stride, padding, kernel,
                                            workspace != nullptr)
                       : LOWBIT_CONV_PATH_ENCODE_GEMM;
    // a BNN map padded with 0 holds zeros im2col encodes: K4 raises ZeroInBinaryInput (core.cpp:23)
    if (path == LOWBIT_CONV_PATH_HALO_FP4 && mode == LOWBIT_BNN && fm_binary && padding > 0 && binary_pad_value == 0)
        path = LOWBIT_CONV_PATH_ENCODE_GEMM;
    if (path == LOWBIT_CONV_PATH_HALO_FP4)
        return lb::launch_conv_halo(fm, batch, h, w, c, kh, kw, padding, mode == LOWBIT_BNN && fm_binary,
                                    fm_binary ? binary_pad_value : 0, weights, b_ternary, cout, out, zero_flag,
                                    (cudaStream_t)stream);
    if (path == LOWBIT_CONV_PATH_IMPLICIT_FP4)
        return lb::launch_conv_fp4(fm, batch, h, w, c, kh, kw, stride, padding, mode == LOWBIT_BNN && fm_binary,
                                   weights, b_ternary, cout, out, workspace, zero_flag, (cudaStream_t)stream);
    if (path == LOWBIT_CONV_PATH_IMPLICIT_I8)
        return lb::launch_conv_pair_im2col(fm, batch, h, w, c, kh, kw, stride, padding, weights, b_ternary, cout, out,
                                           (cudaStream_t)stream);
    if (!workspace) return lbhost::set_error(LOWBIT_INVALID_ARGUMENT, "conv2d: NULL workspace");
    const long long pitch = lowbit_plane_pitch(k);
    uint8_t* p0 = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255));
    const int a_binary = mode == LOWBIT_BNN;
    uint8_t* p1 = a_binary ? nullptr : p0 + rows * pitch;
    // pad with 0 for ternary feature maps, binary_pad_value for binary ones (conv.cpp:13)
    if ((st = lowbit_conv_encode(a_binary, fm, batch, h, w, c, kh, kw, stride, padding,
                                 fm_binary ? binary_pad_value : 0, p0, p1, pitch, zero_flag, stream)))
        return st;
    if (rows > 0x7FFFFFFFLL) return lbhost::set_error(LOWBIT_INVALID_ARGUMENT, "conv2d: too many output pixels");
    return lowbit_gemm(mode, p0, p1, pitch, (int)rows, k, weights, b_ternary, cout, k, (int)rows, cout, k, 4096, out,
                       cout, kernel, stream);
}

extern "C" lowbit_status lowbit_conv2d_host(int mode, const int8_t* fm, int batch, int h, int w, int c, int fm_binary,
                                            const uint8_t* panels, int b_ternary, int cout, int k, int kh, int kw,
                                            int stride, int padding, int binary_pad_value, int32_t* out,
                                            lowbit_stream stream) {
    lowbit_status st = validate_conv(mode, batch, h, w, c, fm_binary, b_ternary, cout, k, kh, kw, stride, padding);
    if (st) return st;
    if (!fm || !panels || !out) return lbhost::set_error(LOWBIT_INVALID_ARGUMENT, "conv2d_host: NULL pointer");
    if ((st = lowbit_device_check())) return st;
    cudaStream_t s = (cudaStream_t)stream;
    const long long rows = lowbit_conv_rows(batch, h, w, kh, kw, stride, padding);
    const size_t fm_bytes = (size_t)batch * h * w * c;
    const size_t pbytes = lowbit_packed_b_bytes(b_ternary, cout, k);
    lbhost::HostCtx* Xp = lbhost::host_ctx();
    if (!Xp) return lbhost::set_error(LOWBIT_INVALID_ARGUMENT, "conv2d_host: device ordinal out of range");
    lbhost::HostCtx& X = *Xp;
    lbhost::DevScratch &g_fm = X.fm, &g_ws = X.ws, &g_pan = X.panels, &g_w = X.conv_w, &g_out = X.out16,
                       &g_out32 = X.out32, &g_flag = X.flag;
    LB_CUDA_TRY(g_fm.ensure(fm_bytes + 16));
    LB_CUDA_TRY(g_ws.ensure(lowbit_conv2d_workspace_bytes(mode, batch, h, w, c, kh, kw, stride, padding)));
    LB_CUDA_TRY(g_pan.ensure(pbytes));
    // the same PackedB as the previous call on this thread and device (a batch of single-image calls):
    // its prepared weights are still in conv_w (byte-exact key; preparation is deterministic)
    const void* w_before = g_w.ptr;
    LB_CUDA_TRY(g_w.ensure(lowbit_weights_bytes(b_ternary, cout, k)));
    const bool same_w = g_w.ptr == w_before && X.conv_w_ternary == b_ternary && X.conv_w_cout == cout &&
                        X.conv_w_k == k && X.conv_w_key.size() == pbytes &&
                        std::memcmp(X.conv_w_key.data(), panels, pbytes) == 0;
    LB_CUDA_TRY(g_out.ensure((size_t)rows * cout * sizeof(int16_t)));
    LB_CUDA_TRY(g_out32.ensure((size_t)rows * cout * sizeof(int32_t)));
    LB_CUDA_TRY(g_flag.ensure(sizeof(int)));
    LB_CUDA_TRY(cudaMemsetAsync(g_flag.ptr, 0, sizeof(int), s));
    LB_CUDA_TRY(cudaMemcpyAsync(g_fm.ptr, fm, fm_bytes, cudaMemcpyHostToDevice, s));
    if (!same_w) {
        X.conv_w_ternary = -1;  // invalid until the new weights are prepared
        LB_CUDA_TRY(cudaMemcpyAsync(g_pan.ptr, panels, pbytes, cudaMemcpyHostToDevice, s));
        if ((st = lowbit_prepare_weights(b_ternary, static_cast<const uint8_t*>(g_pan.ptr), cout, k, g_w.ptr, stream)))
            return st;
        X.conv_w_key.assign(panels, panels + pbytes);
        X.conv_w_ternary = b_ternary;
        X.conv_w_cout = cout;
        X.conv_w_k = k;
    }
    if ((st = lowbit_conv2d(mode, static_cast<const int8_t*>(g_fm.ptr), batch, h, w, c, fm_binary, g_w.ptr, b_ternary,
                            cout, k, kh, kw, stride, padding, binary_pad_value, g_ws.ptr,
                            static_cast<int*>(g_flag.ptr), static_cast<int16_t*>(g_out.ptr), LOWBIT_KERNEL_AUTO,
                            stream)))
        return st;
    const long long n = rows * cout;
    widen_kernel<<<grid_for(n, 256), 256, 0, s>>>(static_cast<const int16_t*>(g_out.ptr),
                                                    static_cast<int32_t*>(g_out32.ptr), n);
    LB_CUDA_TRY(cudaGetLastError());
    int flag = 0;
    LB_CUDA_TRY(cudaMemcpyAsync(&flag, g_flag.ptr, sizeof(int), cudaMemcpyDeviceToHost, s));
    LB_CUDA_TRY(cudaMemcpyAsync(out, g_out32.ptr, (size_t)n * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    LB_CUDA_TRY(cudaStreamSynchronize(s));
    // a 0 among binary activations (or a 0 binary pad value) is what
    // encode_binary(cols) rejects in the reference (conv.cpp:51, core.cpp:23)
    if (mode == LOWBIT_BNN && flag) return lbhost::set_error(LOWBIT_ZERO_IN_BINARY, "binary matrix contains a zero element");
    return LOWBIT_OK;
}
