// encode.cu — HBM-bound packing kernels.
//
//   K1   encode_kernel       int8 sign matrix -> bit plane(s)      (core.cpp:13-58)
//   K1b  pack_b_kernel       K x N planes -> PackedB panels        (pack.cpp:64-127, gemm.cpp:59-77)
//   --   prepare_*_kernel    PackedB panels -> device weight operand (layout.cuh)
//   --   generate_kernel     counter-based synthetic inputs
//
// Algorithmic bytes (roofline denominators):
//   encode: rows*cols int8 read + planes*rows*pitch written.
#include "common.cuh"
#include "encode.cuh"
#include "layout.cuh"

namespace lb {

// One thread -> one 32-bit word of every plane of one row (32 values).
// LAYOUT 0: the reference LSB-first layout; 1: the lane-interleaved B200 layout.
// The (row, word) of each iteration advance by a fixed step (no 64-bit
// division per word: it cost ~20% of the kernel at c5's 67M words).
template <int LAYOUT>
__global__ void encode_kernel(int ternary, const int8_t* __restrict__ values, int rows, int cols, long long ld,
                              uint8_t* __restrict__ plane0, uint8_t* __restrict__ plane1, long long pitch,
                              int* zero_flag) {
    const int words_per_row = (int)(pitch / 4);
    const long long total = (long long)rows * words_per_row;
    bool saw_zero = false;
    const long long first = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long step = (long long)gridDim.x * blockDim.x;
    long long r = first / words_per_row;
    int w = (int)(first - r * words_per_row);
    const long long dr = step / words_per_row;
    const int dw = (int)(step - dr * words_per_row);
    for (long long idx = first; idx < total; idx += step) {
        const int c0 = w * 32;
        uint32_t minus = 0, plus = 0;
        if (c0 < cols) {
            const int nvals = cols - c0 < 32 ? cols - c0 : 32;
            if (LAYOUT == 0) {
                encode_word32(values + r * ld + c0, nvals, plus, minus);
                if (!ternary && ((plus | minus) != valid_mask32(nvals))) saw_zero = true;
            } else if (LAYOUT == 1) {
                encode_word32_lanes(values + r * ld + c0, nvals, plus, minus);
                if (!ternary && ((plus | minus) != valid_mask32_lanes(nvals))) saw_zero = true;
            } else {
                encode_word32_nibbles(values + r * ld + c0, nvals, plus, minus);
                if (!ternary && ((plus | minus) != valid_mask32_nibbles(nvals))) saw_zero = true;
            }
        }
        uint32_t* d0 = reinterpret_cast<uint32_t*>(plane0 + r * pitch);
        if (ternary) {
            d0[w] = plus;
            reinterpret_cast<uint32_t*>(plane1 + r * pitch)[w] = minus;
        } else {
            d0[w] = minus;  // binary: -1 -> 1, +1 -> 0 (core.cpp:24)
        }
        r += dr;
        w += dw;
        if (w >= words_per_row) {
            w -= words_per_row;
            ++r;
        }
    }
    if (saw_zero && zero_flag) atomicOr(zero_flag, 1);
}

// 8x8 bit-matrix transpose: byte i bit j -> byte j bit i (LSB-first).
__device__ __forceinline__ uint64_t transpose8x8(uint64_t x) {
    uint64_t t;
    t = (x ^ (x >> 7)) & 0x00AA00AA00AA00AAull;
    x = x ^ t ^ (t << 7);
    t = (x ^ (x >> 14)) & 0x0000CCCC0000CCCCull;
    x = x ^ t ^ (t << 14);
    t = (x ^ (x >> 28)) & 0x00000000F0F0F0F0ull;
    x = x ^ t ^ (t << 28);
    return x;
}

// One thread -> one (panel p, depth byte d) group of the PackedB stream:
// bnn_b 8 bytes (col j's depth byte), tnn_b 16 bytes (col j plus, minus).
// Rows past k and columns past n read as 0 (gather_col_byte, pack.cpp:22-32).
__global__ void pack_b_kernel(int ternary, const uint8_t* __restrict__ b0, const uint8_t* __restrict__ b1, int k,
                              int n, long long pitch, uint8_t* __restrict__ panels) {
    const int db = (k + 7) / 8;
    const int npanels = (n + 7) / 8;
    const long long total = (long long)npanels * db;
    const int group = ternary ? 16 : 8;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int p = (int)(idx / db);
        const int d = (int)(idx - (long long)p * db);
        const int valid_cols = n - p * 8 < 8 ? n - p * 8 : 8;
        const uint8_t colmask = (uint8_t)((1u << valid_cols) - 1u);
        uint64_t xp = 0, xm = 0;
        for (int i = 0; i < 8; ++i) {
            const int t = d * 8 + i;
            if (t >= k) break;
            xp |= (uint64_t)(b0[(long long)t * pitch + p] & colmask) << (8 * i);
            if (ternary) xm |= (uint64_t)(b1[(long long)t * pitch + p] & colmask) << (8 * i);
        }
        const uint64_t tp = transpose8x8(xp);
        uint8_t* dst = panels + (size_t)p * group * db + (size_t)d * group;
        if (!ternary) {
            // group offset d*8 is 8-byte aligned
            *reinterpret_cast<uint64_t*>(dst) = tp;
        } else {
            const uint64_t tm = transpose8x8(xm);
            // interleave: byte 2j = plus col j, byte 2j+1 = minus col j
            uint64_t lo = 0, hi = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                lo |= ((tp >> (8 * j)) & 0xFF) << (16 * j) | ((tm >> (8 * j)) & 0xFF) << (16 * j + 8);
                hi |= ((tp >> (8 * (j + 4))) & 0xFF) << (16 * j) | ((tm >> (8 * (j + 4))) & 0xFF) << (16 * j + 8);
            }
            reinterpret_cast<uint64_t*>(dst)[0] = lo;
            reinterpret_cast<uint64_t*>(dst)[1] = hi;
        }
    }
}

// PackedB byte of column col, depth byte d, plane (0 = binary/plus, 1 = minus).
__device__ __forceinline__ uint32_t panel_byte(const uint8_t* panels, int ternary, int db, int col, int d,
                                               int plane) {
    const int group = ternary ? 16 : 8;
    const int p = col >> 3, j = col & 7;
    const size_t off = (size_t)p * group * db + (size_t)d * group + (ternary ? 2 * j + plane : j);
    return panels[off];
}

// Bit sections: one thread per (column, word).
__global__ void prepare_bits_kernel(int ternary, const uint8_t* __restrict__ panels, int n, int k, int np, int kw,
                                    uint32_t* __restrict__ sign, uint32_t* __restrict__ nz) {
    const int db = (k + 7) / 8;
    const long long total = (long long)np * kw;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int col = (int)(idx / kw);
        const int w = (int)(idx - (long long)col * kw);
        uint32_t s = 0, z = 0;
        if (col < n) {
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int d = w * 4 + b;
                if (d >= db) break;
                if (ternary) {
                    const uint32_t pb = panel_byte(panels, 1, db, col, d, 0);
                    const uint32_t mb = panel_byte(panels, 1, db, col, d, 1);
                    s |= mb << (8 * b);
                    z |= (pb | mb) << (8 * b);
                } else {
                    s |= panel_byte(panels, 0, db, col, d, 0) << (8 * b);
                }
            }
        }
        sign[idx] = s;
        if (ternary) nz[idx] = z;
    }
}

// int8 section: one thread per (column, 16-value chunk).
__global__ void prepare_i8_kernel(int ternary, const uint8_t* __restrict__ panels, int n, int k, int np, int kp,
                                  int8_t* __restrict__ out) {
    const int db = (k + 7) / 8;
    const int chunks = kp / 16;
    const long long total = (long long)np * chunks;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int col = (int)(idx / chunks);
        const int ch = (int)(idx - (long long)col * chunks);
        uint32_t words[4] = {0, 0, 0, 0};
        if (col < n) {
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const int d = ch * 2 + half;
                if (d >= db) break;
                // bits past k are zero in PackedB (tail-masked by gather_col_byte)
                uint32_t p, m;
                if (ternary) {
                    p = panel_byte(panels, 1, db, col, d, 0);
                    m = panel_byte(panels, 1, db, col, d, 1);
                } else {
                    m = panel_byte(panels, 0, db, col, d, 0);
                    // binary: bit 0 -> +1 only for depths < k
                    const int valid = k - d * 8 < 8 ? k - d * 8 : 8;
                    p = ~m & ((1u << valid) - 1u);
                }
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const uint32_t pq = spread4((p >> (4 * q)) & 0xF);
                    const uint32_t mq = spread4((m >> (4 * q)) & 0xF);
                    words[half * 2 + q] = pq | (mq * 0xFFu);
                }
            }
        }
        reinterpret_cast<uint4*>(out + (size_t)col * kp)[ch] = make_uint4(words[0], words[1], words[2], words[3]);
    }
}

// fp4 (e2m1) sections: one thread per (column, 16-byte chunk = 32 depth
// positions); +1 -> 0x2, -1 -> 0xA, 0 -> 0x0, zero past k.
//   out  (canonical): element 2i in the low nibble of byte i.
//   outr (reference order, layout.cuh): nibble 8q+i holds element 4i+q.
//   outc (conv order, layout.cuh): nibble i of word q holds element 8q + i/2 + 4*(i%2).
__global__ void prepare_fp4_kernel(int ternary, const uint8_t* __restrict__ panels, int n, int k, int np, int kp4,
                                   uint8_t* __restrict__ out, uint8_t* __restrict__ outr, uint8_t* __restrict__ outc) {
    const int db = (k + 7) / 8;
    const int chunks = kp4 / 32;
    const long long total = (long long)np * chunks;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int col = (int)(idx / chunks);
        const int ch = (int)(idx - (long long)col * chunks);
        uint32_t words[4] = {0, 0, 0, 0}, rwords[4] = {0, 0, 0, 0}, cwords[4] = {0, 0, 0, 0};
        if (col < n) {
            uint32_t pw = 0, mw = 0;  // the chunk's 32 plus / minus bits, element e at bit e
#pragma unroll
            for (int q = 0; q < 4; ++q) {  // 8 depth positions (one panel byte) per output word
                const int d = ch * 4 + q;
                if (d >= db) break;
                uint32_t p, m;
                if (ternary) {
                    p = panel_byte(panels, 1, db, col, d, 0);
                    m = panel_byte(panels, 1, db, col, d, 1);
                } else {
                    m = panel_byte(panels, 0, db, col, d, 0);
                    const int valid = k - d * 8 < 8 ? k - d * 8 : 8;
                    p = ~m & ((1u << valid) - 1u);
                }
                pw |= p << (8 * q);
                mw |= m << (8 * q);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint32_t w = 0, wr = 0, wc = 0;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int e = 8 * q + i, er = 4 * i + q, ec = 8 * q + (i >> 1) + 4 * (i & 1);
                    w |= (((pw >> e) & 1u) ? 0x2u : (((mw >> e) & 1u) ? 0xAu : 0x0u)) << (4 * i);
                    wr |= (((pw >> er) & 1u) ? 0x2u : (((mw >> er) & 1u) ? 0xAu : 0x0u)) << (4 * i);
                    wc |= (((pw >> ec) & 1u) ? 0x2u : (((mw >> ec) & 1u) ? 0xAu : 0x0u)) << (4 * i);
                }
                words[q] = w;
                rwords[q] = wr;
                cwords[q] = wc;
            }
        }
        reinterpret_cast<uint4*>(out + (size_t)col * (kp4 / 2))[ch] = make_uint4(words[0], words[1], words[2], words[3]);
        reinterpret_cast<uint4*>(outr + (size_t)col * (kp4 / 2))[ch] =
            make_uint4(rwords[0], rwords[1], rwords[2], rwords[3]);
        reinterpret_cast<uint4*>(outc + (size_t)col * (kp4 / 2))[ch] =
            make_uint4(cwords[0], cwords[1], cwords[2], cwords[3]);
    }
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void generate_kernel(int dist, uint64_t seed, int matrix_id, long long row0, long long rows,
                                long long cols, int8_t* __restrict__ out) {
    const uint64_t base = seed ^ ((uint64_t)(unsigned)matrix_id << 56);
    const long long total = rows * cols;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const uint64_t h = splitmix64(base ^ (uint64_t)(row0 * cols + i));
        int8_t v;
        if (dist == 0) v = (int8_t)((int)(((h >> 32) * 3ull) >> 32) - 1);
        else if (dist == 1) v = (h & 1ull) ? (int8_t)-1 : (int8_t)1;
        else {
            const unsigned u = (unsigned)(h & 3ull);
            v = u < 2 ? (int8_t)0 : (u == 2 ? (int8_t)1 : (int8_t)-1);
        }
        out[i] = v;
    }
}

}  // namespace lb

using namespace lb;

extern "C" lowbit_status lowbit_encode(int ternary, const int8_t* values, int rows, int cols, long long ld,
                                       uint8_t* plane0, uint8_t* plane1, long long pitch, int* zero_flag,
                                       lowbit_stream stream) {
    return lowbit_encode_ex(ternary, LOWBIT_LAYOUT_REFERENCE, values, rows, cols, ld, plane0, plane1, pitch,
                            zero_flag, stream);
}

extern "C" lowbit_status lowbit_encode_ex(int ternary, int layout, const int8_t* values, int rows, int cols,
                                          long long ld, uint8_t* plane0, uint8_t* plane1, long long pitch,
                                          int* zero_flag, lowbit_stream stream) {
    if (layout != LOWBIT_LAYOUT_REFERENCE && layout != LOWBIT_LAYOUT_LANES && layout != LOWBIT_LAYOUT_NIBBLES)
        return lbhost::set_error(LOWBIT_INVALID_ARGUMENT, "encode: unknown plane layout");
    if (rows < 0 || cols < 0) return lbhost::set_error(LOWBIT_INVALID_ARGUMENT, "encode: negative shape");
    if (rows == 0 || cols == 0) return LOWBIT_OK;
    if (!values || !plane0 || (ternary && !plane1))
        return lbhost::set_error(LOWBIT_INVALID_ARGUMENT, "encode: NULL pointer");
    if (ld < cols || pitch < (cols + 7) / 8 || (pitch & 3) || (reinterpret_cast<uintptr_t>(plane0) & 3) ||
        (ternary && (reinterpret_cast<uintptr_t>(plane1) & 3)))
        return lbhost::set_error(LOWBIT_INVALID_ARGUMENT, "encode: pitch must be >= ceil(cols/8) and 4-byte aligned");
    const long long work = (long long)rows * (pitch / 4);
    if (layout == LOWBIT_LAYOUT_REFERENCE)
        encode_kernel<0><<<grid_for(work, 256), 256, 0, (cudaStream_t)stream>>>(ternary, values, rows, cols, ld,
                                                                                 plane0, plane1, pitch, zero_flag);
    else if (layout == LOWBIT_LAYOUT_LANES)
        encode_kernel<1><<<grid_for(work, 256), 256, 0, (cudaStream_t)stream>>>(ternary, values, rows, cols, ld,
                                                                                 plane0, plane1, pitch, zero_flag);
    else
        encode_kernel<2><<<grid_for(work, 256), 256, 0, (cudaStream_t)stream>>>(ternary, values, rows, cols, ld,
                                                                                 plane0, plane1, pitch, zero_flag);
    LB_CUDA_TRY(cudaGetLastError());
    return LOWBIT_OK;
}

extern "C" size_t lowbit_packed_b_bytes(int ternary, int n, int k) {
    if (n <= 0 || k <= 0) return 0;
    return (size_t)((n + 7) / 8) * (ternary ? 16 : 8) * (size_t)((k + 7) / 8);
}

extern "C" lowbit_status lowbit_pack_b(int ternary, const uint8_t* b0, const uint8_t* b1, int k, int n,
                                       long long pitch, uint8_t* panels, lowbit_stream stream) {
    if (k <= 0 || n <= 0) return LOWBIT_OK;  // pack_b of an empty matrix has no panels
    if (!b0 || !panels || (ternary && !b1)) return lbhost::set_error(LOWBIT_INVALID_ARGUMENT, "pack_b: NULL pointer");
    if (pitch < (n + 7) / 8) return lbhost::set_error(LOWBIT_INVALID_ARGUMENT, "pack_b: pitch < ceil(n/8)");
    if (reinterpret_cast<uintptr_t>(panels) & 7)
        return lbhost::set_error(LOWBIT_INVALID_ARGUMENT, "pack_b: panels must be 8-byte aligned");
    const long long work = (long long)((n + 7) / 8) * ((k + 7) / 8);
    pack_b_kernel<<<grid_for(work, 256), 256, 0, (cudaStream_t)stream>>>(ternary, b0, b1, k, n, pitch, panels);
    LB_CUDA_TRY(cudaGetLastError());
    return LOWBIT_OK;
}

extern "C" size_t lowbit_weights_bytes(int ternary, int n, int k) {
    if (n <= 0 || k <= 0) return 0;
    return WeightsLayout(ternary, n, k).bytes;
}

extern "C" lowbit_status lowbit_prepare_weights(int ternary, const uint8_t* panels, int n, int k, void* weights,
                                                lowbit_stream stream) {
    if (n <= 0 || k <= 0) return lbhost::set_error(LOWBIT_OUT_OF_BOUNDS, "prepare_weights: empty B");
    if (!panels || !weights) return lbhost::set_error(LOWBIT_INVALID_ARGUMENT, "prepare_weights: NULL pointer");
    if (reinterpret_cast<uintptr_t>(weights) & 255)
        return lbhost::set_error(LOWBIT_INVALID_ARGUMENT, "prepare_weights: weights must be 256-byte aligned");
    const WeightsLayout L(ternary, n, k);
    uint8_t* base = static_cast<uint8_t*>(weights);
    cudaStream_t s = (cudaStream_t)stream;
    prepare_i8_kernel<<<grid_for((long long)L.np * (L.kp / 16), 256), 256, 0, s>>>(
        ternary, panels, n, k, L.np, L.kp, reinterpret_cast<int8_t*>(base));
    LB_CUDA_TRY(cudaGetLastError());
    prepare_fp4_kernel<<<grid_for((long long)L.np * (L.kp4 / 32), 256), 256, 0, s>>>(
        ternary, panels, n, k, L.np, L.kp4, base + L.off_fp4, base + L.off_fp4r, base + L.off_fp4c);
    LB_CUDA_TRY(cudaGetLastError());
    prepare_bits_kernel<<<grid_for((long long)L.np * L.kw, 256), 256, 0, s>>>(
        ternary, panels, n, k, L.np, L.kw, reinterpret_cast<uint32_t*>(base + L.off_sign),
        reinterpret_cast<uint32_t*>(base + L.off_nz));
    LB_CUDA_TRY(cudaGetLastError());
    return LOWBIT_OK;
}

extern "C" lowbit_status lowbit_generate(int dist, unsigned long long seed, int matrix_id, long long row0,
                                         long long rows, long long cols, int8_t* out, lowbit_stream stream) {
    if (rows <= 0 || cols <= 0) return LOWBIT_OK;
    if (!out) return lbhost::set_error(LOWBIT_INVALID_ARGUMENT, "generate: NULL pointer");
    generate_kernel<<<grid_for(rows * cols / 4 + 1, 256), 256, 0, (cudaStream_t)stream>>>(
        dist, seed, matrix_id, row0, rows, cols, out);
    LB_CUDA_TRY(cudaGetLastError());
    return LOWBIT_OK;
}
