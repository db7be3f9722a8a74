/*
 * lowbit_oracle.c — CPU restatement of the reference low-bit GeMM path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product in paper_2205_09120_b200/.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product path never links, loads or calls it.
 *
 * Parity pinning: every function below is checked (tests/test_oracle.py)
 * against (1) the known-answer vectors of the reference's own unit tests and
 * (2) golden fixtures under tests/golden/ that were produced by the reference
 * library itself, compiled from /root/reference/proj/src by oracle/Makefile
 * into oracle/_ref/ (see tests/golden/make_golden.py).
 *
 * Reference anchors are `proj/<file>:<line>` under /root/reference.
 *
 * Plain C99, single-threaded, no dependencies.
 */
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Status codes: the same numbering as include/lowbit_cuda.h (lowbit_status). */
enum {
    ORC_OK = 0,
    ORC_ERROR = 1,            /* plain lowbit::Error, e.g. bad k_blk (gemm.cpp:9-12) */
    ORC_ZERO_IN_BINARY = 2,   /* errors.hpp:12-14 */
    ORC_INVALID_CODE = 3,     /* errors.hpp:16-18 */
    ORC_OUT_OF_BOUNDS = 4,    /* errors.hpp:20-22 */
    ORC_DEPTH_OVERFLOW = 5,   /* errors.hpp:24-27 */
    ORC_MODE_MISMATCH = 6,    /* errors.hpp:29-31 */
    ORC_CHANNEL_OVERFLOW = 7, /* errors.hpp:33-37 */
    ORC_EMPTY_OUTPUT = 8,     /* errors.hpp:39-41 */
};

enum { ORC_BNN = 0, ORC_TNN = 1, ORC_TBN = 2 };              /* gemm.hpp:24 GemmMode order */
enum { ORC_BNN_A = 0, ORC_BNN_B = 1, ORC_TNN_A = 2, ORC_TNN_B = 3 }; /* pack.hpp:22 BlockMode */

#define ORC_K_MAX16 32767 /* kernels.hpp:24 kMaxDepth16 */

static int popc8(unsigned v) { return __builtin_popcount(v & 0xFFu); }

/* ------------------------------------------------------------------------ */
/* Seeded counter-based generator shared with the GPU generator kernel.     */
/* value(seed, matrix_id, r, c) = f(splitmix64(seed ^ id<<56 ^ (r*cols+c))) */
/* (SURVEY.md §8d).  Not part of the reference; it replaces mt19937 so that */
/* any shard of any config can be regenerated independently on CPU or GPU.  */
/* ------------------------------------------------------------------------ */
uint64_t orc_splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* dist 0: uniform {-1,0,+1}; 1: uniform {-1,+1}; 2: P(0)=.5, P(+-1)=.25 */
static int8_t gen_value(int dist, uint64_t h) {
    switch (dist) {
        case 0: return (int8_t)((int)((((h >> 32) * 3ull) >> 32)) - 1);
        case 1: return (h & 1ull) ? (int8_t)-1 : (int8_t)1;
        default: {
            unsigned u = (unsigned)(h & 3ull);
            return u < 2 ? (int8_t)0 : (u == 2 ? (int8_t)1 : (int8_t)-1);
        }
    }
}

/* Fill rows [row0, row0+nrows) of a logical rows x cols matrix (row-major). */
void orc_generate(int dist, uint64_t seed, int matrix_id, long long row0, long long nrows,
                  long long cols, int8_t* out) {
    uint64_t base = seed ^ ((uint64_t)(unsigned)matrix_id << 56);
    for (long long r = 0; r < nrows; ++r)
        for (long long c = 0; c < cols; ++c) {
            uint64_t idx = (uint64_t)(row0 + r) * (uint64_t)cols + (uint64_t)c;
            out[r * cols + c] = gen_value(dist, orc_splitmix64(base ^ idx));
        }
}

/* ------------------------------------------------------------------------ */
/* Encodings (core.cpp)                                                      */
/* ------------------------------------------------------------------------ */
int orc_stride_bytes(int cols) { return ((cols + 7) & ~7) / 8; } /* core.cpp:9 stride_for */

/* encode_binary, core.cpp:13-28: -1 -> bit 1, +1 -> bit 0, 0 -> ZeroInBinaryInput. */
int orc_encode_binary(const int8_t* v, int rows, int cols, uint8_t* plane) {
    int sb = orc_stride_bytes(cols);
    memset(plane, 0, (size_t)rows * sb);
    for (int r = 0; r < rows; ++r) {
        uint8_t* dst = plane + (size_t)r * sb;
        for (int c = 0; c < cols; ++c) {
            int8_t x = v[(size_t)r * cols + c];
            if (x == 0) return ORC_ZERO_IN_BINARY; /* core.cpp:23 */
            if (x < 0) dst[c >> 3] |= (uint8_t)(1u << (c & 7));
        }
    }
    return ORC_OK;
}

/* encode_ternary, core.cpp:40-58: +1 -> plus bit, -1 -> minus bit. */
int orc_encode_ternary(const int8_t* v, int rows, int cols, uint8_t* plus, uint8_t* minus) {
    int sb = orc_stride_bytes(cols);
    memset(plus, 0, (size_t)rows * sb);
    memset(minus, 0, (size_t)rows * sb);
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) {
            int8_t x = v[(size_t)r * cols + c];
            uint8_t bit = (uint8_t)(1u << (c & 7));
            if (x > 0) plus[(size_t)r * sb + (c >> 3)] |= bit;
            if (x < 0) minus[(size_t)r * sb + (c >> 3)] |= bit;
        }
    return ORC_OK;
}

/* decode_binary / decode_ternary, core.cpp:30-38, 60-71. */
void orc_decode_binary(const uint8_t* plane, int rows, int cols, int8_t* out) {
    int sb = orc_stride_bytes(cols);
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c)
            out[(size_t)r * cols + c] = ((plane[(size_t)r * sb + (c >> 3)] >> (c & 7)) & 1) ? -1 : 1;
}

void orc_decode_ternary(const uint8_t* plus, const uint8_t* minus, int rows, int cols, int8_t* out) {
    int sb = orc_stride_bytes(cols);
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) {
            size_t o = (size_t)r * sb + (c >> 3);
            int p = (plus[o] >> (c & 7)) & 1, n = (minus[o] >> (c & 7)) & 1;
            out[(size_t)r * cols + c] = (int8_t)(p - n);
        }
}

/* ------------------------------------------------------------------------ */
/* Block packing (pack.cpp)                                                  */
/* ------------------------------------------------------------------------ */
int orc_block_group_bytes(int block_mode) { /* pack.cpp:36-44 */
    static const int g[4] = {16, 8, 32, 16};
    return (block_mode >= 0 && block_mode < 4) ? g[block_mode] : 0;
}

static uint8_t tail_mask(int k_eff, int d) { /* pack.cpp:14-18 */
    int rem = k_eff - d * 8;
    return rem >= 8 ? 0xFF : (uint8_t)((1u << rem) - 1);
}

/* gather_col_byte, pack.cpp:22-32: the bit transpose of a K x N plane. */
static uint8_t gather_col_byte(const uint8_t* plane, int sb, int rows_lim, int cols, int t0, int c) {
    if (c >= cols) return 0;
    uint8_t out = 0;
    int lim = rows_lim - t0 < 8 ? rows_lim - t0 : 8;
    for (int j = 0; j < lim; ++j)
        out |= (uint8_t)(((plane[(size_t)(t0 + j) * sb + (c >> 3)] >> (c & 7)) & 1u) << j);
    return out;
}

/* pack.cpp:7-11 */
static int check_depth(int cols, int depth_start, int k_eff) {
    if (depth_start < 0 || (depth_start & 7) != 0) return ORC_OUT_OF_BOUNDS;
    if (k_eff < 1 || depth_start + k_eff > cols) return ORC_OUT_OF_BOUNDS;
    return ORC_OK;
}

/*
 * Block packers pack_{a,b}_{binary,ternary} (pack.cpp:46-127).
 * A matrix: rows x cols planes (row stride ceil(cols/8)); start = row_start.
 * B matrix: rows(=depth) x cols planes; start = col_start.
 * out receives group*ceil(k_eff/8) bytes; *lanes receives the lane count.
 */
int orc_pack_block(int block_mode, const uint8_t* p0, const uint8_t* p1, int rows, int cols,
                   int start, int depth_start, int k_eff, uint8_t* out, int* lanes) {
    int is_a = block_mode == ORC_BNN_A || block_mode == ORC_TNN_A;
    int st = check_depth(is_a ? cols : rows, depth_start, k_eff);
    if (st) return st;
    if (start < 0 || start >= (is_a ? rows : cols)) return ORC_OUT_OF_BOUNDS;
    int sb = orc_stride_bytes(cols);
    int group = orc_block_group_bytes(block_mode);
    int db = (k_eff + 7) / 8;
    int ln = is_a ? (rows - start < 16 ? rows - start : 16) : (cols - start < 8 ? cols - start : 8);
    *lanes = ln;
    memset(out, 0, (size_t)group * db);
    int db0 = depth_start / 8;
    for (int d = 0; d < db; ++d) {
        uint8_t* dst = out + (size_t)d * group;
        if (block_mode == ORC_BNN_A) { /* pack.cpp:46-62 */
            uint8_t mask = tail_mask(k_eff, d);
            for (int i = 0; i < ln; ++i) dst[i] = (uint8_t)(p0[(size_t)(start + i) * sb + db0 + d] & mask);
        } else if (block_mode == ORC_TNN_A) { /* pack.cpp:83-104 */
            uint8_t mask = tail_mask(k_eff, d);
            for (int i = 0; i < ln; ++i) {
                int half = i / 8, sub = i % 8;
                dst[half * 16 + sub] = (uint8_t)(p0[(size_t)(start + i) * sb + db0 + d] & mask);
                dst[half * 16 + 8 + sub] = (uint8_t)(p1[(size_t)(start + i) * sb + db0 + d] & mask);
            }
        } else { /* pack.cpp:64-81, 106-127 */
            int t0 = depth_start + d * 8, lim = depth_start + k_eff;
            for (int j = 0; j < ln; ++j) {
                if (block_mode == ORC_BNN_B) {
                    dst[j] = gather_col_byte(p0, sb, lim, cols, t0, start + j);
                } else {
                    dst[2 * j] = gather_col_byte(p0, sb, lim, cols, t0, start + j);
                    dst[2 * j + 1] = gather_col_byte(p1, sb, lim, cols, t0, start + j);
                }
            }
        }
    }
    return ORC_OK;
}

/*
 * pack_b (gemm.cpp:59-77): one full-depth panel per 8 columns, concatenated.
 * b_ternary selects tnn_b (plus,minus) vs bnn_b (one plane).
 * out size: ceil(n/8) * group * ceil(k/8) bytes.
 */
size_t orc_packed_b_bytes(int b_ternary, int n, int k) {
    return (size_t)((n + 7) / 8) * (b_ternary ? 16 : 8) * (size_t)((k + 7) / 8);
}

int orc_pack_b(int b_ternary, const uint8_t* p0, const uint8_t* p1, int k, int n, uint8_t* out) {
    int mode = b_ternary ? ORC_TNN_B : ORC_BNN_B;
    size_t panel = (size_t)orc_block_group_bytes(mode) * ((k + 7) / 8);
    int lanes;
    for (int c = 0, p = 0; c < n; c += 8, ++p) {
        int st = orc_pack_block(mode, p0, p1, k, n, c, 0, k, out + p * panel, &lanes);
        if (st) return st;
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* 16x8 tiles (kernels.cpp:31-126), restated on depth bytes.                 */
/* tile[i*8+j] += contribution of depth bytes [0, db) of the given blocks.   */
/* ------------------------------------------------------------------------ */
static void bnn_tile(const uint8_t* a, const uint8_t* b, int db, int k_eff, int16_t* tile) {
    for (int i = 0; i < 16; ++i)
        for (int j = 0; j < 8; ++j) {
            int pc = 0;
            for (int d = 0; d < db; ++d) pc += popc8(a[d * 16 + i] ^ b[d * 8 + j]);
            tile[i * 8 + j] = (int16_t)(tile[i * 8 + j] + k_eff - 2 * pc); /* kernels.cpp:49 */
        }
}

static void tnn_tile(const uint8_t* a, const uint8_t* b, int db, int16_t* tile) {
    for (int i = 0; i < 16; ++i) {
        int half = i >> 3, sub = i & 7;
        for (int j = 0; j < 8; ++j) {
            int s = 0;
            for (int d = 0; d < db; ++d) {
                unsigned ap = a[d * 32 + half * 16 + sub], am = a[d * 32 + half * 16 + 8 + sub];
                unsigned bp = b[d * 16 + 2 * j], bm = b[d * 16 + 2 * j + 1];
                unsigned zp = (ap & bp) | (am & bm), zm = (ap & bm) | (am & bp); /* kernels.cpp:83-84 */
                s += popc8(zp) - popc8(zm);
            }
            tile[i * 8 + j] = (int16_t)(tile[i * 8 + j] + s);
        }
    }
}

static void tbn_tile(const uint8_t* a, const uint8_t* b, int db, int16_t* tile) {
    for (int i = 0; i < 16; ++i) {
        int half = i >> 3, sub = i & 7;
        int nnz = 0; /* hoisted per row, kernels.cpp:112-115 */
        for (int d = 0; d < db; ++d) nnz += popc8(a[d * 32 + half * 16 + sub] | a[d * 32 + half * 16 + 8 + sub]);
        for (int j = 0; j < 8; ++j) {
            int plus = 0;
            for (int d = 0; d < db; ++d) {
                unsigned ap = a[d * 32 + half * 16 + sub], am = a[d * 32 + half * 16 + 8 + sub];
                unsigned bb = b[d * 8 + j];
                plus += popc8((ap & ~bb) | (am & bb)); /* kernels.cpp:120 */
            }
            tile[i * 8 + j] = (int16_t)(tile[i * 8 + j] + 2 * plus - nnz);
        }
    }
}

/* ------------------------------------------------------------------------ */
/* gemm_lowbit (gemm.cpp:79-112) with drive() (gemm.cpp:24-55).              */
/* A planes: a_rows x a_cols, stride ceil(a_cols/8).  a1 = minus plane for    */
/* ternary A, ignored for binary A.  pb = pack_b output; pb_ternary selects   */
/* tnn_b vs bnn_b.  Error checks in the reference order.                      */
/* ------------------------------------------------------------------------ */
int orc_check_gemm(int mode, int a_ternary, int pb_ternary, int a_rows, int a_cols, int pb_n, int pb_k,
                   int m, int n, int k, int k_blk) {
    if (k_blk < 8 || (k_blk & 7) != 0) return ORC_ERROR; /* check_cfg gemm.cpp:9-12 */
    if (!a_ternary) {                                    /* gemm.cpp:81-84 */
        if (mode != ORC_BNN) return ORC_MODE_MISMATCH;
        if (pb_ternary) return ORC_MODE_MISMATCH;
    } else { /* gemm.cpp:94-99 */
        if (mode == ORC_BNN) return ORC_MODE_MISMATCH;
        if (mode == ORC_TNN && !pb_ternary) return ORC_MODE_MISMATCH;
        if (mode == ORC_TBN && pb_ternary) return ORC_MODE_MISMATCH;
    }
    /* check_dims gemm.cpp:14-19 */
    if (m <= 0 || n <= 0 || k <= 0) return ORC_OUT_OF_BOUNDS;
    if (a_rows != m || a_cols != k) return ORC_OUT_OF_BOUNDS;
    if (pb_k != k || pb_n != n) return ORC_OUT_OF_BOUNDS;
    if (k > ORC_K_MAX16) return ORC_DEPTH_OVERFLOW;
    return ORC_OK;
}

int orc_gemm_lowbit(int mode, int a_ternary, const uint8_t* a0, const uint8_t* a1, int a_rows, int a_cols,
                    int pb_ternary, const uint8_t* pb, int pb_n, int pb_k, int m, int n, int k, int k_blk,
                    int16_t* c) {
    int st = orc_check_gemm(mode, a_ternary, pb_ternary, a_rows, a_cols, pb_n, pb_k, m, n, k, k_blk);
    if (st) return st;
    int bmode = pb_ternary ? ORC_TNN_B : ORC_BNN_B;
    int amode = a_ternary ? ORC_TNN_A : ORC_BNN_A;
    int group_b = orc_block_group_bytes(bmode), group_a = orc_block_group_bytes(amode);
    size_t panel = (size_t)group_b * ((k + 7) / 8);
    uint8_t* ablock = (uint8_t*)malloc((size_t)group_a * ((k_blk + 7) / 8));
    if (!ablock) return ORC_ERROR;
    memset(c, 0, (size_t)m * n * sizeof(int16_t)); /* gemm.cpp:30 */
    for (int d = 0; d < k; d += k_blk) {           /* depth slice, gemm.cpp:32 */
        int k_eff = k_blk < k - d ? k_blk : k - d;
        int db = (k_eff + 7) / 8;
        for (int r = 0; r < m; r += 16) { /* gemm.cpp:35 */
            int lanes;
            orc_pack_block(amode, a0, a1, m, k, r, d, k_eff, ablock, &lanes);
            int m_e = m - r < 16 ? m - r : 16;
            for (int cg = 0; cg < n; cg += 8) { /* gemm.cpp:38 */
                const uint8_t* bptr = pb + (size_t)(cg / 8) * panel + (size_t)(d / 8) * group_b;
                int16_t tile[128];
                memset(tile, 0, sizeof tile);
                if (mode == ORC_BNN) bnn_tile(ablock, bptr, db, k_eff, tile);
                else if (mode == ORC_TNN) tnn_tile(ablock, bptr, db, tile);
                else tbn_tile(ablock, bptr, db, tile);
                int n_e = n - cg < 8 ? n - cg : 8;
                for (int i = 0; i < m_e; ++i) /* masked writeback gemm.cpp:43-50 */
                    for (int j = 0; j < n_e; ++j) {
                        int16_t* e = c + (size_t)(r + i) * n + cg + j;
                        *e = (int16_t)(*e + tile[i * 8 + j]);
                    }
            }
        }
    }
    free(ablock);
    return ORC_OK;
}

/* dot_binary, kernels.cpp:8-16. */
int orc_dot_binary(const uint8_t* a, const uint8_t* b, int nbytes, int k_logical, int16_t* out) {
    if (k_logical > ORC_K_MAX16) return ORC_DEPTH_OVERFLOW;
    int pc = 0;
    for (int i = 0; i < nbytes; ++i) pc += popc8(a[i] ^ b[i]);
    *out = (int16_t)(k_logical - 2 * pc);
    return ORC_OK;
}

/* reference_gemm_int, gemm.cpp:210-223: naive int32 triple loop, skips zero A. */
void orc_reference_gemm_int(const int8_t* a, const int8_t* b, int m, int n, int k, int32_t* c) {
    memset(c, 0, (size_t)m * n * sizeof(int32_t));
    for (int i = 0; i < m; ++i)
        for (int t = 0; t < k; ++t) {
            int av = a[(size_t)i * k + t];
            if (av == 0) continue;
            const int8_t* brow = b + (size_t)t * n;
            int32_t* crow = c + (size_t)i * n;
            for (int j = 0; j < n; ++j) crow[j] += av * brow[j];
        }
}

/* k_max family, gemm.cpp:198-208. */
long long orc_k_max(int p, int q) {
    unsigned long long acc_max = (q >= 64) ? ~0ull : ((1ull << q) - 1);
    unsigned long long prod = ((1ull << p) - 1) * ((1ull << p) - 1);
    return (long long)(acc_max / prod);
}
long long orc_k_max_sign(int q) { return (long long)((1ull << (q - 1)) - 1); }
long long orc_c_in_max(long long k_max, int kh, int kw) { return k_max / ((long long)kh * kw); }

/* ------------------------------------------------------------------------ */
/* Convolution (conv.cpp)                                                    */
/* ------------------------------------------------------------------------ */
int orc_conv_out_dim(int in, int kernel, int stride, int padding) { /* conv.cpp:5-7 */
    return (in + 2 * padding - kernel) / stride + 1;
}

/* im2col, conv.cpp:9-31: row = oy*ow+ox, col = (ky*kw+kx)*C + c. fm is HWC. */
int orc_im2col(const int8_t* fm, int h, int w, int ch, int fm_binary, int kh, int kw, int stride,
               int padding, int binary_pad_value, int8_t* out) {
    int oh = orc_conv_out_dim(h, kh, stride, padding), ow = orc_conv_out_dim(w, kw, stride, padding);
    if (oh < 1 || ow < 1) return ORC_EMPTY_OUTPUT;
    int8_t pad = fm_binary ? (int8_t)binary_pad_value : (int8_t)0;
    int kcols = kh * kw * ch;
    for (int oy = 0; oy < oh; ++oy)
        for (int ox = 0; ox < ow; ++ox) {
            int8_t* row = out + (size_t)(oy * ow + ox) * kcols;
            int col = 0;
            for (int ky = 0; ky < kh; ++ky) {
                int y = oy * stride + ky - padding;
                for (int kx = 0; kx < kw; ++kx) {
                    int x = ox * stride + kx - padding;
                    int inside = y >= 0 && y < h && x >= 0 && x < w;
                    for (int c = 0; c < ch; ++c, ++col)
                        row[col] = inside ? fm[((size_t)y * w + x) * ch + c] : pad;
                }
            }
        }
    return ORC_OK;
}

/*
 * conv2d_lowbit, conv.cpp:33-59, as im2col + encode + pack_b + gemm_lowbit,
 * widened to int32.  weights: (kh*kw*ch) x cout sign matrix.
 * fm_binary / w_binary are the SignMatrix / FeatureMap modes.
 */
int orc_conv2d_lowbit(int mode, const int8_t* fm, int h, int w, int ch, int fm_binary, const int8_t* wts,
                      int w_rows, int w_cols, int w_binary, int kh, int kw, int stride, int padding,
                      int cout, int binary_pad_value, int32_t* out) {
    long long k = (long long)kh * kw * ch;
    if (k > ORC_K_MAX16) return ORC_CHANNEL_OVERFLOW; /* conv.cpp:35-37 */
    if (w_rows != k || w_cols != cout) return ORC_OUT_OF_BOUNDS;
    int a_binary = mode == ORC_BNN, b_binary = mode != ORC_TNN;
    if (a_binary && !fm_binary) return ORC_MODE_MISMATCH;
    if (b_binary && !w_binary) return ORC_MODE_MISMATCH;
    if (!b_binary && w_binary) return ORC_MODE_MISMATCH;
    int oh = orc_conv_out_dim(h, kh, stride, padding), ow = orc_conv_out_dim(w, kw, stride, padding);
    if (oh < 1 || ow < 1) return ORC_EMPTY_OUTPUT;
    int m = oh * ow, kk = (int)k, sb = orc_stride_bytes(kk), sbn = orc_stride_bytes(cout);
    int8_t* cols = (int8_t*)malloc((size_t)m * kk);
    uint8_t* a0 = (uint8_t*)malloc((size_t)m * sb);
    uint8_t* a1 = (uint8_t*)malloc((size_t)m * sb);
    uint8_t* b0 = (uint8_t*)malloc((size_t)kk * sbn);
    uint8_t* b1 = (uint8_t*)malloc((size_t)kk * sbn);
    uint8_t* pb = (uint8_t*)malloc(orc_packed_b_bytes(!b_binary, cout, kk));
    int16_t* c16 = (int16_t*)malloc((size_t)m * cout * sizeof(int16_t));
    int st = ORC_ERROR;
    if (cols && a0 && a1 && b0 && b1 && pb && c16) {
        orc_im2col(fm, h, w, ch, fm_binary, kh, kw, stride, padding, binary_pad_value, cols);
        st = b_binary ? orc_encode_binary(wts, kk, cout, b0) : orc_encode_ternary(wts, kk, cout, b0, b1);
        if (!st) st = orc_pack_b(!b_binary, b0, b1, kk, cout, pb);
        if (!st) st = a_binary ? orc_encode_binary(cols, m, kk, a0) : orc_encode_ternary(cols, m, kk, a0, a1);
        if (!st)
            st = orc_gemm_lowbit(mode, !a_binary, a0, a1, m, kk, !b_binary, pb, cout, kk, m, cout, kk, 4096, c16);
        if (!st)
            for (size_t i = 0; i < (size_t)m * cout; ++i) out[i] = c16[i]; /* conv.cpp:57 */
    }
    free(cols); free(a0); free(a1); free(b0); free(b1); free(pb); free(c16);
    return st;
}

/* 6-loop direct convolution (the test oracle of test_conv.cpp:22-47). */
void orc_direct_conv(const int8_t* fm, int h, int w, int ch, int fm_binary, const int8_t* wts, int kh, int kw,
                     int stride, int padding, int cout, int binary_pad_value, int32_t* out) {
    int oh = orc_conv_out_dim(h, kh, stride, padding), ow = orc_conv_out_dim(w, kw, stride, padding);
    int8_t pad = fm_binary ? (int8_t)binary_pad_value : (int8_t)0;
    for (int oy = 0; oy < oh; ++oy)
        for (int ox = 0; ox < ow; ++ox)
            for (int f = 0; f < cout; ++f) {
                int32_t s = 0;
                for (int ky = 0; ky < kh; ++ky)
                    for (int kx = 0; kx < kw; ++kx)
                        for (int c = 0; c < ch; ++c) {
                            int y = oy * stride + ky - padding, x = ox * stride + kx - padding;
                            int8_t v = (y >= 0 && y < h && x >= 0 && x < w) ? fm[((size_t)y * w + x) * ch + c] : pad;
                            s += v * wts[(size_t)((ky * kw + kx) * ch + c) * cout + f];
                        }
                out[((size_t)oy * ow + ox) * cout + f] = s;
            }
}
