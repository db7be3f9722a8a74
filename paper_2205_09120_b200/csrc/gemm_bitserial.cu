// gemm_bitserial.cu — K2: the bit-serial low-bit GeMM (LOP3 + POPC on the
// integer pipes), replacing detail::{bnn,tnn,tbn}_tile (kernels.cpp:31-126)
// and the Algorithm-2 driver (gemm.cpp:24-55).
//
// Device-internal form: every operand is a pair of
// K-major bit words (nz, sign); binary operands have nz == all-ones within K.
//   BNN:  C = K - 2 * sum popc(sA ^ sB)                         (kernels.cpp:49)
//   TNN:  C = sum popc(nzA & nzB) - 2 * sum popc(nzA & nzB & (sA ^ sB))
//         == popc(z+) - popc(z-)                                 (kernels.cpp:83-87)
//   TBN:  C = nnz(A_i) - 2 * sum popc(nzA & (sA ^ bB))           (kernels.cpp:114-123)
// int32 register accumulators, narrowed to int16 at the store (exact:
// |C| <= K <= 32767, gemm.cpp:18).
//
// Tiling: CTA 128 x 128 outputs, 256 threads, 8 x 8 outputs per thread laid
// out as two 4-wide groups per dimension (conflict-free 128-bit LDS).  Depth
// advances 8 words (256 bits) per stage; global -> register -> shared double
// buffering; A arrives as the reference plus/minus (or binary) planes and is
// turned into (nz, sign) on the way into shared memory.
#include "common.cuh"
#include "layout.cuh"

namespace lb {

constexpr int K2_BM = 128, K2_BN = 128, K2_KC = 8, K2_LD = 132;  // K2_LD: padded row length (words)
// Depth words unrolled per step of the inner loop.  Fully unrolled, TNN's four
// operand sets for all 8 words hoist into 255 registers and spill (1 CTA per
// SM); not unrolled it takes 128 registers, 2 CTAs per SM: c5-shaped TNN 129.9
// -> 141.0 TOPS, 0.947 of the TNN POPC peak (unroll 2: 177 registers, 129.2;
// tools/k2_time.py).  BNN / TBN stay fully unrolled (126 / 172 registers).
#ifndef K2_TNN_UNROLL
#define K2_TNN_UNROLL 1
#endif

template <int MODE>  // 0 = BNN, 1 = TNN, 2 = TBN
__global__ void __launch_bounds__(256) gemm_bitserial_kernel(const uint8_t* __restrict__ a0,
                                                             const uint8_t* __restrict__ a1, long long a_pitch,
                                                             int m, int n, int k,
                                                             const uint32_t* __restrict__ b_sign,
                                                             const uint32_t* __restrict__ b_nz, int kw,
                                                             int16_t* __restrict__ c, long long ldc) {
    constexpr bool A_TER = MODE != 0;
    constexpr bool B_TER = MODE == 1;
    constexpr int UW = MODE == 1 ? K2_TNN_UNROLL : K2_KC;
    __shared__ __align__(16) uint32_t As_s[2][K2_KC][K2_LD];
    __shared__ __align__(16) uint32_t As_n[A_TER ? 2 : 1][K2_KC][K2_LD];
    __shared__ __align__(16) uint32_t Bs_s[2][K2_KC][K2_LD];
    __shared__ __align__(16) uint32_t Bs_n[B_TER ? 2 : 1][K2_KC][K2_LD];

    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    const int m0 = blockIdx.y * K2_BM, n0 = blockIdx.x * K2_BN;
    const int kwords = (k + 31) / 32;
    const int nstages = (kwords + K2_KC - 1) / K2_KC;
    const long long a_words = a_pitch / 4;

    // loader mapping: 128 rows x 8 words = 256 threads x one uint4
    const int lrow = tid >> 1, lq = (tid & 1) * 4;

    uint4 ra_s, ra_n, rb_s, rb_n;
    auto load_global = [&](int st) {
        const int w0 = st * K2_KC + lq;  // first word of this thread's quad
        // ---- A (reference layout: row-major planes, pitch multiple of 16) ----
        uint4 p = make_uint4(0, 0, 0, 0), q = make_uint4(0, 0, 0, 0);
        const int row = m0 + lrow;
        if (row < m && w0 < a_words) {
            const uint4* src0 = reinterpret_cast<const uint4*>(a0 + (long long)row * a_pitch) + (w0 >> 2);
            p = __ldg(src0);
            if (A_TER) q = __ldg(reinterpret_cast<const uint4*>(a1 + (long long)row * a_pitch) + (w0 >> 2));
        }
        // mask depth tail (bits >= k), like tail_mask (pack.cpp:14-18)
        uint32_t pw[4] = {p.x, p.y, p.z, p.w}, qw[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int bit0 = (w0 + j) * 32;
            const uint32_t mask = bit0 >= k ? 0u : (k - bit0 >= 32 ? 0xFFFFFFFFu : ((1u << (k - bit0)) - 1u));
            pw[j] &= mask;
            qw[j] &= mask;
        }
        if (A_TER) {  // (plus, minus) -> (nz, sign)
            ra_s = make_uint4(qw[0], qw[1], qw[2], qw[3]);
            ra_n = make_uint4(pw[0] | qw[0], pw[1] | qw[1], pw[2] | qw[2], pw[3] | qw[3]);
        } else {
            ra_s = make_uint4(pw[0], pw[1], pw[2], pw[3]);
        }
        // ---- B (prepared: column-major words, kw a multiple of 8) ----
        const long long boff = (long long)(n0 + lrow) * kw + w0;
        rb_s = __ldg(reinterpret_cast<const uint4*>(b_sign + boff));
        if (B_TER) rb_n = __ldg(reinterpret_cast<const uint4*>(b_nz + boff));
    };
    auto store_shared = [&](int buf) {
        As_s[buf][lq + 0][lrow] = ra_s.x;
        As_s[buf][lq + 1][lrow] = ra_s.y;
        As_s[buf][lq + 2][lrow] = ra_s.z;
        As_s[buf][lq + 3][lrow] = ra_s.w;
        if (A_TER) {
            As_n[buf][lq + 0][lrow] = ra_n.x;
            As_n[buf][lq + 1][lrow] = ra_n.y;
            As_n[buf][lq + 2][lrow] = ra_n.z;
            As_n[buf][lq + 3][lrow] = ra_n.w;
        }
        Bs_s[buf][lq + 0][lrow] = rb_s.x;
        Bs_s[buf][lq + 1][lrow] = rb_s.y;
        Bs_s[buf][lq + 2][lrow] = rb_s.z;
        Bs_s[buf][lq + 3][lrow] = rb_s.w;
        if (B_TER) {
            Bs_n[buf][lq + 0][lrow] = rb_n.x;
            Bs_n[buf][lq + 1][lrow] = rb_n.y;
            Bs_n[buf][lq + 2][lrow] = rb_n.z;
            Bs_n[buf][lq + 3][lrow] = rb_n.w;
        }
    };

    int acc[8][8];
    int nnz[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        nnz[i] = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0;
    }

    if (nstages > 0) {
        load_global(0);
        store_shared(0);
    }
    __syncthreads();
    for (int st = 0; st < nstages; ++st) {
        const int buf = st & 1;
        if (st + 1 < nstages) load_global(st + 1);
#pragma unroll UW
        for (int w = 0; w < K2_KC; ++w) {
            uint32_t as[8], an[8], bs[8], bn[8];
            *reinterpret_cast<uint4*>(&as[0]) = *reinterpret_cast<const uint4*>(&As_s[buf][w][ty * 4]);
            *reinterpret_cast<uint4*>(&as[4]) = *reinterpret_cast<const uint4*>(&As_s[buf][w][64 + ty * 4]);
            *reinterpret_cast<uint4*>(&bs[0]) = *reinterpret_cast<const uint4*>(&Bs_s[buf][w][tx * 4]);
            *reinterpret_cast<uint4*>(&bs[4]) = *reinterpret_cast<const uint4*>(&Bs_s[buf][w][64 + tx * 4]);
            if (A_TER) {
                *reinterpret_cast<uint4*>(&an[0]) = *reinterpret_cast<const uint4*>(&As_n[buf][w][ty * 4]);
                *reinterpret_cast<uint4*>(&an[4]) = *reinterpret_cast<const uint4*>(&As_n[buf][w][64 + ty * 4]);
            }
            if (B_TER) {
                *reinterpret_cast<uint4*>(&bn[0]) = *reinterpret_cast<const uint4*>(&Bs_n[buf][w][tx * 4]);
                *reinterpret_cast<uint4*>(&bn[4]) = *reinterpret_cast<const uint4*>(&Bs_n[buf][w][64 + tx * 4]);
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (MODE == 2) nnz[i] += __popc(an[i]);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (MODE == 0) {
                        acc[i][j] += __popc(as[i] ^ bs[j]);
                    } else if (MODE == 1) {
                        const uint32_t mm = an[i] & bn[j];
                        acc[i][j] += __popc(mm) - 2 * __popc(mm & (as[i] ^ bs[j]));
                    } else {
                        acc[i][j] += __popc(an[i] & (as[i] ^ bs[j]));
                    }
                }
            }
        }
        if (st + 1 < nstages) store_shared(buf ^ 1);
        __syncthreads();
    }

    // epilogue: finish the mode formula, narrow to int16, store 4-wide groups
    const bool vec_ok = ((ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(c) & 7) == 0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int row = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
        if (row >= m) continue;
#pragma unroll
        for (int g = 0; g < 2; ++g) {
            const int col0 = n0 + g * 64 + tx * 4;
            int v[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int a = acc[i][g * 4 + j];
                v[j] = MODE == 0 ? k - 2 * a : (MODE == 1 ? a : nnz[i] - 2 * a);
            }
            int16_t* dst = c + (long long)row * ldc + col0;
            if (vec_ok && col0 + 4 <= n) {
                const uint32_t lo = (uint32_t)(v[0] & 0xFFFF) | ((uint32_t)v[1] << 16);
                const uint32_t hi = (uint32_t)(v[2] & 0xFFFF) | ((uint32_t)v[3] << 16);
                *reinterpret_cast<uint2*>(dst) = make_uint2(lo, hi);
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (col0 + j < n) dst[j] = (int16_t)v[j];
            }
        }
    }
}

lowbit_status launch_bitserial(int mode, const uint8_t* a0, const uint8_t* a1, long long a_pitch, int m, int n,
                               int k, const void* weights, int b_ternary, int16_t* c, long long ldc,
                               cudaStream_t stream) {
    const WeightsLayout L(b_ternary, n, k);
    const uint8_t* base = static_cast<const uint8_t*>(weights);
    const uint32_t* bs = reinterpret_cast<const uint32_t*>(base + L.off_sign);
    const uint32_t* bn = reinterpret_cast<const uint32_t*>(base + L.off_nz);
    dim3 grid((n + K2_BN - 1) / K2_BN, (m + K2_BM - 1) / K2_BM);
    if (grid.y > 65535) return lbhost::set_error(LOWBIT_INVALID_ARGUMENT, "bitserial: m too large for grid");
    switch (mode) {
        case 0:
            gemm_bitserial_kernel<0><<<grid, 256, 0, stream>>>(a0, a1, a_pitch, m, n, k, bs, bn, L.kw, c, ldc);
            break;
        case 1:
            gemm_bitserial_kernel<1><<<grid, 256, 0, stream>>>(a0, a1, a_pitch, m, n, k, bs, bn, L.kw, c, ldc);
            break;
        default:
            gemm_bitserial_kernel<2><<<grid, 256, 0, stream>>>(a0, a1, a_pitch, m, n, k, bs, bn, L.kw, c, ldc);
            break;
    }
    LB_CUDA_TRY(cudaGetLastError());
    return LOWBIT_OK;
}

}  // namespace lb
