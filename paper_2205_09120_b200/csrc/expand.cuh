// expand.cuh — bit planes -> int8 UMMA operand rows (converter warps of K3).
#pragma once
#include "common.cuh"

namespace lb {

// One converter thread: A row r, raw bytes [8h, 8h+8) of the row's 16-byte
// k-block chunk (64 elements) -> int8 UMMA chunks 4h..4h+3 (16 B each) of the
// K-major 128B-swizzled tile.  ~2 integer ops per element:
//   nibble isolate (PRMT) -> spread4 (IMAD+LOP) -> minus*0xFF + plus (IMAD).
// 32 raw bits of each plane (one word) -> two 16-byte UMMA chunks (ch0, ch0+1).
template <bool A_TER, int DBG = 0>
__device__ __forceinline__ void expand_word(uint32_t pw, uint32_t mw, uint32_t row, int sw, int ch0) {
    {
        const uint32_t p_lo = pw & 0x0F0F0F0Fu, p_hi = (pw >> 4) & 0x0F0F0F0Fu;
        const uint32_t m_lo = mw & 0x0F0F0F0Fu, m_hi = (mw >> 4) & 0x0F0F0F0Fu;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            uint32_t w[4];
#pragma unroll
            for (int bb = 0; bb < 2; ++bb) {
                const uint32_t sel = 0x4440u | (uint32_t)(2 * c + bb);
                const uint32_t P0 = spread4(__byte_perm(p_lo, 0, sel));
                const uint32_t P1 = spread4(__byte_perm(p_hi, 0, sel));
                if (A_TER) {
                    const uint32_t M0 = spread4(__byte_perm(m_lo, 0, sel));
                    const uint32_t M1 = spread4(__byte_perm(m_hi, 0, sel));
                    w[2 * bb] = M0 * 0xFFu + P0;  // +1 -> 0x01, -1 -> 0xFF, 0 -> 0x00 (disjoint planes)
                    w[2 * bb + 1] = M1 * 0xFFu + P1;
                } else {
                    w[2 * bb] = (P0 * 0xFEu) ^ 0x01010101u;  // bit 1 -> 0xFF (-1), bit 0 -> 0x01 (+1)
                    w[2 * bb + 1] = (P1 * 0xFEu) ^ 0x01010101u;
                }
            }
            const int ch = ch0 + c;
            if (DBG == 2) {  // timing experiment: keep the ALU work, drop the stores
                if ((w[0] ^ w[1] ^ w[2] ^ w[3]) == 0x9E3779B9u && pw == 0x7F4A7C15u) sts_v4(row, w[0], 0, 0, 0);
            } else {
                sts_v4(row + ((ch ^ sw) << 4), w[0], w[1], w[2], w[3]);
            }
        }
    }
}

template <bool A_TER>
__device__ __forceinline__ void expand_half(uint32_t raw_p, uint32_t raw_m, uint32_t a_tile, int r, int h) {
    const uint2 p = lds_v2(raw_p + r * 16 + 8 * h);
    uint2 m = make_uint2(0, 0);
    if (A_TER) m = lds_v2(raw_m + r * 16 + 8 * h);
    const uint32_t row = a_tile + r * 128;
    expand_word<A_TER>(p.x, m.x, row, r & 7, 4 * h);
    expand_word<A_TER>(p.y, m.y, row, r & 7, 4 * h + 2);
}

// Whole row: 16 raw bytes per plane -> the row's 8 chunks (128 int8).
template <bool A_TER, int DBG = 0>
__device__ __forceinline__ void expand_row(uint32_t raw_p, uint32_t raw_m, uint32_t a_tile, int r) {
    const uint4 p = lds_v4(raw_p + r * 16);
    uint4 m = make_uint4(0, 0, 0, 0);
    if (A_TER) m = lds_v4(raw_m + r * 16);
    const uint32_t row = a_tile + r * 128;
    expand_word<A_TER, DBG>(p.x, m.x, row, r & 7, 0);
    expand_word<A_TER, DBG>(p.y, m.y, row, r & 7, 2);
    expand_word<A_TER, DBG>(p.z, m.z, row, r & 7, 4);
    expand_word<A_TER, DBG>(p.w, m.w, row, r & 7, 6);
}

// ---------------------------------------------------------------------------
// B200 ("lane-interleaved") plane layout, produced by lowbit_encode_ex with
// LOWBIT_LAYOUT_LANES: within each 32-bit word (32 consecutive depth
// positions) element j sits at bit 8*(j%4) + j/4, i.e. byte b holds elements
// b, b+4, ..., b+28.  Expanding to int8 is then a shift and a mask per output
// word: bytes of ((w >> q) & 0x01010101) are elements 4q..4q+3 in order.
// Popcounts of whole words are unchanged by the permutation.
// ---------------------------------------------------------------------------
template <bool A_TER>
__device__ __forceinline__ void expand_word_lanes(uint32_t pw, uint32_t mw, uint32_t row, int sw, int ch0) {
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        uint32_t w[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int q = 4 * c + j;
            const uint32_t P = (pw >> q) & 0x01010101u;
            if (A_TER) {
                const uint32_t M = (mw >> q) & 0x01010101u;
                w[j] = M * 0xFFu + P;  // +1 -> 0x01, -1 -> 0xFF, 0 -> 0x00
            } else {
                w[j] = P * 0xFEu + 0x01010101u;  // bit 1 -> 0xFF (-1), bit 0 -> 0x01 (+1)
            }
        }
        const int ch = ch0 + c;
        sts_v4(row + ((ch ^ sw) << 4), w[0], w[1], w[2], w[3]);
    }
}

template <bool A_TER, int LAYOUT>
__device__ __forceinline__ void expand_half_layout(uint32_t raw_p, uint32_t raw_m, uint32_t a_tile, int r, int h) {
    if (LAYOUT == 0) {
        expand_half<A_TER>(raw_p, raw_m, a_tile, r, h);
        return;
    }
    const uint2 p = lds_v2(raw_p + r * 16 + 8 * h);
    uint2 m = make_uint2(0, 0);
    if (A_TER) m = lds_v2(raw_m + r * 16 + 8 * h);
    const uint32_t row = a_tile + r * 128;
    expand_word_lanes<A_TER>(p.x, m.x, row, r & 7, 4 * h);
    expand_word_lanes<A_TER>(p.y, m.y, row, r & 7, 4 * h + 2);
}

template <bool A_TER, int LAYOUT>
__device__ __forceinline__ void expand_row_layout(uint32_t raw_p, uint32_t raw_m, uint32_t a_tile, int r) {
    if (LAYOUT == 0) {
        expand_row<A_TER>(raw_p, raw_m, a_tile, r);
        return;
    }
    const uint4 p = lds_v4(raw_p + r * 16);
    uint4 m = make_uint4(0, 0, 0, 0);
    if (A_TER) m = lds_v4(raw_m + r * 16);
    const uint32_t row = a_tile + r * 128;
    expand_word_lanes<A_TER>(p.x, m.x, row, r & 7, 0);
    expand_word_lanes<A_TER>(p.y, m.y, row, r & 7, 2);
    expand_word_lanes<A_TER>(p.z, m.z, row, r & 7, 4);
    expand_word_lanes<A_TER>(p.w, m.w, row, r & 7, 6);
}

// Timing experiment helper: the expansion ALU work on register-resident data,
// stores suppressed (never-true guard keeps the work alive).
template <bool A_TER, int LAYOUT>
__device__ __forceinline__ void expand_row_regs(uint32_t seed_p, uint32_t seed_m, uint32_t a_tile, int r) {
    const uint32_t row = a_tile + r * 128;
#pragma unroll
    for (int wi = 0; wi < 4; ++wi) {
        const uint32_t pw = seed_p * (wi + 1), mw = seed_m * (wi + 3);
        if (LAYOUT == 0) expand_word<A_TER, 2>(pw, mw & ~pw, row, r & 7, 2 * wi);
        else {
            uint32_t acc = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint32_t P = (pw >> q) & 0x01010101u, M = (mw >> q) & 0x01010101u;
                acc ^= A_TER ? M * 0xFFu + P : P * 0xFEu + 0x01010101u;
            }
            if (acc == 0x9E3779B9u && pw == 0x7F4A7C15u) sts_v4(row, acc, 0, 0, 0);
        }
    }
}

}  // namespace lb
