// encode.cuh — shared pieces of the HBM-bound packing kernels (K1, K4).
#pragma once
#include "common.cuh"

namespace lb {

__device__ __forceinline__ uint32_t valid_mask32(int nvals) { return nvals >= 32 ? 0xFFFFFFFFu : ((1u << nvals) - 1u); }

// 32 int8 values already in registers (two 16-byte vectors) -> plus / minus words
// (bit j <-> value j, by sign: core.cpp:40-58).  Per word: the sign flags
// ((v >> 7) & 0x01010101) and the positive flags ((low7 != 0) & !sign, bit 7 of
// ((v & 0x7f..) + 0x7f..) & ~v) sit at bit 0 of each byte; two words' flags go
// to the top byte of one product, a*0x01020408 + b*0x10204080 (partial
// products land on distinct bits below 24: no carries), and PRMT collects the
// four top bytes: ~9 ops per word instead of ~17 for a per-word gather.
__device__ __forceinline__ uint32_t top8_of_pair(uint32_t a, uint32_t b) { return a * 0x01020408u + b * 0x10204080u; }
__device__ __forceinline__ void encode_word32_regs(const uint4 lo, const uint4 hi, uint32_t& plus, uint32_t& minus) {
    const uint32_t v[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    uint32_t rn[4], rp[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint32_t a = v[2 * q], b = v[2 * q + 1];
        const uint32_t na = (a >> 7) & 0x01010101u, nb = (b >> 7) & 0x01010101u;
        const uint32_t pa = ((((a & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) & ~a & 0x80808080u) >> 7);
        const uint32_t pb = ((((b & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) & ~b & 0x80808080u) >> 7);
        rn[q] = top8_of_pair(na, nb);
        rp[q] = top8_of_pair(pa, pb);
    }
    minus = __byte_perm(__byte_perm(rn[0], rn[1], 0x0073), __byte_perm(rn[2], rn[3], 0x0073), 0x5410);
    plus = __byte_perm(__byte_perm(rp[0], rp[1], 0x0073), __byte_perm(rp[2], rp[3], 0x0073), 0x5410);
}
// 32 (or fewer) consecutive int8 sign values -> plus / minus bit words
// (bit j <-> value j; LSB-first, core.cpp:13-58).  Vector path when the 32
// values are complete and 16-byte aligned.
__device__ __forceinline__ void encode_word32(const int8_t* src, int nvals, uint32_t& plus, uint32_t& minus) {
    plus = 0;
    minus = 0;
    if (nvals == 32 && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
        encode_word32_regs(__ldg(reinterpret_cast<const uint4*>(src)), __ldg(reinterpret_cast<const uint4*>(src) + 1),
                           plus, minus);
    } else {
        for (int j = 0; j < nvals; ++j) {
            const int8_t x = src[j];
            if (x < 0) minus |= 1u << j;
            if (x > 0) plus |= 1u << j;
        }
    }
}

// Same as encode_word32 but producing the lane-interleaved layout
// (element j -> bit 8*(j%4) + j/4, see expand.cuh).  With 4 values per
// 32-bit lane word x_i (values 4i..4i+3), the per-byte flags of x_i land in
// bit i of each byte: word |= flags_i << i.
__device__ __forceinline__ void encode_word32_lanes(const int8_t* src, int nvals, uint32_t& plus, uint32_t& minus) {
    plus = 0;
    minus = 0;
    uint32_t v[8];
    if (nvals == 32 && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
        const uint4 lo = __ldg(reinterpret_cast<const uint4*>(src));
        const uint4 hi = __ldg(reinterpret_cast<const uint4*>(src) + 1);
        v[0] = lo.x, v[1] = lo.y, v[2] = lo.z, v[3] = lo.w, v[4] = hi.x, v[5] = hi.y, v[6] = hi.z, v[7] = hi.w;
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            uint32_t x = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int j = 4 * i + b;
                if (j < nvals) x |= (uint32_t)(uint8_t)src[j] << (8 * b);
            }
            v[i] = x;
        }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint32_t neg = (v[i] >> 7) & 0x01010101u;
        const uint32_t nz = nonzero_msb(v[i]) >> 7;
        minus |= neg << i;
        plus |= (nz & ~neg) << i;
    }
}

// Same for the nibble-interleaved layout (LOWBIT_LAYOUT_NIBBLES): element j at
// bit 4*(j%8) + j/8, so (w >> q) & 0x11111111 holds elements 8q..8q+7, one per
// nibble — the packed-e2m1 order of the fp4 tensor-core path.  Built from the
// per-byte flags of 4-value lane words: pairs (2t, 2t+1) interleave by
// nibble at bit t, then one perfect unshuffle of the 8 nibbles.
__device__ __forceinline__ uint32_t unshuffle_nibbles(uint32_t x) {
    uint32_t t = (x ^ (x >> 4)) & 0x00F000F0u;
    x = x ^ t ^ (t << 4);
    t = (x ^ (x >> 8)) & 0x0000FF00u;
    return x ^ t ^ (t << 8);
}

__device__ __forceinline__ void encode_word32_nibbles(const int8_t* src, int nvals, uint32_t& plus,
                                                      uint32_t& minus) {
    uint32_t v[8];
    if (nvals == 32 && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
        const uint4 lo = __ldg(reinterpret_cast<const uint4*>(src));
        const uint4 hi = __ldg(reinterpret_cast<const uint4*>(src) + 1);
        v[0] = lo.x, v[1] = lo.y, v[2] = lo.z, v[3] = lo.w, v[4] = hi.x, v[5] = hi.y, v[6] = hi.z, v[7] = hi.w;
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            uint32_t x = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int j = 4 * i + b;
                if (j < nvals) x |= (uint32_t)(uint8_t)src[j] << (8 * b);
            }
            v[i] = x;
        }
    }
    uint32_t pa = 0, ma = 0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const uint32_t ne = (v[2 * t] >> 7) & 0x01010101u, no = (v[2 * t + 1] >> 7) & 0x01010101u;
        const uint32_t ze = nonzero_msb(v[2 * t]) >> 7, zo = nonzero_msb(v[2 * t + 1]) >> 7;
        ma |= (ne | (no << 4)) << t;
        pa |= ((ze & ~ne) | ((zo & ~no) << 4)) << t;
    }
    plus = unshuffle_nibbles(pa);
    minus = unshuffle_nibbles(ma);
}

__device__ __forceinline__ uint32_t valid_mask32_nibbles(int nvals) {
    uint32_t m = 0;
    for (int j = 0; j < nvals && j < 32; ++j) m |= 1u << (4 * (j & 7) + (j >> 3));
    return m;
}

// Bit mask of the first nvals elements in the lane-interleaved layout.
__device__ __forceinline__ uint32_t valid_mask32_lanes(int nvals) {
    uint32_t m = 0;
    for (int j = 0; j < nvals && j < 32; ++j) m |= 1u << (8 * (j & 3) + (j >> 2));
    return m;
}

inline int grid_for(long long work, int threads) {
    long long g = (work + threads - 1) / threads;
    const long long cap = 148LL * 16;  // 16 resident 256-thread blocks per SM
    if (g > cap) g = cap;
    return (int)(g < 1 ? 1 : g);
}

}  // namespace lb
