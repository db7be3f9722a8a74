// halo_common.cuh — device helpers shared by the fused halo convolutions
// (K7 conv_fp4_halo.cu and K7T conv_fp4_ts.cu): the UMMA descriptor of a
// 64-byte-swizzled tile, the int8 -> e2m1 converters with their sign-domain
// check (core.cpp:40-58), and division-free ring / tile bookkeeping.
#pragma once
#include "common.cuh"

namespace lb {

LB_DEV uint64_t h7_desc_sw64(uint32_t smem_addr, uint32_t sbo = 512) {  // K-major, 64-byte rows, 8-row atoms every sbo B
    uint64_t d = 0;
    d |= (uint64_t)((smem_addr >> 4) & 0x3FFFu);
    d |= (uint64_t)1u << 16;
    d |= (uint64_t)(sbo >> 4) << 32;
    d |= (uint64_t)1u << 46;
    d |= (uint64_t)4u << 61;  // SWIZZLE_64B
    return d;
}

// 8 int8 {-1, 0, +1} (two words) -> 8 packed e2m1 codes encoding +-1 as +-0.5
// (0x1 / 0x9): the code is the int8 byte ANDed with 0x09 (0x01 -> 0x1,
// 0xFF -> 0x9, 0x00 -> 0x0).  Byte i of the result pairs channel i of x0 (low
// nibble) with channel i of x1 (high nibble) — the "conv order" of the
// prepared filter (layout.cuh) — so the whole conversion is two ANDs and one
// multiply-add per word pair, no byte permute; the multiply-add (by a
// register operand, so ptxas keeps it an IMAD) runs on the FMA pipe, next to
// the ALU pipe the ANDs and the domain check use.  The filter stays +-1.0,
// every product is +-0.5, and the f32 sums are half-integers of magnitude
// <= 16383.5 (exact); the epilogue doubles them.
LB_DEV uint32_t h7_mad(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
LB_DEV uint32_t h7_pack8(uint32_t x0, uint32_t x1, uint32_t k16) {
    return h7_mad(x1 & 0x09090909u, k16, x0 & 0x09090909u);
}
// Any int8 value, by SIGN as encode_ternary maps it (core.cpp:40-58: v > 0 -> +1,
// v < 0 -> -1): the code is the nonzero flag in bit 0 and the sign bit in bit 3.
// The converters take this path only for a batch that holds a value outside
// {-1, 0, +1}.
LB_DEV uint32_t h7_code4(uint32_t x) { return (nonzero_msb(x) >> 7) | ((x >> 4) & 0x08080808u); }
LB_DEV uint32_t h7_pack8_sign(uint32_t x0, uint32_t x1) { return (h7_code4(x1) << 4) | h7_code4(x0); }
// Domain check of four int8: bits 1..7 of the result are all zero iff every byte is in
// {-1, 0, +1} (bit 0 of each byte is garbage: the caller masks with 0xFEFEFEFE once per
// batch).  With y = x << 1 (an IMAD on the FMA pipe), bits 2..7 of x ^ y are zero iff
// bits 1..7 of the byte are equal (0x00, 0x01, 0xFE, 0xFF), and bit 1 of x & ~y picks out
// 0xFE: one multiply and one LOP3 per word.
LB_DEV uint32_t h7_bad4(uint32_t x, uint32_t k2) {
    const uint32_t y = h7_mad(x, k2, 0u);
    uint32_t f;  // bit 1 of each byte: x & ~y; the other bits: x ^ y (one LOP3; written as asm so
                 // the caller's final mask is not folded in, which split it into three)
    asm("lop3.b32 %0, %1, %2, %3, 0x34;" : "=r"(f) : "r"(x), "r"(y), "r"(0x02020202u));
    return f;
}
LB_DEV uint32_t h7_bad16(uint4 v, uint32_t k2) {
    return h7_bad4(v.x, k2) | h7_bad4(v.y, k2) | h7_bad4(v.z, k2) | h7_bad4(v.w, k2);
}
// all 16 bytes nonzero (a binary map holds no 0, core.cpp:23)
LB_DEV bool h7_all_nonzero(uint4 v) {
    return (nonzero_msb(v.x) & nonzero_msb(v.y) & nonzero_msb(v.z) & nonzero_msb(v.w)) == 0x80808080u;
}

// Slot index and phase bit of a ring walked one step per tile (t % n and (t / n) & 1 without the
// divisions: the ring depths are run-time values).
struct H7Ring {
    uint32_t idx, phase, n;
    LB_DEV void init(int depth) { idx = 0, phase = 0, n = (uint32_t)depth; }
    LB_DEV void next() {
        if (++idx == n) idx = 0, phase ^= 1;
    }
};
// A CTA's tiles ct = first + i * step decoded to (image, tile of the image) without a division
// per tile (the divisions sat in front of every halo load and every epilogue pass).
struct H7Walk {
    int img, rem, dimg, drem, tpi;
    LB_DEV void init(int first, int step, int tiles_per_image) {
        tpi = tiles_per_image;
        img = first / tpi;
        rem = first - img * tpi;
        dimg = step / tpi;
        drem = step - dimg * tpi;
    }
    LB_DEV void next() {
        img += dimg;
        rem += drem;
        if (rem >= tpi) rem -= tpi, ++img;
    }
};

}  // namespace lb
