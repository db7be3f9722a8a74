// layout.cuh — device layout of prepared weights (the GPU form of PackedB).
//
//   [ int8 section ]  np rows (output columns n) x kp int8 (depth), K-major,
//                     values in {-1,0,+1}, zero for n >= N or t >= K.
//                     Read by K3 through TMA (128-byte swizzle) as the UMMA
//                     B operand.
//   [ sign words   ]  np x kw uint32, K-major: bit t%32 of word t/32 = the
//                     element's minus bit (binary: its only bit).
//   [ nz words     ]  ternary only: np x kw uint32, plus|minus bits.
//                     Read by K2 (bit-serial).
//   [ fp4 section  ]  np x kp4/2 bytes, K-major packed e2m1 (+1 = 0x2,
//                     -1 = 0xA, 0 = 0x0; element 2i in the low nibble of
//                     byte i), kp4 a multiple of 256: the UMMA B operand of
//                     the kind::mxf4 path.
//   [ fp4 section, reference order ]
//                     the same codes with the 32 depth positions of every
//                     16-byte chunk permuted: byte-nibble position 8q+i holds
//                     depth element 4i+q of the chunk.  That is the order in
//                     which ((w >> q) & 0x11111111) lays a plane word of the
//                     REFERENCE bit order (element j at bit j, core.hpp:3-10)
//                     into nibbles, so K5 turns reference planes into its A
//                     operand with the same one shift + mask per plane as the
//                     NIBBLES layout, and the MMA's depth sum is unchanged
//                     (A and B are permuted alike; padding is 0 in both).
//   [ fp4 section, conv order ]
//                     the same codes with every 8 depth positions paired
//                     across their halves: byte i of the 4-byte word holds
//                     depth elements i (low nibble) and 4+i (high nibble) of
//                     the word's 8.  K7's converters build that word from two
//                     int8 words with two ANDs and one multiply-add
//                     ((x1 & 0x09..) * 16 + (x0 & 0x09..)), with no byte
//                     permute; the MMA's depth sum is unchanged.
#pragma once
#include <cstddef>

namespace lb {

struct WeightsLayout {
    int ternary, n, k;
    int np;  // rows padded to a multiple of 256
    int kp;  // int8 row length, multiple of 128 bytes (one UMMA k-block)
    int kw;  // words per column in the bit sections, multiple of 8 (one K2 stage)
    int kp4; // fp4 row length in elements, multiple of 256 (one 128-byte fp4 k-block)
    size_t off_sign, off_nz, off_fp4, off_fp4r, off_fp4c, bytes;

    __host__ __device__ WeightsLayout(int ternary_, int n_, int k_) : ternary(ternary_), n(n_), k(k_) {
        np = (n + 255) / 256 * 256;
        kp = (k + 127) / 128 * 128;
        kw = ((k + 31) / 32 + 7) / 8 * 8;
        kp4 = (k + 255) / 256 * 256;
        off_sign = (size_t)np * kp;
        off_nz = off_sign + (size_t)np * kw * 4;
        off_fp4 = (off_nz + (ternary ? (size_t)np * kw * 4 : 0) + 1023) / 1024 * 1024;
        off_fp4r = off_fp4 + (size_t)np * kp4 / 2;
        off_fp4c = off_fp4r + (size_t)np * kp4 / 2;
        bytes = off_fp4c + (size_t)np * kp4 / 2;
    }
};

}  // namespace lb
