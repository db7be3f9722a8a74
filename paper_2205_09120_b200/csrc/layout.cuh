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
#pragma once
#include <cstddef>

namespace lb {

struct WeightsLayout {
    int ternary, n, k;
    int np;  // rows padded to a multiple of 256
    int kp;  // int8 row length, multiple of 128 bytes (one UMMA k-block)
    int kw;  // words per column in the bit sections, multiple of 8 (one K2 stage)
    size_t off_sign, off_nz, bytes;

    __host__ __device__ WeightsLayout(int ternary_, int n_, int k_) : ternary(ternary_), n(n_), k(k_) {
        np = (n + 255) / 256 * 256;
        kp = (k + 127) / 128 * 128;
        kw = ((k + 31) / 32 + 7) / 8 * 8;
        off_sign = (size_t)np * kp;
        off_nz = off_sign + (size_t)np * kw * 4;
        bytes = off_nz + (ternary ? (size_t)np * kw * 4 : 0);
    }
};

}  // namespace lb
