// encode.cuh — shared pieces of the HBM-bound packing kernels (K1, K4).
#pragma once
#include "common.cuh"

namespace lb {

__device__ __forceinline__ uint32_t valid_mask32(int nvals) { return nvals >= 32 ? 0xFFFFFFFFu : ((1u << nvals) - 1u); }

// 32 (or fewer) consecutive int8 sign values -> plus / minus bit words
// (bit j <-> value j; LSB-first, core.cpp:13-58).  Vector path when the 32
// values are complete and 16-byte aligned.
__device__ __forceinline__ void encode_word32(const int8_t* src, int nvals, uint32_t& plus, uint32_t& minus) {
    plus = 0;
    minus = 0;
    if (nvals == 32 && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
        const uint4 lo = __ldg(reinterpret_cast<const uint4*>(src));
        const uint4 hi = __ldg(reinterpret_cast<const uint4*>(src) + 1);
        const uint32_t v[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint32_t neg = gather_msb4(v[q]);
            const uint32_t nz = gather_msb4(nonzero_msb(v[q]));
            minus |= neg << (4 * q);
            plus |= (nz & ~neg) << (4 * q);
        }
    } else {
        for (int j = 0; j < nvals; ++j) {
            const int8_t x = src[j];
            if (x < 0) minus |= 1u << j;
            if (x > 0) plus |= 1u << j;
        }
    }
}

inline int grid_for(long long work, int threads) {
    long long g = (work + threads - 1) / threads;
    const long long cap = 148LL * 16;  // 16 resident 256-thread blocks per SM
    if (g > cap) g = cap;
    return (int)(g < 1 ? 1 : g);
}

}  // namespace lb
