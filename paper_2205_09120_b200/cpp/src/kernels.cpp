// kernels.cpp — drop-in 16x8 tile kernels (host code; the formulas of
// /root/reference/proj/src/kernels.cpp:8-158 evaluated directly on the
// depth-byte-major block layouts, no lane transpose).  GeMM-sized work runs
// on the B200 via gemm_lowbit.
#include <bit>

#include "lowbit/kernels.hpp"

namespace lowbit {

// kernels.cpp:8-16
std::int16_t dot_binary(std::span<const std::uint8_t> a_bits, std::span<const std::uint8_t> b_bits, int k_logical) {
    if (k_logical > kMaxDepth16) throw DepthOverflow(k_logical, kMaxDepth16);
    const size_t n = a_bits.size() < b_bits.size() ? a_bits.size() : b_bits.size();
    int diff = 0;
    for (size_t i = 0; i < n; ++i) diff += std::popcount(static_cast<unsigned>(a_bits[i] ^ b_bits[i]));
    return static_cast<std::int16_t>(k_logical - 2 * diff);
}

namespace detail {

// acc(i,j) += k_eff - 2 * popc(a_i ^ b_j)    (kernels.cpp:43-51)
void bnn_tile(const std::uint8_t* a, const std::uint8_t* b, int depth_bytes, int k_eff, AccumulatorTile& acc) {
    for (int i = 0; i < kTileRows; ++i)
        for (int j = 0; j < kTileCols; ++j) {
            int diff = 0;
            for (int d = 0; d < depth_bytes; ++d) diff += std::popcount(static_cast<unsigned>(a[d * 16 + i] ^ b[d * 8 + j]));
            acc.at(i, j) = static_cast<std::int16_t>(acc.at(i, j) + k_eff - 2 * diff);
        }
}

// acc += popc((a+&b+)|(a-&b-)) - popc((a+&b-)|(a-&b+))    (kernels.cpp:75-89)
void tnn_tile(const std::uint8_t* a, const std::uint8_t* b, int depth_bytes, AccumulatorTile& acc) {
    for (int i = 0; i < kTileRows; ++i) {
        const int off = (i / 8) * 16 + i % 8;
        for (int j = 0; j < kTileCols; ++j) {
            int s = 0;
            for (int d = 0; d < depth_bytes; ++d) {
                const unsigned ap = a[d * 32 + off], am = a[d * 32 + off + 8];
                const unsigned bp = b[d * 16 + 2 * j], bm = b[d * 16 + 2 * j + 1];
                s += std::popcount((ap & bp) | (am & bm)) - std::popcount((ap & bm) | (am & bp));
            }
            acc.at(i, j) = static_cast<std::int16_t>(acc.at(i, j) + s);
        }
    }
}

// acc += 2*popc((a+ & ~b) | (a- & b)) - popc(a+ | a-)    (kernels.cpp:109-125)
void tbn_tile(const std::uint8_t* a, const std::uint8_t* b, int depth_bytes, AccumulatorTile& acc) {
    for (int i = 0; i < kTileRows; ++i) {
        const int off = (i / 8) * 16 + i % 8;
        int nnz = 0;
        for (int d = 0; d < depth_bytes; ++d) nnz += std::popcount(static_cast<unsigned>(a[d * 32 + off] | a[d * 32 + off + 8]));
        for (int j = 0; j < kTileCols; ++j) {
            int agree = 0;
            for (int d = 0; d < depth_bytes; ++d) {
                const unsigned ap = a[d * 32 + off], am = a[d * 32 + off + 8], bb = b[d * 8 + j];
                agree += std::popcount((ap & ~bb & 0xFFu) | (am & bb));
            }
            acc.at(i, j) = static_cast<std::int16_t>(acc.at(i, j) + 2 * agree - nnz);
        }
    }
}

}  // namespace detail

namespace {
// kernels.cpp:132-140
void validate_blocks(const PackedBlock& a, BlockMode want_a, const PackedBlock& b, BlockMode want_b, int k_eff) {
    if (a.mode != want_a || b.mode != want_b) throw ModeMismatch("packed block mode");
    if (k_eff > kMaxDepth16) throw DepthOverflow(k_eff, kMaxDepth16);
    const int need = (k_eff + 7) / 8;
    if (need > a.depth_bytes || need > b.depth_bytes) throw OutOfBounds("k_eff exceeds packed depth");
}
}  // namespace

void microkernel_bnn(const PackedBlock& a_block, const PackedBlock& b_block, int k_eff, AccumulatorTile& acc) {
    validate_blocks(a_block, BlockMode::bnn_a, b_block, BlockMode::bnn_b, k_eff);
    detail::bnn_tile(a_block.buffer.data(), b_block.buffer.data(), (k_eff + 7) / 8, k_eff, acc);
}

void microkernel_tnn(const PackedBlock& a_block, const PackedBlock& b_block, int k_eff, AccumulatorTile& acc) {
    validate_blocks(a_block, BlockMode::tnn_a, b_block, BlockMode::tnn_b, k_eff);
    detail::tnn_tile(a_block.buffer.data(), b_block.buffer.data(), (k_eff + 7) / 8, acc);
}

void microkernel_tbn(const PackedBlock& a_block, const PackedBlock& b_block, int k_eff, AccumulatorTile& acc) {
    validate_blocks(a_block, BlockMode::tnn_a, b_block, BlockMode::bnn_b, k_eff);
    detail::tbn_tile(a_block.buffer.data(), b_block.buffer.data(), (k_eff + 7) / 8, acc);
}

}  // namespace lowbit
