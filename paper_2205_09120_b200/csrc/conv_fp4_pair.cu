// conv_fp4_pair.cu — K6: implicit-GeMM convolution on the fp4 tensor cores.
//
// conv2d_lowbit (conv.cpp:33-59) is im2col -> encode -> pack_b -> gemm_lowbit
// with k = (ky*kw + kx)*C + c (conv.cpp:18-27).  Here:
//   1. one HBM pass packs the NHWC int8 feature map into packed e2m1 (+1 ->
//      0x2, -1 -> 0xA, 0 -> 0x0; two channels per byte): the "fm4" map;
//   2. the GeMM's A tiles never exist in memory: an im2col TMA map over fm4,
//      viewed as NHWC uint8 with C/2 "channels", brings 128 output pixels x
//      128 channels of one filter tap (64 bytes per pixel, 64-byte swizzle)
//      straight into the UMMA A operand; TMA zero-fill is exactly the
//      ternary padding value;
//   3. the filter (prepared weights, fp4 section, K-major) stays resident in
//      shared memory for all the output tiles of a pair;
//   4. tcgen05.mma.cta_group::2.kind::mxf4.block_scale with unit scales and
//      f32 accumulators (exact: |partial sums| <= k <= 32767), int16 out by
//      TMA stores — bit-identical to the reference's int16 GeMM.
// Against the int8 implicit GeMM (gemm_tc_pair.cu LAYOUT 3, L2-bound on the
// taps' re-reads) the im2col traffic halves and the MMA rate doubles.
//
// Applies to TNN/TBN (ternary activations) or any conv without padding,
// c % 128 == 0, and a filter that fits (k-blocks x BN/2 rows x 64 B).
//
// Warp roles per CTA (352 threads): 0-7 epilogue (two warps per TMEM lane
// quarter, each draining half of the tile's columns), 8 A (im2col) producer,
// 9 B producer, 10 TMEM allocation + UMMA issuer (leader CTA).
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "encode.cuh"
#include "layout.cuh"
#include "tmap.cuh"

namespace lb {

constexpr int C6_BM = 128;                    // output pixels per CTA (256 per pair)
constexpr int C6_MAX_BN = 240;                // cout per tile: 2 accumulators + scales <= 512 TMEM columns
constexpr int C6_KB_BYTES = C6_BM * 64;       // one k-block of A: 128 pixels x 128 fp4 channels = 8 KB
constexpr int C6_MAX_A_ST = 12;               // A ring stages (runtime depth: what the filter leaves)
constexpr int C6_B_MAX = 96 * 1024;           // resident filter budget per CTA
constexpr int C6_THREADS = 352;
constexpr int C6_W_A = 8, C6_W_B = 9, C6_W_MMA = 10;
constexpr int C6_EPI_BYTES = 32 * 32;         // 32 rows x 16 int16
constexpr int C6_EPI_ALL = 8 * 2 * C6_EPI_BYTES;
constexpr uint32_t C6_SF_COL = 2 * C6_MAX_BN; // 480: unit scales, 8 columns
constexpr int C6_SMEM = 227 * 1024;           // filter + A ring + staging + barriers (+1 KB alignment)
constexpr int C6_RING_BUDGET = C6_SMEM - 1024 - C6_EPI_ALL - 1024;

struct ConvF4Params {
    int rows, cout, kblocks, g, bn, m_tiles, n_tiles;
    int ow, ohw, stride, pad, kw, cblocks;
    int breg;  // bytes of one resident B k-block region (1 KB aligned)
    int a_st;  // A ring depth (stages of g k-blocks)
    long long ldc;
    int16_t* c;
};

// UMMA shared-memory descriptor, K-major operand, 64-byte swizzle: rows of
// 64 bytes, 8-row atoms every 512 bytes.
LB_DEV uint64_t umma_desc_k_sw64(uint32_t smem_addr) {
    uint64_t d = 0;
    d |= (uint64_t)((smem_addr >> 4) & 0x3FFFu);
    d |= (uint64_t)1u << 16;            // LBO (unused for swizzled K-major)
    d |= (uint64_t)(512u >> 4) << 32;   // SBO
    d |= (uint64_t)1u << 46;            // version
    d |= (uint64_t)4u << 61;            // SWIZZLE_64B
    return d;
}

// PT ("tap pair", 3-wide filters, stride 1, padding 1, c = 128): a k-block is two
// horizontally adjacent taps = one 128-byte virtual pixel of the padded fm4 map
// (make_map_im2col_pairtap): (zero dummy, tap (ky,0)) and (tap (ky,1), tap (ky,2)),
// the filter side read straight from the prepared weights by a 3-D map whose
// out-of-bounds half row is zero-filled (make_map_filter_pairtap).  6 loads of
// 128-byte rows replace 9 of 64 bytes per output tile (the im2col TMA's cost
// is per pixel row).
template <bool PT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(C6_THREADS, 1)
    conv_fp4_pair_kernel(const __grid_constant__ CUtensorMap tmap_b, const __grid_constant__ CUtensorMap tmap_a,
                         const __grid_constant__ CUtensorMap tmap_c, const ConvF4Params prm) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int A_ST = prm.a_st;
    constexpr int KB_BYTES = PT ? 2 * C6_KB_BYTES : C6_KB_BYTES;  // one k-block of A (128 or 64-byte rows)
    const int a_stage = prm.g * KB_BYTES;
    uint8_t* sB = smem;                                  // resident filter: kblocks x breg
    uint8_t* sA = sB + prm.kblocks * prm.breg;           // A ring: A_ST x g k-blocks (1 KB multiples)
    uint8_t* sEpi = smem + C6_RING_BUDGET;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sEpi + C6_EPI_ALL);
    uint64_t* a_full = bars;            // leader: a stage's im2col tiles of both CTAs landed
    uint64_t* a_empty = bars + 16;      // local: pair MMAs done with the stage
    uint64_t* b_full = bars + 32;       // leader: resident filter of this n tile landed
    uint64_t* b_empty = bars + 33;      // local: pair MMAs done with the filter
    uint64_t* tmem_full = bars + 34;    // local (2)
    uint64_t* tmem_empty = bars + 36;   // leader: 16 epilogue warps drained (2)
    uint64_t* sf_ready = bars + 38;     // leader: unit scales written (16 warps)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 39);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int bn = prm.bn, bnh = bn >> 1;
    const int G = prm.g;                               // k-blocks per stage
    const int stages_per_tile = prm.kblocks / G;
    const int my_m = prm.m_tiles > pair ? (prm.m_tiles - pair + npairs - 1) / npairs : 0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < A_ST; ++s) {
            mbar_init(&a_full[s], 1);
            mbar_init(&a_empty[s], 1);
        }
        mbar_init(b_full, 1);
        mbar_init(b_empty, 1);
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tmem_full[a], 1);
            mbar_init(&tmem_empty[a], 16);
        }
        mbar_init(sf_ready, 16);
        fence_barrier_init();
    }
    if (warp == C6_W_A && lane == 0) {
        tma_prefetch_desc(&tmap_a);
        tma_prefetch_desc(&tmap_b);
        tma_prefetch_desc(&tmap_c);
    }
    if (warp == C6_W_MMA) tmem_alloc_pair<512>(tmem_slot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == C6_W_A) {
        // ===================== im2col A producer (both CTAs; bytes land on the leader) =====================
        if (lane == 0) {
            const uint32_t a_full0 = mapa_shared(smem_u32(&a_full[0]), 0);
            uint32_t t = 0;
            for (int nt = 0; nt < prm.n_tiles; ++nt)
                for (int i = 0; i < my_m; ++i) {
                    const int mt = pair + i * npairs;
                    const int row = mt * 2 * C6_BM + (int)rank * C6_BM;  // this CTA's first output pixel
                    const int img = row / prm.ohw, rem = row - img * prm.ohw;
                    const int oy = rem / prm.ow, ox = rem - oy * prm.ow;
                    for (int sg = 0; sg < stages_per_tile; ++sg, ++t) {
                        const uint32_t s = t % A_ST;
                        mbar_wait_sleep(&a_empty[s], ((t / A_ST) & 1) ^ 1);
                        if (leader) mbar_arrive_expect_tx(&a_full[s], 2u * G * KB_BYTES);
                        for (int j = 0; j < G; ++j) {
                            const int kb = sg * G + j;
                            int cb, ky, kx;
                            if (PT) {  // k-block 2*ky + g: (dummy, tap (ky,0)) at offset 0, taps (ky,1),(ky,2) at 2
                                cb = 0;
                                ky = kb >> 1;
                                kx = 2 * (kb & 1);
                            } else {
                                const int tap = kb / prm.cblocks;
                                cb = kb - tap * prm.cblocks;
                                ky = tap / prm.kw;
                                kx = tap - ky * prm.kw;
                            }
                            tma_load_im2col_4d_pair(smem_u32(sA + s * a_stage + j * KB_BYTES), &tmap_a,
                                                    a_full0 + s * 8, cb * 64, ox * prm.stride - prm.pad,
                                                    oy * prm.stride - prm.pad, img, (uint16_t)kx, (uint16_t)ky);
                        }
                    }
                }
        }
    } else if (warp == C6_W_B) {
        // ===================== resident filter producer (both CTAs) =====================
        if (lane == 0) {
            const uint32_t b_full0 = mapa_shared(smem_u32(b_full), 0);
            for (int nt = 0; nt < prm.n_tiles; ++nt) {
                if (my_m == 0) break;
                mbar_wait_sleep(b_empty, (nt & 1) ^ 1);
                if (leader) mbar_arrive_expect_tx(b_full, (uint32_t)prm.kblocks * bn * (PT ? 128 : 64));
                const int brow = nt * bn + (int)rank * bnh;
                for (int kb = 0; kb < prm.kblocks; ++kb) {
                    if (PT)  // (zero, tap (ky,0)) at byte -64, (tap (ky,1), tap (ky,2)) at byte 64
                        tma_load_3d_pair(smem_u32(sB + kb * prm.breg), &tmap_b, b_full0, (kb & 1) ? 64 : -64, kb >> 1,
                                         brow);
                    else
                        tma_load_2d_pair(smem_u32(sB + kb * prm.breg), &tmap_b, b_full0, kb * 64, brow);
                }
            }
        }
    } else if (warp == C6_W_MMA) {
        // ===================== UMMA issuer (leader CTA only) =====================
        if (leader && my_m > 0) {
            const uint32_t idesc = idesc_mxf4(2 * C6_BM, (uint32_t)bn);
            const uint32_t sf = tmem_base + C6_SF_COL;
            mbar_wait(sf_ready, 0);
            tc_fence_after();
            uint32_t t = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int nt = 0; nt < prm.n_tiles; ++nt) {
                mbar_wait(b_full, nt & 1);
                tc_fence_after();
                for (int i = 0; i < my_m; ++i) {
                    mbar_wait_sleep(&tmem_empty[acc], acc_phase ^ 1);
                    tc_fence_after();
                    const uint32_t d_tmem = tmem_base + (uint32_t)acc * C6_MAX_BN;
                    for (int sg = 0; sg < stages_per_tile; ++sg, ++t) {
                        const uint32_t s = t % A_ST;
                        mbar_wait(&a_full[s], (t / A_ST) & 1);
                        tc_fence_after();
                        if (lane == 0) {
                            for (int j = 0; j < G; ++j) {
                                const int kb = sg * G + j;
                                const uint32_t a_addr = smem_u32(sA + s * a_stage + j * KB_BYTES);
                                const uint32_t b_addr = smem_u32(sB + kb * prm.breg);
#pragma unroll
                                for (int h = 0; h < (PT ? 4 : 2); ++h)  // K = 64 per MMA = 32 bytes of the row
                                    umma_mxf4_pair(d_tmem,
                                                   PT ? umma_desc_k_sw128(a_addr + h * 32) : umma_desc_k_sw64(a_addr + h * 32),
                                                   PT ? umma_desc_k_sw128(b_addr + h * 32) : umma_desc_k_sw64(b_addr + h * 32),
                                                   idesc, sf, sf, (kb | h) != 0);
                            }
                            umma_commit_pair(&a_empty[s], 0x3);
                        }
                        __syncwarp();
                    }
                    if (lane == 0) umma_commit_pair(&tmem_full[acc], 0x3);
                    __syncwarp();
                    if (++acc == 2) { acc = 0; acc_phase ^= 1; }
                }
                if (lane == 0) umma_commit_pair(b_empty, 0x3);
                __syncwarp();
            }
        }
    } else {
        // ===================== epilogue (both CTAs): warps 0-7 =====================
        const int wq = warp & 3;     // TMEM lane quarter
        const int half = warp >> 2;  // which half of the tile's 16-column chunks
        const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
        tmem_st_32x32b_x8_fill(tmem_base + lane_base + C6_SF_COL, 0x7F7F7F7Fu);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(sf_ready), 0));
        const uint32_t tmem_empty0 = mapa_shared(smem_u32(&tmem_empty[0]), 0);
        const uint32_t epi = smem_u32(sEpi) + (uint32_t)warp * 2 * C6_EPI_BYTES;
        int acc = 0, nbuf = 0;
        uint32_t acc_phase = 0;
        const int nch = bn / 16;
        const int ch0 = half * ((nch + 1) / 2), ch1 = half ? nch : (nch + 1) / 2;
        for (int nt = 0; nt < prm.n_tiles; ++nt)
            for (int i = 0; i < my_m; ++i) {
                const int mt = pair + i * npairs;
                const int row0 = mt * 2 * C6_BM + (int)rank * C6_BM + wq * 32;
                mbar_wait_sleep(&tmem_full[acc], acc_phase);
                tc_fence_after();
                const uint32_t tacc = tmem_base + lane_base + (uint32_t)acc * C6_MAX_BN;
                for (int ch = ch0; ch < ch1; ++ch) {
                    uint32_t v[16];
                    tmem_ld_32x32b_x16(tacc + ch * 16, v);
                    tmem_ld_wait();
                    uint32_t h[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j)  // exact f32 integer -> int16 (see gemm_fp4_pair.cu)
                        h[j] = __byte_perm(__float_as_uint(__uint_as_float(v[2 * j]) + 12582912.0f),
                                           __float_as_uint(__uint_as_float(v[2 * j + 1]) + 12582912.0f), 0x5410);
                    const uint32_t buf = epi + (uint32_t)nbuf * C6_EPI_BYTES;
                    if (lane == 0) bulk_wait_read<1>();
                    __syncwarp();
                    const uint32_t rowaddr = buf + lane * 32;
                    const uint32_t sw = (uint32_t)(lane >> 2) & 1;  // TMA SWIZZLE_32B
                    sts_v4(rowaddr + (sw << 4), h[0], h[1], h[2], h[3]);
                    sts_v4(rowaddr + ((sw ^ 1) << 4), h[4], h[5], h[6], h[7]);
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        tma_store_2d(&tmap_c, buf, nt * bn + ch * 16, row0);
                        bulk_commit();
                    }
                    nbuf ^= 1;
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(tmem_empty0 + acc * 8);
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
        if (lane == 0) bulk_wait<0>();
    }

    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (warp == C6_W_MMA) {
        tc_fence_after();
        tmem_dealloc_pair<512>(tmem_base);
    }
}

// fm int8 NHWC -> packed e2m1 (two channels per byte, channel 2i in the low
// nibble).  One thread per 32 channels.  A 0 in a binary feature map sets
// *zero_flag (core.cpp:23).
// pad_w > 0: the output rows carry one extra zero pixel (row pitch pad_w + 1
// pixels, pad_w = the map's width) for the tap-pair map.
__global__ void conv_pack_fp4_kernel(const int8_t* __restrict__ fm, long long groups, int check_zero,
                                     uint8_t* __restrict__ out, int* __restrict__ zero_flag, int pad_w, int gpp) {
    for (long long gi = blockIdx.x * (long long)blockDim.x + threadIdx.x; gi < groups;
         gi += (long long)gridDim.x * blockDim.x) {
        const uint4 lo = __ldg(reinterpret_cast<const uint4*>(fm) + 2 * gi);
        const uint4 hi = __ldg(reinterpret_cast<const uint4*>(fm) + 2 * gi + 1);
        const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
        uint32_t o[4];
        uint32_t nz_all = 0x01010101u;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t half[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t x = w[2 * q + h];
                const uint32_t nz = nonzero_msb(x) >> 7;             // per-byte nonzero (bit 0 of each byte)
                nz_all &= nz;
                // per-byte code 0x2 (+1) / 0xA (-1) / 0x0, then bytes -> nibbles:
                // c | c >> 4 puts bytes 0,1 in byte 0 and bytes 2,3 in byte 2
                const uint32_t c = nz * 2u + ((x >> 4) & 0x08080808u);
                const uint32_t t = c | (c >> 4);
                half[h] = __byte_perm(t, 0, 0x4420);                    // bytes 0 and 2 -> 16 bits
            }
            o[q] = half[0] | (half[1] << 16);
        }
        const bool zero = check_zero && nz_all != 0x01010101u;
        long long oi = gi;
        if (pad_w > 0) {  // group gi = (pixel, channel group); pixel = row * pad_w + x (32-bit: < 2^31 groups)
            // rows of pad_w + 1 pixels, a zero pixel first; one more zero pixel after the last row
            const uint32_t g32 = (uint32_t)gi, pix = g32 / (uint32_t)gpp, cg = g32 - pix * (uint32_t)gpp;
            const uint32_t row = pix / (uint32_t)pad_w, x = pix - row * (uint32_t)pad_w;
            oi = ((long long)row * (pad_w + 1) + x + 1) * gpp + cg;
            if (x == 0) reinterpret_cast<uint4*>(out)[oi - gpp] = make_uint4(0, 0, 0, 0);
            if (gi >= groups - gpp) reinterpret_cast<uint4*>(out)[oi + gpp] = make_uint4(0, 0, 0, 0);
        }
        reinterpret_cast<uint4*>(out)[oi] = make_uint4(o[0], o[1], o[2], o[3]);
        if (zero && zero_flag) atomicOr(zero_flag, 1);
    }
}

static int pick_bn_conv(int cout) {
    const int tiles = (cout + C6_MAX_BN - 1) / C6_MAX_BN;
    const int per = (cout + tiles - 1) / tiles;
    return (per + 15) / 16 * 16;
}

static bool pairtap_ok(int c, int kw, int stride, int pad, int cout) {
    (void)cout;
    return c == 128 && kw == 3 && stride == 1 && pad == 1;
}

// fm4, with the tap-pair map's one zero pixel per row
size_t conv_fp4_workspace_bytes(int batch, int h, int w, int c) { return (size_t)batch * h * (w + 1) * c / 2 + 1024; }

// Whether K6 takes a conv: the im2col map's zero fill must be the padding
// value, channels tile into 128-channel k-blocks, and the filter fits the
// resident budget.
bool conv_fp4_applies(int mode, int fm_binary, int c, int cout, int kh, int kw, int padding, long long rows,
                      int stride) {
    if (!(padding == 0 || !fm_binary) || c % 128 != 0 || cout % 8 != 0 || rows > 0x7FFFFFFFLL) return false;
    (void)mode;
    const bool pt = pairtap_ok(c, kw, stride, padding, cout);
    const int kblocks = pt ? 2 * kh : kh * kw * (c / 128);
    const int kbb = pt ? 2 * C6_KB_BYTES : C6_KB_BYTES;
    const int bn = pick_bn_conv(cout);
    const int breg = ((bn / 2) * (pt ? 128 : 64) + 1023) / 1024 * 1024;
    const int g = kblocks % 4 == 0 ? 4 : (kblocks % 3 == 0 ? 3 : (kblocks % 2 == 0 ? 2 : 1));
    return kblocks * breg <= C6_B_MAX && (C6_RING_BUDGET - kblocks * breg) / (g * kbb) >= 2;
}

lowbit_status launch_conv_fp4(const int8_t* fm, int batch, int h, int w, int cch, int kh, int kw, int stride,
                              int pad, int check_zero, const void* weights, int b_ternary, int cout, int16_t* out,
                              void* workspace, int* zero_flag, cudaStream_t stream) {
    const int oh = (h + 2 * pad - kh) / stride + 1, ow = (w + 2 * pad - kw) / stride + 1;
    const long long rows = (long long)batch * oh * ow;
    const int k = kh * kw * cch;
    static const bool no_pt = getenv("LOWBIT_CONV_NO_PAIRTAP") != nullptr;  // tuning experiment knob
    const bool pt = pairtap_ok(cch, kw, stride, pad, cout) && !no_pt;
    uint8_t* fm4 = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(workspace) + 1023) & ~uintptr_t(1023));
    const long long groups = (long long)batch * h * w * cch / 32;
    conv_pack_fp4_kernel<<<grid_for(groups, 256), 256, 0, stream>>>(fm, groups, check_zero, fm4, zero_flag,
                                                                     pt ? w : 0, cch / 32);
    LB_CUDA_TRY(cudaGetLastError());

    const WeightsLayout L(b_ternary, cout, k);
    const uint8_t* wfp4 = static_cast<const uint8_t*>(weights) + L.off_fp4;

    ConvF4Params prm{};
    prm.rows = (int)rows;
    prm.cout = cout;
    prm.kblocks = pt ? 2 * kh : kh * kw * (cch / 128);
    prm.g = prm.kblocks % 4 == 0 ? 4 : (prm.kblocks % 3 == 0 ? 3 : (prm.kblocks % 2 == 0 ? 2 : 1));
    prm.bn = pick_bn_conv(cout);
    prm.m_tiles = (int)((rows + 2 * C6_BM - 1) / (2 * C6_BM));
    prm.n_tiles = (cout + prm.bn - 1) / prm.bn;
    prm.ow = ow;
    prm.ohw = oh * ow;
    prm.stride = stride;
    prm.pad = pad;
    prm.kw = kw;
    prm.cblocks = cch / 128;
    const int row_bytes = pt ? 128 : 64;  // bytes of one k-block per filter row / output pixel
    prm.breg = ((prm.bn / 2) * row_bytes + 1023) / 1024 * 1024;
    prm.a_st = (C6_RING_BUDGET - prm.kblocks * prm.breg) / (prm.g * C6_BM * row_bytes);
    if (prm.a_st > C6_MAX_A_ST) prm.a_st = C6_MAX_A_ST;
    prm.ldc = cout;
    prm.c = out;
    CUtensorMap mb, ma, mc;
    if (pt) {
        if (!make_map_filter_pairtap(&mb, wfp4, kh, (uint64_t)L.np, (uint64_t)L.kp4 / 2, (uint32_t)(prm.bn / 2)))
            return lbhost::set_error(LOWBIT_CUDA_ERROR, "cuTensorMapEncodeTiled failed for the conv filter");
        if (!make_map_im2col_pairtap(&ma, fm4, batch, h, w, kh, pad, C6_BM))
            return lbhost::set_error(LOWBIT_CUDA_ERROR, "cuTensorMapEncodeIm2col failed (tap-pair map)");
    } else {
        if (!make_map_2d(&mb, wfp4, (uint64_t)L.kp4 / 2, (uint64_t)L.np, (uint64_t)L.kp4 / 2, 64,
                         (uint32_t)(prm.bn / 2), CU_TENSOR_MAP_SWIZZLE_64B))
            return lbhost::set_error(LOWBIT_CUDA_ERROR, "cuTensorMapEncodeTiled failed for the conv filter");
        if (!make_map_im2col(&ma, fm4, batch, h, w, cch / 2, kh, kw, stride, pad, 64, C6_BM,
                             CU_TENSOR_MAP_SWIZZLE_64B))
            return lbhost::set_error(LOWBIT_CUDA_ERROR, "cuTensorMapEncodeIm2col failed (fp4 feature map)");
    }
    if (!make_map_2d(&mc, out, (uint64_t)cout, (uint64_t)rows, (uint64_t)cout * 2, 16, 32, CU_TENSOR_MAP_SWIZZLE_32B,
                     CU_TENSOR_MAP_DATA_TYPE_UINT16))
        return lbhost::set_error(LOWBIT_CUDA_ERROR, "cuTensorMapEncodeTiled failed for the conv output");
    static bool attr[2] = {false, false};
    if (!attr[pt]) {
        LB_CUDA_TRY(cudaFuncSetAttribute(pt ? conv_fp4_pair_kernel<true> : conv_fp4_pair_kernel<false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C6_SMEM));
        attr[pt] = true;
    }
    const int pairs = prm.m_tiles < num_sms() / 2 ? prm.m_tiles : num_sms() / 2;
    if (pt) conv_fp4_pair_kernel<true><<<2 * pairs, C6_THREADS, C6_SMEM, stream>>>(mb, ma, mc, prm);
    else conv_fp4_pair_kernel<false><<<2 * pairs, C6_THREADS, C6_SMEM, stream>>>(mb, ma, mc, prm);
    LB_CUDA_TRY(cudaGetLastError());
    return LOWBIT_OK;
}

}  // namespace lb
