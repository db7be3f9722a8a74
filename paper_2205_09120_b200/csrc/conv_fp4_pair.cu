// conv_fp4_pair.cu — K6: implicit-GeMM convolution on the fp4 tensor cores.
//
// conv2d_lowbit (conv.cpp:33-59) is im2col -> encode -> pack_b -> gemm_lowbit
// with k = (ky*kw + kx)*C + c (conv.cpp:18-27).  Here:
//   1. one HBM pass packs the NHWC int8 feature map into packed e2m1 (+1 ->
//      0x2, -1 -> 0xA, 0 -> 0x0; two channels per byte): the "fm4" map;
//   2. the GeMM's A tiles never exist in memory.  Stride 1 ("halo" form):
//      fm4 is written spatially padded (zero border, (H+2p) x (W+2p) pixels
//      per image) and the GeMM runs over every padded pixel position q, so
//      filter tap (ky,kx) of output q is fm4 pixel q + ky*(W+2p) + kx.  A
//      CTA's 128 positions need the 128 + (kh-1)*(W+2p) + kw-1 consecutive
//      pixels from q0 on — one "halo" tile, loaded once by plain 2-D TMA
//      boxes (64-byte rows, 64-byte swizzle) — and the A operand of tap
//      (ky,kx) is that tile's UMMA descriptor advanced by ky*(W+2p) + kx
//      rows: the swizzle is a function of the absolute smem address (base
//      offset 0), so any 64-byte row can start an operand
//      (tools/micro/halo_check.cu).  The border positions (no output) are
//      computed and dropped by the epilogue.  Other strides: an im2col TMA
//      map over fm4 (NHWC uint8 with C/2 "channels"), whose zero fill is the
//      padding — one TMA row per output pixel and tap, the im2col unit's
//      ~5 cycles per row being ~5x the MMA time of a 3x3 tile;
//   3. the filter (prepared weights, fp4 section, K-major) stays resident in
//      shared memory for all the output tiles of a pair;
//   4. tcgen05.mma.cta_group::2.kind::mxf4.block_scale with unit scales and
//      f32 accumulators (exact: |partial sums| <= k <= 32767), int16 out by
//      TMA stores (im2col form) or per-row direct stores (tiled form: a tile's
//      rows are not contiguous in the output) — bit-identical to the
//      reference's int16 GeMM.
// Against the int8 implicit GeMM (gemm_tc_pair.cu LAYOUT 3, L2-bound on the
// taps' re-reads) the im2col traffic halves and the MMA rate doubles.
//
// Applies to TNN/TBN (ternary activations) or any conv without padding,
// c % 128 == 0, and a filter that fits (k-blocks x BN/2 rows x 64 B).
//
// Warp roles per CTA (384 threads): 0-7 epilogue (two warps per TMEM lane
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
constexpr int C6_THREADS = 384;
constexpr int C6_W_A = 8, C6_W_B = 9, C6_W_MMA = 10, C6_W_MMA2 = 11;
constexpr int C6_EPI_BYTES = 32 * 128;        // 32 rows x 64 int16 (one 64-column box; 16-column boxes use 1 KB)
constexpr int C6_EPI_BUFS = 2;                // staging buffers per epilogue warp (TMA store in flight)
constexpr int C6_EPI_ALL = 8 * C6_EPI_BUFS * C6_EPI_BYTES;
constexpr uint32_t C6_SF_COL = 2 * C6_MAX_BN; // 480: unit scales, 8 columns
constexpr int C6_SMEM = 227 * 1024;           // filter + A ring + staging + barriers (+1 KB alignment)
constexpr int C6_RING_BUDGET = C6_SMEM - 1024 - C6_EPI_ALL - 1024;

struct ConvF4Params {
    int rows, cout, kblocks, g, bn, m_tiles, n_tiles;
    int ow, ohw, stride, pad, kw, cblocks;
    int oh, wp, hpwp;  // halo form: output height, row pitch of the padded map, its pixels per image
    int hloads;        // halo form: 128-row TMA boxes per channel block of a halo tile
    int oh_kh;         // filter height
    int epi_split;       // 1: every tile drained by all 8 epilogue warps (column halves)
    int nacc, acc_cols;  // accumulators in TMEM (3 when 3 x bn fits below the scale columns) and their stride
    int dbg;  // tuning experiments (LOWBIT_CONV_DEBUG): 1 no output stores, 2 no MMAs, 4 no A loads, 8 no TMEM loads
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

// Timing experiments (ConvF4Params::dbg) exist only in -DLOWBIT_TUNING builds: C6_DBG is the
// constant 0 in the product kernel (as in K5 / K7).
#ifdef LOWBIT_TUNING
#define C6_DBG(bits) (prm.dbg & (bits))
#define C6_DBGV(v, bits) ((v) & (bits))
#else
#define C6_DBG(bits) 0
#define C6_DBGV(v, bits) 0
#endif

// dbg & 32: per-tile event times of pair 0's leader CTA (clock64), read by lowbit_debug_conv_trace
__device__ unsigned long long g_conv_trace[16 * 64];
#define C6_TRACE(ev, i)                                                                  \
    if (C6_DBG(32) && pair == 0 && leader && (i) < 64) g_conv_trace[(ev) * 64 + (i)] = clock64()

LB_DEV void cwait(int dbg, uint64_t* bar, uint32_t parity) {
    if (C6_DBGV(dbg, 16)) mbar_wait(bar, parity);
    else mbar_wait_sleep(bar, parity);
}
// the MMA thread's waits: polled (dbg & 128: try_wait)
LB_DEV void mwait(int dbg, uint64_t* bar, uint32_t parity) {
    if (C6_DBGV(dbg, 128)) mbar_wait(bar, parity);
    else if (C6_DBGV(dbg, 8192)) mbar_wait_sleep(bar, parity);
    else mbar_wait_poll(bar, parity);
}

// TL: the halo form (stride 1, padded fm4, rows = padded pixel positions,
// one halo tile per A stage).
template <bool TL>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(C6_THREADS, 1)
    conv_fp4_pair_kernel(const __grid_constant__ CUtensorMap tmap_b, const __grid_constant__ CUtensorMap tmap_a,
                         const __grid_constant__ CUtensorMap tmap_c, const __grid_constant__ CUtensorMap tmap_c64,
                         const ConvF4Params prm) {
    if (C6_DBG(256)) return;  // launch-overhead probe
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int A_ST = prm.a_st;
    constexpr int KB_BYTES = C6_KB_BYTES;  // one k-block of A: 128 pixels x 64 bytes
    const int a_stage = TL ? prm.cblocks * prm.hloads * KB_BYTES : prm.g * KB_BYTES;
    uint8_t* sB = smem;                                  // resident filter: kblocks x breg
    uint8_t* sA = sB + prm.kblocks * prm.breg;           // A ring: A_ST x g k-blocks (1 KB multiples)
    uint8_t* sEpi = smem + C6_RING_BUDGET;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sEpi + C6_EPI_ALL);
    uint64_t* a_full = bars;            // leader: a stage's im2col tiles of both CTAs landed
    uint64_t* a_empty = bars + 16;      // local: pair MMAs done with the stage
    uint64_t* b_full = bars + 32;       // leader: resident filter of this n tile landed
    uint64_t* b_empty = bars + 33;      // local: pair MMAs done with the filter
    uint64_t* tmem_full = bars + 34;    // local (3)
    uint64_t* tmem_empty = bars + 37;   // leader: the accumulator's 8 epilogue warps drained (3)
    uint64_t* sf_ready = bars + 40;     // leader: unit scales written (16 warps)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 41);
    uint32_t* kb_aoff = reinterpret_cast<uint32_t*>(bars + 42);  // halo form: A row offset per k-block (<= 96)

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int bn = prm.bn, bnh = bn >> 1;
    const int G = prm.g;                               // k-blocks per stage
    const int stages_per_tile = TL ? 1 : prm.kblocks / G;
    const int my_m = prm.m_tiles > pair ? (prm.m_tiles - pair + npairs - 1) / npairs : 0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < A_ST; ++s) {
            mbar_init(&a_full[s], 1);
            mbar_init(&a_empty[s], 1);
        }
        mbar_init(b_full, 1);
        mbar_init(b_empty, TL ? 2 : 1);  // one commit per issuer
        for (int a = 0; a < 3; ++a) {
            mbar_init(&tmem_full[a], 1);
            mbar_init(&tmem_empty[a], prm.epi_split ? 16 : 8);
        }
        mbar_init(sf_ready, 16);
        fence_barrier_init();
    }
    if (warp == C6_W_A && lane == 0) {
        tma_prefetch_desc(&tmap_a);
        tma_prefetch_desc(&tmap_b);
        tma_prefetch_desc(&tmap_c);
        tma_prefetch_desc(&tmap_c64);
    }
    if (warp == C6_W_MMA) tmem_alloc_pair<512>(tmem_slot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const bool probe_only = C6_DBG(512) != 0;  // setup/teardown probe

    if (probe_only) {
    } else if (warp == C6_W_A) {
        // ===================== im2col A producer (both CTAs; bytes land on the leader) =====================
        if (lane == 0) {
            const uint32_t a_full0 = mapa_shared(smem_u32(&a_full[0]), 0);
            uint32_t t = 0;
            for (int nt = 0; nt < prm.n_tiles; ++nt)
                for (int i = 0; i < my_m; ++i) {
                    const int mt = pair + i * npairs;
                    const int row = mt * 2 * C6_BM + (int)rank * C6_BM;  // this CTA's first output pixel
                    int img = 0, oy = 0, ox = 0;
                    if (!TL) {
                        img = row / prm.ohw;
                        const int rem = row - img * prm.ohw;
                        oy = rem / prm.ow;
                        ox = rem - oy * prm.ow;
                    }
                    if (TL) {  // the tile's halo: cblocks x hloads boxes of 128 pixel rows
                        const uint32_t s = t % A_ST;
                        cwait(prm.dbg, &a_empty[s], ((t / A_ST) & 1) ^ 1);
                        C6_TRACE(5, i);
                        if (!C6_DBG(4))
                            for (int cb = 0; cb < prm.cblocks; ++cb)
                                for (int l = 0; l < prm.hloads; ++l)
                                    tma_load_2d_pair(smem_u32(sA + s * a_stage + (cb * prm.hloads + l) * KB_BYTES),
                                                     &tmap_a, a_full0 + s * 8, cb * 64, row + l * C6_BM);
                        if (leader) {
                            // a_full also carries "the tile's accumulator is drained": the MMA
                            // thread then waits once per tile (a wait costs it ~300 cycles with
                            // only a few MMAs queued behind it)
                            const int u = (int)t;
                            cwait(prm.dbg, &tmem_empty[u % prm.nacc], ((uint32_t)(u / prm.nacc) & 1) ^ 1);
                            mbar_arrive_expect_tx(&a_full[s], C6_DBG(4) ? 0u : 2u * a_stage);
                        }
                        C6_TRACE(6, i);
                        ++t;
                        continue;
                    }
                    for (int sg = 0; sg < stages_per_tile; ++sg, ++t) {
                        const uint32_t s = t % A_ST;
                        cwait(prm.dbg, &a_empty[s], ((t / A_ST) & 1) ^ 1);
                        if (leader) mbar_arrive_expect_tx(&a_full[s], 2u * G * KB_BYTES);
                        for (int j = 0; j < G; ++j) {
                            const int kb = sg * G + j;
                            const int tap = kb / prm.cblocks;
                            const int cb = kb - tap * prm.cblocks;
                            const int ky = tap / prm.kw;
                            const int kx = tap - ky * prm.kw;
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
                cwait(prm.dbg, b_empty, (nt & 1) ^ 1);
                if (leader) mbar_arrive_expect_tx(b_full, (uint32_t)prm.kblocks * bn * 64);
                const int brow = nt * bn + (int)rank * bnh;
                for (int kb = 0; kb < prm.kblocks; ++kb)
                    tma_load_2d_pair(smem_u32(sB + kb * prm.breg), &tmap_b, b_full0, kb * 64, brow);
            }
        }
    } else if (warp == C6_W_MMA || warp == C6_W_MMA2) {
        // ===================== UMMA issuers (leader CTA only) =====================
        // Halo form: two issuer warps take alternate tiles.  An issuing thread's
        // mbarrier wait costs it ~300-400 cycles, while only a few 64-cycle
        // (N = 128) MMAs sit queued in the tensor pipe: one issuer left the pipe
        // idle for most of every wait; two keep it fed.
        const int which = warp - C6_W_MMA, nissuers = TL ? 2 : 1;
        if (leader && my_m > 0 && which < nissuers) {
            const uint32_t idesc = idesc_mxf4(2 * C6_BM, (uint32_t)bn);
            const uint32_t sf = tmem_base + C6_SF_COL;
            // the loop's parameters in registers, and the halo row offset of each
            // k-block in smem: re-reading them from the constant bank inside the
            // issue loop stalled it for ~250 cycles per k-block
            const int nkb = prm.kblocks;
            const uint32_t breg = (uint32_t)prm.breg, sB32 = smem_u32(sB), breg16 = breg >> 4;
            const uint64_t bd0 = umma_desc_k_sw64(sB32);
            const bool skip_mma = C6_DBG(2) != 0;
            const bool k33 = prm.oh_kh == 3 && prm.kw == 3 && prm.cblocks == 1;
            const int wp4 = prm.wp * 4;  // one padded pixel row in 16-byte units
            if (TL) {  // k-block kb -> A start offset in 16-byte descriptor units
                for (int kb = lane; kb < nkb; kb += 32) {
                    const int tap = kb / prm.cblocks, cb = kb - tap * prm.cblocks;
                    const int ky = tap / prm.kw, kx = tap - ky * prm.kw;
                    kb_aoff[kb] = ((uint32_t)(cb * prm.hloads * KB_BYTES) + (uint32_t)(ky * prm.wp + kx) * 64u) >> 4;
                }
                __syncwarp();
            }
            mbar_wait(sf_ready, 0);
            tc_fence_after();
            uint32_t t = 0;
            int acc = 0, u = 0;  // tile u uses accumulator u % nacc for the (u / nacc)-th time
            for (int nt = 0; nt < prm.n_tiles; ++nt) {
                mbar_wait(b_full, nt & 1);
                tc_fence_after();
                for (int i = 0; i < my_m; ++i) {
                    if (TL && (u % nissuers) != which) {  // the other issuer's tile
                        t += stages_per_tile;
                        ++u;
                        if (++acc == prm.nacc) acc = 0;
                        continue;
                    }
                    if (!TL) {  // (halo form: folded into a_full by the producer)
                        const uint32_t acc_phase = (uint32_t)(u / prm.nacc) & 1;
                        mwait(prm.dbg, &tmem_empty[acc], acc_phase ^ 1);
                        tc_fence_after();
                    }
                    C6_TRACE(0, i);
                    const uint32_t d_tmem = tmem_base + (uint32_t)(acc * prm.acc_cols);
                    for (int sg = 0; sg < stages_per_tile; ++sg, ++t) {
                        const uint32_t s = t % A_ST;
                        if (!C6_DBG(4096)) mwait(prm.dbg, &a_full[s], (t / A_ST) & 1);
                        tc_fence_after();
                        C6_TRACE(1, i);
                        if (TL && lane == 0) {  // tap (ky,kx): the halo advanced by ky*wp + kx pixel rows
                            // (descriptor start-address fields advanced directly, in 16-byte units)
                            const uint64_t ad0 = umma_desc_k_sw64(smem_u32(sA + s * a_stage));
                            if (k33) {  // 3x3, 128 channels: straight-line, addresses scheduled ahead
#pragma unroll
                                for (int kb = 0; kb < 9; ++kb) {
                                    const uint64_t ad = ad0 + (uint32_t)((kb / 3) * wp4 + (kb % 3) * 4);
                                    const uint64_t bd = bd0 + (uint32_t)(kb * breg16);
                                    if (!skip_mma || kb == 0) {
                                        umma_mxf4_pair(d_tmem, ad, bd, idesc, sf, sf, kb != 0);
                                        umma_mxf4_pair(d_tmem, ad + 2, bd + 2, idesc, sf, sf, 1);
                                    }
                                }
                            } else {
                                for (int kb = 0; kb < nkb; ++kb) {
                                    const uint64_t ad = ad0 + kb_aoff[kb];
                                    const uint64_t bd = bd0 + (uint64_t)kb * breg16;
                                    if (!skip_mma || kb == 0) {
                                        umma_mxf4_pair(d_tmem, ad, bd, idesc, sf, sf, kb != 0);
                                        umma_mxf4_pair(d_tmem, ad + 2, bd + 2, idesc, sf, sf, 1);
                                    }
                                }
                            }
                            C6_TRACE(7, i);
                            umma_commit_pair(&a_empty[s], 0x3);
                        } else if (lane == 0) {
                            for (int j = 0; j < G; ++j) {
                                const int kb = sg * G + j;
                                const uint32_t a_addr = smem_u32(sA + s * a_stage + j * KB_BYTES);
                                const uint32_t b_addr = sB32 + (uint32_t)kb * breg;
#pragma unroll
                                for (int h = 0; h < 2; ++h)  // K = 64 per MMA = 32 bytes of the row
                                    umma_mxf4_pair(d_tmem, umma_desc_k_sw64(a_addr + h * 32),
                                                   umma_desc_k_sw64(b_addr + h * 32), idesc, sf, sf, (kb | h) != 0);
                            }
                            umma_commit_pair(&a_empty[s], 0x3);
                        }
                        __syncwarp();
                    }
                    if (lane == 0) umma_commit_pair(&tmem_full[acc], 0x3);
                    __syncwarp();
                    C6_TRACE(2, i);
                    ++u;
                    if (++acc == prm.nacc) acc = 0;
                }
                if (lane == 0) umma_commit_pair(b_empty, 0x3);
                __syncwarp();
            }
        }
    } else {
        // ===================== epilogue (both CTAs): warps 0-7 =====================
        const int wq = warp & 3;     // TMEM lane quarter
        const int half = warp >> 2;  // which accumulator (alternate tiles): two tiles drain concurrently
        const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
        tmem_st_32x32b_x8_fill(tmem_base + lane_base + C6_SF_COL, 0x7F7F7F7Fu);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(sf_ready), 0));
        const uint32_t tmem_empty0 = mapa_shared(smem_u32(&tmem_empty[0]), 0);
        const uint32_t epi = smem_u32(sEpi) + (uint32_t)warp * C6_EPI_BUFS * C6_EPI_BYTES;
        int nbuf = 0, u = 0;

        const int nch = bn / 16;
        const int nimg = TL ? prm.rows / prm.hpwp : 0;
        // epi_split: all 8 warps drain every tile, the two warps of a lane quarter
        // splitting its columns (whole 64-column groups first); else the two warp
        // groups take alternate tiles
        const int nch0 = (nch / 2 + 3) / 4 * 4 < nch ? (nch / 2 + 3) / 4 * 4 : nch;
        const int ch0 = prm.epi_split ? (half ? nch0 : 0) : 0, ch1 = prm.epi_split ? (half ? nch : nch0) : nch;
        for (int nt = 0; nt < prm.n_tiles; ++nt)
            for (int i = 0; i < my_m; ++i) {
                const int tu = u++;
                if (!prm.epi_split && (tu & 1) != half) continue;  // the two warp groups take alternate tiles
                const int acc = tu % prm.nacc;   // the MMA cycles through the accumulators
                const uint32_t acc_phase = (uint32_t)(tu / prm.nacc) & 1;
                const int mt = pair + i * npairs;
                const int row0 = mt * 2 * C6_BM + (int)rank * C6_BM + wq * 32;
                // halo form: the warp's 32 positions are padded pixels (img0, y0, x0 .. x0+31)
                // of one row (the pitch is a multiple of 32): one 4-D box store, the
                // border columns / rows clipped by the map's bounds
                int x0 = 0, y0 = 0, img0 = 0;
                if (TL) {
                    img0 = row0 / prm.hpwp;
                    const int rem = row0 - img0 * prm.hpwp;
                    y0 = rem / prm.wp;
                    x0 = rem - y0 * prm.wp;
                }
                cwait(prm.dbg, &tmem_full[acc], acc_phase);
                tc_fence_after();
                if ((warp & 3) == 0 && lane == 0) C6_TRACE(3, i);
                const uint32_t tacc = tmem_base + lane_base + (uint32_t)(acc * prm.acc_cols);
                // groups of 4 chunks = 64 columns: one 128-byte-swizzled box store
                // (TMA cost is per box row); a tail of fewer chunks: 16-column boxes
                for (int g = ch0; g < ch1; g += 4) {
                    const int nc = ch1 - g < 4 ? ch1 - g : 4;
                    uint32_t v[4][16];
                    if (C6_DBG(8)) {
#pragma unroll
                        for (int c = 0; c < 4; ++c)
#pragma unroll
                            for (int j = 0; j < 16; ++j) v[c][j] = (uint32_t)c;
                    } else {
#pragma unroll
                        for (int c = 0; c < 4; ++c)
                            if (c < nc) tmem_ld_32x32b_x16(tacc + (g + c) * 16, v[c]);
                        tmem_ld_wait();
                    }
                    if ((warp & 3) == 0 && lane == 0 && g == 0) C6_TRACE(9, i);
                    const uint32_t buf = epi + (uint32_t)nbuf * C6_EPI_BYTES;
                    if (lane == 0) bulk_wait_read<C6_EPI_BUFS - 1>();
                    __syncwarp();
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        if (c >= nc || C6_DBG(2048)) break;
                        uint32_t h[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j)  // exact f32 integer -> int16 (see gemm_fp4_pair.cu)
                            h[j] = __byte_perm(__float_as_uint(__uint_as_float(v[c][2 * j]) + 12582912.0f),
                                               __float_as_uint(__uint_as_float(v[c][2 * j + 1]) + 12582912.0f), 0x5410);
                        if (nc == 4) {  // SW128: 16-byte unit u of row lane at ((u ^ (lane & 7)) << 4)
                            const uint32_t rowaddr = buf + lane * 128;
                            sts_v4(rowaddr + (((2 * c) ^ (lane & 7)) << 4), h[0], h[1], h[2], h[3]);
                            sts_v4(rowaddr + (((2 * c + 1) ^ (lane & 7)) << 4), h[4], h[5], h[6], h[7]);
                        } else {        // SW32 1 KB boxes
                            const uint32_t rowaddr = buf + c * 1024 + lane * 32;
                            const uint32_t sw = (uint32_t)(lane >> 2) & 1;
                            sts_v4(rowaddr + (sw << 4), h[0], h[1], h[2], h[3]);
                            sts_v4(rowaddr + ((sw ^ 1) << 4), h[4], h[5], h[6], h[7]);
                        }
                    }
                    if ((warp & 3) == 0 && lane == 0 && g == 0) C6_TRACE(10, i);
                    if (!C6_DBG(1024)) fence_proxy_async_smem();
                    __syncwarp();
                    if ((warp & 3) == 0 && lane == 0 && g == 0) C6_TRACE(11, i);
                    if (lane == 0 && !C6_DBG(1)) {
                        const int col = nt * bn + g * 16;
                        if (TL) {  // (a box wholly outside the output is not issued)
                            if (y0 < prm.oh && img0 < nimg && x0 < prm.ow) {
                                if (nc == 4) tma_store_4d(&tmap_c64, buf, col, x0, y0, img0);
                                else
                                    for (int c = 0; c < nc; ++c)
                                        tma_store_4d(&tmap_c, buf + c * 1024, col + c * 16, x0, y0, img0);
                            }
                        } else if (nc == 4) {
                            tma_store_2d(&tmap_c64, buf, col, row0);
                        } else {
                            for (int c = 0; c < nc; ++c) tma_store_2d(&tmap_c, buf + c * 1024, col + c * 16, row0);
                        }
                        bulk_commit();
                    }
                    if ((warp & 3) == 0 && lane == 0 && g == 0) C6_TRACE(12, i);
                    nbuf = (nbuf + 1) % C6_EPI_BUFS;
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(tmem_empty0 + acc * 8);
                if ((warp & 3) == 0 && lane == 0) C6_TRACE(4, i);
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
LB_DEV uint4 pack_fp4_group(const int8_t* __restrict__ src, uint32_t& nz_all) {
    const uint4 lo = __ldg(reinterpret_cast<const uint4*>(src));
    const uint4 hi = __ldg(reinterpret_cast<const uint4*>(src) + 1);
    const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    uint32_t o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        uint32_t half[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t x = w[2 * q + h];
            const uint32_t nz = nonzero_msb(x) >> 7;  // per-byte nonzero (bit 0 of each byte)
            nz_all &= nz;
            // per-byte code 0x2 (+1) / 0xA (-1) / 0x0, then bytes -> nibbles:
            // c | c >> 4 puts bytes 0,1 in byte 0 and bytes 2,3 in byte 2
            const uint32_t c = nz * 2u + ((x >> 4) & 0x08080808u);
            const uint32_t t = c | (c >> 4);
            half[h] = __byte_perm(t, 0, 0x4420);  // bytes 0 and 2 -> 16 bits
        }
        o[q] = half[0] | (half[1] << 16);
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
}

// Halo form: fm4 spatially padded — pad zero rows above and below, pad zero
// pixels left, zeros right up to the row pitch — one block-stride loop
// iteration per padded pixel row (b, yp), threads over the row's (pixel,
// 32-channel group) pairs.
__global__ void conv_pack_fp4_padded_kernel(const int8_t* __restrict__ fm, int batch, int h, int w, int pad, int pitch,
                                            int gpp, int check_zero, uint8_t* __restrict__ out,
                                            int* __restrict__ zero_flag) {
    const int hp = h + 2 * pad, per_row = pitch * gpp;
    bool zero = false;
    for (int prow = blockIdx.x; prow < batch * hp; prow += gridDim.x) {
        const int img = prow / hp, y = prow - img * hp - pad;
        uint4* orow = reinterpret_cast<uint4*>(out) + (long long)prow * per_row;
        const bool yin = y >= 0 && y < h;
        for (int t = threadIdx.x; t < per_row; t += blockDim.x) {
            const int xp = t / gpp, cg = t - xp * gpp, x = xp - pad;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (yin && x >= 0 && x < w) {
                uint32_t nz_all = 0x01010101u;
                v = pack_fp4_group(fm + (((long long)img * h + y) * w + x) * gpp * 32 + cg * 32, nz_all);
                zero |= nz_all != 0x01010101u;
            }
            orow[t] = v;
        }
    }
    if (check_zero && zero && zero_flag) atomicOr(zero_flag, 1);
}

__global__ void conv_pack_fp4_kernel(const int8_t* __restrict__ fm, long long groups, int check_zero,
                                     uint8_t* __restrict__ out, int* __restrict__ zero_flag) {
    for (long long gi = blockIdx.x * (long long)blockDim.x + threadIdx.x; gi < groups;
         gi += (long long)gridDim.x * blockDim.x) {
        uint32_t nz_all = 0x01010101u;
        reinterpret_cast<uint4*>(out)[gi] = pack_fp4_group(fm + 32 * gi, nz_all);
        if (check_zero && nz_all != 0x01010101u && zero_flag) atomicOr(zero_flag, 1);
    }
}

static int pick_bn_conv(int cout) {
    const int tiles = (cout + C6_MAX_BN - 1) / C6_MAX_BN;
    const int per = (cout + tiles - 1) / tiles;
    return (per + 15) / 16 * 16;
}

// Halo form row pitch: the padded width rounded up to 32 pixels, so a warp's
// 32 consecutive positions never straddle two rows (one box store each).
static int halo_pitch(int w, int pad) { return (w + 2 * pad + 31) / 32 * 32; }

// 128-row boxes of one channel block of a halo tile
static int halo_loads(int w, int pad, int kh, int kw) {
    const int rows = C6_BM + (kh - 1) * halo_pitch(w, pad) + kw - 1;
    return (rows + C6_BM - 1) / C6_BM;
}

// The halo form: stride 1, padded pixel positions indexable in 32 bits, at
// least 60% of them real outputs (the rest is border and pitch padding), and
// two halo tiles fit next to the resident filter.
static bool halo_ok(int batch, int h, int w, int c, int cout, int kh, int kw, int stride, int pad) {
    const int hp = h + 2 * pad, pitch = halo_pitch(w, pad);
    if (stride != 1 || (long long)batch * hp * pitch >= 0x7FFFFFFFLL - 65536) return false;
    const long long outs = (long long)(hp - kh + 1) * (w + 2 * pad - kw + 1);
    if (outs * 10 < (long long)hp * pitch * 6) return false;
    const int kblocks = kh * kw * (c / 128);
    const int breg = ((pick_bn_conv(cout) / 2) * 64 + 1023) / 1024 * 1024;
    const long long stage = (long long)(c / 128) * halo_loads(w, pad, kh, kw) * C6_KB_BYTES;
    return kblocks * breg <= C6_B_MAX && (C6_RING_BUDGET - kblocks * breg) / stage >= 2;
}

// fm4: the halo form's padded map (the larger of the two layouts)
size_t conv_fp4_workspace_bytes(int batch, int h, int w, int c, int pad) {
    return (size_t)batch * (h + 2 * pad) * halo_pitch(w, pad) * c / 2 + 1024;
}

// Whether K6 takes a conv (in the im2col form at least; the halo form is
// picked when it also fits): the zero fill must be the padding value,
// channels tile into 128-channel k-blocks, and the filter fits the resident
// budget.
bool conv_fp4_applies(int mode, int fm_binary, int c, int cout, int kh, int kw, int padding, long long rows,
                      int stride) {
    if (!(padding == 0 || !fm_binary) || c % 128 != 0 || cout % 8 != 0 || rows > 0x7FFFFFFFLL) return false;
    (void)mode;
    (void)stride;
    const int kblocks = kh * kw * (c / 128);
    const int bn = pick_bn_conv(cout);
    const int breg = ((bn / 2) * 64 + 1023) / 1024 * 1024;
    const int g = kblocks % 4 == 0 ? 4 : (kblocks % 3 == 0 ? 3 : (kblocks % 2 == 0 ? 2 : 1));
    return kblocks * breg <= C6_B_MAX && (C6_RING_BUDGET - kblocks * breg) / (g * C6_KB_BYTES) >= 2;
}

lowbit_status launch_conv_fp4(const int8_t* fm, int batch, int h, int w, int cch, int kh, int kw, int stride,
                              int pad, int check_zero, const void* weights, int b_ternary, int cout, int16_t* out,
                              void* workspace, int* zero_flag, cudaStream_t stream) {
    const int oh = (h + 2 * pad - kh) / stride + 1, ow = (w + 2 * pad - kw) / stride + 1;
    const long long rows = (long long)batch * oh * ow;
    const int k = kh * kw * cch;
    static const bool no_tl = lb::tuning_env("LOWBIT_CONV_IM2COL") != nullptr;  // tuning experiment knob
    const bool tl = halo_ok(batch, h, w, cch, cout, kh, kw, stride, pad) && !no_tl;
    const int hp = h + 2 * pad, wp = halo_pitch(w, pad);
    uint8_t* fm4 = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(workspace) + 1023) & ~uintptr_t(1023));
    static std::atomic<bool> carve[kMaxDevices] = {};  // idempotent attribute: racing setters agree
    const int cdev = current_device();
    if (cdev >= kMaxDevices || !carve[cdev].load(std::memory_order_relaxed)) {  // run the pack passes with K6's shared-memory carveout: no L1/smem reconfiguration between them
        cudaFuncSetAttribute(conv_pack_fp4_padded_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
        cudaFuncSetAttribute(conv_pack_fp4_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
        if (cdev < kMaxDevices) carve[cdev].store(true, std::memory_order_relaxed);
    }
    if (tl) {
        const int prows = batch * hp;
        const int blocks = prows < 64 * num_sms() ? prows : 64 * num_sms();
        conv_pack_fp4_padded_kernel<<<blocks, 256, 0, stream>>>(fm, batch, h, w, pad, wp, cch / 32, check_zero, fm4,
                                                                 zero_flag);
    } else {
        const long long groups = (long long)batch * h * w * cch / 32;
        conv_pack_fp4_kernel<<<grid_for(groups, 256), 256, 0, stream>>>(fm, groups, check_zero, fm4, zero_flag);
    }
    LB_CUDA_TRY(cudaGetLastError());

    const WeightsLayout L(b_ternary, cout, k);
    const uint8_t* wfp4 = static_cast<const uint8_t*>(weights) + L.off_fp4;

    ConvF4Params prm{};
    const long long grows = tl ? (long long)batch * hp * wp : rows;  // GeMM rows: padded positions when tiled
    prm.rows = (int)grows;
    prm.cout = cout;
    prm.kblocks = kh * kw * (cch / 128);
    prm.g = prm.kblocks % 4 == 0 ? 4 : (prm.kblocks % 3 == 0 ? 3 : (prm.kblocks % 2 == 0 ? 2 : 1));
    prm.bn = pick_bn_conv(cout);
    prm.m_tiles = (int)((grows + 2 * C6_BM - 1) / (2 * C6_BM));
    prm.n_tiles = (cout + prm.bn - 1) / prm.bn;
    prm.ow = ow;
    prm.ohw = oh * ow;
    prm.stride = stride;
    prm.pad = pad;
    prm.kw = kw;
    prm.cblocks = cch / 128;
    prm.oh = oh;
    prm.wp = wp;
    prm.hpwp = hp * wp;
    prm.hloads = halo_loads(w, pad, kh, kw);
    prm.oh_kh = kh;
    static const int epi_split = lb::tuning_env("LOWBIT_CONV_EPI_ALT") ? 0 : 1;  // tuning experiment knob
    prm.epi_split = epi_split;
    prm.nacc = 3 * prm.bn <= (int)C6_SF_COL ? 3 : 2;
    prm.acc_cols = prm.nacc == 3 ? (int)C6_SF_COL / 3 : C6_MAX_BN;
    static const int dbg = lb::tuning_env("LOWBIT_CONV_DEBUG") ? atoi(lb::tuning_env("LOWBIT_CONV_DEBUG")) : 0;
    prm.dbg = dbg;
    prm.breg = ((prm.bn / 2) * 64 + 1023) / 1024 * 1024;
    prm.a_st = (C6_RING_BUDGET - prm.kblocks * prm.breg) /
               (tl ? prm.cblocks * prm.hloads * C6_KB_BYTES : prm.g * C6_KB_BYTES);
    if (prm.a_st > C6_MAX_A_ST) prm.a_st = C6_MAX_A_ST;
    prm.ldc = cout;
    prm.c = out;
    CUtensorMap mb, ma, mc, mc64;
    if (!make_map_2d(&mb, wfp4, (uint64_t)L.kp4 / 2, (uint64_t)L.np, (uint64_t)L.kp4 / 2, 64, (uint32_t)(prm.bn / 2),
                     CU_TENSOR_MAP_SWIZZLE_64B))
        return lbhost::set_error(LOWBIT_CUDA_ERROR, "cuTensorMapEncodeTiled failed for the conv filter");
    if (tl) {  // padded fm4 as rows of pixels; boxes past the end read zeros
        if (!make_map_2d(&ma, fm4, (uint64_t)cch / 2, (uint64_t)grows, (uint64_t)cch / 2, 64, C6_BM,
                         CU_TENSOR_MAP_SWIZZLE_64B))
            return lbhost::set_error(LOWBIT_CUDA_ERROR, "cuTensorMapEncodeTiled failed for the padded feature map");
    } else if (!make_map_im2col(&ma, fm4, batch, h, w, cch / 2, kh, kw, stride, pad, 64, C6_BM,
                                CU_TENSOR_MAP_SWIZZLE_64B)) {
        return lbhost::set_error(LOWBIT_CUDA_ERROR, "cuTensorMapEncodeIm2col failed (fp4 feature map)");
    }
    const bool mc_ok = tl ? make_map_conv_out(&mc, out, batch, oh, ow, cout, 16) &&
                                make_map_conv_out(&mc64, out, batch, oh, ow, cout, 64)
                          : make_map_2d(&mc, out, (uint64_t)cout, (uint64_t)rows, (uint64_t)cout * 2, 16, 32,
                                        CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_DATA_TYPE_UINT16) &&
                                make_map_2d(&mc64, out, (uint64_t)cout, (uint64_t)rows, (uint64_t)cout * 2, 64, 32,
                                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_UINT16);
    if (!mc_ok) return lbhost::set_error(LOWBIT_CUDA_ERROR, "cuTensorMapEncodeTiled failed for the conv output");
    static SmemOptIn attr[2];
    LB_CUDA_TRY(attr[tl].ensure(tl ? conv_fp4_pair_kernel<true> : conv_fp4_pair_kernel<false>, C6_SMEM));
    const int pairs = prm.m_tiles < num_sms() / 2 ? prm.m_tiles : num_sms() / 2;
    if (tl) conv_fp4_pair_kernel<true><<<2 * pairs, C6_THREADS, C6_SMEM, stream>>>(mb, ma, mc, mc64, prm);
    else conv_fp4_pair_kernel<false><<<2 * pairs, C6_THREADS, C6_SMEM, stream>>>(mb, ma, mc, mc64, prm);
    LB_CUDA_TRY(cudaGetLastError());
    return LOWBIT_OK;
}

}  // namespace lb

extern "C" int lowbit_debug_conv_trace(unsigned long long* out1024) {
    return cudaMemcpyFromSymbol(out1024, lb::g_conv_trace, sizeof(unsigned long long) * 1024) != cudaSuccess;
}
