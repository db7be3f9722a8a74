// conv_fp4_halo.cu — K7: fused halo convolution on the fp4 tensor cores
// (stride 1, the int8 feature map read once, no packed copy, no im2col).
//
// conv2d_lowbit (conv.cpp:33-59) is im2col -> encode -> pack_b -> gemm_lowbit
// with GeMM depth index k = (ky*kw + kx)*C + c (conv.cpp:18-27).  Here one
// kernel does all of it:
//
//   * Output positions are laid out on a padded grid of pitch P = 32, 64 or
//     128 >= W + 2*pad: a CTA tile is R = 128/P whole output rows of one
//     image (position i = ry*P + ox).  Its input "halo" is the R + kh - 1
//     padded input rows starting at y0 - pad, P pixels each starting at
//     x = -pad: ONE 4-D TMA box of the int8 NHWC map per 128-channel block,
//     whose out-of-image elements read as zero — the padding.  Rows wider
//     than 128 padded pixels (or whenever it takes fewer tiles) are cut into
//     column blocks of P = 32 positions with 32 - (kw - 1) valid outputs.
//   * Converter warps turn the int8 halo into packed e2m1 (two channels per
//     byte) in a 64-byte-swizzled shared-memory tile: halo position j is
//     UMMA row j.
//   * Filter tap (ky, kx) of output position i reads halo position
//     i + ky*P + kx, so the A operand of that tap is the halo tile's UMMA
//     descriptor advanced by ky*P + kx rows (the swizzle is a function of
//     the absolute address; tools/micro/halo_check.cu) — no im2col exists
//     anywhere.  Positions with ox >= OW (or rows past OH) are computed and
//     dropped; their taps may read a few rows past the halo (garbage-in,
//     never stored).
//   * The filter (prepared weights, fp4 section, K-major) stays resident in
//     shared memory; tcgen05.mma.cta_group::2.kind::mxf4.block_scale with
//     f32 accumulators.
//   * Encoding: +-1 activations become +-0.5 (e2m1 0x1 / 0x9 = the int8 byte
//     AND 0x09; a chunk holding any value outside {-1, 0, +1} is mapped by
//     sign, as encode_ternary does), the filter stays +-1.0: every product is
//     +-0.5.  A bias MMA first sets every accumulator element to 1.5 * 2^22
//     (uniform operands under a 2^16 block scale), so the exact partial sums
//     live in [2^22, 2^23) — f32 spacing 0.5 — and the low 16 bits of each
//     f32 are the int16 result.
//   * The epilogue: two warps per TMEM lane quarter and tile, each half of the
//     tile's columns; tcgen05.ld.pack::16b loads those low halves as packed
//     words (releasing the accumulator at once), which go into a 128-byte-
//     swizzled staging box and out by TMA store: 32 pixels x 64 columns,
//     clipped at the image edges by the tensor map.
//
// Warp roles per CTA (NEPI = 16: 864 threads, or 8: 608): 0 .. NEPI-1
// epilogue (two warps per TMEM lane quarter and tile, each half of the tile's
// columns; with 16, two groups on alternate tiles), then 8 converters, the
// TMA producer (raw halo + filter) and two UMMA issuers on alternate tiles
// (leader CTA; the first also owns TMEM).
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "encode.cuh"
#include "halo_common.cuh"
#include "layout.cuh"
#include "tmap.cuh"

namespace lb {

constexpr int H7_BM = 128;        // output positions per CTA tile (256 per pair)
// Epilogue warps NEPI (a kernel template parameter): 16 — two groups of 8 drain
// alternate tiles, two tiles in flight (5% faster on config 4) — when their 64 KB
// of staging fits next to the filter and the halo rings, else 8.
#ifndef H7_NCONV_WARPS
#define H7_NCONV_WARPS 8
#endif
constexpr int H7_NCONV = H7_NCONV_WARPS;  // converter warps
__host__ __device__ constexpr int h7_threads(int nepi) { return 32 * (nepi + H7_NCONV + 4); }
constexpr int H7_MAX_BN = 240;    // cout per tile: accumulators + scales <= 512 TMEM columns
constexpr uint32_t H7_SF_COL = 480;       // unit UE8M0 scales (8 columns)
constexpr uint32_t H7_SFBIAS_COL = 488;   // the bias MMA's A scales, 2^16 (8 columns)
// Bias MMA operands: every A element e2m1 1.0, every B element 1.5.  Uniform bytes, so one 8-row
// swizzle atom (512 B) stands for every atom of the operand: the descriptors' stride between atoms is 0.
#ifndef H7_BIAS_FULL
constexpr int H7_BIAS_A = 512, H7_BIAS_B = 512;
constexpr uint32_t H7_BIAS_SBO = 0;
#else
constexpr int H7_BIAS_A = 8 * 1024, H7_BIAS_B = 8 * 1024;  // 128 / up to 120 rows x 64 B
constexpr uint32_t H7_BIAS_SBO = 512;
#endif
#ifndef H7_RAW_CAP
#define H7_RAW_CAP 4
#endif
#ifndef H7_NEPI_MAX
#define H7_NEPI_MAX 16
#endif
constexpr int H7_SMEM = 227 * 1024;
constexpr int H7_BAR_BYTES = 1024;  // barriers + the k-block offset table
__host__ __device__ constexpr int h7_epi_bytes(int nepi) { return nepi * 4096; }  // one 32 px x 64 col box per warp
constexpr int H7_MAX_KB = 96;       // k-blocks (taps x channel blocks) the offset table holds
constexpr int H7_MAX_ST = 4;        // raw / fp4 ring depth cap
constexpr int H7_RAW_MAX = 64 * 1024;

struct HaloParams {
    int batch, h, w, oh, ow, pad, kw, cblocks;
    int P, log2p, R, rows_h;   // position pitch (32, 64 or 128), output rows per CTA tile, halo rows
    int tpi, ctiles, ptiles;   // CTA tiles per image, CTA tiles, pair tiles
    int nxb, vx;               // column blocks per row of tiles and output pixels per block (ow when one block)
    int cout, bn, n_tiles, kblocks;
    int breg;                  // bytes of one resident filter k-block (1 KB aligned)
    int raw_cb;                // bytes of one channel block of a raw stage
    int f4_cb;                 // bytes of one channel block of an fp4 halo (1 KB aligned)
    int raw_st, f4_st;         // ring depths
    int nacc, acc_cols;        // TMEM accumulators and their column stride
    int k33;                   // 3x3 filter over one channel block: the unrolled issue loop
    uint32_t mul16;            // 16: the converters' multiplier (a register operand keeps their shifts IMADs)
    int check_zero;            // binary map: a 0 activation sets *zero_flag (core.cpp:23)
    uint32_t pad_word;         // binary map padded with +-1 (binary_pad_value, conv.cpp:13): 4 int8 pad values;
                               // 0 when the padding reads as 0 (the TMA's out-of-bounds fill)
    int dbg;                   // timing experiments (LOWBIT_HALO_DEBUG): 1 no stores, 2 no MMAs, 4 no conversion,
                               // 8 no TMEM loads, 16 no staging stores,
                               // 64 epilogue ignores tmem_full, 128 epilogue drains nothing, 32 trace,
                               // 512 no raw halo loads, 2048 no tiles (setup + teardown only), 4096 one MMA issuer,
                               // 32768 return at entry (launch cost)
    int16_t* out;
    int* zero_flag;
};

// Timing experiments (HaloParams::dbg) exist only in -DLOWBIT_TUNING builds: in the product
// kernel H7_DBG is the constant 0, so the experiments' branches and constants are compiled out
// (left in, their hoisted register set-ups cost the epilogue ~90 instructions per tile).
#ifdef LOWBIT_TUNING
#define H7_DBG(bits) (prm.dbg & (bits))
#else
#define H7_DBG(bits) 0
#endif

// dbg & 32: per-tile event times (clock64) of pair 0's leader CTA, read by lowbit_debug_halo_trace
__device__ unsigned long long g_halo_trace[16 * 64];
// dbg & 32: kernel phases in %globaltimer ns over all CTAs: first entry, last end of setup,
// last end of work, last exit
__device__ unsigned long long g_halo_phase[4];
LB_DEV unsigned long long h7_gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define H7_TRACE(ev, i) \
    if (H7_DBG(32) && pair == 0 && leader && (i) < 64) g_halo_trace[(ev) * 64 + (i)] = clock64()

// waits of the non-issuing roles: suspend-hinted try_wait (dbg & 1024: plain try_wait)
LB_DEV void h7_wait(int dbg, uint64_t* bar, uint32_t parity) {
#ifdef LOWBIT_TUNING
    if (dbg & 1024) mbar_wait(bar, parity);
    else mbar_wait_sleep(bar, parity);
#else
    (void)dbg;
    mbar_wait_sleep(bar, parity);
#endif
}


// FLAGS bit 0 (PADFILL): a binary map padded with +-1 — the converters write the pad codes;
// bit 1 (CHECKZ): a binary BNN map — a 0 in a real pixel raises ZeroInBinaryInput (core.cpp:23).
// Both are folded into the converters' load/convert batch.
template <int NEPI, int FLAGS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(h7_threads(NEPI), 1)
    conv_fp4_halo_kernel(const __grid_constant__ CUtensorMap tmap_b, const __grid_constant__ CUtensorMap tmap_raw,
                         const __grid_constant__ CUtensorMap tmap_c64, const __grid_constant__ CUtensorMap tmap_c16,
                         const HaloParams prm) {
    constexpr int H7_W_CONV = NEPI, H7_W_PROD = H7_W_CONV + H7_NCONV, H7_W_MMA = H7_W_PROD + 1,
                  H7_W_WAIT = H7_W_MMA + 2;
    constexpr bool PADFILL = (FLAGS & 1) != 0, CHECKZ = (FLAGS & 2) != 0;
    if (H7_DBG(32768)) return;  // launch-overhead probe

    if (H7_DBG(32) && threadIdx.x == 0) atomicMin(&g_halo_phase[0], h7_gtime());
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int CB = prm.cblocks;
    const int raw_stage = CB * prm.raw_cb, f4_stage = CB * prm.f4_cb;
    uint8_t* sB = smem;                                      // resident filter: kblocks x breg
    uint8_t* sRaw = sB + prm.kblocks * prm.breg;             // raw int8 halo ring
    uint8_t* sF4 = sRaw + prm.raw_st * raw_stage;            // fp4 halo ring (the UMMA A operand)
    uint8_t* sEpi = sF4 + prm.f4_st * f4_stage;             // epilogue staging: 4 KB per epilogue warp
    uint8_t* sBiasA = sEpi + h7_epi_bytes(NEPI);             // the bias MMA's operands (uniform bytes)
    uint8_t* sBiasB = sBiasA + H7_BIAS_A;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sBiasB + H7_BIAS_B);
    uint64_t* raw_full = bars;            // local: TMA landed the raw halo
    uint64_t* raw_empty = bars + 4;       // local: the converter warps are done with it
    uint64_t* a_full = bars + 8;          // leader: fp4 halos of both CTAs written (all converter warps)
    uint64_t* a_empty = bars + 12;        // local: the pair's MMAs are done with the fp4 halo
    uint64_t* b_full = bars + 16;         // leader: the filter of this n tile landed (both CTAs)
    uint64_t* b_empty = bars + 17;        // local: both issuers' MMAs done with the filter
    uint64_t* tmem_full = bars + 18;      // local (3): accumulator complete
    uint64_t* tmem_empty = bars + 21;     // leader (3): the 16 epilogue warps (8 per CTA) drained it
    uint64_t* sf_ready = bars + 24;       // leader: unit scales written (16 warps)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 25);
    uint32_t* kb_aoff = reinterpret_cast<uint32_t*>(bars + 32);  // k-block -> A row offset (16-byte units)

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int bn = prm.bn, bnh = bn >> 1;
    const int my_tiles = (prm.ptiles > pair && !H7_DBG(2048)) ? (prm.ptiles - pair + npairs - 1) / npairs : 0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < H7_MAX_ST; ++s) {
            mbar_init(&raw_full[s], 1);
            mbar_init(&raw_empty[s], H7_NCONV);
            mbar_init(&a_full[s], 2 * H7_NCONV);
            mbar_init(&a_empty[s], 1);
        }
        mbar_init(b_full, 1);
        mbar_init(b_empty, 2);
        for (int a = 0; a < 3; ++a) {
            mbar_init(&tmem_full[a], 1);
            mbar_init(&tmem_empty[a], 16);
        }
        mbar_init(sf_ready, 16);
        fence_barrier_init();
    }
    // The bias MMA (see the issuers): every A element 1.0 (0x22), every B element 1.5 (0x33);
    // uniform bytes, so the swizzle does not matter.
    for (int i = threadIdx.x; i < (H7_BIAS_A + H7_BIAS_B) / 16; i += h7_threads(NEPI)) {
        const uint32_t w = i < H7_BIAS_A / 16 ? 0x22222222u : 0x33333333u;
        sts_v4(smem_u32(sBiasA) + i * 16, w, w, w, w);
    }
    fence_proxy_async_smem();
    if (warp == H7_W_PROD && lane == 0) {
        tma_prefetch_desc(&tmap_raw);
        tma_prefetch_desc(&tmap_b);
        tma_prefetch_desc(&tmap_c64);
        tma_prefetch_desc(&tmap_c16);
    }
    if (warp == H7_W_MMA) {
        tmem_alloc_pair<512>(tmem_slot);
        for (int kb = lane; kb < prm.kblocks; kb += 32) {  // tap (ky,kx), channel block cb
            const int tap = kb / CB, cb = kb - tap * CB;
            const int ky = tap / prm.kw, kx = tap - ky * prm.kw;
            kb_aoff[kb] = ((uint32_t)(cb * prm.f4_cb) + (uint32_t)(ky * prm.P + kx) * 64u) >> 4;
        }
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // programmatic dependent launch: the setup above (barriers, TMEM, the k-block table)
    // overlaps the previous kernel's tail; global memory is touched only after this
    // The next kernel in the stream may begin launching now: its CTAs take each SM as this grid's
    // CTA leaves it and run their own setup, then block in griddepcontrol.wait until this grid has
    // completed (c4 back to back: 20.2 -> 19.9 us).
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (H7_DBG(32) && threadIdx.x == 0) atomicMax(&g_halo_phase[1], h7_gtime());

    if (warp == H7_W_PROD) {
        // ===================== TMA producer (both CTAs): filter + raw halos =====================
        if (lane == 0 && my_tiles > 0) {
            const uint32_t b_full0 = mapa_shared(smem_u32(b_full), 0);
            uint32_t t = 0;
            H7Ring rr;
            rr.init(prm.raw_st);
            auto load_filter = [&](int nt) {
                h7_wait(prm.dbg, b_empty, (nt & 1) ^ 1);
                if (leader) mbar_arrive_expect_tx(b_full, (uint32_t)prm.kblocks * bn * 64);
                const int brow = nt * bn + (int)rank * bnh;
                for (int kb = 0; kb < prm.kblocks; ++kb)
                    tma_load_2d_pair(smem_u32(sB + kb * prm.breg), &tmap_b, b_full0, kb * 64, brow);
            };
            for (int nt = 0; nt < prm.n_tiles; ++nt) {
                // the kernel's first halo comes from HBM and gates the first tile: it goes out before
                // the filter (an L2 hit for all but the first CTAs)
                if (nt > 0) load_filter(nt);
                H7Walk wk;
                wk.init(pair * 2 + (int)rank, 2 * npairs, prm.tpi);
                for (int i = 0; i < my_tiles; ++i, ++t, wk.next(), rr.next()) {
                    const uint32_t s = rr.idx;
                    h7_wait(prm.dbg, &raw_empty[s], rr.phase ^ 1);
                    if (nt == 0) H7_TRACE(0, i);
                    if (H7_DBG(512)) {  // timing experiment: no raw loads (stale halo)
                        mbar_arrive(&raw_full[s]);
                        if (t == 0) load_filter(0);
                        continue;
                    }
                    mbar_arrive_expect_tx(&raw_full[s], (uint32_t)raw_stage);
                    const int ct = (pair + i * npairs) * 2 + (int)rank;  // this CTA's tile
                    int img = wk.img;
                    const int rem = wk.rem, yb = prm.nxb == 1 ? rem : rem / prm.nxb;
                    int y0 = yb * prm.R, x0 = (rem - yb * prm.nxb) * prm.vx;
                    if (ct >= prm.ctiles) img = prm.batch - 1, y0 = 0, x0 = 0;  // odd tail: any real box, never stored
                    for (int cb = 0; cb < CB; ++cb)
                        tma_load_4d(smem_u32(sRaw + s * raw_stage + cb * prm.raw_cb), &tmap_raw,
                                    smem_u32(&raw_full[s]), cb * 128, x0 - prm.pad, y0 - prm.pad, img);
                    if (t == 0) load_filter(0);
                }
            }
        }
    } else if (warp >= H7_W_CONV && warp < H7_W_PROD) {
        // ===================== converters (both CTAs): raw int8 halo -> fp4 halo =====================
        const int cw = warp - H7_W_CONV;
        const uint32_t a_full0 = mapa_shared(smem_u32(&a_full[0]), 0);
        // loop constants in registers (kernel parameters would be re-read after
        // every shared-memory store: the stores' asm clobbers memory)
        const int P = prm.P, lp = prm.log2p, rows_h = prm.rows_h, raw_st = prm.raw_st, f4_st = prm.f4_st;
        const int raw_cb = prm.raw_cb, f4_cb = prm.f4_cb, tpi = prm.tpi, R = prm.R, ctiles = prm.ctiles;
        const bool convert = !H7_DBG(4);
        const int npos = rows_h * P;             // a multiple of 32
        constexpr int STEP = 4 * H7_NCONV;     // positions per iteration of all converter warps
        const int nfull = npos / (8 * STEP), nrem = (npos % (8 * STEP)) / STEP;  // batches of 8 loads, a last partial one
        const int nbatch = nfull + (nrem != 0);
        const int chunk = lane & 7;              // 16 channels of one position
        const int j0 = cw * 4 + (lane >> 3);     // this lane's first position; then every STEP-th
        auto raw_off = [](int j) -> uint32_t { return (uint32_t)j << 7; };  // raw layout: [position] x 128 B
        // SW64: 16-byte unit u of row j at j*64 + ((u ^ ((j >> 1) & 3)) << 4); (j >> 1) & 3 is the
        // same for all of this lane's positions (they step by a multiple of 8)
        const uint32_t swz = ((((uint32_t)chunk >> 1) ^ (((uint32_t)j0 >> 1) & 3u)) << 4) + (chunk & 1) * 8;
        // multipliers held in registers (from a kernel parameter), so the converters'
        // shifts stay IMADs on the FMA pipe instead of ALU-pipe shifts
        const uint32_t k16 = prm.mul16, k2 = k16 >> 3;
        bool zero = false;
        uint32_t t = 0;
        H7Ring rr, fr;
        rr.init(raw_st);
        fr.init(f4_st);
        for (int nt = 0; nt < prm.n_tiles; ++nt)
            for (int i = 0; i < my_tiles; ++i, ++t, rr.next(), fr.next()) {
                const uint32_t rs = rr.idx, fs = fr.idx;
                // the waiter warp saw this tile's raw halo land and its fp4 slot free (an mbarrier
                // try_wait costs the waiting thread ~270 cycles even on a completed phase: two per
                // tile were on the converters' critical path); one named barrier per raw slot
                named_bar_sync(3 + rs, 32 * (H7_NCONV + 1));
                if (cw == 0 && lane == 0) H7_TRACE(2, t);
                int ytop = 0, xleft = 0;  // image row / column of halo position 0 (binary maps: padding / zero checks)
                if (PADFILL || CHECKZ) {
                    const int ct = (pair + i * npairs) * 2 + (int)rank;
                    const int img = ct / tpi;
                    const int rem = ct - img * tpi, yb = prm.nxb == 1 ? rem : rem / prm.nxb;
                    const bool tail = ct >= ctiles;  // odd tail: the box at the image's corner
                    ytop = (tail ? 0 : yb * R) - prm.pad;
                    xleft = (tail ? 0 : (rem - yb * prm.nxb) * prm.vx) - prm.pad;
                }
                const bool chk = CHECKZ && nt == 0;
                if (convert)
                    for (int cb = 0; cb < CB; ++cb) {
                        const uint32_t src = smem_u32(sRaw + rs * raw_stage + cb * raw_cb) + chunk * 16;
                        const uint32_t dst = smem_u32(sF4 + fs * f4_stage + cb * f4_cb) + swz;
                        // a batch: NQ loads in flight (NQ a compile-time count: with a run-time count the
                        // loads serialise behind their predicates), then as many stores
                        auto batch = [&](auto nq_c, int bi) {
                            constexpr int NQ = decltype(nq_c)::value;
                            const int jb = j0 + bi * 8 * STEP;
                            uint4 v[NQ];
#pragma unroll
                            for (int q = 0; q < NQ; ++q) v[q] = lds_v4(src + raw_off(jb + STEP * q));
                            // The tile's last loads are issued: hand the raw slot back now, not after the
                            // conversion (the arrive follows the loads through the same in-order queue), so
                            // the producer's next halo load — ~1,800 cycles from issue to landing with the
                            // epilogue's TMA stores in the same queue — starts ~1,000 cycles earlier.
                            if (cb == CB - 1 && bi == nbatch - 1) {
                                __syncwarp();
                                if (lane == 0) mbar_arrive(&raw_empty[rs]);
                            }
                            if (PADFILL || chk) {
#pragma unroll
                                for (int q = 0; q < NQ; ++q) {
                                    const int j = jb + STEP * q;
                                    const int y = ytop + (j >> lp), x = (j & (P - 1)) + xleft;
                                    const bool real = (unsigned)y < (unsigned)prm.h && (unsigned)x < (unsigned)prm.w;
                                    if (chk && real && !h7_all_nonzero(v[q])) zero = true;
                                    if (PADFILL && !real) v[q] = make_uint4(prm.pad_word, prm.pad_word, prm.pad_word, prm.pad_word);
                                }
                            }
                            uint32_t bad = 0;
#pragma unroll
                            for (int q = 0; q < NQ; ++q) {
                                sts_v2(dst + (uint32_t)(jb + STEP * q) * 64u, h7_pack8(v[q].x, v[q].y, k16),
                                       h7_pack8(v[q].z, v[q].w, k16));
                                bad |= h7_bad16(v[q], k2);
                            }
                            if ((bad & 0xFEFEFEFEu) != 0) {  // a value outside {-1, 0, +1}: rewrite the chunks by sign
#pragma unroll
                                for (int q = 0; q < NQ; ++q)
                                    sts_v2(dst + (uint32_t)(jb + STEP * q) * 64u, h7_pack8_sign(v[q].x, v[q].y),
                                           h7_pack8_sign(v[q].z, v[q].w));
                            }
                        };
                        for (int bi = 0; bi < nfull; ++bi) batch(std::integral_constant<int, 8>{}, bi);
                        // the last, partial batch: 2, 4 or 6 loads at once (the halo sizes 3x3 / 5x5 / 1x1 filters
                        // give on each pitch), any other count one load at a time
                        if (nrem == 6) batch(std::integral_constant<int, 6>{}, nfull);
                        else if (nrem == 4) batch(std::integral_constant<int, 4>{}, nfull);
                        else if (nrem == 2) batch(std::integral_constant<int, 2>{}, nfull);
                        else if (nrem != 0) {
                            for (int q = 0; q < nrem; ++q) {
                                const int j = j0 + nfull * 8 * STEP + STEP * q;
                                uint4 v = lds_v4(src + raw_off(j));
                                if (PADFILL || chk) {
                                    const int y = ytop + (j >> lp), x = (j & (P - 1)) + xleft;
                                    const bool real = (unsigned)y < (unsigned)prm.h && (unsigned)x < (unsigned)prm.w;
                                    if (chk && real && !h7_all_nonzero(v)) zero = true;
                                    if (PADFILL && !real) v = make_uint4(prm.pad_word, prm.pad_word, prm.pad_word, prm.pad_word);
                                }
                                sts_v2(dst + (uint32_t)j * 64u, h7_pack8_sign(v.x, v.y), h7_pack8_sign(v.z, v.w));
                            }
                            if (cb == CB - 1) {
                                __syncwarp();
                                if (lane == 0) mbar_arrive(&raw_empty[rs]);
                            }
                        }
                    }
                if (cw == 0 && lane == 0) H7_TRACE(15, t);
                fence_proxy_async_smem();
                __syncwarp();
                if (cw == 0 && lane == 0) H7_TRACE(3, t);
                if (lane == 0) {
                    if (!convert) mbar_arrive(&raw_empty[rs]);  // else released after the last loads
                    mbar_arrive_cluster(a_full0 + fs * 8);
                }
            }
        if (zero && prm.zero_flag) atomicOr(prm.zero_flag, 1);
    } else if (warp == H7_W_WAIT) {
        // ===================== converter waiter (both CTAs) =====================
        // Waits for tile t's raw halo (raw_full) and its free fp4 slot (a_empty), then
        // releases the converters through named barrier 3 + t % raw_st.  It cannot run more
        // than raw_st tiles ahead (raw_full of tile t needs the converters' raw_empty of tile
        // t - raw_st, arrived after their bar.sync on the same barrier), so each barrier
        // generation pairs one waiter arrival with one converter pass.
        const int raw_st = prm.raw_st, f4_st = prm.f4_st;
        uint32_t t = 0;
        H7Ring rr, fr;
        rr.init(raw_st);
        fr.init(f4_st);
        for (int nt = 0; nt < prm.n_tiles; ++nt)
            for (int i = 0; i < my_tiles; ++i, ++t, rr.next(), fr.next()) {
                const uint32_t rs = rr.idx, fs = fr.idx;
                h7_wait(prm.dbg, &raw_full[rs], rr.phase);
                if (lane == 0) H7_TRACE(1, t);
                h7_wait(prm.dbg, &a_empty[fs], fr.phase ^ 1);
                __syncwarp();
                named_bar_arrive(3 + rs, 32 * (H7_NCONV + 1));
            }
    } else if (warp >= H7_W_MMA) {
        // ===================== UMMA issuers (leader CTA): alternate tiles =====================
        // A waiting issuer thread stalls for ~300 cycles per mbarrier wait while
        // only a few 64-cycle (N = 128) MMAs are queued; two issuers keep the
        // tensor pipe fed across each other's waits.
        const int which = warp - H7_W_MMA;
        if (leader && my_tiles > 0) {
            const uint32_t idesc = idesc_mxf4(2 * H7_BM, (uint32_t)bn);
            const uint32_t sf = tmem_base + H7_SF_COL;
            const int nkb = prm.kblocks;
            const uint32_t breg16 = (uint32_t)prm.breg >> 4;
            const uint64_t bd0 = h7_desc_sw64(smem_u32(sB));
            const uint64_t bias_ad = h7_desc_sw64(smem_u32(sBiasA), H7_BIAS_SBO), bias_bd = h7_desc_sw64(smem_u32(sBiasB), H7_BIAS_SBO);
            const uint32_t sf_bias = tmem_base + H7_SFBIAS_COL;
            const uint32_t p4 = (uint32_t)prm.P * 4;  // one halo row of positions in 16-byte units
            const bool skip_mma = H7_DBG(2) != 0;
            const bool single = H7_DBG(4096) != 0;      // timing experiment: one issuer for all tiles
            mbar_wait(sf_ready, 0);
            tc_fence_after();
            uint32_t t = 0;
            H7Ring ar, fr;  // accumulator and fp4-halo rings: slot and phase of tile t (no divisions on the issue path)
            ar.init(prm.nacc);
            fr.init(prm.f4_st);
            for (int nt = 0; nt < prm.n_tiles; ++nt) {
                mbar_wait(b_full, nt & 1);
                tc_fence_after();
                for (int i = 0; i < my_tiles; ++i, ++t, ar.next(), fr.next()) {
                    const int u = (int)t;
                    const int a = (int)ar.idx;
                    if (single ? which != 0 : (u & 1) != which) continue;  // the other issuer's tile
                    mbar_wait_poll(&tmem_empty[a], ar.phase ^ 1);
                    if (lane == 0) H7_TRACE(4, t);
                    const uint32_t fs = fr.idx;
                    mbar_wait_poll(&a_full[fs], fr.phase);
                    tc_fence_after();
                    if (lane == 0) H7_TRACE(5, t);
                    // lane 0 issues (a converged warp with elect.sync issued fewer instructions per MMA
                    // but ran c4 4% slower, as it did in K5)
                    if (lane == 0) {
                        const uint32_t d_tmem = tmem_base + (uint32_t)(a * prm.acc_cols);
                        const uint64_t ad0 = h7_desc_sw64(smem_u32(sF4 + fs * f4_stage));
                        // The bias MMA sets every accumulator element to 64 * (1.0 * 2^16) * 1.5 = 1.5 * 2^22.
                        // The taps then add half-integers of magnitude <= 16383.5: every partial sum stays in
                        // [2^22, 2^23), where the f32 spacing is 0.5 — exact — and the low 16 bits of the
                        // f32's mantissa are the int16 result (2 * sum mod 2^16), so the epilogue has no
                        // arithmetic left (tcgen05.ld.pack::16b takes those halves).
                        if (!H7_DBG(8192)) umma_mxf4_pair(d_tmem, bias_ad, bias_bd, idesc, sf_bias, sf, 0);
                        if (prm.k33) {
#pragma unroll
                            for (int kb = 0; kb < 9; ++kb) {
                                const uint64_t ad = ad0 + (uint32_t)((kb / 3) * p4 + (kb % 3) * 4);
                                const uint64_t bd = bd0 + (uint32_t)(kb * breg16);
                                if (!skip_mma) {
                                    umma_mxf4_pair(d_tmem, ad, bd, idesc, sf, sf, kb != 0 || !H7_DBG(8192));
                                    umma_mxf4_pair(d_tmem, ad + 2, bd + 2, idesc, sf, sf, 1);
                                }
                            }
                        } else {
                            for (int kb = 0; kb < nkb; ++kb) {
                                const uint64_t ad = ad0 + kb_aoff[kb];
                                const uint64_t bd = bd0 + (uint64_t)kb * breg16;
                                if (!skip_mma) {
                                    umma_mxf4_pair(d_tmem, ad, bd, idesc, sf, sf, kb != 0 || !H7_DBG(8192));
                                    umma_mxf4_pair(d_tmem, ad + 2, bd + 2, idesc, sf, sf, 1);
                                }
                            }
                        }
                        umma_commit_pair(&a_empty[fs], 0x3);
                        umma_commit_pair(&tmem_full[a], 0x3);
                        H7_TRACE(6, t);
                    }
                    __syncwarp();
                }
                if (lane == 0) umma_commit_pair(b_empty, 0x3);
                __syncwarp();
            }
        }
    } else {
        // ===================== epilogue (both CTAs): warps 0 .. NEPI-1 =====================
        // two warps per TMEM lane quarter and tile, each half of the columns; with 16 warps
        // two such groups of 8 drain alternate tiles (two tiles in flight)
        const int wq = warp & 3;     // TMEM lane quarter = 32 output positions
        const int half = (warp >> 2) & 1;          // which half of the tile's columns
        const int tgrp = NEPI == 16 ? warp >> 3 : 0;  // 16 warps: two groups on alternate tiles
        const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
        if (warp < 8) {  // unit UE8M0 scales (sf_ready counts 8 warps x 2 CTAs)
            tmem_st_32x32b_x8_fill(tmem_base + lane_base + H7_SF_COL, 0x7F7F7F7Fu);
            tmem_st_32x32b_x8_fill(tmem_base + lane_base + H7_SFBIAS_COL, 0x8F8F8F8Fu);  // 2^16: the bias MMA's A scales
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(sf_ready), 0));
        }
        const uint32_t tmem_empty0 = mapa_shared(smem_u32(&tmem_empty[0]), 0);
        const int nch = bn / 16, nch0 = (nch + 1) / 2;
        const int ch0 = half ? nch0 : 0, ch1 = half ? nch : nch0;  // this warp's 16-column chunks
        // The warp's 32 positions are 32 consecutive pixels of one output row (P
        // is a multiple of 32): one TMA store box of 32 pixels x 64 columns (the block's
        // valid pixels when rows are cut into column blocks: P = 32, the first vx of the warp's rows).
        const int ry = (wq * 32) / prm.P, ox0 = (wq * 32) % prm.P;
        const uint32_t stg = smem_u32(sEpi) + (uint32_t)warp * 4096u;  // this warp's staging box
        int u = 0;
        H7Ring ar;
        ar.init(prm.nacc);
        for (int nt = 0; nt < prm.n_tiles; ++nt) {
            H7Walk wk;
            wk.init(pair * 2 + (int)rank, 2 * npairs, prm.tpi);
            for (int i = 0; i < my_tiles; ++i, ++u, wk.next(), ar.next()) {
                if (NEPI == 16 && (u & 1) != tgrp) continue;  // the other group's tile
                const int acc = (int)ar.idx;
                const uint32_t acc_phase = ar.phase;
                const int ct = (pair + i * npairs) * 2 + (int)rank;
                const int img = wk.img;
                const int rem = wk.rem, yb = prm.nxb == 1 ? rem : rem / prm.nxb;
                const int oy = yb * prm.R + ry, ox = (rem - yb * prm.nxb) * prm.vx + ox0;
                const bool store_ok = ct < prm.ctiles && oy < prm.oh && ox < prm.ow && !H7_DBG(1);
                // one warp of the group waits on the mbarrier, the other seven block on a named
                // barrier: sixteen wait loops cost issue slots the converters need
                if (!H7_DBG(64) && (warp & 7) == 0) h7_wait(prm.dbg, &tmem_full[acc], acc_phase);
                named_bar_sync(1 + tgrp, 256);
                tc_fence_after();
                if (wq == 0 && lane == 0) H7_TRACE(7, u);
                if (H7_DBG(128)) {  // timing experiment: drain nothing
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(tmem_empty0 + acc * 8);
                    continue;
                }
                const uint32_t tacc = tmem_base + lane_base + (uint32_t)(acc * prm.acc_cols);
                auto release = [&]() {  // the tile's last TMEM read is done: hand the accumulator back
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(tmem_empty0 + acc * 8);
                    if (wq == 0 && lane == 0) H7_TRACE(8, u);
                };
                // Groups of up to 4 chunks (64 columns) go through this warp's 4 KB staging box
                // (128-byte swizzle; 16-column boxes with 32-byte swizzle for a tail) and out by
                // TMA store: 32 pixels x 64 columns per instruction, clipped at the image's
                // right / bottom edge by the tensor map.  Direct per-lane 32-byte stores cost 32
                // L1 lines per instruction and their stalls delayed the accumulator's release.
                // the accumulator holds 1.5 * 2^22 + sum (see the bias MMA): the low 16 bits of each
                // f32 are the int16 result, and pack::16b loads 16 columns as 8 packed words
                auto load16 = [&](int chunk, uint32_t (&w8)[8]) {
                    if (!H7_DBG(8)) {
                        tmem_ld_32x32b_x8_pack16(tacc + chunk * 16, w8);
                    } else {
#pragma unroll
                        for (int q = 0; q < 8; ++q) w8[q] = (uint32_t)q;
                    }
                };
                for (int g = ch0; g < ch1; g += 4) {
                    const int nc = ch1 - g < 4 ? ch1 - g : 4;
                    const bool last_box = g + 4 >= ch1;
                    if (lane == 0) bulk_wait_read<0>();  // the previous box left the staging buffer
                    __syncwarp();
                    if (nc == 4) {  // a full box: SW128, 16-byte unit q of row `lane` at ((q ^ (lane & 7)) << 4)
                        const uint32_t row = stg + lane * 128;
                        uint32_t w[4][8];
#pragma unroll
                        for (int c = 0; c < 4; ++c) load16(g + c, w[c]);
                        tmem_ld_wait();
                        if (last_box) release();
                        if (!H7_DBG(16)) {
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                sts_v4(row + (((2 * c) ^ (lane & 7)) << 4), w[c][0], w[c][1], w[c][2], w[c][3]);
                                sts_v4(row + (((2 * c + 1) ^ (lane & 7)) << 4), w[c][4], w[c][5], w[c][6], w[c][7]);
                            }
                        }
                    } else {  // a tail of 1-3 chunks: SW32 1 KB boxes
                        const uint32_t sw = (uint32_t)(lane >> 2) & 1;
                        for (int c = 0; c < nc; ++c) {
                            uint32_t w8[8];
                            load16(g + c, w8);
                            tmem_ld_wait();
                            if (c == nc - 1 && last_box) release();
                            if (!H7_DBG(16)) {
                                const uint32_t row = stg + c * 1024 + lane * 32;
                                sts_v4(row + (sw << 4), w8[0], w8[1], w8[2], w8[3]);
                                sts_v4(row + ((sw ^ 1) << 4), w8[4], w8[5], w8[6], w8[7]);
                            }
                        }
                    }
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0 && store_ok) {
                        const int col = nt * bn + g * 16;
                        if (nc == 4) tma_store_4d(&tmap_c64, stg, col, ox, oy, img);
                        else
                            for (int c = 0; c < nc; ++c) tma_store_4d(&tmap_c16, stg + c * 1024, col + c * 16, ox, oy, img);
                        bulk_commit();
                    }
                }
                if (wq == 0 && lane == 0) H7_TRACE(9, u);
            }
        }
        // the staging buffers must outlive the stores' reads; their writes are complete when the grid is
        if (lane == 0) bulk_wait_read<0>();
    }

    tc_fence_before();
    __syncthreads();
    if (H7_DBG(32) && threadIdx.x == 0) atomicMax(&g_halo_phase[2], h7_gtime());
    cluster_sync();
    if (warp == H7_W_MMA) {
        tc_fence_after();
        tmem_dealloc_pair<512>(tmem_base);
    }
    if (H7_DBG(32) && threadIdx.x == 0) atomicMax(&g_halo_phase[3], h7_gtime());
}

static int h7_pick_bn(int cout) {
    const int tiles = (cout + H7_MAX_BN - 1) / H7_MAX_BN;
    const int per = (cout + tiles - 1) / tiles;
    return (per + 15) / 16 * 16;
}

namespace {
struct HaloGeom {
    int P, R, rows_h, nxb, vx, bn, breg, raw_cb, f4_cb, raw_st, f4_st, kblocks, nepi;
    bool ok;
};
HaloGeom halo_geom(int h, int w, int c, int cout, int kh, int kw, int stride, int pad) {
    HaloGeom g{};
    g.ok = false;
    const int wp = w + 2 * pad;
    if (stride != 1 || c % 128 != 0 || cout % 8 != 0 || kw > 9 || h + 2 * pad < kh || wp < kw) return g;
    const int oh = h + 2 * pad - kh + 1, ow = wp - kw + 1;
    // Whole padded rows on a pitch of 32, 64 or 128 positions — or, when that takes fewer tiles
    // (or the row is wider than 128), rows cut into column blocks of 32 positions with 32 - (kw - 1)
    // valid outputs each, 4 output rows per tile.  (Config 4 needs 28 tiles per image either way and
    // keeps whole rows: blocks move 25% less halo through shared memory but ran 4% slower, 19.6 us
    // against 18.9 back to back.)
    g.P = wp <= 32 ? 32 : (wp <= 64 ? 64 : 128);
    g.nxb = 1;
    g.vx = ow;
    if (wp > 32) {
        const int vx = 32 - (kw - 1), nxb = (ow + vx - 1) / vx;
        const long long tiles_blocked = (long long)((oh + 3) / 4) * nxb;
        const long long tiles_rows = wp <= 128 ? (oh + H7_BM / g.P - 1) / (H7_BM / g.P) : -1;
        static const bool no_blocks = lb::tuning_env("LOWBIT_HALO_NOBLOCKS") != nullptr;  // tuning knob
        if (tiles_rows < 0 || (tiles_blocked < tiles_rows && !no_blocks)) g.P = 32, g.nxb = nxb, g.vx = vx;
    }
    g.R = H7_BM / g.P;
    g.rows_h = g.R + kh - 1;
    if (g.rows_h > 256) return g;
    const int cb = c / 128;
    g.kblocks = kh * kw * cb;
    g.bn = h7_pick_bn(cout);
    g.breg = ((g.bn / 2) * 64 + 1023) / 1024 * 1024;
    g.raw_cb = g.rows_h * g.P * 128;
    g.f4_cb = ((g.rows_h * g.P + 8) * 64 + 1023) / 1024 * 1024;  // + the taps' over-read past the halo
    if (g.kblocks > H7_MAX_KB || cb * g.raw_cb > H7_RAW_MAX) return g;
    // 16 epilogue warps when their staging fits, else 8; ring depths: fp4 3 (2 if tight),
    // raw whatever is left (<= 4, >= 2)
    static const int f4_max = lb::tuning_env("LOWBIT_HALO_F4ST") ? atoi(lb::tuning_env("LOWBIT_HALO_F4ST")) : 3;  // tuning knob
    static const int nepi_max = lb::tuning_env("LOWBIT_HALO_NEPI8") ? 8 : H7_NEPI_MAX;                            // tuning knob
    for (int nepi = nepi_max; nepi >= 8; nepi -= 8) {
        const int budget = H7_SMEM - 1024 - H7_BAR_BYTES - H7_BIAS_A - H7_BIAS_B - h7_epi_bytes(nepi) - g.kblocks * g.breg;
        for (int f4 = f4_max; f4 >= 2; --f4) {
            const int raw = (budget - f4 * cb * g.f4_cb) / (cb * g.raw_cb);
            if (raw >= 2) {
                g.f4_st = f4;
                static const int raw_max = lb::tuning_env("LOWBIT_HALO_RAWST") ? atoi(lb::tuning_env("LOWBIT_HALO_RAWST")) : H7_RAW_CAP;
                g.raw_st = raw < raw_max ? raw : raw_max;  // (tuning knob: LOWBIT_HALO_RAWST caps the raw ring)
                g.nepi = nepi;
                g.ok = true;
                return g;
            }
        }
    }
    return g;
}
}  // namespace

// Whether K7 takes a conv: stride 1, 128-channel blocks, any map width (column
// blocks past 128 padded pixels), and a filter + two raw and two fp4 halo
// stages that fit in shared memory.
bool conv_halo_applies(int fm_binary, int h, int w, int c, int cout, int kh, int kw, int stride, int pad,
                       long long batch) {
    (void)fm_binary;  // binary maps padded with +-1: the converters write the pad codes
    const HaloGeom g = halo_geom(h, w, c, cout, kh, kw, stride, pad);
    if (!g.ok) return false;
    const long long tpi = (long long)((h + 2 * pad - kh + 1 + g.R - 1) / g.R) * g.nxb;
    return batch * tpi < 0x7FFFFFFFLL;
}

bool conv_ts_applies(int h, int w, int c, int cout, int kh, int kw, int stride, int pad, long long batch);
lowbit_status launch_conv_ts(const int8_t* fm, int batch, int h, int w, int cch, int kh, int kw, int pad,
                             int check_zero, int pad_value, const void* weights, int b_ternary, int cout,
                             int16_t* out, int* zero_flag, cudaStream_t stream);

lowbit_status launch_conv_halo(const int8_t* fm, int batch, int h, int w, int cch, int kh, int kw, int pad,
                               int check_zero, int pad_value, const void* weights, int b_ternary, int cout,
                               int16_t* out, int* zero_flag, cudaStream_t stream) {
    // cout <= 128 and <= 14 k-blocks: the filter-in-TMEM variant (conv_fp4_ts.cu)
    if (conv_ts_applies(h, w, cch, cout, kh, kw, 1, pad, batch))
        return launch_conv_ts(fm, batch, h, w, cch, kh, kw, pad, check_zero, pad_value, weights, b_ternary, cout,
                              out, zero_flag, stream);
    const HaloGeom g = halo_geom(h, w, cch, cout, kh, kw, 1, pad);
    if (!g.ok) return lbhost::set_error(LOWBIT_INVALID_ARGUMENT, "conv halo kernel: unsupported shape");
    const int oh = h + 2 * pad - kh + 1, ow = w + 2 * pad - kw + 1;
    const int k = kh * kw * cch;
    const WeightsLayout L(b_ternary, cout, k);
    const uint8_t* wfp4 = static_cast<const uint8_t*>(weights) + L.off_fp4c;  // conv order (layout.cuh)

    HaloParams prm{};
    prm.batch = batch;
    prm.h = h;
    prm.w = w;
    prm.oh = oh;
    prm.ow = ow;
    prm.pad = pad;
    prm.kw = kw;
    prm.cblocks = cch / 128;
    prm.P = g.P;
    prm.log2p = g.P == 32 ? 5 : (g.P == 64 ? 6 : 7);
    prm.R = g.R;
    prm.rows_h = g.rows_h;
    prm.nxb = g.nxb;
    prm.vx = g.vx;
    prm.tpi = (oh + g.R - 1) / g.R * g.nxb;
    prm.ctiles = batch * prm.tpi;
    prm.ptiles = (prm.ctiles + 1) / 2;
    prm.cout = cout;
    prm.bn = g.bn;
    prm.n_tiles = (cout + g.bn - 1) / g.bn;
    prm.kblocks = g.kblocks;
    prm.breg = g.breg;
    prm.raw_cb = g.raw_cb;
    prm.f4_cb = g.f4_cb;
    prm.raw_st = g.raw_st;
    prm.f4_st = g.f4_st;
    prm.nacc = 3 * g.bn <= (int)H7_SF_COL ? 3 : 2;
    prm.acc_cols = prm.nacc == 3 ? (int)H7_SF_COL / 3 : H7_MAX_BN;
    prm.k33 = kh == 3 && kw == 3 && prm.cblocks == 1;
    prm.check_zero = check_zero;
    prm.mul16 = 16;
    prm.pad_word = pad > 0 ? (pad_value > 0 ? 0x01010101u : (pad_value < 0 ? 0xFFFFFFFFu : 0u)) : 0u;
    static const int dbg = lb::tuning_env("LOWBIT_HALO_DEBUG") ? atoi(lb::tuning_env("LOWBIT_HALO_DEBUG")) : 0;
    prm.dbg = dbg;
    prm.out = out;
    prm.zero_flag = zero_flag;

    CUtensorMap mb, mraw, mc64, mc16;
    const uint32_t box_px = g.nxb > 1 ? (uint32_t)g.vx : 32u;  // column blocks: a warp stores its block's valid pixels
    if (!make_map_conv_out_box(&mc64, out, batch, oh, ow, cout, 64, box_px, 1, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !make_map_conv_out_box(&mc16, out, batch, oh, ow, cout, 16, box_px, 1, CU_TENSOR_MAP_SWIZZLE_32B))
        return lbhost::set_error(LOWBIT_CUDA_ERROR, "cuTensorMapEncodeTiled failed for the conv output");
    if (!make_map_2d(&mb, wfp4, (uint64_t)L.kp4 / 2, (uint64_t)L.np, (uint64_t)L.kp4 / 2, 64, (uint32_t)(g.bn / 2),
                     CU_TENSOR_MAP_SWIZZLE_64B))
        return lbhost::set_error(LOWBIT_CUDA_ERROR, "cuTensorMapEncodeTiled failed for the conv filter");
    if (!make_map_nhwc_box(&mraw, fm, batch, h, w, cch, (uint32_t)g.P, (uint32_t)g.rows_h))
        return lbhost::set_error(LOWBIT_CUDA_ERROR, "cuTensorMapEncodeTiled failed for the feature-map halo");
    const int flags = (prm.pad_word != 0 ? 1 : 0) | (check_zero ? 2 : 0);
    using KernT = decltype(&conv_fp4_halo_kernel<16, 0>);
    const KernT kerns[2][4] = {{conv_fp4_halo_kernel<8, 0>, conv_fp4_halo_kernel<8, 1>, conv_fp4_halo_kernel<8, 2>,
                                conv_fp4_halo_kernel<8, 3>},
                               {conv_fp4_halo_kernel<16, 0>, conv_fp4_halo_kernel<16, 1>, conv_fp4_halo_kernel<16, 2>,
                                conv_fp4_halo_kernel<16, 3>}};
    const KernT kern = kerns[g.nepi == 16][flags];
    static SmemOptIn attr[2][4];
    LB_CUDA_TRY(attr[g.nepi == 16][flags].ensure(kern, H7_SMEM));
    const int pairs = prm.ptiles < num_sms() / 2 ? prm.ptiles : num_sms() / 2;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(h7_threads(g.nepi));
    cfg.dynamicSmemBytes = H7_SMEM;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    static const bool no_pdl = lb::tuning_env("LOWBIT_NO_PDL") != nullptr;  // tuning experiment knob
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = no_pdl ? 0 : 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    LB_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, mb, mraw, mc64, mc16, prm));
    LB_CUDA_TRY(cudaGetLastError());
    return LOWBIT_OK;
}

}  // namespace lb

extern "C" int lowbit_debug_halo_trace(unsigned long long* out1024) {
    return cudaMemcpyFromSymbol(out1024, lb::g_halo_trace, sizeof(unsigned long long) * 1024) != cudaSuccess;
}
// phases of the last K7 launch with LOWBIT_HALO_DEBUG & 32 (ns); reset = 1 re-arms them
extern "C" int lowbit_debug_halo_phases(unsigned long long* out4, int reset) {
    if (cudaMemcpyFromSymbol(out4, lb::g_halo_phase, sizeof(unsigned long long) * 4) != cudaSuccess) return 1;
    if (reset) {
        const unsigned long long init[4] = {~0ull, 0, 0, 0};
        return cudaMemcpyToSymbol(lb::g_halo_phase, init, sizeof init) != cudaSuccess;
    }
    return 0;
}
